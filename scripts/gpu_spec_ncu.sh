timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t11.log 2>&1; echo "exit $?" >> gpurun_out/t11.log
PDB_TRACE=1 python scripts/setup_one.py > gpurun_out/spec_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spectral_tile -s 40 -c 2 -o gpurun_out/spec_src python scripts/setup_one.py > gpurun_out/spec_ncu.log 2>&1
