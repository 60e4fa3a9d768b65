timeout 900 python -m pytest tests/ -q -m gpu -k "pcg" > gpurun_out/t_pcg.log 2>&1; echo "exit $?" >> gpurun_out/t_pcg.log
VARIANTS=exact,spectral timeout 900 python scripts/pcg_probe.py > gpurun_out/pcg.log 2>&1; echo "exit $?" >> gpurun_out/pcg.log
PDB_PCG_LOOKAHEAD=0 VARIANTS=exact timeout 900 python scripts/pcg_probe.py > gpurun_out/pcg0.log 2>&1; echo "exit $?" >> gpurun_out/pcg0.log
