PDB_TRACE=1 REPS=1 python scripts/setup_c3_phases.py > gpurun_out/setup2_trace.log 2>&1
python scripts/setup_c3_phases.py > gpurun_out/setup2.log 2>&1
CONFIGS="3 2" scripts/sweep_ab.sh "DEFAULT=1" > gpurun_out/ab2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q >> gpurun_out/ab2.log 2>&1
