python scripts/setup_c3_phases.py > gpurun_out/setup1.log 2>&1
PDB_TRACE=1 REPS=1 python scripts/setup_c3_phases.py > gpurun_out/setup1_trace.log 2>&1
PDB_DEVBUF_POOL=0 python scripts/setup_c3_phases.py > gpurun_out/setup1_nopool.log 2>&1
