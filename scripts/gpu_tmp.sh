REPS=3 PDB_TRACE=1 python scripts/setup_c3_phases.py > gpurun_out/ext.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "extract or detect or exact or lu or fullsize or configs45 or slab" >> gpurun_out/ext.log 2>&1; echo "exit $?" >> gpurun_out/ext.log
