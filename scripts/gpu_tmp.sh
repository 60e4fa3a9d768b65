PDB_KMEANS_TRACE=1 python scripts/setup_one.py > gpurun_out/kmtrace2.log 2>&1
REPS=3 python scripts/lib_ab.py >> gpurun_out/kmtrace2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "kmeans or bootstrap or varmin or fullsize_pins or slab or configs45" >> gpurun_out/kmtrace2.log 2>&1; echo "exit $?" >> gpurun_out/kmtrace2.log
