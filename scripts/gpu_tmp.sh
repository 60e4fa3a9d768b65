for b in 0 2 3 1; do PDB_DIAG_BPS=$b TAG=bps$b REPS=2 python scripts/lib_ab.py >> gpurun_out/bps.log 2>&1; done
