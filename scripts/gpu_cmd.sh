for r in 0 1 0 1; do
PDB_SPECTRAL_RECIP=$r ITERS=10 timeout 300 python scripts/setup_small.py 256 >> gpurun_out/setup_rc.log 2>&1
done
