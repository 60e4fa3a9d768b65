for pf in 0 1 2 3; do
  PDB_SPECTRAL_PF=$pf ITERS=10 timeout 300 python scripts/setup_small.py 256 >> gpurun_out/setup_pf.log 2>&1
done
PDB_SPECTRAL_PF=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spectral" >> gpurun_out/setup_pf.log 2>&1
