for cfg in "" "PDB_SPECTRAL_LSMEM=1" "PDB_SPECTRAL_TE=4" "PDB_SPECTRAL_TE=4 PDB_SPECTRAL_LSMEM=1"; do
  echo "== $cfg" >> gpurun_out/setup_ls.log
  env $cfg timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_configs45.py -x -q -m gpu -k "spectral" >> gpurun_out/setup_ls.log 2>&1
  env $cfg ITERS=10 timeout 300 python scripts/setup_small.py 256 >> gpurun_out/setup_ls.log 2>&1
done
