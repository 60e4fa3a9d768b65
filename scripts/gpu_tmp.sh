timeout 1200 python -m pytest tests/test_configs45.py tests/test_slab.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/tma_pytest.log 2>&1; echo "exit $?" >> gpurun_out/tma_pytest.log
for c in 5 2 3; do timeout 900 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/tma_c$c.log 2>&1; echo "exit $?" >> gpurun_out/tma_c$c.log; done
CELLS=32 SWEEPS=2 timeout 900 python scripts/sweep_c5_once.py > gpurun_out/tma_once.log 2>&1 && \
CELLS=32 SWEEPS=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:patch_apply_dmma_tma -c 1 -s 1 \
  -o gpurun_out/apply_tma_c5 -f python scripts/sweep_c5_once.py > gpurun_out/tma_ncu.log 2>&1
CELLS=32 SWEEPS=2 PDB_APPLY_TMA=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:patch_apply_dmma_large -c 1 -s 1 \
  -o gpurun_out/apply_large_c5 -f python scripts/sweep_c5_once.py >> gpurun_out/tma_ncu.log 2>&1
