# The round's GPU evidence in one gpurun call (run from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2700 -- 'bash scripts/gpu_round.sh'
# GPU tests, the default bench line (config 3) and the reference arm, then the
# launch list of a config-3 build + 5 sweeps (ncu, after the runs above exited 0).
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/round_smi.txt
timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/round_smoke.log 2>&1; echo "exit $?" >> gpurun_out/round_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/round_pytest.log 2>&1; echo "exit $?" >> gpurun_out/round_pytest.log
T0=$SECONDS; timeout 900 python bench.py > gpurun_out/round_bench.log 2>&1; echo "exit $?" >> gpurun_out/round_bench.log; echo "bench.py default run: $((SECONDS - T0)) s wall" > gpurun_out/round_bench_wall.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/round_ref.log 2>&1; echo "exit $?" >> gpurun_out/round_ref.log
SWEEPS=5 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/round_launches.csv python scripts/sweep_c3_once.py > gpurun_out/round_ncu.log 2>&1
for c in 1 2 4 5; do timeout 900 python bench.py --config $c --steps 100 --warmup 10 > gpurun_out/round_c$c.log 2>&1; echo "exit $?" >> gpurun_out/round_c$c.log; done
# the N>1 bench path as a one-rank job (rank-local slab API + NCCL communicator of one rank)
BENCH_SLABS=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29511 RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/round_slab1.log 2>&1; echo "exit $?" >> gpurun_out/round_slab1.log
# ncu --set full of the TMA-staged 192-DoF tile apply (config 5 at 32^3 cells), after the plain run exits 0
CELLS=32 SWEEPS=2 timeout 900 python scripts/sweep_c5_once.py > gpurun_out/round_c5_once.log 2>&1 && \
CELLS=32 SWEEPS=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:patch_apply_dmma_tma -c 1 -s 1 \
  -o gpurun_out/round_apply_tma_c5 -f python scripts/sweep_c5_once.py > gpurun_out/round_ncu_tma.log 2>&1
