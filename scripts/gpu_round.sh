# The round's GPU evidence in one gpurun call (run from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2700 -- 'bash scripts/gpu_round.sh'
# GPU tests, the default bench line (config 3) and the reference arm, then the
# launch list of a config-3 build + 5 sweeps (ncu, after the runs above exited 0).
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/round_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/round_pytest.log 2>&1; echo "exit $?" >> gpurun_out/round_pytest.log
timeout 900 python bench.py > gpurun_out/round_bench.log 2>&1; echo "exit $?" >> gpurun_out/round_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/round_ref.log 2>&1; echo "exit $?" >> gpurun_out/round_ref.log
SWEEPS=5 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/round_launches.csv python scripts/sweep_c3_once.py > gpurun_out/round_ncu.log 2>&1
for c in 1 2 4 5; do timeout 900 python bench.py --config $c --steps 100 --warmup 10 > gpurun_out/round_c$c.log 2>&1; echo "exit $?" >> gpurun_out/round_c$c.log; done
