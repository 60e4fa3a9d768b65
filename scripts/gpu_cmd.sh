set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo "exit $?" >> gpurun_out/t_all.log
for c in 1 3; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "exit $?" >> gpurun_out/bench_c$c.err
done
