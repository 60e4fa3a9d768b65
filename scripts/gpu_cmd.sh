set -x
for c in 3 4 5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "exit $?" >> gpurun_out/bench_c$c.err
done
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "exit $?" >> gpurun_out/bench_r02.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err; echo "exit $?" >> gpurun_out/bench_ref_r02.err
