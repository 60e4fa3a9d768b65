set -x
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/t_gpu_pipe.log 2>&1; echo "exit $?" >> gpurun_out/t_gpu_pipe.log
B="python bench.py --method kmeans-entrywise --no-cpu-baseline --steps 200 --warmup 20"
timeout 300 $B > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err; echo "exit $?" >> gpurun_out/bench_pipe.err
PDB_PIPELINE=0 timeout 300 $B > gpurun_out/bench_nopipe.json 2> gpurun_out/bench_nopipe.err
