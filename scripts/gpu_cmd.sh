set -x
timeout 600 python -m pytest tests/test_shard.py -x -q -m gpu > gpurun_out/t_shard.log 2>&1; echo "exit $?" >> gpurun_out/t_shard.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 --method kmeans-entrywise --no-cpu-baseline > gpurun_out/bench_tr1.json 2> gpurun_out/bench_tr1.err; echo "exit $?" >> gpurun_out/bench_tr1.err
