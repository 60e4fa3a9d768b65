timeout 900 python -m pytest tests/test_shard.py -x -q -m gpu > gpurun_out/t_shard2.log 2>&1; echo "exit $?" >> gpurun_out/t_shard2.log
