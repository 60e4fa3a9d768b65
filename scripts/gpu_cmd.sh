timeout 900 python -m pytest tests/test_configs45.py -x -q -m gpu > gpurun_out/t_c45b.log 2>&1; echo "exit $?" >> gpurun_out/t_c45b.log
