timeout 900 python -m pytest tests/test_fullsize.py -x -q -m gpu --durations=3 > gpurun_out/t_full3.log 2>&1; echo "exit $?" >> gpurun_out/t_full3.log
