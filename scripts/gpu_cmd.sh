timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_imp.log 2>&1; echo "exit $?" >> gpurun_out/t_imp.log
