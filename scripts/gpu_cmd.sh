timeout 300 python scripts/spmv_ab.py 2 > gpurun_out/ab_clean2.log 2>&1
timeout 300 python scripts/spmv_ab.py 3 >> gpurun_out/ab_clean2.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_clean2.log 2>&1; echo "exit $?" >> gpurun_out/t_clean2.log
