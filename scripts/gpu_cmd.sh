set -x
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/t_gpu_po.log 2>&1; echo "exit $?" >> gpurun_out/t_gpu_po.log
timeout 300 python scripts/spmv_ab.py 2 > gpurun_out/ab8.log 2>&1; echo "exit $?" >> gpurun_out/ab8.log
timeout 300 python scripts/spmv_ab.py 3 > gpurun_out/ab8_c3.log 2>&1; echo "exit $?" >> gpurun_out/ab8_c3.log
