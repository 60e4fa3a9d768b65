set -x
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/t_gpu_pdl.log 2>&1; echo "exit $?" >> gpurun_out/t_gpu_pdl.log
timeout 300 python scripts/spmv_ab.py 2 > gpurun_out/ab9.log 2>&1; echo "exit $?" >> gpurun_out/ab9.log
timeout 300 python scripts/spmv_ab.py 3 > gpurun_out/ab9_c3.log 2>&1; echo "exit $?" >> gpurun_out/ab9_c3.log
