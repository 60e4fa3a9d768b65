PDB_APPLY_PIPE=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_configs45.py tests/test_fullsize.py -x -q -m gpu > gpurun_out/t_pipe.log 2>&1; echo "exit $?" >> gpurun_out/t_pipe.log
PDB_APPLY_PIPE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "apply or relax" >> gpurun_out/t_pipe.log 2>&1; echo "exit $?" >> gpurun_out/t_pipe.log
timeout 300 python scripts/spmv_ab.py 2 > gpurun_out/ab_pipe.log 2>&1
timeout 300 python scripts/spmv_ab.py 3 >> gpurun_out/ab_pipe.log 2>&1
