timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_fuse.log 2>&1; echo "exit $?" >> gpurun_out/t_fuse.log
for c in 2 3 4; do timeout 300 python scripts/spmv_ab.py $c >> gpurun_out/ab_fuse.log 2>&1; done
