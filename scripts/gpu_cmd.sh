for c in 2 3 4; do timeout 300 python scripts/spmv_ab.py $c >> gpurun_out/ab_head.log 2>&1; done
