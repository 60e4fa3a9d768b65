timeout 900 python scripts/combo_bench.py 256,4 > gpurun_out/combo_bench2.log 2>&1; echo "exit $?" >> gpurun_out/combo_bench2.log
