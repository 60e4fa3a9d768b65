timeout 900 python -m pytest tests/test_combo.py -q -m gpu -x > gpurun_out/t_combo.log 2>&1; echo "exit $?" >> gpurun_out/t_combo.log
timeout 900 python scripts/combo_bench.py > gpurun_out/combo_bench.log 2>&1; echo "exit $?" >> gpurun_out/combo_bench.log
