timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_combo.py -q -m gpu -k "greedy or experiment1" > gpurun_out/t_gr.log 2>&1; echo "exit $?" >> gpurun_out/t_gr.log
timeout 900 python scripts/greedy_prune_probe.py > gpurun_out/gr.log 2>&1; echo "exit $?" >> gpurun_out/gr.log
