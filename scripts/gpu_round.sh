nvidia-smi -L > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/g1_pytest.log 2>&1; echo "exit $?" >> gpurun_out/g1_pytest.log
timeout 600 python bench.py > gpurun_out/g1_bench.log 2>&1; echo "exit $?" >> gpurun_out/g1_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g1_ref.log 2>&1; echo "exit $?" >> gpurun_out/g1_ref.log
