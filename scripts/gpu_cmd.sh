set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "exit $?" >> gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "exit $?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "exit $?" >> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "exit $?" >> gpurun_out/final_bench_ref.err
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/final_gpu.txt
