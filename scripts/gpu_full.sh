timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1; echo "exit $?" >> gpurun_out/full_tests.log
REPS=3 python scripts/setup_c3_phases.py > gpurun_out/full_setup.log 2>&1
timeout 600 python bench.py > gpurun_out/full_bench.log 2>&1; echo "exit $?" >> gpurun_out/full_bench.log
