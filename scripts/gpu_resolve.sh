REPS=3 python scripts/setup_c3_phases.py > gpurun_out/resolve.log 2>&1
PCT=5 REPS=2 python scripts/setup_c3_phases.py >> gpurun_out/resolve.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "greedy or bisect or fullsize or slab or dropin or combo or objective" >> gpurun_out/resolve.log 2>&1; echo "exit $?" >> gpurun_out/resolve.log
