timeout 2400 python -m pytest tests/ -q -m gpu -x --durations=15 > gpurun_out/t_all.log 2>&1; echo "exit $?" >> gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
