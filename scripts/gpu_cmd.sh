timeout 900 python scripts/setup_c2.py > gpurun_out/setup_c2.log 2>&1; echo "exit $?" >> gpurun_out/setup_c2.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup_launches.csv python scripts/setup_one.py > gpurun_out/setup_ncu.log 2>&1; echo "exit $?" >> gpurun_out/setup_ncu.log
