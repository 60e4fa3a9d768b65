python scripts/setup_c3_phases.py > gpurun_out/setup3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "detect or greedy or fullsize or slab or dropin or parity" > gpurun_out/setup3_tests.log 2>&1
REPS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:l1_tile_kernel -s 9 -c 2 -o gpurun_out/l1scan python scripts/setup_c3_phases.py > gpurun_out/setup3_ncu.log 2>&1
