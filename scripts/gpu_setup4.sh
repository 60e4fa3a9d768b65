for te in 32 64 128; do PDB_L1_TE=$te REPS=3 python scripts/setup_c3_phases.py > gpurun_out/setup4_te$te.log 2>&1; done
PDB_L1_TE=64 timeout 900 python -m pytest tests -m gpu -x -q -k "greedy or l1 or kmeans or fullsize_pins or slab" > gpurun_out/setup4_tests64.log 2>&1
PDB_L1_TE=128 timeout 900 python -m pytest tests -m gpu -x -q -k "greedy or l1 or kmeans or fullsize_pins or slab" > gpurun_out/setup4_tests128.log 2>&1
REPS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:l1_tile_kernel -s 3 -c 1 -o gpurun_out/l1scan_big python scripts/setup_c3_phases.py > gpurun_out/setup4_ncu.log 2>&1
