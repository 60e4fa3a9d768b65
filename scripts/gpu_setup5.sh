for te in 32 64; do PCT=5 PDB_L1_TE=$te REPS=2 python scripts/setup_c3_phases.py > gpurun_out/s5_te$te.log 2>&1; done
PCT=5 PDB_TRACE=1 REPS=1 python scripts/setup_c3_phases.py > gpurun_out/s5_trace.log 2>&1
for v in 0 1; do PDB_L2_PERSIST=$v PDB_TRACE=$v CONFIGS=3 STEPS=200 scripts/sweep_ab.sh "PDB_L2_PERSIST=$v" >> gpurun_out/s5_l2.log 2>&1; done
