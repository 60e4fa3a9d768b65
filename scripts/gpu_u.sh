for i in 1 2; do CONFIGS="3 2" STEPS=300 scripts/sweep_ab.sh "PDB_SCATTER_U=1" "PDB_SCATTER_U=2" "PDB_SCATTER_U=4" >> gpurun_out/u.log 2>&1; done
