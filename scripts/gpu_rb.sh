for i in 1 2; do for v in 1 2; do CONFIGS="3 2" STEPS=300 scripts/sweep_ab.sh "PDB_APPLY_RB=$v" >> gpurun_out/rb.log 2>&1; done; done
CONFIGS=4 scripts/sweep_ab.sh "PDB_APPLY_RB=1" "PDB_APPLY_RB=2" >> gpurun_out/rb.log 2>&1
PDB_APPLY_RB=2 timeout 900 python -m pytest tests -m gpu -x -q -k "relax or apply or history or pcg or identity or front" >> gpurun_out/rb.log 2>&1
