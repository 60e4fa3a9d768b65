for i in 1 2; do CONFIGS="3 2 4" STEPS=300 scripts/sweep_ab.sh "PDB_APPLY_TILE=32" "PDB_APPLY_TILE=64" >> gpurun_out/tile64.log 2>&1; done
PDB_APPLY_TILE=64 timeout 900 python -m pytest tests -m gpu -x -q -k "relax or apply or history or pcg or identity" >> gpurun_out/tile64.log 2>&1
