scripts/sweep_ab.sh "PDB_APPLY_SP=0 PDB_SCATTER=pad" "PDB_APPLY_SP=1 PDB_SCATTER=pad" "PDB_APPLY_SP=1 PDB_SCATTER=csr" "PDB_APPLY_SP=0 PDB_SCATTER=pad" "PDB_APPLY_SP=1 PDB_SCATTER=csr" > gpurun_out/ab1.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "sweep or relax or history or apply or pcg" >> gpurun_out/ab1.log 2>&1
