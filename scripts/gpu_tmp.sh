for i in 1 2; do CONFIGS="5" STEPS=100 scripts/sweep_ab.sh "PDB_LARGE_TILE=32" "PDB_LARGE_TILE=64" >> gpurun_out/large64.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q -k "configs45 or c5 or lu_large or entrywise_kmeans_matches_reference or slab" >> gpurun_out/large64.log 2>&1; echo "exit $?" >> gpurun_out/large64.log
