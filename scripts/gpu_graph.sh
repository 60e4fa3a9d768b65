for i in 1 2; do CONFIGS="1 3 2" STEPS=200 scripts/sweep_ab.sh "PDB_GRAPH=0" "PDB_GRAPH=1" >> gpurun_out/graph.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q >> gpurun_out/graph.log 2>&1; echo "exit $?" >> gpurun_out/graph.log
