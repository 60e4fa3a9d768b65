timeout 1200 python -m pytest tests -m gpu -x -q -k "slab or shard or sell_device or spmv or mirror" > gpurun_out/slab2.log 2>&1; echo "exit $?" >> gpurun_out/slab2.log
PDB_TRACE=1 timeout 1200 python scripts/c5_rank.py > gpurun_out/c5trace3.log 2>&1; echo "exit $?" >> gpurun_out/c5trace3.log
