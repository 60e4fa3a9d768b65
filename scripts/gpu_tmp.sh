timeout 1200 python -m pytest tests -m gpu -x -q -k "sell_device or spmv or fem_rows or fullsize or slab or mirror" > gpurun_out/sell.log 2>&1; echo "exit $?" >> gpurun_out/sell.log
PDB_TRACE=1 timeout 1200 python scripts/c5_rank.py > gpurun_out/c5trace2.log 2>&1; echo "exit $?" >> gpurun_out/c5trace2.log
