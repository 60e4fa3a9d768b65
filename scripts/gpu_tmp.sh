PDB_TRACE=1 timeout 1200 python scripts/c5_rank.py > gpurun_out/c5trace4.log 2>&1; echo "exit $?" >> gpurun_out/c5trace4.log
BENCH_SLABS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 5 > gpurun_out/slabs1c.log 2>&1; echo "exit $?" >> gpurun_out/slabs1c.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "slab or spmv or fullsize or mmio or abi or generator" > gpurun_out/staged.log 2>&1; echo "exit $?" >> gpurun_out/staged.log
