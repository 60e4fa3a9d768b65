for c in 1 2 4 5; do timeout 900 python bench.py --config $c --steps 100 --warmup 10 > gpurun_out/allcfg_c$c.log 2>&1; echo "exit $?" >> gpurun_out/allcfg_c$c.log; done
