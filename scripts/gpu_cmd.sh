set -x
ITERS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:spectral_tile -c 12 -o gpurun_out/prof_spec_il python scripts/setup_small.py 256 > gpurun_out/ncu_spec.log 2>&1
tail -3 gpurun_out/ncu_spec.log
