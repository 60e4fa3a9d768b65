#!/bin/bash
# A/B of sweep-kernel switches on the bench configs: one line per (config, env).
# usage: scripts/sweep_ab.sh "ENV1=a ENV2=b" "ENV1=c" ...   (CONFIGS="3 2" by default)
cd "$(dirname "$0")/.."
for cfg in ${CONFIGS:-3 2}; do
  for envs in "$@"; do
    env $envs timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps ${STEPS:-200} --warmup 20 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c$cfg', '$envs', round(d['ms_per_step']*1e3,1), 'us/sweep', {k: round(v*1e3,1) for k,v in d['sweep_roofline']['kernel_ms'].items()}, 'resid', round(d['roofline']['frac'],3), 'sweep', round(d['sweep_roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])"
  done
done
