#!/bin/bash
# Sweep-kernel variant timing on config 2 (entrywise k-means for a short setup).
cd "$(dirname "$0")/.."
run() {
  env "$@" python bench.py --method kmeans-entrywise --no-cpu-baseline --steps 200 --warmup 20 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step']*1e3,1), 'us/sweep', {k: round(v*1e3,1) for k,v in d['sweep_roofline']['kernel_ms'].items()}, 'resid frac', round(d['roofline']['frac'],3), 'sweep frac', round(d['sweep_roofline']['frac'],3))"
}
run DEFAULT=1
run PDB_SPMV_VERSION=2 PDB_SPMV_GROUP=8 PDB_SPMV_ENTRIES=8
run PDB_PADDED=0
run PDB_GROUPED=0
