# A/B of the 192-DoF tile apply at config 5 (32^3 cells): persistent pipelined TMA kernel (default),
# one-tile-per-block TMA kernel (PDB_APPLY_TMA_PERSISTENT=0), register-streamed kernel (PDB_APPLY_TMA=0).
# Run on the GPU box from the repo root.
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 900 python bench.py --config 5 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ab_tma_$name.log 2>&1; echo "exit $?" >> gpurun_out/ab_tma_$name.log
  python - "$name" <<'P'
import json, sys
l = [x for x in open(f"gpurun_out/ab_tma_{sys.argv[1]}.log") if x.startswith("{")]
if l:
    d = json.loads(l[-1])
    print(sys.argv[1], d["ms_per_step"], d["sweep_roofline"]["kernel_ms"], file=open("gpurun_out/ab_tma_summary.txt", "a"))
P
}
rm -f gpurun_out/ab_tma_summary.txt
timeout 900 python -m pytest tests/test_configs45.py tests/test_slab.py -m gpu -x -q > gpurun_out/ab_tma_pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab_tma_pytest.log
run persistent PDB_APPLY_TMA_PERSISTENT=1
run persistent_st1 PDB_APPLY_TMA_STAGES=1
run tile PDB_APPLY_TMA_PERSISTENT=0
run off PDB_APPLY_TMA=0
run persistent2 PDB_APPLY_TMA_PERSISTENT=1
