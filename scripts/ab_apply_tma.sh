# A/B of the 192-DoF tile apply: TMA-staged inverse (default) vs the register-streamed kernel
# (PDB_APPLY_TMA=0), config 5 at 32^3 cells.  Run on the GPU box from the repo root.
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
run st3_c0 PDB_RES_CARVEOUT=0
run off_c0 PDB_APPLY_TMA=0 PDB_RES_CARVEOUT=0
run st3 PDB_APPLY_TMA_STAGES=3
run off PDB_APPLY_TMA=0
