"""Config-3 headline setup, phase by phase (detect / greedy-l1 pass at the
committed 1 % eps / preconditioner), REPS repetitions after a warm-up; run
with PDB_TRACE=1 for the library's scope timings on stderr."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(3, 0)
A = prob.matrix()
eps = float(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"c3_l1_{os.environ.get('PCT', '1')}.npz"))["eps"])
for rep in range(1 + int(os.environ.get("REPS", "4"))):
    ps = db = pc = None
    gc.collect()
    t0 = time.perf_counter(); ps = P.PatchSet.detect(A, 27)
    t1 = time.perf_counter(); db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps)
    t2 = time.perf_counter(); pc = P.Preconditioner.create(A, ps, db, omega=1.0)
    t3 = time.perf_counter()
    print(f"rep {rep} detect {1e3*(t1-t0):.1f} build {1e3*(t2-t1):.1f} precond {1e3*(t3-t2):.1f} total {1e3*(t3-t0):.1f} ms m={db.size}", flush=True)
if os.environ.get("BISECT", "0") == "1":
    # greedy_bisect_to_size at the band of the committed fixture (BASELINE retention)
    g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"c3_l1_{os.environ.get('PCT', '1')}.npz"))
    lo, hi = (int(v) for v in g["target"])
    for rep in range(2):
        t = time.perf_counter(); dbb, e = P.Database.build_to_size(A, ps, lo, hi, P.GREEDY_L1); t = time.perf_counter() - t
        print(f"bisect {t:.3f} s eps {e!r} m={dbb.size} same_eps={e == float(g['eps'])}", flush=True)
