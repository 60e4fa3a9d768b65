"""PCG to 1e-8 on config 2 (BASELINE: 'CG preconditioned by patch relaxation to 1e-8')."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
method = {"entrywise": P.KMEANS_ENTRYWISE, "spectral": P.KMEANS_SPECTRAL}[sys.argv[2] if len(sys.argv) > 2 else "entrywise"]
prob = P.Problem.generate(cfg, 0)
A = prob.matrix()
ps = P.PatchSet.detect(A, 25)
db = P.Database.build(A, ps, method, db_size=64, seed=42, max_iters=50)
pc = P.Preconditioner.create(A, ps, db, omega=1.0)
b = prob.rhs()
for rep in range(2):
    t = time.perf_counter()
    x, r = P.pcg(A, b, pc, tol=1e-8, max_iters=int(os.environ.get("MAXIT", "500")))
    dt = time.perf_counter() - t
    print(f"rep {rep}: converged={r.converged} iterations={r.iterations} rel={r.final_relative_residual:.3e} "
          f"time {dt * 1e3:.1f} ms ({dt / max(r.iterations, 1) * 1e6:.0f} us/iteration)")
