"""PCG to 1e-8 on BASELINE config 2 with the one-level patch preconditioner
(exact, k-means entrywise k=64, k-means spectral k=64): iterations and time."""
import json, os, sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(2, 0)
A = prob.matrix(); ps = P.PatchSet.detect(A, 25); b = prob.rhs()
maxit = int(os.environ.get("MAXIT", "40000"))
for name in os.environ.get("VARIANTS", "exact,entrywise,spectral").split(","):
    t = time.perf_counter()
    db = None if name == "exact" else P.Database.build(A, ps, {"entrywise": P.KMEANS_ENTRYWISE, "spectral": P.KMEANS_SPECTRAL}[name], db_size=64, seed=42, max_iters=50)
    pc = P.Preconditioner.create(A, ps, db, omega=1.0)
    t_setup = time.perf_counter() - t
    t = time.perf_counter(); x, r = P.pcg(A, b, pc, tol=1e-8, max_iters=maxit); dt = time.perf_counter() - t
    h = np.array(r.residual_history)
    print(json.dumps(dict(config=2, precond=name, setup_s=round(t_setup, 2), pcg_iters=r.iterations, converged=r.converged,
                          final_rel=r.final_relative_residual, solve_s=round(dt, 3), us_per_iter=round(1e6 * dt / max(r.iterations, 1), 1),
                          history_every_10pct=[float(f"{h[i]:.2e}") for i in range(0, len(h), max(1, len(h) // 10))])), flush=True)
