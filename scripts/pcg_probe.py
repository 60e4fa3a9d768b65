"""PCG on config 2 with the Dirichlet columns eliminated (symmetric system) vs row replacement only."""
import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(2, 0)
rp, ci, v = prob.csr()
b = prob.rhs()
n = len(rp) - 1
cnt = np.diff(rp)
bnd = np.zeros(n, bool)
# boundary rows: single stored entry on the diagonal
one = np.flatnonzero(cnt == 1)
bnd[one] = ci[rp[one]] == one
rows = np.repeat(np.arange(n), cnt)
mask = (~bnd[rows]) & bnd[ci]
bs = b.copy()
np.subtract.at(bs, rows[mask], v[mask] * b[ci[mask]])
vs = v.copy(); vs[mask] = 0.0
As = P.Matrix.from_csr(rp, ci, vs)
A = prob.matrix()
ps = P.PatchSet.detect(As, 25)
for name, M, rhs in [("sym", As, bs), ("rowrep", A, b)]:
    db = P.Database.build(M, ps, P.KMEANS_ENTRYWISE, db_size=64, seed=42, max_iters=50)
    for pname, pc in [("compressed", P.Preconditioner.create(M, ps, db, omega=1.0)), ("exact", P.Preconditioner.create(M, ps, None, omega=1.0))]:
        t = time.perf_counter(); x, r = P.pcg(M, rhs, pc, tol=1e-8, max_iters=8000); dt = time.perf_counter() - t
        h = np.array(r.residual_history)
        print(name, pname, "pcg", r.converged, r.iterations, f"{dt:.2f}s", [f"{h[i]:.1e}" for i in range(0, len(h), max(1, len(h)//10))], flush=True)
