"""Small instances of every hot-path entry point, for compute-sanitizer
(memcheck / racecheck / synccheck): detection, all seven database methods,
exact and compressed preconditioners, sweeps, PCG, GMRES, and a 3-rank
emulated slab group (device sweep), on reduced meshes of configs 1-5."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

CASES = [(1, 0, 9), (2, 8, 25), (3, 4, 27), (4, 8, 22), (5, 2, 192)]
for cfg, cells, ps in CASES:
    prob = P.Problem.generate(cfg, cells)
    A = prob.matrix()
    b = prob.rhs()
    pset = P.PatchSet.detect(A, ps)
    k = max(2, min(16, pset.count // 4))
    methods = [(P.EXACT, {}), (P.GREEDY_L1, dict(eps=0.5)), (P.KMEANS_ENTRYWISE, dict(db_size=k, seed=42, max_iters=5))]
    if ps <= 27:
        methods += [(P.GREEDY_SPECTRAL, dict(eps=0.5)), (P.KMEANS_SPECTRAL, dict(db_size=k, seed=42, max_iters=3)),
                    (P.KMEANS_VARMIN, dict(db_size=k, seed=42, max_iters=2)), (P.BOOTSTRAP, dict(eps=0.5, max_iters=2))]
    for meth, kw in methods:
        db = P.Database.build(A, pset, meth, **kw)
        pc = P.Preconditioner.create(A, pset, db if meth != P.EXACT else None, omega=0.8)
        x, hist = pc.relax(A, b, np.zeros_like(b), 3)
        print(f"c{cfg} method {meth} m={db.size} hist {hist[0]:.3e} -> {hist[-1]:.3e}", flush=True)
    if cfg in (1, 2):
        pc = P.Preconditioner.create(A, pset, None, omega=1.0)
        _, rep = P.pcg(A, b, pc, tol=1e-6, max_iters=50)
        print(f"c{cfg} pcg {rep.iterations} it", flush=True)
        _, rep = P.gmres(A, b, pc, restart=10, tol=1e-6, max_iters=40)
        print(f"c{cfg} gmres {rep.iterations} it", flush=True)

# emulated 3-rank slab group, device sweeps (config 3 at 6^3)
import torch  # noqa: E402
slabs = [P.Problem.generate_slab(3, 6, r, 3) for r in range(3)]
sl = P.Slab.create(slabs, 0, 3, 27, None, omega=0.9)
bs, xs = [], []
for i in range(3):
    nloc = sl.info(i)["n_local"]
    bs.append(torch.rand(nloc, dtype=torch.float64, device="cuda"))
    xs.append(torch.zeros(nloc, dtype=torch.float64, device="cuda"))
sl.relax_device([t.data_ptr() for t in bs], [t.data_ptr() for t in xs], 2)
torch.cuda.synchronize()
print("slab group ok", flush=True)
