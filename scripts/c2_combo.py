"""BASELINE config 2 solved with the two-level method (patch term + coarse
correction, pdb_precond_create_combo) under GMRES(20) to 1e-8, against the
one-level preconditioner, and the reference's combo on the same CSR
(oracle/_ref, one thread) when REF=1.  One JSON line per variant."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from paper_2306_10025_b200 import patchdb as P  # noqa: E402
import oracle as O  # noqa: E402

cells = int(os.environ.get("CELLS", "0"))
prob = P.Problem.generate(2, cells)
A = prob.matrix()
ps = P.PatchSet.detect(A, 25)
b = prob.rhs()
n = prob.ndofs
C = int(round(((np.sqrt(n) - 1) / 4)))
variants = os.environ.get("VARIANTS", "entrywise,exact").split(",")
dbs = {}
t_db = {}
for v in variants:
    if v == "exact":
        dbs[v] = None
        continue
    method = {"entrywise": P.KMEANS_ENTRYWISE, "spectral": P.KMEANS_SPECTRAL}[v]
    t = time.perf_counter()
    dbs[v] = P.Database.build(A, ps, method, db_size=64, seed=42, max_iters=50)
    t_db[v] = time.perf_counter() - t
for name in variants:
    dbx = dbs[name]
    t = time.perf_counter()
    pc = P.Preconditioner.create_combo(prob, ps, dbx)
    t_pc = time.perf_counter() - t
    for _ in range(2):
        t = time.perf_counter()
        x, rep = P.gmres(A, b, pc, restart=20, tol=1e-8, max_iters=400)
        t_s = time.perf_counter() - t
    row = dict(config=2, n=n, precond=f"combo/{name}", nc=pc.coarse_size()[0], setup_s=round(t_pc, 3),
               db_build_s=round(t_db[name], 3) if dbx is not None else None, gmres_iters=rep.iterations,
               converged=rep.converged, solve_s=round(t_s, 4), us_per_iter=round(1e6 * t_s / max(rep.iterations, 1), 1))
    if os.environ.get("REF") == "1" and name != "spectral":
        ref = O.RefLib()
        rp = ref.problem_from_csr(prob.csr(), b, 2, C, 4)
        rA = rp.matrix()
        rps = rA.detect(25)
        rdb = None
        if dbx is not None:
            lu, piv = dbx.factors()
            rdb = ref.database(dbx.representatives(), lu, piv, dbx.phi())
        t = time.perf_counter()
        rpc = rp.combo(rA, rps, rdb)
        row["ref_setup_s"] = round(time.perf_counter() - t, 3)
        t = time.perf_counter()
        _, rr = rpc.gmres(b, restart=20, tol=1e-8, max_iters=400)
        row["ref_solve_s"] = round(time.perf_counter() - t, 3)
        row["ref_iters"] = rr["iterations"]
        h, hr = np.array(rep.residual_history), np.array(rr["residual_history"])
        row["history_max_rel_diff"] = float(np.max(np.abs(h - hr) / np.abs(hr))) if len(h) == len(hr) else None
    print(json.dumps(row), flush=True)
    pc1 = P.Preconditioner.create(A, ps, dbx)
    t = time.perf_counter()
    x, rep = P.gmres(A, b, pc1, restart=20, tol=1e-8, max_iters=400)
    print(json.dumps(dict(config=2, precond=f"one-level/{name}", gmres_iters=rep.iterations, converged=rep.converged,
                          final_rel=rep.final_relative_residual, solve_s=round(time.perf_counter() - t, 3))), flush=True)
