"""Greedy-spectral bisection timing (paper Experiment 1 sizes) with and without pruning."""
import json, os, sys, time
sys.path.insert(0, ".")
from paper_2306_10025_b200 import patchdb as P
for cells, deg, target in [(60, 2, 35), (60, 3, 35)]:
    p = P.Problem.assemble(dict(cells=cells, degree=deg, coefficient=dict(kind="smooth")))
    A = p.matrix(); ps = P.PatchSet.detect(A, (deg + 1) ** 2)
    lo, hi = int(0.9 * target), int(1.1 * target) + 1
    for prune in ("1", "0"):
        os.environ["PDB_GREEDY_PRUNE"] = prune
        t = time.perf_counter()
        db, eps = P.Database.build_to_size(A, ps, lo, hi, P.GREEDY_SPECTRAL)
        dt = time.perf_counter() - t
        print(json.dumps(dict(cells=cells, degree=deg, prune=prune, seconds=round(dt, 3), size=db.size, eps=eps,
                              **db.work(), phi_sum=int(db.phi().sum()))), flush=True)
