import sys, time, json, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from paper_2306_10025_b200 import patchdb as P
for cells, deg in [(60, 2), (120, 2)]:
    p = P.Problem.assemble(dict(cells=cells, degree=deg, coefficient=dict(kind="smooth")))
    A = p.matrix(); ps = P.PatchSet.detect(A, (deg+1)**2)
    pc = P.Preconditioner.create_combo(p, ps)
    plain = P.Preconditioner.create(A, ps)
    b = p.rhs()
    for name, pp in [("combo", pc), ("plain", plain), ("none", None)]:
        ts = []
        for _ in range(4):
            t = time.time(); x, rep = P.gmres(A, b, pp, max_iters=300); ts.append(time.time() - t)
        print(cells, deg, name, rep.iterations, [round(1e3*t, 2) for t in ts], "ms; per-iter us", round(1e6*min(ts)/max(rep.iterations,1), 1))
