"""Config-5 exact setup at a reduced mesh (default 32^3: 32,768 x 192-DoF
patches): exact database (extract + LU) and exact preconditioner (streamed
extract + LU + inverse), best of 3, per LU kernel variant."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

cells = int(os.environ.get("CELLS", "32"))
prob = P.Problem.generate(5, cells)
A = prob.matrix()
ps = P.PatchSet.detect(A, 192)
P.Database.build(A, ps, P.EXACT)  # warm-up (pools, modules)
for variant in ("blocked", "cta"):
    for k in ("PDB_LU_CTA", "PDB_LU_WARP"):
        os.environ.pop(k, None)
    if variant == "cta":
        os.environ["PDB_LU_CTA"] = "1"
    tb, tp = [], []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        db = P.Database.build(A, ps, P.EXACT)
        torch.cuda.synchronize()
        tb.append(time.perf_counter() - t)
        del db
        t = time.perf_counter()
        pc = P.Preconditioner.create(A, ps, None, omega=1.0)
        torch.cuda.synchronize()
        tp.append(time.perf_counter() - t)
        del pc
    print(f"{variant}: exact database (extract + LU) {min(tb):.3f} s, exact preconditioner (streamed extract + LU + "
          f"inverse) {min(tp):.3f} s  (runs {[round(v, 3) for v in tb]} / {[round(v, 3) for v in tp]})", flush=True)
