"""Config-3 headline sweep, a few sweeps only (for ncu): 64^3 Q2, greedy-l1 at
the committed 1 % eps (tests/golden/c3_l1_1.npz), omega 1, SWEEPS sweeps on
device-resident b / x."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

pct = int(os.environ.get("PCT", "1"))
sweeps = int(os.environ.get("SWEEPS", "5"))
prob = P.Problem.generate(3, 0)
A = prob.matrix()
ps = P.PatchSet.detect(A, 27)
eps = float(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"c3_l1_{pct}.npz"))["eps"])
db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps) if pct > 0 else None
pc = P.Preconditioner.create(A, ps, db, omega=1.0)
b = torch.from_numpy(prob.rhs()).cuda()
x = torch.zeros_like(b)
pc.relax_device(A, b.data_ptr(), x.data_ptr(), sweeps)
torch.cuda.synchronize()
print("ok", db.size if db else "exact", float(x.abs().max()))
