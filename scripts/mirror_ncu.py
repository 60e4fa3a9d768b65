"""Config-3 sweeps through the half-storage layout only (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

prob = P.Problem.generate(3, 0)
os.environ["PDB_SELL_MIRROR"] = "1"
A = prob.matrix()
ps = P.PatchSet.detect(A, 27)
eps = float(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c3_l1_1.npz"))["eps"])
db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps)
pc = P.Preconditioner.create(A, ps, db, omega=1.0)
b = torch.from_numpy(prob.rhs()).cuda()
x = torch.zeros_like(b)
pc.relax_device(A, b.data_ptr(), x.data_ptr(), int(os.environ.get("SWEEPS", "3")))
torch.cuda.synchronize()
print("ok", A.mirror_info())
