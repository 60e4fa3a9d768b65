"""Config-5 compressed sweep at a reduced mesh (CELLS^3 cells, default 16), a
few sweeps only (for ncu of the TMA-staged 192-DoF tile apply): k-means
entrywise database with K entries, omega 1, SWEEPS sweeps on device-resident
b / x."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

cells = int(os.environ.get("CELLS", "16"))
k = int(os.environ.get("K", "256"))
sweeps = int(os.environ.get("SWEEPS", "3"))
prob = P.Problem.generate(5, cells)
A = prob.matrix()
ps = P.PatchSet.detect(A, 192)
db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=k, seed=42, max_iters=10)
pc = P.Preconditioner.create(A, ps, db, omega=1.0)
b = torch.from_numpy(prob.rhs()).cuda()
x = torch.zeros_like(b)
pc.relax_device(A, b.data_ptr(), x.data_ptr(), sweeps)
torch.cuda.synchronize()
print("ok", db.size, float(x.abs().max()))
