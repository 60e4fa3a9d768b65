"""Probe: does an apply + scatter on a high-priority stream hide under a
concurrently running residual?  Prints per-sweep ms for the overlapped pair,
the residual alone and apply + scatter alone (config 2 by default)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2306_10025_b200 import patchdb as P

cfg = int(os.environ.get("CFG", "2"))
ps_size = {1: 9, 2: 25, 3: 27, 4: 22}[cfg]
prob = P.Problem.generate(cfg, int(os.environ.get("CELLS", "0")))
A = prob.matrix()
ps = P.PatchSet.detect(A, ps_size)
db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=64, seed=42, max_iters=10)
pc = P.Preconditioner.create(A, ps, db, omega=1.0)
b = torch.from_numpy(prob.rhs()).cuda()
x = torch.zeros_like(b)
os.environ["PDB_PROFILE_OVERLAP"] = "1"
for _ in range(3):
    ms = P.relax_profile(pc, A, b.data_ptr(), x.data_ptr(), 100)
    print(json.dumps({"cfg": cfg, "overlapped_ms": ms[0], "residual_ms": ms[1], "apply_scatter_ms": ms[2]}))
