"""Interleaved A/B timing of sweep-kernel variants (env-selected) on one process.

Usage: python scripts/spmv_ab.py [config] [cells]
Variants are chosen through the PDB_* environment knobs read at launch time.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cells = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ps_size = {1: 9, 2: 25, 3: 27, 4: 22, 5: 192}[cfg]
prob = P.Problem.generate(cfg, cells)
A = prob.matrix()
ps = P.PatchSet.detect(A, ps_size)
db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size={3: 128, 4: 128}.get(cfg, 64), max_iters=5)
pc = P.Preconditioner.create(A, ps, db)
b = torch.from_numpy(prob.rhs()).cuda()
x = torch.zeros_like(b)
s = torch.cuda.current_stream().cuda_stream
variants = {
    "two_kernel": {"PDB_FUSE": "0"},
    "fused": {},
}
extra = [v for v in os.environ.get("AB_VARIANTS", "").split(";") if v]
for v in extra:  # NAME=K1:V1,K2:V2
    name, kv = v.split("=", 1)
    variants[name] = dict(p.split(":") for p in kv.split(","))
keys = {k for d in variants.values() for k in d}
res = {k: [] for k in variants}
for rnd in range(3):
    for name, env in variants.items():
        for k in keys:
            os.environ.pop(k, None)
        os.environ.update(env)
        P.relax_profile(pc, A, b.data_ptr(), x.data_ptr(), 20, stream=s)
        ms = P.relax_profile(pc, A, b.data_ptr(), x.data_ptr(), 200, stream=s)
        # whole sweeps back to back (kernels may overlap through PDL)
        pc.relax_device(A, b.data_ptr(), x.data_ptr(), 20, stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pc.relax_device(A, b.data_ptr(), x.data_ptr(), 200, stream=s)
        e1.record()
        torch.cuda.synchronize()
        res[name].append([round(v * 1e3, 1) for v in ms] + [round(e0.elapsed_time(e1) / 200 * 1e3, 1)])
n, nnz = prob.ndofs, prob.nnz
rb = 12 * nnz + 4 * (n + 1) + 24 * n
for name, r in res.items():
    best = min(x[0] for x in r)
    print(f"{name:12s} residual us {[x[0] for x in r]}  best {best} -> {rb / best / 1e3:.0f} GB/s; patch {[x[1] for x in r]} scatter {[x[2] for x in r]} SWEEP {[x[3] for x in r]}")
