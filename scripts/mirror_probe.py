"""Config-3 residual through the half-storage (mirror) layout vs the plain
classed SELL copy: per-phase sweep times (relax_profile, CUDA events) for
kernel variants; greedy-l1 at the committed 1 % eps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

prob = P.Problem.generate(3, 0)
csr = prob.csr()
B = P.Matrix.from_csr(*csr)
os.environ["PDB_SELL_MIRROR"] = "1"
A = P.Matrix.from_csr(*csr)
del os.environ["PDB_SELL_MIRROR"]
print("mirror", A.mirror_info(), A.sell_info(), "plain", B.sell_info(), flush=True)
ps = P.PatchSet.detect(A, 27)
eps = float(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c3_l1_1.npz"))["eps"])
db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps)
b = torch.from_numpy(prob.rhs()).cuda()
x = torch.zeros_like(b)
x2 = torch.zeros_like(b)
pa = P.Preconditioner.create(A, ps, db, omega=1.0)
pb = P.Preconditioner.create(B, ps, db, omega=1.0)
pa.relax_device(A, b.data_ptr(), x.data_ptr(), 5)
pb.relax_device(B, b.data_ptr(), x2.data_ptr(), 5)
torch.cuda.synchronize()
print("iterates equal:", bool(torch.equal(x, x2)), flush=True)
for name, M, pc, ahead, u in (("plain", B, pb, "0", "8"), ("mirror", A, pa, "0", "8"), ("mirror", A, pa, "2048", "8"),
                              ("mirror", A, pa, "4096", "8"), ("mirror", A, pa, "0", "4"), ("mirror", A, pa, "2048", "4"),
                              ("mirror", A, pa, "4096", "4")):
    os.environ["PDB_MIRROR_AHEAD"] = ahead
    os.environ["PDB_MIRROR_U"] = u
    ms = P.relax_profile(pc, M, b.data_ptr(), x.data_ptr(), 50)
    print(f"{name:6s} ahead {ahead:>5s} U {u}: residual {ms[0]*1e3:7.1f} us  apply {ms[1]*1e3:6.1f}  "
          f"scatter {ms[2]*1e3:6.1f}", flush=True)
os.environ["PDB_MIRROR_AHEAD"] = "4096"
# whole sweep (no per-phase events)
for name, M, pc in (("plain", B, pb), ("mirror", A, pa)):
    os.environ["PDB_MIRROR_VARIANT"] = "0"
    os.environ["PDB_SELL_PF"] = "1"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pc.relax_device(M, b.data_ptr(), x.data_ptr(), 10)
    e0.record()
    pc.relax_device(M, b.data_ptr(), x.data_ptr(), 100)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 100 * 1e3:.1f} us per sweep", flush=True)
