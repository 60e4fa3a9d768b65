"""Config-3 rank-local setup of a W-rank emulated slab group on one GPU
(pdb_slab_create_built, greedy-l1 at the committed 1 % eps): the whole
group's setup time, i.e. roughly W x one rank's, and the database size
(equal to the single-GPU build's)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2306_10025_b200 import patchdb as P
W = int(os.environ.get("W", "8"))
eps = float(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c3_l1_1.npz"))["eps"])
t = time.perf_counter()
slabs = [P.Problem.generate_slab(3, 0, r, W) for r in range(W)]
print(f"W={W} generate {time.perf_counter() - t:.2f} s", flush=True)
for rep in range(2):
    t = time.perf_counter()
    sl = P.Slab.create_built(slabs, 0, W, 27, P.GREEDY_L1, eps=eps, omega=1.0)
    dt = time.perf_counter() - t
    print(f"W={W} group setup {dt:.3f} s (per rank ~{dt / W * 1e3:.0f} ms), m={sl.database_size}", flush=True)
    sl = None
