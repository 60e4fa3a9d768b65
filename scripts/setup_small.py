"""Small setup run (config-2 generator at reduced size) for profiling the
compression kernels: python scripts/setup_small.py [cells] [method]."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
method = int(sys.argv[2]) if len(sys.argv) > 2 else P.KMEANS_SPECTRAL
prob = P.Problem.generate(2, cells)
A = prob.matrix()
ps = P.PatchSet.detect(A, 25)
t = time.perf_counter()
db = P.Database.build(A, ps, method, db_size=64, seed=42, max_iters=int(os.environ.get("ITERS", "50")))
dt = time.perf_counter() - t
w = db.work()
print(f"cells={cells} np={ps.count} m={db.size} setup {dt:.3f}s pairs={w['pair_evals']} power_iters={w['power_iters']} "
      f"-> {w['power_iters'] / dt / 1e6:.1f} M pair-iterations/s, {ps.count / dt:.0f} patches/s")
