"""One config-3 greedy-l1 build at the committed 1 % eps (for ncu launch lists)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

prob = P.Problem.generate(3, 0)
A = prob.matrix()
ps = P.PatchSet.detect(A, 27)
pct = int(os.environ.get("PCT", "1"))
eps = float(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"c3_l1_{pct}.npz"))["eps"])
t = time.perf_counter()
db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps)
print("build", time.perf_counter() - t, db.size)
