"""One config-2 spectral k-means build (for profiling)."""
import os, sys, time
sys.path.insert(0, ".")
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(2, int(os.environ.get("CELLS", "0")))
A = prob.matrix(); ps = P.PatchSet.detect(A, 25)
t = time.perf_counter()
db = P.Database.build(A, ps, P.KMEANS_SPECTRAL, db_size=64, seed=42, max_iters=50)
print("build s", time.perf_counter() - t, db.work())
