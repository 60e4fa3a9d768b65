import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(3, 0)
A = prob.matrix()
ps = P.PatchSet.detect(A, 27)
eps = float(np.load('/root/repo/tests/golden/c3_l1_1.npz')['eps'])
for tiled in ("1", "0", "1"):
    os.environ["PDB_L1_TILED"] = tiled
    for rep in range(2):
        t = time.perf_counter(); db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps); t = time.perf_counter() - t
        print("tiled", tiled, "build", round(t, 4), "m", db.size, "pairs", db.work()["pair_evals"], flush=True)
    t = time.perf_counter(); dbb, e = P.Database.build_to_size(A, ps, 2358, 2884, P.GREEDY_L1); t = time.perf_counter() - t
    print("tiled", tiled, "bisect", round(t, 3), e, dbb.size, flush=True)
for k in (128,):
    for tiled in ("1", "0"):
        os.environ["PDB_L1_TILED"] = tiled
        P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=k, seed=42, max_iters=10)
        t = time.perf_counter(); db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=k, seed=42, max_iters=10); t = time.perf_counter() - t
        print("kmeans-entrywise tiled", tiled, round(t, 3), db.work(), flush=True)
