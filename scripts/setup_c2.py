"""Config-2 spectral k-means setup timing with and without assignment pruning."""
import json, os, sys, time
sys.path.insert(0, ".")
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(2, int(os.environ.get("CELLS", "0")))
A = prob.matrix(); ps = P.PatchSet.detect(A, 25)
for prune in ("1", "0"):
    os.environ["PDB_KMEANS_PRUNE"] = prune
    t = time.perf_counter()
    db = P.Database.build(A, ps, P.KMEANS_SPECTRAL, db_size=64, seed=42, max_iters=50)
    dt = time.perf_counter() - t
    print(json.dumps(dict(prune=prune, seconds=round(dt, 3), **db.work(), phi_sum=int(db.phi().sum()))), flush=True)
