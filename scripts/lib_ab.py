"""Config-2 spectral k-means build with the library named by PDB_LIB_PATH:
REPS timed builds after one warm-up, and a digest of phi / representatives,
for A/B runs of kernel build variants and environment switches."""
import hashlib, json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(int(os.environ.get("CFG", "2")), int(os.environ.get("CELLS", "0")))
A = prob.matrix(); ps = P.PatchSet.detect(A, int(os.environ.get("PS", "25")))
times = []
for rep in range(1 + int(os.environ.get("REPS", "3"))):
    t = time.perf_counter()
    db = P.Database.build(A, ps, P.KMEANS_SPECTRAL, db_size=int(os.environ.get("K", "64")), seed=42, max_iters=50)
    times.append(round(time.perf_counter() - t, 3))
dig = hashlib.sha1(db.phi().tobytes() + db.representatives().tobytes()).hexdigest()[:16]
print(json.dumps(dict(lib=os.environ.get("PDB_LIB_PATH", "default"), tag=os.environ.get("TAG", ""), seconds=times,
                      digest=dig, **db.work())), flush=True)
