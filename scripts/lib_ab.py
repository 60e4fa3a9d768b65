"""Config-2 spectral k-means build with the library named by PDB_LIB_PATH:
warm timing (second of two builds) and a digest of phi / representatives,
for A/B runs of kernel build variants."""
import hashlib, json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2306_10025_b200 import patchdb as P
prob = P.Problem.generate(int(os.environ.get("CFG", "2")), int(os.environ.get("CELLS", "0")))
A = prob.matrix(); ps = P.PatchSet.detect(A, int(os.environ.get("PS", "25")))
for rep in range(2):
    t = time.perf_counter()
    db = P.Database.build(A, ps, P.KMEANS_SPECTRAL, db_size=int(os.environ.get("K", "64")), seed=42, max_iters=50)
    dt = time.perf_counter() - t
dig = hashlib.sha1(db.phi().tobytes() + db.representatives().tobytes()).hexdigest()[:16]
print(json.dumps(dict(lib=os.environ.get("PDB_LIB_PATH", "default"), seconds=round(dt, 3), digest=dig, **db.work())), flush=True)
