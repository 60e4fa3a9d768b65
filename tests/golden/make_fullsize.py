"""Full-size golden fixtures from the compiled reference (oracle/_ref).

TEST INFRASTRUCTURE ONLY.  Runs here (where /root/reference exists and
oracle/_ref/libpdbref.so was built from it), takes hours, and writes small
fixtures under tests/golden/ that the `-m gpu` tests in
tests/test_fullsize_pins.py compare the GPU path with:

  c3_l1_{1,2,5}.npz   config 3 at 64^3 (262,144 x 27-DoF patches): the
                      reference's greedy_bisect_to_size (experiments.cpp:
                      168-204) for the BASELINE retentions 1/2/5 %
                      (targets 2,621 / 5,243 / 13,107, band [0.9t, 1.1t]),
                      greedy-l1 first match, threads = 1 (the serial scan
                      of compress.cpp:71-80): eps, size, creators, sha256 of
                      phi; then 10 sweeps of the reference smooth()
                      (precond.cpp:90-101) from x = 0 with omega 1 and the
                      residual history ||b - A x_k||_2, k = 0..10.
  c3_exact.npz        the same 10 sweeps with PatchPreconditioner::exact.
  c2_pcg_exact.npz    config 2, exact patch preconditioner: the oracle's PCG
                      restatement to 1e-8, iteration count and history.
  c2_kmeans.npz       config 2 at 256^2 (65,536 x 25-DoF patches):
                      KMEANS_SPECTRAL through the reference's
                      partitioned_build (capi.cpp:268-271), k = 64, seed 42,
                      max_iters 50: phi, sha256 of the representatives,
                      cluster sizes; then the oracle's PCG restatement
                      (orc_pcg, the reference has no CG) with
                      that database to 1e-8: iteration count and history.

    python tests/golden/make_fullsize.py c3 1      # one band per process
    python tests/golden/make_fullsize.py c3exact
    python tests/golden/make_fullsize.py c2 [threads]
    python tests/golden/make_fullsize.py c2pcg     # exact patches, PCG only
    python tests/golden/make_fullsize.py c2pcgfix  # PCG part of c2_kmeans.npz from its phi
    python tests/golden/make_fullsize.py c4 [threads]
    python tests/golden/make_fullsize.py c5 CELLS [threads]

  c4_kmeans.npz       config 4 at 512^2 (262,144 x 22-DoF Vanka patches):
                      KMEANS_ENTRYWISE through partitioned_build, k = 128,
                      seed 42, max_iters 50: phi, sha256 of representatives
                      and factors; then 10 reference smooth() sweeps (omega 1)
                      with that database: the residual history.
  c5_kmeans_<cells>.npz  config 5 (3D Q3 elasticity, 192-DoF patches) at
                      CELLS^3: KMEANS_ENTRYWISE k = 256, seed 42, max_iters
                      50, as c4, and 10 smooth() sweeps.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
from paper_2306_10025_b200 import patchdb as P  # noqa: E402

C3_TARGETS = {1: 2621, 2: 5243, 5: 13107}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_digest(csr) -> str:
    h = hashlib.sha256()
    for a in csr:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def history(rm, pc, b, sweeps, threads):
    """x_{k+1} = smooth(x_k) by the reference; ||b - A x_k|| after each."""
    x = np.zeros_like(b)
    hist = [float(np.linalg.norm(b - rm.spmv(x, threads)))]
    for _ in range(sweeps):
        x = pc.smooth(x, b, 1, threads)
        hist.append(float(np.linalg.norm(b - rm.spmv(x, threads))))
    return np.array(hist), x


def c3_setup():
    prob = P.Problem.generate(3, 0)
    csr = prob.csr()
    b = prob.rhs()
    ref = O.RefLib()
    rm = ref.matrix(csr)
    rps = rm.detect(27)
    return prob, csr, b, ref, rm, rps


def job_c3(pct: int):
    t = C3_TARGETS[pct]
    lo, hi = int(np.floor(0.9 * t)), int(np.ceil(1.1 * t))
    prob, csr, b, ref, rm, rps = c3_setup()
    log(f"c3 {pct}%: n={prob.ndofs} patches={rps.count} band=[{lo},{hi}]")
    t0 = time.time()
    db, eps = rps.bisect(rm, False, lo, hi, False, 1)
    tb = time.time() - t0
    phi = db.phi()
    m = db.size
    # creators: first patch of each entry in phi order (greedy appends the
    # unmatched patch itself, compress.cpp:91)
    _, first = np.unique(phi, return_index=True)
    creators = first[np.argsort(phi[first])]
    log(f"c3 {pct}%: eps={eps!r} m={m} bisect {tb:.0f} s")
    pc = rps.precond(rm, db, 1.0, 8)
    hist, x = history(rm, pc, b, 10, 8)
    np.savez_compressed(os.path.join(HERE, f"c3_l1_{pct}.npz"), csr_sha256=np.array(csr_digest(csr)),
                        rhs_sha256=np.array(sha(b)), target=np.array([lo, hi]), eps=np.array(eps), m=np.array(m),
                        creators=creators.astype(np.int64), phi_sha256=np.array(sha(phi.astype(np.int64))),
                        reps_sha256=np.array(sha(db.reps(27))), hist=hist, x10_sample=x[::997].copy(),
                        bisect_seconds=np.array(tb))
    log(f"c3 {pct}%: wrote; hist {hist[0]:.6e} -> {hist[-1]:.6e}")


def job_c3exact():
    prob, csr, b, ref, rm, rps = c3_setup()
    pc = rps.precond(rm, None, 1.0, 8)
    hist, x = history(rm, pc, b, 10, 8)
    np.savez_compressed(os.path.join(HERE, "c3_exact.npz"), csr_sha256=np.array(csr_digest(csr)),
                        rhs_sha256=np.array(sha(b)), hist=hist, x10_sample=x[::997].copy())
    log(f"c3 exact: hist {hist[0]:.6e} -> {hist[-1]:.6e}")


def job_c2(threads: int):
    prob = P.Problem.generate(2, 0)
    csr = prob.csr()
    b = prob.rhs()
    ref = O.RefLib()
    rm = ref.matrix(csr)
    rps = rm.detect(25)
    log(f"c2: n={prob.ndofs} patches={rps.count}")
    t0 = time.time()
    db = rps.build(rm, 4, db_size=64, seed=42, max_iters=50, threads=threads)  # PDB_METHOD_KMEANS_SPECTRAL
    tk = time.time() - t0
    phi = db.phi()
    reps = db.reps(25)
    lu, piv = db.factors(25)
    log(f"c2: k-means m={db.size} in {tk:.0f} s")
    np.savez_compressed(os.path.join(HERE, "c2_kmeans.npz"), csr_sha256=np.array(csr_digest(csr)),
                        rhs_sha256=np.array(sha(b)), m=np.array(db.size), phi=phi.astype(np.int32),
                        reps_sha256=np.array(sha(reps)), lu_sha256=np.array(sha(lu)), piv_sha256=np.array(sha(piv)),
                        sizes=np.bincount(phi, minlength=db.size), kmeans_seconds=np.array(tk))
    orc = O.Oracle()
    patches = rps.patches()
    w = rps.weights(prob.ndofs)
    t0 = time.time()
    _, rep = orc.pcg(csr, b, dict(patches=patches, weights=w, omega=1.0, lu=lu, piv=piv, phi=phi), tol=1e-8,
                     max_iters=20000)
    tp = time.time() - t0
    log(f"c2: pcg {rep['iterations']} iterations converged={rep['converged']} in {tp:.0f} s")
    d = dict(np.load(os.path.join(HERE, "c2_kmeans.npz")))
    d.update(pcg_iterations=np.array(rep["iterations"]), pcg_converged=np.array(rep["converged"]),
             pcg_history=rep["residual_history"], pcg_seconds=np.array(tp))
    np.savez_compressed(os.path.join(HERE, "c2_kmeans.npz"), **d)
    log("c2: wrote")


def job_c2pcg_exact():
    """Config 2, exact patch preconditioner (one LU per patch, the reference's
    exact_database), the oracle's PCG restatement to 1e-8 from x = 0."""
    prob = P.Problem.generate(2, 0)
    csr = prob.csr()
    b = prob.rhs()
    ref = O.RefLib()
    rm = ref.matrix(csr)
    rps = rm.detect(25)
    db = rps.build(rm, 0, threads=4)  # PDB_METHOD_EXACT
    lu, piv = db.factors(25)
    orc = O.Oracle()
    t0 = time.time()
    _, rep = orc.pcg(csr, b, dict(patches=rps.patches(), weights=rps.weights(prob.ndofs), omega=1.0, lu=lu, piv=piv,
                                  phi=None), tol=1e-8, max_iters=20000)
    tp = time.time() - t0
    log(f"c2 exact pcg: {rep['iterations']} iterations converged={rep['converged']} in {tp:.0f} s")
    np.savez_compressed(os.path.join(HERE, "c2_pcg_exact.npz"), csr_sha256=np.array(csr_digest(csr)),
                        rhs_sha256=np.array(sha(b)), pcg_iterations=np.array(rep["iterations"]),
                        pcg_converged=np.array(rep["converged"]), pcg_history=rep["residual_history"],
                        pcg_seconds=np.array(tp))


def job_c2pcg_from_phi():
    """Completes c2_kmeans.npz with the PCG part without re-running the
    3.2 h reference k-means: the final representatives are the in-order
    entrywise means of the final clusters (entrywise_mean_indexed,
    dense.cpp:211-223, after the last Lloyd update, compress.cpp:221-262),
    rebuilt here from the recorded phi and checked against the recorded
    sha256 of the reference's representatives, LU factors and pivots before
    the oracle's PCG restatement runs with them."""
    path = os.path.join(HERE, "c2_kmeans.npz")
    d = dict(np.load(path))
    prob = P.Problem.generate(2, 0)
    csr = prob.csr()
    b = prob.rhs()
    assert csr_digest(csr) == str(d["csr_sha256"]) and sha(b) == str(d["rhs_sha256"])
    orc = O.Oracle()
    patches, w = orc.detect(csr, 25)
    mats = orc.extract_all(csr, patches)
    phi = d["phi"].astype(np.int64)
    m = int(d["m"])
    reps = np.zeros((m, 25, 25))
    for j in range(m):
        members = np.flatnonzero(phi == j)  # ascending patch order
        acc = np.zeros((25, 25))
        for k in members:
            acc += mats[k]  # left fold, one entry at a time (elementwise numpy add)
        reps[j] = acc * (1.0 / float(len(members)))
    assert sha(reps) == str(d["reps_sha256"]), "rebuilt representatives differ from the reference's"
    lu = np.empty_like(reps)
    piv = np.empty((m, 25), np.int64)
    for j in range(m):
        lu[j], piv[j] = orc.lu_factor(reps[j])
    assert sha(lu) == str(d["lu_sha256"]) and sha(piv) == str(d["piv_sha256"])
    log(f"c2pcgfix: database rebuilt from phi, sha256 of reps / LU / pivots equal the reference's")
    t0 = time.time()
    _, rep = orc.pcg(csr, b, dict(patches=patches, weights=w, omega=1.0, lu=lu, piv=piv, phi=phi), tol=1e-8,
                     max_iters=20000)
    tp = time.time() - t0
    log(f"c2pcgfix: pcg {rep['iterations']} iterations converged={rep['converged']} in {tp:.0f} s")
    d.update(pcg_iterations=np.array(rep["iterations"]), pcg_converged=np.array(rep["converged"]),
             pcg_history=rep["residual_history"], pcg_seconds=np.array(tp))
    np.savez_compressed(path, **d)
    log("c2pcgfix: wrote")


def job_kmeans_entrywise(cfg: int, cells: int, ps: int, k: int, name: str, threads: int):
    """KMEANS_ENTRYWISE (capi.cpp:268-271 -> partitioned_build) at the given
    size, then 10 smooth() sweeps from x = 0 with omega 1."""
    prob = P.Problem.generate(cfg, cells)
    csr = prob.csr()
    b = prob.rhs()
    ref = O.RefLib()
    rm = ref.matrix(csr)
    rps = rm.detect(ps)
    log(f"{name}: n={prob.ndofs} nnz={len(csr[1])} patches={rps.count}")
    t0 = time.time()
    db = rps.build(rm, 3, db_size=k, seed=42, max_iters=50, threads=threads)  # PDB_METHOD_KMEANS_ENTRYWISE
    tk = time.time() - t0
    phi = db.phi()
    lu, piv = db.factors(ps)
    log(f"{name}: k-means m={db.size} in {tk:.0f} s")
    pc = rps.precond(rm, db, 1.0, threads)
    hist, x = history(rm, pc, b, 10, threads)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), csr_sha256=np.array(csr_digest(csr)),
                        rhs_sha256=np.array(sha(b)), m=np.array(db.size), phi=phi.astype(np.int32),
                        reps_sha256=np.array(sha(db.reps(ps))), lu_sha256=np.array(sha(lu)),
                        piv_sha256=np.array(sha(piv)), sizes=np.bincount(phi, minlength=db.size), hist=hist,
                        x10_sample=x[::997].copy(), kmeans_seconds=np.array(tk), cells=np.array(cells))
    log(f"{name}: wrote; hist {hist[0]:.6e} -> {hist[-1]:.6e}")


if __name__ == "__main__":
    job = sys.argv[1]
    if job == "c3":
        job_c3(int(sys.argv[2]))
    elif job == "c3exact":
        job_c3exact()
    elif job == "c2":
        job_c2(int(sys.argv[2]) if len(sys.argv) > 2 else 4)
    elif job == "c2pcg":
        job_c2pcg_exact()
    elif job == "c2pcgfix":
        job_c2pcg_from_phi()
    elif job == "c4":
        job_kmeans_entrywise(4, 0, 22, 128, "c4_kmeans", int(sys.argv[2]) if len(sys.argv) > 2 else 8)
    elif job == "c5":
        cells = int(sys.argv[2])
        job_kmeans_entrywise(5, cells, 192, 256, f"c5_kmeans_{cells}", int(sys.argv[3]) if len(sys.argv) > 3 else 8)
    else:
        raise SystemExit(__doc__)
