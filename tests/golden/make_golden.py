"""Regenerate tests/golden/*.npz from the compiled reference (oracle/_ref).

The reference ships no tests or golden vectors (proj/tests/CMakeLists.txt:1),
so the goldens are outputs of the unmodified reference library, compiled in
place by oracle/Makefile, on the repo's seeded config-1 input (and a reduced
config-3 input).  Run here (where /root/reference exists):

    python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
from paper_2306_10025_b200 import patchdb as P  # noqa: E402


def csr_digest(csr):
    h = hashlib.sha256()
    for a in csr:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def make_c1(ref):
    prob = P.Problem.generate(1)
    csr = prob.csr()
    b = prob.rhs()
    rm = ref.matrix(csr)
    rps = rm.detect(9)
    out = dict(csr_sha256=np.array(csr_digest(csr)), rhs=b, patches=rps.patches(), weights=rps.weights(len(b)))
    # size targeting (5% of 1024 patches: band 46-57) for both greedy flavours
    for spectral, tag in ((False, "l1"), (True, "spec")):
        db, eps = rps.bisect(rm, spectral, 46, 57)
        out[f"greedy_{tag}_eps"] = np.array(eps)
        out[f"greedy_{tag}_phi"] = db.phi()
        bm = rps.build(rm, 1 if spectral else 2, eps=eps, best_match=True)
        out[f"greedy_{tag}_best_phi"] = bm.phi()
    for method, tag in ((3, "entrywise"), (4, "spectral"), (5, "varmin")):
        db = rps.build(rm, method, db_size=51, seed=42, max_iters=50)
        out[f"kmeans_{tag}_phi"] = db.phi()
        out[f"kmeans_{tag}_reps_sha256"] = np.array(hashlib.sha256(db.reps(9).tobytes()).hexdigest())
    # relaxation: exact and compressed (greedy-l1 at the bisected eps), omega 0.8, 20 sweeps
    ex = rps.precond(rm, None, 0.8)
    x0 = np.zeros_like(b)
    out["relax_exact_x20"] = ex.smooth(x0, b, 20)
    db, _ = rps.bisect(rm, False, 46, 57)
    cp = rps.precond(rm, db, 0.8)
    out["relax_comp_x20"] = cp.smooth(x0, b, 20)
    # GMRES(20) with the exact patch preconditioner (omega 1)
    pc1 = rps.precond(rm, None, 1.0)
    x, rep = pc1.gmres(b)
    out["gmres_iterations"] = np.array(rep["iterations"])
    out["gmres_history"] = rep["residual_history"]
    out["gmres_x"] = x
    return out


def make_c3s(ref):
    prob = P.Problem.generate(3, 6)
    csr = prob.csr()
    rm = ref.matrix(csr)
    rps = rm.detect(27)
    mats = rps.extract(rm)
    out = dict(csr_sha256=np.array(csr_digest(csr)), patches=rps.patches(), weights=rps.weights(prob.ndofs))
    g = np.zeros(len(mats), np.int64)
    masks = np.zeros((len(mats), 27), np.uint8)
    import ctypes as C
    ng = C.c_int64()
    ref._check(ref.lib.refh_boundary_partition(len(mats), 27, mats.ctypes.data_as(C.POINTER(C.c_double)),
                                               g.ctypes.data_as(C.POINTER(C.c_int64)),
                                               masks.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(ng)))
    out["partition_of"] = g
    out["partition_count"] = np.array(ng.value)
    db, eps = rps.bisect(rm, False, 9, 13)
    out["greedy_l1_eps"] = np.array(eps)
    out["greedy_l1_phi"] = db.phi()
    return out


def main():
    ref = O.RefLib()
    np.savez_compressed(os.path.join(HERE, "c1_reference.npz"), **make_c1(ref))
    np.savez_compressed(os.path.join(HERE, "c3s_reference.npz"), **make_c3s(ref))
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
