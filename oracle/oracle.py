"""TEST INFRASTRUCTURE ONLY -- ctypes front-end to the two CPU checkers.

* ``Oracle``  -> lib/liboracle.so, the plain-C restatement (pdb_oracle.c).
* ``RefLib``  -> _ref/libpdbref.so, the unmodified reference sources compiled
  in place by oracle/Makefile plus ref_harness.cpp.  Absent on a machine
  where it was never built (the GPU box only has the prebuilt copy that
  travelled with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(HERE, "lib", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libpdbref.so")

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_P = C.c_void_p


def _dp(a):
    return None if a is None else a.ctypes.data_as(_D)


def _ip(a):
    return None if a is None else a.ctypes.data_as(_I64)


class CheckerError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"[{status}] {message}")
        self.status = status
        self.message = message


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """The C restatement.  CSR arrays are int64 (reference Index)."""

    def __init__(self, path: str = ORACLE_PATH):
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_lu_factor.argtypes = [C.c_int64, _D, _D, _I64]
        L.orc_lu_solve.argtypes = [C.c_int64, _D, _I64, _D, _D]
        L.orc_lu_solve_t.argtypes = [C.c_int64, _D, _I64, _D, _D]
        L.orc_spectral_distance.argtypes = [C.c_int64, _D, _D, _I64, C.POINTER(C.c_int)]
        L.orc_spectral_distance.restype = C.c_double
        L.orc_l1_distance.argtypes = [C.c_int64, _D, _D]
        L.orc_l1_distance.restype = C.c_double
        L.orc_spmv.argtypes = [C.c_int64, _I64, _I64, _D, _D, _D]
        L.orc_detect.argtypes = [C.c_int64, _I64, _I64, C.c_int64, _I64, C.POINTER(_I64), _D]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_extract_all.argtypes = [C.c_int64, _I64, _I64, _D, C.c_int64, C.c_int64, _I64, _D]
        L.orc_boundary_partition.argtypes = [C.c_int64, C.c_int64, _D, _I64, C.POINTER(C.c_uint8), _I64]
        L.orc_greedy.argtypes = [C.c_int64, C.c_int64, _D, C.c_double, C.c_int, C.c_int, C.c_int64, _I64, _I64, _D,
                                 _D, _I64, _I64, C.POINTER(C.c_int)]
        L.orc_split_budget.argtypes = [C.c_int64, C.c_int64, _I64, _I64]
        L.orc_partitioned_build.argtypes = [C.c_int64, C.c_int64, _D, C.c_int64, C.c_int, C.c_uint64, C.c_int, _I64,
                                            _D, _D, _I64, _I64]
        L.orc_kmeans.argtypes = L.orc_partitioned_build.argtypes
        L.orc_bootstrapped.argtypes = [C.c_int64, C.c_int64, _D, C.c_double, C.c_int, C.c_int, _I64, _D, _D, _I64,
                                       _I64]
        L.orc_greedy_bisect.argtypes = [C.c_int64, C.c_int64, _D, C.c_int, C.c_int64, C.c_int64, C.c_int, _I64, _I64,
                                        _D, _D, _I64, _I64, _D]
        L.orc_mt19937_64_first.argtypes = [C.c_uint64, C.c_int64]
        L.orc_mt19937_64_first.restype = C.c_uint64
        L.orc_precond_apply.argtypes = [C.c_int64, C.c_int64, C.c_int64, _I64, _D, C.c_double, _D, _I64, _I64, _D, _D]
        L.orc_relax.argtypes = [C.c_int64, _I64, _I64, _D, C.c_int64, C.c_int64, _I64, _D, C.c_double, _D, _I64,
                                _I64, _D, _D, C.c_int64, _D]
        L.orc_gmres.argtypes = [C.c_int64, _I64, _I64, _D, _D, C.c_int64, C.c_int64, _I64, _D, C.c_double, _D, _I64,
                                _I64, C.c_int, C.c_int64, C.c_double, C.c_int64, C.c_int, _D, _I64, _I64,
                                C.POINTER(C.c_int), _D, _D, _I64]
        L.orc_pcg.argtypes = [C.c_int64, _I64, _I64, _D, _D, C.c_int64, C.c_int64, _I64, _D, C.c_double, _D, _I64,
                              _I64, C.c_int, C.c_double, C.c_int64, _D, _I64, C.POINTER(C.c_int), _D, _I64]

    def _check(self, st):
        if st != 0:
            raise CheckerError(st, self.lib.orc_last_error().decode())

    # dense
    def lu_factor(self, a):
        a = _f64(a)
        n = a.shape[0]
        lu = np.empty_like(a)
        piv = np.empty(n, np.int64)
        self._check(self.lib.orc_lu_factor(n, _dp(a), _dp(lu), _ip(piv)))
        return lu, piv

    def lu_solve(self, lu, piv, rhs, transpose=False):
        lu, piv, rhs = _f64(lu), _i64(piv), _f64(rhs)
        out = np.empty_like(rhs)
        f = self.lib.orc_lu_solve_t if transpose else self.lib.orc_lu_solve
        f(lu.shape[0], _dp(lu), _ip(piv), _dp(rhs), _dp(out))
        return out

    def spectral_distance(self, a, lu, piv):
        a, lu, piv = _f64(a), _f64(lu), _i64(piv)
        it = C.c_int()
        d = self.lib.orc_spectral_distance(a.shape[0], _dp(a), _dp(lu), _ip(piv), C.byref(it))
        return d, it.value

    def l1_distance(self, a, b):
        a, b = _f64(a), _f64(b)
        return self.lib.orc_l1_distance(a.size, _dp(a), _dp(b))

    # sparse / patches
    def spmv(self, csr, x):
        rp, ci, v = csr
        x = _f64(x)
        y = np.empty(len(rp) - 1)
        self.lib.orc_spmv(len(rp) - 1, _ip(rp), _ip(ci), _dp(v), _dp(x), _dp(y))
        return y

    def detect(self, csr, ps):
        rp, ci, _ = csr
        n = len(rp) - 1
        npo = C.c_int64()
        out = _I64()
        w = np.empty(n)
        self._check(self.lib.orc_detect(n, _ip(rp), _ip(ci), ps, C.byref(npo), C.byref(out), _dp(w)))
        np_ = npo.value
        patches = np.ctypeslib.as_array(out, shape=(np_ * ps,)).copy().reshape(np_, ps)
        self.lib.orc_free(out)
        return patches, w

    def extract_all(self, csr, patches):
        rp, ci, v = csr
        patches = _i64(patches)
        np_, ps = patches.shape
        out = np.empty((np_, ps, ps))
        self._check(self.lib.orc_extract_all(len(rp) - 1, _ip(rp), _ip(ci), _dp(v), np_, ps, _ip(patches), _dp(out)))
        return out

    def boundary_partition(self, mats):
        mats = _f64(mats)
        np_, ps = mats.shape[0], mats.shape[1]
        g = np.empty(np_, np.int64)
        masks = np.zeros((np_, ps), np.uint8)
        ng = C.c_int64()
        self._check(self.lib.orc_boundary_partition(np_, ps, _dp(mats), _ip(g),
                                                    masks.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(ng)))
        return g, masks[:ng.value]

    # compression
    def _db_arrays(self, np_, ps):
        return (np.empty(np_, np.int64), np.empty((np_, ps, ps)), np.empty((np_, ps, ps)),
                np.empty((np_, ps), np.int64))

    def greedy(self, mats, eps, spectral=False, best_match=False, abort_above=-1):
        mats = _f64(mats)
        np_, ps = mats.shape[0], mats.shape[1]
        phi, reps, lu, piv = self._db_arrays(np_, ps)
        cre = np.empty(np_, np.int64)
        m = C.c_int64()
        ab = C.c_int()
        self._check(self.lib.orc_greedy(np_, ps, _dp(mats), eps, int(spectral), int(best_match), abort_above, _ip(phi),
                                        _ip(cre), _dp(reps), _dp(lu), _ip(piv), C.byref(m), C.byref(ab)))
        if ab.value:
            return None
        k = m.value
        return dict(phi=phi, creators=cre[:k], reps=reps[:k], lu=lu[:k], piv=piv[:k], m=k)

    def greedy_bisect(self, mats, target_lo, target_hi, spectral=False, best_match=False):
        mats = _f64(mats)
        np_, ps = mats.shape[0], mats.shape[1]
        phi, reps, lu, piv = self._db_arrays(np_, ps)
        cre = np.empty(np_, np.int64)
        m = C.c_int64()
        eps = C.c_double()
        self._check(self.lib.orc_greedy_bisect(np_, ps, _dp(mats), int(spectral), target_lo, target_hi,
                                               int(best_match), _ip(phi), _ip(cre), _dp(reps), _dp(lu), _ip(piv),
                                               C.byref(m), C.byref(eps)))
        k = m.value
        return dict(phi=phi, creators=cre[:k], reps=reps[:k], lu=lu[:k], piv=piv[:k], m=k, eps=eps.value)

    def partitioned_build(self, mats, m_p, variant, seed=42, max_iters=50):
        mats = _f64(mats)
        np_, ps = mats.shape[0], mats.shape[1]
        phi, reps, lu, piv = self._db_arrays(np_, ps)
        m = C.c_int64()
        self._check(self.lib.orc_partitioned_build(np_, ps, _dp(mats), m_p, variant, seed, max_iters, _ip(phi),
                                                   _dp(reps), _dp(lu), _ip(piv), C.byref(m)))
        k = m.value
        return dict(phi=phi, reps=reps[:k], lu=lu[:k], piv=piv[:k], m=k)

    def bootstrapped(self, mats, eps, variant=2, max_iters=50):
        mats = _f64(mats)
        np_, ps = mats.shape[0], mats.shape[1]
        phi, reps, lu, piv = self._db_arrays(np_, ps)
        m = C.c_int64()
        self._check(self.lib.orc_bootstrapped(np_, ps, _dp(mats), eps, variant, max_iters, _ip(phi), _dp(reps),
                                              _dp(lu), _ip(piv), C.byref(m)))
        k = m.value
        return dict(phi=phi, reps=reps[:k], lu=lu[:k], piv=piv[:k], m=k)

    def split_budget(self, m_p, sizes):
        sizes = _i64(sizes)
        out = np.empty(len(sizes), np.int64)
        self._check(self.lib.orc_split_budget(m_p, len(sizes), _ip(sizes), _ip(out)))
        return out

    def mt19937_64(self, seed, k):
        return self.lib.orc_mt19937_64_first(seed, k)

    # preconditioner / sweeps
    def precond_apply(self, patches, weights, omega, lu, piv, phi, r):
        patches, weights, lu, piv, r = _i64(patches), _f64(weights), _f64(lu), _i64(piv), _f64(r)
        phi = None if phi is None else _i64(phi)
        z = np.empty(len(weights))
        self.lib.orc_precond_apply(len(weights), patches.shape[0], patches.shape[1], _ip(patches), _dp(weights), omega,
                                   _dp(lu), _ip(piv), _ip(phi), _dp(r), _dp(z))
        return z

    def relax(self, csr, patches, weights, omega, lu, piv, phi, b, x, sweeps):
        rp, ci, v = csr
        patches, weights, lu, piv, b = _i64(patches), _f64(weights), _f64(lu), _i64(piv), _f64(b)
        phi = None if phi is None else _i64(phi)
        x = _f64(x).copy()
        hist = np.empty(sweeps + 1)
        self.lib.orc_relax(len(rp) - 1, _ip(rp), _ip(ci), _dp(v), patches.shape[0], patches.shape[1], _ip(patches),
                           _dp(weights), omega, _dp(lu), _ip(piv), _ip(phi), _dp(b), _dp(x), sweeps, _dp(hist))
        return x, hist

    def gmres(self, csr, b, pc=None, restart=20, tol=1e-8, max_iters=2000, left=False):
        rp, ci, v = csr
        b = _f64(b)
        n = len(rp) - 1
        x = np.empty(n)
        cap = max_iters + 64
        hist = np.empty(cap)
        hl = C.c_int64(cap)
        it, rs, cv, rr = C.c_int64(), C.c_int64(), C.c_int(), C.c_double()
        if pc is None:
            pc = dict(patches=np.zeros((0, 1), np.int64), weights=np.zeros(n), omega=1.0, lu=np.zeros(1),
                      piv=np.zeros(1, np.int64), phi=None)
            have = 0
        else:
            have = 1
        pt = _i64(pc["patches"])
        phi = None if pc["phi"] is None else _i64(pc["phi"])
        self._check(self.lib.orc_gmres(n, _ip(rp), _ip(ci), _dp(v), _dp(b), pt.shape[0], pt.shape[1], _ip(pt),
                                       _dp(_f64(pc["weights"])), pc["omega"], _dp(_f64(pc["lu"])),
                                       _ip(_i64(pc["piv"])), _ip(phi), have, restart, tol, max_iters, int(left),
                                       _dp(x), C.byref(it), C.byref(rs), C.byref(cv), C.byref(rr), _dp(hist),
                                       C.byref(hl)))
        return x, dict(iterations=it.value, restarts=rs.value, converged=bool(cv.value),
                       final_relative_residual=rr.value, residual_history=hist[:min(hl.value, cap)].copy())

    def pcg(self, csr, b, pc=None, tol=1e-8, max_iters=10000):
        rp, ci, v = csr
        b = _f64(b)
        n = len(rp) - 1
        x = np.empty(n)
        cap = max_iters + 2
        hist = np.empty(cap)
        hl = C.c_int64(cap)
        it, cv = C.c_int64(), C.c_int()
        have = pc is not None
        if pc is None:
            pc = dict(patches=np.zeros((0, 1), np.int64), weights=np.zeros(n), omega=1.0, lu=np.zeros(1),
                      piv=np.zeros(1, np.int64), phi=None)
        pt = _i64(pc["patches"])
        phi = None if pc["phi"] is None else _i64(pc["phi"])
        self._check(self.lib.orc_pcg(n, _ip(rp), _ip(ci), _dp(v), _dp(b), pt.shape[0], pt.shape[1], _ip(pt),
                                     _dp(_f64(pc["weights"])), pc["omega"], _dp(_f64(pc["lu"])), _ip(_i64(pc["piv"])),
                                     _ip(phi), int(have), tol, max_iters, _dp(x), C.byref(it), C.byref(cv), _dp(hist),
                                     C.byref(hl)))
        return x, dict(iterations=it.value, converged=bool(cv.value), residual_history=hist[:hl.value].copy())


class RefLib:
    """The compiled reference (unmodified sources + ref_harness.cpp)."""

    def __init__(self, path: str = REF_PATH):
        self.lib = C.CDLL(path)
        L = self.lib
        L.refh_last_error.restype = C.c_char_p
        L.refh_matrix_new.restype = _P
        L.refh_matrix_new.argtypes = [C.c_int64, _I64, _I64, _D]
        L.refh_matrix_free.argtypes = [_P]
        L.refh_spmv.argtypes = [_P, _D, _D, C.c_int]
        L.refh_detect.argtypes = [_P, C.c_int64, C.POINTER(_P)]
        for f in ("refh_ps_count", "refh_ps_size", "refh_db_size", "refh_db_n_patches", "refh_db_n_patterns",
                  "refh_matrix_n", "refh_matrix_nnz"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [_P]
        L.refh_ps_patches.argtypes = [_P, _I64]
        L.refh_ps_weights.argtypes = [_P, _D]
        L.refh_ps_free.argtypes = [_P]
        L.refh_ps_new.restype = _P
        L.refh_ps_new.argtypes = [C.c_int64, C.c_int64, C.c_int64, _I64]
        L.refh_extract_all.argtypes = [_P, _P, C.c_int, _D]
        L.refh_db_build.argtypes = [_P, _P, C.c_int, C.c_double, C.c_int64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(_P)]
        L.refh_db_greedy_capped.argtypes = [_P, _P, C.c_int, C.c_double, C.c_int64, C.c_int, C.c_int, C.POINTER(_P)]
        L.refh_db_bisect.argtypes = [_P, _P, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int, C.POINTER(_P), _D]
        L.refh_evaluate_objective.argtypes = [_P, _P, _P, C.c_double, C.c_int, _D]
        L.refh_compressibility_curve.argtypes = [_P, _P, C.c_int, _D, C.c_int64, C.c_int, _I64, _D]
        L.refh_db_eps.restype = C.c_double
        L.refh_db_eps.argtypes = [_P]
        L.refh_db_phi.argtypes = [_P, _I64]
        L.refh_db_reps.argtypes = [_P, _D]
        L.refh_db_factors.argtypes = [_P, _D, _I64]
        L.refh_db_patterns.argtypes = [_P, C.POINTER(C.c_uint8)]
        L.refh_db_method.argtypes = [_P, C.c_char_p, C.c_int64]
        L.refh_db_free.argtypes = [_P]
        L.refh_pc_new.argtypes = [_P, _P, _P, C.c_double, C.c_int, C.POINTER(_P)]
        L.refh_pc_apply.argtypes = [_P, _D, _D]
        L.refh_pc_free.argtypes = [_P]
        L.refh_smooth.argtypes = [_P, _P, _D, _D, C.c_int64, C.c_int]
        L.refh_gmres.argtypes = [_P, _D, _P, C.c_int64, C.c_double, C.c_int64, C.c_int, C.c_int, _D, _I64, _I64,
                                 C.POINTER(C.c_int), _D, _D, _I64]
        L.refh_lu_factor.argtypes = [C.c_int64, _D, _D, _I64]
        L.refh_lu_solve.argtypes = [C.c_int64, _D, _I64, _D, _D, C.c_int]
        L.refh_spectral_distance.argtypes = [C.c_int64, _D, _D, _D]
        L.refh_l1_distance.argtypes = [C.c_int64, _D, _D]
        L.refh_l1_distance.restype = C.c_double
        L.refh_split_budget.argtypes = [C.c_int64, C.c_int64, _I64, _I64]
        L.refh_boundary_partition.argtypes = [C.c_int64, C.c_int64, _D, _I64, C.POINTER(C.c_uint8), _I64]
        L.refh_assemble.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_int64, _D,
                                    C.c_int64, C.POINTER(_P), _D]
        L.refh_matrix_csr.argtypes = [_P, _I64, _I64, _D]
        L.refh_db_from_arrays.restype = _P
        L.refh_db_from_arrays.argtypes = [C.c_int64, C.c_int64, C.c_int64, _D, _D, _I64, _I64]
        L.refh_problem_assemble.argtypes = [C.c_char_p, C.POINTER(_P)]
        L.refh_problem_free.argtypes = [_P]
        for f in ("refh_problem_n", "refh_problem_nnz"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [_P]
        L.refh_problem_csr.argtypes = [_P, _I64, _I64, _D]
        L.refh_problem_rhs.argtypes = [_P, _D]
        L.refh_problem_exact.argtypes = [_P, _D]
        L.refh_problem_l2_error.argtypes = [_P, _D, _D]
        L.refh_problem_matrix.restype = _P
        L.refh_problem_matrix.argtypes = [_P]
        L.refh_coarse_sizes.argtypes = [_P, _I64, _I64, _I64, _I64]
        L.refh_coarse_csr.argtypes = [_P, _I64, _I64, _D, _I64, _I64, _D]
        L.refh_coarse_factor.argtypes = [_P, _I64, _I64, _D, _I64]
        L.refh_combo_new.argtypes = [_P, _P, _P, C.c_double, C.c_int, C.POINTER(_P)]
        L.refh_export_matrix.argtypes = [C.c_char_p, C.c_char_p]
        L.refh_read_mm.argtypes = [C.c_char_p, C.POINTER(_P)]
        L.refh_write_mm.argtypes = [_P, C.c_char_p]
        L.refh_problem_from_csr.restype = _P
        L.refh_problem_from_csr.argtypes = [C.c_int64, _I64, _I64, _D, _D, C.c_int, C.c_int64, C.c_int]

    def read_matrix_market(self, path: str):
        """read_matrix_market (matrix_market.cpp:29-91): CSR arrays, or CheckerError."""
        out = _P()
        self._check(self.lib.refh_read_mm(path.encode(), C.byref(out)))
        m = out.value
        n, nnz = self.lib.refh_matrix_n(m), self.lib.refh_matrix_nnz(m)
        rp, ci, v = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        self.lib.refh_matrix_csr(m, _ip(rp), _ip(ci), _dp(v))
        self.lib.refh_matrix_free(m)
        return rp, ci, v

    def write_matrix_market(self, csr, path: str):
        m = self.matrix(csr)
        self._check(self.lib.refh_write_mm(m.ptr, path.encode()))

    def problem_from_csr(self, csr, rhs, dim, cells, degree):
        rp, ci, v = (_i64(csr[0]), _i64(csr[1]), _f64(csr[2]))
        return RefProblem(self, self.lib.refh_problem_from_csr(len(rp) - 1, _ip(rp), _ip(ci), _dp(v), _dp(_f64(rhs)),
                                                               dim, cells, degree))

    def export_matrix(self, config_json: str, path: str):
        self._check(self.lib.refh_export_matrix(config_json.encode(), path.encode()))

    def problem(self, config_json: str = ""):
        """pdb_problem_assemble's recipe on the reference (capi.cpp:169-179)."""
        out = _P()
        self._check(self.lib.refh_problem_assemble(config_json.encode(), C.byref(out)))
        return RefProblem(self, out.value)

    def database(self, reps, lu, piv, phi):
        reps, lu, piv, phi = _f64(reps), _f64(lu), _i64(piv), _i64(phi)
        m, ps = reps.shape[0], reps.shape[1]
        return RefDatabase(self, self.lib.refh_db_from_arrays(m, ps, len(phi), _dp(reps), _dp(lu), _ip(piv),
                                                             _ip(phi)))

    def _check(self, st):
        if st != 0:
            raise CheckerError(st, self.lib.refh_last_error().decode())

    def matrix(self, csr):
        rp, ci, v = _i64(csr[0]), _i64(csr[1]), _f64(csr[2])
        return RefMatrix(self, self.lib.refh_matrix_new(len(rp) - 1, _ip(rp), _ip(ci), _dp(v)))

    def lu_factor(self, a):
        a = _f64(a)
        n = a.shape[0]
        lu = np.empty_like(a)
        piv = np.empty(n, np.int64)
        self._check(self.lib.refh_lu_factor(n, _dp(a), _dp(lu), _ip(piv)))
        return lu, piv

    def lu_solve(self, lu, piv, rhs, transpose=False):
        lu, piv, rhs = _f64(lu), _i64(piv), _f64(rhs)
        out = np.empty_like(rhs)
        self._check(self.lib.refh_lu_solve(lu.shape[0], _dp(lu), _ip(piv), _dp(rhs), _dp(out), int(transpose)))
        return out

    def spectral_distance(self, a, b):
        a, b = _f64(a), _f64(b)
        d = C.c_double()
        self._check(self.lib.refh_spectral_distance(a.shape[0], _dp(a), _dp(b), C.byref(d)))
        return d.value

    def l1_distance(self, a, b):
        a, b = _f64(a), _f64(b)
        return self.lib.refh_l1_distance(a.shape[0], _dp(a), _dp(b))

    def split_budget(self, m_p, sizes):
        sizes = _i64(sizes)
        out = np.empty(len(sizes), np.int64)
        self._check(self.lib.refh_split_budget(m_p, len(sizes), _ip(sizes), _ip(out)))
        return out

    def assemble(self, dim, cells, degree, coeff_kind=0, value=1.0, blocks=(4, 4), block_values=None):
        bv = _f64(block_values) if block_values is not None else np.zeros(1)
        m = _P()
        self._check(self.lib.refh_assemble(dim, cells, degree, coeff_kind, value, blocks[0], blocks[1], _dp(bv),
                                           0 if block_values is None else len(bv), C.byref(m), None))
        n, nnz = self.lib.refh_matrix_n(m), self.lib.refh_matrix_nnz(m)
        rp, ci, v = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        self.lib.refh_matrix_csr(m, _ip(rp), _ip(ci), _dp(v))
        self.lib.refh_matrix_free(m)
        return rp, ci, v


class RefMatrix:
    def __init__(self, ref: RefLib, ptr):
        self.ref, self.ptr, self.L = ref, ptr, ref.lib

    def __del__(self):
        try:
            self.L.refh_matrix_free(self.ptr)
        except Exception:
            pass

    def spmv(self, x, threads=1):
        x = _f64(x)
        y = np.empty_like(x)
        self.ref._check(self.L.refh_spmv(self.ptr, _dp(x), _dp(y), threads))
        return y

    def detect(self, ps):
        out = _P()
        self.ref._check(self.L.refh_detect(self.ptr, ps, C.byref(out)))
        return RefPatchSet(self.ref, out.value)

    def patchset(self, n, patches):
        patches = _i64(patches)
        return RefPatchSet(self.ref, self.L.refh_ps_new(n, patches.shape[0], patches.shape[1], _ip(patches)))


class RefPatchSet:
    def __init__(self, ref: RefLib, ptr):
        self.ref, self.ptr, self.L = ref, ptr, ref.lib

    def __del__(self):
        try:
            self.L.refh_ps_free(self.ptr)
        except Exception:
            pass

    @property
    def count(self):
        return self.L.refh_ps_count(self.ptr)

    @property
    def patch_size(self):
        return self.L.refh_ps_size(self.ptr)

    def patches(self):
        out = np.empty((self.count, self.patch_size), np.int64)
        self.L.refh_ps_patches(self.ptr, _ip(out))
        return out

    def weights(self, n):
        out = np.empty(n)
        self.L.refh_ps_weights(self.ptr, _dp(out))
        return out

    def extract(self, m: RefMatrix, threads=1):
        out = np.empty((self.count, self.patch_size, self.patch_size))
        self.ref._check(self.L.refh_extract_all(m.ptr, self.ptr, threads, _dp(out)))
        return out

    def build(self, m: RefMatrix, method, eps=1e-7, db_size=0, seed=42, max_iters=50, best_match=False, threads=1):
        out = _P()
        self.ref._check(self.L.refh_db_build(m.ptr, self.ptr, method, eps, db_size, seed, max_iters, int(best_match),
                                             threads, C.byref(out)))
        return RefDatabase(self.ref, out.value)

    def greedy_capped(self, m: RefMatrix, spectral, eps, abort_above, best_match=False, threads=1):
        out = _P()
        self.ref._check(self.L.refh_db_greedy_capped(m.ptr, self.ptr, int(spectral), eps, abort_above,
                                                     int(best_match), threads, C.byref(out)))
        return None if not out.value else RefDatabase(self.ref, out.value)

    def bisect(self, m: RefMatrix, spectral, lo, hi, best_match=False, threads=1):
        out = _P()
        eps = C.c_double()
        self.ref._check(self.L.refh_db_bisect(m.ptr, self.ptr, int(spectral), lo, hi, int(best_match), threads,
                                              C.byref(out), C.byref(eps)))
        return RefDatabase(self.ref, out.value), eps.value

    def objective(self, m: RefMatrix, db, beta, threads=1):
        """evaluate_objective (compress.cpp:423-440)."""
        out = C.c_double()
        self.ref._check(self.L.refh_evaluate_objective(m.ptr, self.ptr, db.ptr, beta, threads, C.byref(out)))
        return out.value

    def curve(self, m: RefMatrix, spectral, grid, threads=1):
        """compressibility_curve (compress.cpp:442-456): [(eps, db_size, ratio)]."""
        g = np.ascontiguousarray(grid, dtype=np.float64)
        sizes = np.zeros(len(g), np.int64)
        ratios = np.zeros(len(g))
        self.ref._check(self.L.refh_compressibility_curve(m.ptr, self.ptr, int(spectral), _dp(g), len(g), threads,
                                                          _ip(sizes), _dp(ratios)))
        return [(float(e), int(n), float(r)) for e, n, r in zip(g, sizes, ratios)]

    def precond(self, m: RefMatrix, db=None, omega=1.0, threads=1):
        out = _P()
        self.ref._check(self.L.refh_pc_new(m.ptr, self.ptr, None if db is None else db.ptr, omega, threads,
                                           C.byref(out)))
        return RefPrecond(self.ref, out.value, m)


class RefDatabase:
    def __init__(self, ref: RefLib, ptr):
        self.ref, self.ptr, self.L = ref, ptr, ref.lib

    def __del__(self):
        try:
            self.L.refh_db_free(self.ptr)
        except Exception:
            pass

    @property
    def size(self):
        return self.L.refh_db_size(self.ptr)

    @property
    def n_patches(self):
        return self.L.refh_db_n_patches(self.ptr)

    @property
    def eps(self):
        return self.L.refh_db_eps(self.ptr)

    def phi(self):
        out = np.empty(self.n_patches, np.int64)
        self.L.refh_db_phi(self.ptr, _ip(out))
        return out

    def reps(self, ps):
        out = np.empty((self.size, ps, ps))
        self.L.refh_db_reps(self.ptr, _dp(out))
        return out

    def factors(self, ps):
        lu = np.empty((self.size, ps, ps))
        piv = np.empty((self.size, ps), np.int64)
        self.L.refh_db_factors(self.ptr, _dp(lu), _ip(piv))
        return lu, piv

    def method(self):
        buf = C.create_string_buffer(128)
        self.L.refh_db_method(self.ptr, buf, 128)
        return buf.value.decode()


class RefProblem:
    """Reference DiscreteProblem (fem.hpp:55-61) with its coarse space."""

    def __init__(self, ref: RefLib, ptr):
        self.ref, self.ptr, self.L = ref, ptr, ref.lib

    def __del__(self):
        try:
            self.L.refh_problem_free(self.ptr)
        except Exception:
            pass

    @property
    def n(self):
        return self.L.refh_problem_n(self.ptr)

    def csr(self):
        n, nnz = self.n, self.L.refh_problem_nnz(self.ptr)
        rp, ci, v = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        self.L.refh_problem_csr(self.ptr, _ip(rp), _ip(ci), _dp(v))
        return rp, ci, v

    def rhs(self):
        out = np.empty(self.n)
        self.L.refh_problem_rhs(self.ptr, _dp(out))
        return out

    def exact(self):
        out = np.empty(self.n)
        self.L.refh_problem_exact(self.ptr, _dp(out))
        return out

    def l2_error(self, u):
        out = np.zeros(1)
        self.ref._check(self.L.refh_problem_l2_error(self.ptr, _dp(_f64(u)), _dp(out)))
        return float(out[0])

    def matrix(self) -> "RefMatrix":
        return RefMatrix(self.ref, self.L.refh_problem_matrix(self.ptr))

    def coarse(self):
        """(P0 csr, R0 A P0 csr) as int64/fp64 arrays (fem.cpp:433-479)."""
        sz = np.zeros(4, np.int64)
        self.ref._check(self.L.refh_coarse_sizes(self.ptr, _ip(sz[0:]), _ip(sz[1:]), _ip(sz[2:]), _ip(sz[3:])))
        fine_n, nc, pnnz, cnnz = (int(v) for v in sz)
        p_rp, p_ci, p_v = np.empty(fine_n + 1, np.int64), np.empty(pnnz, np.int64), np.empty(pnnz)
        c_rp, c_ci, c_v = np.empty(nc + 1, np.int64), np.empty(cnnz, np.int64), np.empty(cnnz)
        self.ref._check(self.L.refh_coarse_csr(self.ptr, _ip(p_rp), _ip(p_ci), _dp(p_v), _ip(c_rp), _ip(c_ci),
                                               _dp(c_v)))
        return (p_rp, p_ci, p_v), (c_rp, c_ci, c_v)

    def coarse_factor(self):
        """band_factor(R0 A P0): (kl, ku, ab[(2kl+ku+1), n], ipiv[n])."""
        kk = np.zeros(2, np.int64)
        self.ref._check(self.L.refh_coarse_factor(self.ptr, _ip(kk[0:]), _ip(kk[1:]), None, None))
        kl, ku = int(kk[0]), int(kk[1])
        nc = self.coarse()[1][0].shape[0] - 1
        ab, ipiv = np.empty((2 * kl + ku + 1, nc)), np.empty(nc, np.int64)
        self.ref._check(self.L.refh_coarse_factor(self.ptr, _ip(kk[0:]), _ip(kk[1:]), _dp(ab), _ip(ipiv)))
        return kl, ku, ab, ipiv

    def combo(self, m: "RefMatrix", ps: "RefPatchSet", db=None, omega=1.0, threads=1):
        out = _P()
        self.ref._check(self.L.refh_combo_new(self.ptr, ps.ptr, None if db is None else db.ptr, omega, threads,
                                              C.byref(out)))
        return RefPrecond(self.ref, out.value, m)


class RefPrecond:
    def __init__(self, ref: RefLib, ptr, m: RefMatrix):
        self.ref, self.ptr, self.L, self.m = ref, ptr, ref.lib, m

    def __del__(self):
        try:
            self.L.refh_pc_free(self.ptr)
        except Exception:
            pass

    def apply(self, r):
        r = _f64(r)
        z = np.empty_like(r)
        self.ref._check(self.L.refh_pc_apply(self.ptr, _dp(r), _dp(z)))
        return z

    def smooth(self, x, b, sweeps=1, threads=1):
        x = _f64(x).copy()
        b = _f64(b)
        self.ref._check(self.L.refh_smooth(self.ptr, self.m.ptr, _dp(x), _dp(b), sweeps, threads))
        return x

    def gmres(self, b, restart=20, tol=1e-8, max_iters=2000, left=False, threads=1):
        b = _f64(b)
        x = np.empty_like(b)
        cap = max_iters + 64
        hist = np.empty(cap)
        hl = C.c_int64(cap)
        it, rs, cv, rr = C.c_int64(), C.c_int64(), C.c_int(), C.c_double()
        self.ref._check(self.L.refh_gmres(self.m.ptr, _dp(b), self.ptr, restart, tol, max_iters, int(left), threads,
                                          _dp(x), C.byref(it), C.byref(rs), C.byref(cv), C.byref(rr), _dp(hist),
                                          C.byref(hl)))
        return x, dict(iterations=it.value, restarts=rs.value, converged=bool(cv.value),
                       final_relative_residual=rr.value, residual_history=hist[:min(hl.value, cap)].copy())


def have_ref() -> bool:
    return os.path.exists(REF_PATH)
