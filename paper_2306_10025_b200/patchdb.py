"""Python mirror of the patchdb C-ABI, backed by the B200 library.

Thin ctypes bindings over ``lib/libpatchdb.so.0`` (built from ``csrc/``).
The classes mirror the reference handles one-to-one (``pdb_matrix``,
``pdb_patchset``, ``pdb_database``, ``pdb_precond``, ``pdb_report``; see
/root/reference/proj/include/patchdb/patchdb.h) and raise :class:`PatchdbError`
with the reference status code and message whenever a call returns non-OK.

There is no fallback: if the shared library is missing this module fails
to import, and on a machine without an sm_100 GPU every compute call raises
``PatchdbError(PDB_ERR_INTERNAL, "CUDA device unavailable ...")``.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDB_LIB_PATH") or os.path.join(_HERE, "lib", "libpatchdb.so.0")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(no CPU fallback exists)")

_lib = C.CDLL(LIB_PATH)

# ---- status codes (patchdb.h:25-41) -------------------------------------
PDB_OK = 0
PDB_ERR_INVALID_ARGUMENT = 1
PDB_ERR_DIMENSION_MISMATCH = 2
PDB_ERR_SINGULAR_MATRIX = 3
PDB_ERR_INDEX_OUT_OF_RANGE = 4
PDB_ERR_DUPLICATE_INDEX = 5
PDB_ERR_PARSE = 6
PDB_ERR_NON_SQUARE_MATRIX = 7
PDB_ERR_NO_PATCHES_FOUND = 8
PDB_ERR_EMPTY_CLUSTER = 9
PDB_ERR_BUDGET_TOO_SMALL = 10
PDB_ERR_INVALID_DEGREE = 11
PDB_ERR_NON_POSITIVE_COEFFICIENT = 12
PDB_ERR_IO = 13
PDB_ERR_INTERNAL = 14

# ---- methods (patchdb.h:88-96) -------------------------------------------
EXACT, GREEDY_SPECTRAL, GREEDY_L1, KMEANS_ENTRYWISE, KMEANS_SPECTRAL, KMEANS_VARMIN, BOOTSTRAP = range(7)


class PatchdbError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status
        self.message = message


class CompressOptions(C.Structure):
    """pdb_compress_options: 48 bytes, offsets 0/8/16/24/32/36/40 (patchdb.h:98-106)."""
    _fields_ = [("method", C.c_int), ("eps", C.c_double), ("db_size", C.c_int64), ("seed", C.c_uint64),
                ("max_iters", C.c_int), ("best_match", C.c_int), ("threads", C.c_int)]


class GmresOptions(C.Structure):
    """pdb_gmres_options: 32 bytes, offsets 0/8/16/24/28 (patchdb.h:134-140)."""
    _fields_ = [("restart", C.c_int64), ("tol", C.c_double), ("max_iters", C.c_int64), ("left_precond", C.c_int),
                ("threads", C.c_int)]


class GenOptions(C.Structure):
    _fields_ = [("physics", C.c_int), ("dim", C.c_int), ("degree", C.c_int), ("bc_mode", C.c_int),
                ("cells", C.c_int64), ("jitter", C.c_double), ("seed", C.c_uint64), ("coeff_kind", C.c_int),
                ("n_levels", C.c_int), ("coeff_value", C.c_double), ("block_cells", C.c_int64),
                ("levels", C.c_double * 8), ("threads", C.c_int), ("reserved", C.c_int),
                ("poisson_ratio", C.c_double)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


# Every symbol of include/patchdb/patchdb.h.
_sig("pdb_status_string", C.c_char_p, C.c_int)
_sig("pdb_last_error", C.c_char_p)
_sig("pdb_build_info", C.c_char_p)
_sig("pdb_matrix_read_matrix_market", C.c_int, C.c_char_p, C.POINTER(_P))
_sig("pdb_matrix_write_matrix_market", C.c_int, _P, C.c_char_p)
_sig("pdb_matrix_rows", C.c_int64, _P)
_sig("pdb_matrix_nnz", C.c_int64, _P)
_sig("pdb_matrix_spmv", C.c_int, _P, _D, _D)
_sig("pdb_matrix_spmv_device", C.c_int, _P, C.c_void_p, C.c_void_p, C.c_void_p)
_sig("pdb_matrix_free", None, _P)
_sig("pdb_matrix_from_csr", C.c_int, C.c_int64, _I64, _I64, _D, C.POINTER(_P))
_sig("pdb_matrix_sell_info", C.c_int, _P, _I64)
_sig("pdb_matrix_mirror_info", C.c_int, _P, _I64, C.POINTER(C.c_char_p))
_sig("pdb_debug_mirror_check", C.c_int, C.c_int64, _I64, _I64, _D, _D, _D, _I64)
_sig("pdb_matrix_csr", C.c_int, _P, _I64, _I64, _D)
_sig("pdb_problem_assemble", C.c_int, C.c_char_p, C.POINTER(_P))
_sig("pdb_problem_ndofs", C.c_int64, _P)
_sig("pdb_problem_nnz", C.c_int64, _P)
_sig("pdb_problem_matrix", C.c_int, _P, C.POINTER(_P))
_sig("pdb_problem_rhs", C.c_int, _P, _D)
_sig("pdb_problem_csr", C.c_int, _P, _I64, _I64, _D)
_sig("pdb_problem_exact_solution", C.c_int, _P, _D)
_sig("pdb_problem_l2_error", C.c_int, _P, _D, _D)
_sig("pdb_problem_free", None, _P)
_sig("pdb_gen_options_init", None, C.POINTER(GenOptions))
_sig("pdb_gen_options_config", C.c_int, C.c_int, C.c_int64, C.POINTER(GenOptions))
_sig("pdb_problem_generate", C.c_int, C.POINTER(GenOptions), C.POINTER(_P))
_sig("pdb_problem_generate_slab", C.c_int, C.POINTER(GenOptions), C.c_int, C.c_int, C.POINTER(_P))
_sig("pdb_problem_rows_global", C.c_int64, _P)
_sig("pdb_problem_row_range_count", C.c_int64, _P)
_sig("pdb_problem_row_ranges", C.c_int, _P, _I64)
_sig("pdb_patchset_detect", C.c_int, _P, C.c_int64, C.POINTER(_P))
_sig("pdb_patchset_count", C.c_int64, _P)
_sig("pdb_patchset_patch_size", C.c_int64, _P)
_sig("pdb_patchset_rows", C.c_int64, _P)
_sig("pdb_patchset_write_json", C.c_int, _P, C.c_char_p)
_sig("pdb_patchset_patches", C.c_int, _P, _I64)
_sig("pdb_patchset_weights", C.c_int, _P, _D)
_sig("pdb_patchset_extract", C.c_int, _P, _P, _D)
_sig("pdb_patchset_free", None, _P)
_sig("pdb_compress_options_init", None, C.POINTER(CompressOptions))
_sig("pdb_database_build", C.c_int, _P, _P, C.POINTER(CompressOptions), C.POINTER(_P))
_sig("pdb_database_build_to_size", C.c_int, _P, _P, C.POINTER(CompressOptions), C.c_int64, C.c_int64,
     C.POINTER(_P), _D)
_sig("pdb_database_objective", C.c_int, _P, _P, _P, C.c_double, _D)
_sig("pdb_compressibility_curve", C.c_int, _P, _P, C.c_int, _D, C.c_int64, _I64, _D)
_sig("pdb_database_size", C.c_int64, _P)
_sig("pdb_database_n_patches", C.c_int64, _P)
_sig("pdb_database_patch_size", C.c_int64, _P)
_sig("pdb_database_eps", C.c_double, _P)
_sig("pdb_database_phi", C.c_int, _P, _I64)
_sig("pdb_database_representatives", C.c_int, _P, _D)
_sig("pdb_database_factors", C.c_int, _P, _D, _I64)
_sig("pdb_database_work", C.c_int, _P, _I64, _I64, _I64)
_sig("pdb_database_export", C.c_int, _P, C.c_char_p, C.c_char_p)
_sig("pdb_database_import", C.c_int, C.c_char_p, C.c_char_p, C.POINTER(_P))
_sig("pdb_database_free", None, _P)
_sig("pdb_precond_create", C.c_int, _P, _P, _P, C.c_double, C.c_int, C.POINTER(_P))
_sig("pdb_precond_create_combo", C.c_int, _P, _P, _P, C.c_double, C.c_int, C.POINTER(_P))
_sig("pdb_precond_apply", C.c_int, _P, _D, _D)
_sig("pdb_precond_apply_device", C.c_int, _P, C.c_void_p, C.c_void_p, C.c_void_p)
_sig("pdb_relax", C.c_int, _P, _P, _D, _D, C.c_int64, _D)
_sig("pdb_relax_device", C.c_int, _P, _P, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)
_sig("pdb_precond_free", None, _P)
_sig("pdb_gmres_options_init", None, C.POINTER(GmresOptions))
_sig("pdb_gmres_solve", C.c_int, _P, _D, _P, C.POINTER(GmresOptions), _D, C.POINTER(_P))
_sig("pdb_pcg_solve", C.c_int, _P, _D, _P, C.c_double, C.c_int64, _D, C.POINTER(_P))
_sig("pdb_report_iterations", C.c_int64, _P)
_sig("pdb_report_restarts", C.c_int64, _P)
_sig("pdb_report_converged", C.c_int, _P)
_sig("pdb_report_final_relative_residual", C.c_double, _P)
_sig("pdb_report_residual_history_size", C.c_int64, _P)
_sig("pdb_report_residual_history", C.c_int, _P, _D)
_sig("pdb_report_free", None, _P)
_sig("pdb_precond_coarse_size", C.c_int, _P, _I64, _I64, _I64)
_sig("pdb_precond_coarse_factor", C.c_int, _P, _D, _I64)
_sig("pdb_run_experiment", C.c_int, C.c_char_p, C.c_char_p)
_sig("pdb_run_analyze", C.c_int, C.c_char_p, C.c_char_p, C.c_char_p)
_sig("pdb_run_benchmark", C.c_int, C.c_char_p, C.c_char_p)
_sig("pdb_export_matrix", C.c_int, C.c_char_p, C.c_char_p)

lib = _lib


def _check(status: int) -> None:
    if status != PDB_OK:
        raise PatchdbError(status, _lib.pdb_last_error().decode())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def build_info() -> str:
    return _lib.pdb_build_info().decode()


class _Handle:
    _free = None

    def __init__(self, ptr: C.c_void_p):
        self._ptr = ptr

    @property
    def ptr(self):
        return self._ptr

    def close(self):
        if self._ptr:
            type(self)._free(self._ptr)
            self._ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Matrix(_Handle):
    """Device CSR matrix (pdb_matrix)."""
    _free = _lib.pdb_matrix_free

    @classmethod
    def from_csr(cls, row_ptr, col_idx, values) -> "Matrix":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        v = _f64(values)
        out = C.c_void_p()
        _check(_lib.pdb_matrix_from_csr(len(rp) - 1, _ip(rp), _ip(ci), _dp(v), C.byref(out)))
        return cls(out)

    @classmethod
    def read_matrix_market(cls, path: str) -> "Matrix":
        out = C.c_void_p()
        _check(_lib.pdb_matrix_read_matrix_market(path.encode(), C.byref(out)))
        return cls(out)

    def write_matrix_market(self, path: str) -> None:
        _check(_lib.pdb_matrix_write_matrix_market(self._ptr, path.encode()))

    @property
    def rows(self) -> int:
        return _lib.pdb_matrix_rows(self._ptr)

    @property
    def nnz(self) -> int:
        return _lib.pdb_matrix_nnz(self._ptr)

    def sell_info(self) -> dict:
        """Residual storage: column-pattern classes (0: explicit column
        indices), column indices and values stored, slices."""
        out = np.zeros(4, dtype=np.int64)
        _check(_lib.pdb_matrix_sell_info(self._ptr, _ip(out)))
        return {"classes": int(out[0]), "col_entries": int(out[1]), "slices": int(out[2]),
                "val_entries": int(out[3])}

    def mirror_info(self) -> dict:
        """Half-storage residual layout: in use or why
        not, values stored, identity rows storing mirrored values, class
        offsets."""
        out = np.zeros(4, dtype=np.int64)
        why = C.c_char_p()
        _check(_lib.pdb_matrix_mirror_info(self._ptr, _ip(out), C.byref(why)))
        return {"mirror": bool(out[0]), "values": int(out[1]), "virtual_rows": int(out[2]),
                "class_offsets": int(out[3]), "why": (why.value or b"").decode()}

    def spmv(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(self.rows)
        _check(_lib.pdb_matrix_spmv(self._ptr, _dp(x), _dp(y)))
        return y

    def csr(self):
        n, nnz = self.rows, self.nnz
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.int64)
        v = np.empty(nnz)
        _check(_lib.pdb_matrix_csr(self._ptr, _ip(rp), _ip(ci), _dp(v)))
        return rp, ci, v


class Problem(_Handle):
    """Host-side problem (pdb_problem): the reference's uniform-mesh model
    problem (assemble) or a seeded BASELINE configuration (generate)."""
    _free = _lib.pdb_problem_free

    @classmethod
    def assemble(cls, config=None, **keys) -> "Problem":
        """pdb_problem_assemble(config_json): `config` is a JSON string or a
        dict (keys as the reference's ExperimentConfig: dim, cells, degree,
        coefficient={kind, value, blocks, values}); keyword arguments are
        merged into it."""
        if config is None or isinstance(config, dict):
            cfg = dict(config or {})
            cfg.update(keys)
            config = json.dumps(cfg) if cfg else ""
        out = C.c_void_p()
        _check(_lib.pdb_problem_assemble(config.encode(), C.byref(out)))
        return cls(out)

    def exact_solution(self) -> np.ndarray:
        u = np.empty(self.ndofs)
        _check(_lib.pdb_problem_exact_solution(self._ptr, _dp(u)))
        return u

    def l2_error(self, u) -> float:
        u = _f64(u)
        out = C.c_double()
        _check(_lib.pdb_problem_l2_error(self._ptr, _dp(u), C.byref(out)))
        return out.value

    @staticmethod
    def _options(config, cells, overrides):
        o = GenOptions()
        _check(_lib.pdb_gen_options_config(config, cells, C.byref(o)))
        for k, v in overrides.items():
            if k == "levels":
                for i, x in enumerate(v):
                    o.levels[i] = x
                o.n_levels = len(v)
            else:
                setattr(o, k, v)
        return o

    @classmethod
    def generate(cls, config: int = 1, cells: int = 0, **overrides) -> "Problem":
        o = cls._options(config, cells, overrides)
        out = C.c_void_p()
        _check(_lib.pdb_problem_generate(C.byref(o), C.byref(out)))
        return cls(out)

    @classmethod
    def generate_slab(cls, config: int, cells: int, rank: int, nranks: int, **overrides) -> "Problem":
        """Rows of rank `rank`'s slab only (global column ids); pdb_problem_generate_slab."""
        o = cls._options(config, cells, overrides)
        out = C.c_void_p()
        _check(_lib.pdb_problem_generate_slab(C.byref(o), rank, nranks, C.byref(out)))
        return cls(out)

    @classmethod
    def generate_cells(cls, config: int, cells: int, c0: int, c1: int, rank: int, nranks: int,
                       **overrides) -> "Problem":
        """Rows of the cell layers [c0, c1) (pdb_problem_generate_cells)."""
        o = cls._options(config, cells, overrides)
        out = C.c_void_p()
        _check(_lib.pdb_problem_generate_cells(C.byref(o), c0, c1, rank, nranks, C.byref(out)))
        return cls(out)

    @property
    def rows_global(self) -> int:
        return _lib.pdb_problem_rows_global(self._ptr)

    def row_ranges(self) -> np.ndarray:
        k = _lib.pdb_problem_row_range_count(self._ptr)
        out = np.empty(2 * k, np.int64)
        _check(_lib.pdb_problem_row_ranges(self._ptr, _ip(out)))
        return out.reshape(k, 2)

    def row_ids(self) -> np.ndarray:
        return np.concatenate([np.arange(lo, hi) for lo, hi in self.row_ranges()])

    @property
    def ndofs(self) -> int:
        return _lib.pdb_problem_ndofs(self._ptr)

    @property
    def nnz(self) -> int:
        return _lib.pdb_problem_nnz(self._ptr)

    def rhs(self) -> np.ndarray:
        b = np.empty(self.ndofs)
        _check(_lib.pdb_problem_rhs(self._ptr, _dp(b)))
        return b

    def csr(self):
        n, nnz = self.ndofs, self.nnz
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.int64)
        v = np.empty(nnz)
        _check(_lib.pdb_problem_csr(self._ptr, _ip(rp), _ip(ci), _dp(v)))
        return rp, ci, v

    def matrix(self) -> Matrix:
        out = C.c_void_p()
        _check(_lib.pdb_problem_matrix(self._ptr, C.byref(out)))
        return Matrix(out)


def export_matrix(config, path: str) -> None:
    """pdb_export_matrix: assemble the experiment's model problem (smooth
    coefficient for experiment 1, piecewise for 2 unless given) and write it
    as Matrix Market."""
    if isinstance(config, dict):
        config = json.dumps(config)
    _check(_lib.pdb_export_matrix(config.encode(), path.encode()))


class PatchSet(_Handle):
    """Detected cell patches (pdb_patchset)."""
    _free = _lib.pdb_patchset_free

    @classmethod
    def detect(cls, m: Matrix, patch_size: int) -> "PatchSet":
        out = C.c_void_p()
        _check(_lib.pdb_patchset_detect(m.ptr, patch_size, C.byref(out)))
        return cls(out)

    @property
    def count(self) -> int:
        return _lib.pdb_patchset_count(self._ptr)

    @property
    def patch_size(self) -> int:
        return _lib.pdb_patchset_patch_size(self._ptr)

    @property
    def rows(self) -> int:
        return _lib.pdb_patchset_rows(self._ptr)

    def patches(self) -> np.ndarray:
        out = np.empty((self.count, self.patch_size), np.int64)
        _check(_lib.pdb_patchset_patches(self._ptr, _ip(out)))
        return out

    def weights(self) -> np.ndarray:
        out = np.empty(self.rows)
        _check(_lib.pdb_patchset_weights(self._ptr, _dp(out)))
        return out

    def extract(self, m: Matrix) -> np.ndarray:
        out = np.empty((self.count, self.patch_size, self.patch_size))
        _check(_lib.pdb_patchset_extract(m.ptr, self._ptr, _dp(out)))
        return out

    def write_json(self, path: str) -> None:
        _check(_lib.pdb_patchset_write_json(self._ptr, path.encode()))


def compress_options(method: int = GREEDY_L1, **kw) -> CompressOptions:
    o = CompressOptions()
    _lib.pdb_compress_options_init(C.byref(o))
    o.method = method
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Database(_Handle):
    """Factorization database + assignment phi (pdb_database)."""
    _free = _lib.pdb_database_free

    @classmethod
    def build(cls, m: Matrix, ps: PatchSet, method: int = GREEDY_L1, comm: "Comm" = None, **kw) -> "Database":
        """comm: a Comm over the participating ranks -> the sharded build
        (k-means assignment split across ranks, same database on every rank)."""
        o = compress_options(method, **kw)
        out = C.c_void_p()
        if comm is None:
            _check(_lib.pdb_database_build(m.ptr, ps.ptr, C.byref(o), C.byref(out)))
        else:
            _check(_lib.pdb_database_build_sharded(m.ptr, ps.ptr, C.byref(o), comm.ptr, C.byref(out)))
        return cls(out)

    @classmethod
    def build_to_size(cls, m: Matrix, ps: PatchSet, target_lo: int, target_hi: int, method: int = GREEDY_L1,
                      comm: "Comm" = None, **kw):
        o = compress_options(method, **kw)
        out = C.c_void_p()
        eps = C.c_double()
        if comm is None:
            _check(_lib.pdb_database_build_to_size(m.ptr, ps.ptr, C.byref(o), target_lo, target_hi, C.byref(out),
                                                   C.byref(eps)))
        else:
            _check(_lib.pdb_database_build_to_size_sharded(m.ptr, ps.ptr, C.byref(o), target_lo, target_hi, comm.ptr,
                                                           C.byref(out), C.byref(eps)))
        return cls(out), eps.value

    @property
    def size(self) -> int:
        return _lib.pdb_database_size(self._ptr)

    @property
    def n_patches(self) -> int:
        return _lib.pdb_database_n_patches(self._ptr)

    @property
    def patch_size(self) -> int:
        return _lib.pdb_database_patch_size(self._ptr)

    @property
    def eps(self) -> float:
        return _lib.pdb_database_eps(self._ptr)

    def phi(self) -> np.ndarray:
        out = np.empty(self.n_patches, np.int64)
        _check(_lib.pdb_database_phi(self._ptr, _ip(out)))
        return out

    def representatives(self) -> np.ndarray:
        ps = self.patch_size
        out = np.empty((self.size, ps, ps))
        _check(_lib.pdb_database_representatives(self._ptr, _dp(out)))
        return out

    def factors(self):
        ps = self.patch_size
        lu = np.empty((self.size, ps, ps))
        piv = np.empty((self.size, ps), np.int64)
        _check(_lib.pdb_database_factors(self._ptr, _dp(lu), _ip(piv)))
        return lu, piv

    def work(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.pdb_database_work(self._ptr, C.byref(a), C.byref(b), C.byref(c)))
        return {"pair_evals": a.value, "power_iters": b.value, "lu_count": c.value}

    def objective(self, m: Matrix, ps: "PatchSet", beta: float) -> float:
        """Reference evaluate_objective: beta |B| + sum_k d(A_k, B_phi(k))^2."""
        out = C.c_double()
        _check(_lib.pdb_database_objective(m.ptr, ps.ptr, self._ptr, float(beta), C.byref(out)))
        return out.value

    def export(self, json_path: str, bin_path: str) -> None:
        _check(_lib.pdb_database_export(self._ptr, json_path.encode(), bin_path.encode()))

    @classmethod
    def load(cls, json_path: str, bin_path: str) -> "Database":
        """pdb_database_import: a database written by export (setup reuse)."""
        out = C.c_void_p()
        _check(_lib.pdb_database_import(json_path.encode(), bin_path.encode(), C.byref(out)))
        return cls(out)


class Preconditioner(_Handle):
    """Patch preconditioner (pdb_precond); db=None selects the exact variant."""
    _free = _lib.pdb_precond_free

    def __init__(self, ptr, n: int):
        super().__init__(ptr)
        self.n = n

    @classmethod
    def create(cls, m: Optional[Matrix], ps: PatchSet, db: Optional[Database] = None, omega: float = 1.0,
               threads: int = 1) -> "Preconditioner":
        out = C.c_void_p()
        _check(_lib.pdb_precond_create(m.ptr if m is not None else None, ps.ptr, db.ptr if db is not None else None,
                                       omega, threads, C.byref(out)))
        return cls(out, ps.rows)

    @classmethod
    def create_combo(cls, problem: "Problem", ps: PatchSet, db: Optional[Database] = None, omega: float = 1.0,
                     threads: int = 1) -> "Preconditioner":
        """Patch term plus the coarse correction P0 (R0 A P0)^-1 R0
        (pdb_precond_create_combo; reference ComboPreconditioner)."""
        out = C.c_void_p()
        _check(_lib.pdb_precond_create_combo(problem.ptr, ps.ptr, db.ptr if db is not None else None, omega, threads,
                                             C.byref(out)))
        return cls(out, ps.rows)

    def coarse_size(self):
        """(n_c, kl, ku) of the coarse band LU; (0, 0, 0) without one."""
        v = np.zeros(3, np.int64)
        _check(_lib.pdb_precond_coarse_size(self._ptr, _ip(v[0:]), _ip(v[1:]), _ip(v[2:])))
        return tuple(int(x) for x in v)

    def coarse_factor(self):
        """The device band LU in the reference layout: (ab[(2kl+ku+1), n_c], ipiv)."""
        nc, kl, ku = self.coarse_size()
        ab, ipiv = np.empty((2 * kl + ku + 1, nc)), np.empty(nc, np.int64)
        _check(_lib.pdb_precond_coarse_factor(self._ptr, _dp(ab), _ip(ipiv)))
        return ab, ipiv

    def apply(self, r) -> np.ndarray:
        r = _f64(r)
        z = np.empty(self.n)
        _check(_lib.pdb_precond_apply(self._ptr, _dp(r), _dp(z)))
        return z

    def apply_device(self, d_r: int, d_z: int, stream: int = 0) -> None:
        _check(_lib.pdb_precond_apply_device(self._ptr, d_r, d_z, stream or None))

    def relax(self, m: Matrix, b, x, sweeps: int, history: bool = True):
        """`sweeps` smooth() steps from x (copied); returns (x_new, history or None)."""
        b = _f64(b)
        xn = _f64(x).copy()
        hist = np.empty(sweeps + 1) if history else None
        _check(_lib.pdb_relax(m.ptr, self._ptr, _dp(b), _dp(xn), sweeps, _dp(hist) if history else None))
        return xn, hist

    def relax_device(self, m: Matrix, d_b: int, d_x: int, sweeps: int, d_hist: int = 0, stream: int = 0) -> None:
        _check(_lib.pdb_relax_device(m.ptr, self._ptr, d_b, d_x, sweeps, d_hist or None, stream or None))


@dataclass
class Report:
    iterations: int
    restarts: int
    converged: bool
    final_relative_residual: float
    residual_history: np.ndarray


def _report(ptr) -> Report:
    try:
        n = _lib.pdb_report_residual_history_size(ptr)
        h = np.empty(n)
        if n:
            _check(_lib.pdb_report_residual_history(ptr, _dp(h)))
        return Report(_lib.pdb_report_iterations(ptr), _lib.pdb_report_restarts(ptr),
                      bool(_lib.pdb_report_converged(ptr)), _lib.pdb_report_final_relative_residual(ptr), h)
    finally:
        _lib.pdb_report_free(ptr)


def gmres(m: Matrix, b, pc: Optional[Preconditioner] = None, restart: int = 20, tol: float = 1e-8,
          max_iters: int = 2000, left_precond: bool = False):
    o = GmresOptions()
    _lib.pdb_gmres_options_init(C.byref(o))
    o.restart, o.tol, o.max_iters, o.left_precond = restart, tol, max_iters, int(left_precond)
    b = _f64(b)
    x = np.empty(m.rows)
    rep = C.c_void_p()
    _check(_lib.pdb_gmres_solve(m.ptr, _dp(b), pc.ptr if pc is not None else None, C.byref(o), _dp(x),
                                C.byref(rep)))
    return x, _report(rep)


def pcg(m: Matrix, b, pc: Optional[Preconditioner] = None, tol: float = 1e-8, max_iters: int = 10000,
        reproducible: bool = False):
    """pdb_pcg_solve; reproducible=True: pdb_pcg_solve_ex(PDB_PCG_REPRODUCIBLE), the
    oracle's sequence bit for bit (the preconditioner must be created with PDB_APPLY=lu)."""
    b = _f64(b)
    x = np.empty(m.rows)
    rep = C.c_void_p()
    if reproducible:
        _check(_lib.pdb_pcg_solve_ex(m.ptr, _dp(b), pc.ptr if pc is not None else None, tol, max_iters, 1, _dp(x),
                                     C.byref(rep)))
    else:
        _check(_lib.pdb_pcg_solve(m.ptr, _dp(b), pc.ptr if pc is not None else None, tol, max_iters, _dp(x),
                                  C.byref(rep)))
    return x, _report(rep)


_sig("pdb_pcg_solve_ex", C.c_int, _P, _D, _P, C.c_double, C.c_int64, C.c_int, _D, C.POINTER(_P))
_sig("pdb_relax_profile", C.c_int, _P, _P, C.c_void_p, C.c_void_p, C.c_int64, _D, C.c_void_p)
_sig("pdb_precond_stored_factors", C.c_int64, _P)
_sig("pdb_precond_patch_count", C.c_int64, _P)
_sig("pdb_precond_patch_size", C.c_int64, _P)


def relax_profile(pc: Preconditioner, m: Matrix, d_b: int, d_x: int, sweeps: int, stream: int = 0):
    """Average ms per sweep of (residual, patch_solve, scatter_update), timed with CUDA events."""
    ms = np.zeros(3)
    _check(_lib.pdb_relax_profile(m.ptr, pc.ptr, d_b, d_x, sweeps, _dp(ms), stream or None))
    return ms


def precond_sizes(pc: Preconditioner):
    return (_lib.pdb_precond_stored_factors(pc.ptr), _lib.pdb_precond_patch_count(pc.ptr),
            _lib.pdb_precond_patch_size(pc.ptr))


# ---- multi-GPU shards ----------------------------------------------------
PLAN_ARRAYS = dict(dofs=0, row_ptr=1, cols=2, values=3, patches=4, weights=5, owned=6, up=7, up_peer=8, pin=9,
                   pin_peer=10, xs=11, xs_peer=12, xr=13, xr_peer=14, patch_range=15)
_sig("pdb_shard_plan_create", C.c_int, C.c_int64, _I64, _I64, _D, C.c_int64, C.c_int64, _I64, _D, C.c_int, C.c_int,
     C.POINTER(_P))
_sig("pdb_shard_plan_size", C.c_int64, _P, C.c_int)
_sig("pdb_shard_plan_get", C.c_int, _P, C.c_int, C.c_void_p)
_sig("pdb_shard_plan_free", None, _P)
_sig("pdb_comm_unique_id", C.c_int, C.c_void_p)
_sig("pdb_shard_create", C.c_int, _P, _P, _P, C.c_double, C.c_int, C.c_int, C.POINTER(_P))
_sig("pdb_shard_attach_comm", C.c_int, _P, C.c_void_p)
_sig("pdb_shard_local_size", C.c_int64, _P)
_sig("pdb_shard_local_dofs", C.c_int, _P, _I64)
_sig("pdb_shard_owned_count", C.c_int64, _P)
_sig("pdb_shard_owned", C.c_int, _P, _I64)
_sig("pdb_shard_relax_device", C.c_int, _P, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
_sig("pdb_shard_free", None, _P)


def shard_plan(csr, patches, weights, rank: int, nranks: int) -> dict:
    """Host-only exchange schedule of one rank (no GPU needed)."""
    rp = np.ascontiguousarray(csr[0], np.int64)
    ci = np.ascontiguousarray(csr[1], np.int64)
    v = _f64(csr[2])
    pt = np.ascontiguousarray(patches, np.int64)
    w = _f64(weights)
    h = C.c_void_p()
    _check(_lib.pdb_shard_plan_create(len(rp) - 1, _ip(rp), _ip(ci), _dp(v), pt.shape[0], pt.shape[1], _ip(pt), _dp(w),
                                      rank, nranks, C.byref(h)))
    try:
        out = {}
        for name, which in PLAN_ARRAYS.items():
            size = _lib.pdb_shard_plan_size(h, which)
            arr = np.empty(size, np.float64 if name in ("values", "weights") else np.int64)
            if size:
                _check(_lib.pdb_shard_plan_get(h, which, arr.ctypes.data_as(C.c_void_p)))
            out[name] = arr
        return out
    finally:
        _lib.pdb_shard_plan_free(h)


def comm_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(_lib.pdb_comm_unique_id(buf))
    return bytes(buf)


_sig("pdb_comm_create", C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(_P))
_sig("pdb_comm_free", None, _P)
_sig("pdb_database_build_sharded", C.c_int, _P, _P, C.POINTER(CompressOptions), _P, C.POINTER(_P))
_sig("pdb_database_build_to_size_sharded", C.c_int, _P, _P, C.POINTER(CompressOptions), C.c_int64, C.c_int64, _P,
     C.POINTER(_P), C.POINTER(C.c_double))


class Comm(_Handle):
    """NCCL communicator for the sharded setup (one process per GPU)."""
    _free = _lib.pdb_comm_free

    @classmethod
    def create(cls, uid: bytes, rank: int, nranks: int) -> "Comm":
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        out = C.c_void_p()
        _check(_lib.pdb_comm_create(buf, rank, nranks, C.byref(out)))
        return cls(out)


class Shard(_Handle):
    """One rank's slab of the sweep on this process's GPU."""
    _free = _lib.pdb_shard_free

    @classmethod
    def create(cls, m: Matrix, ps: PatchSet, db: Optional[Database], omega: float, rank: int,
               nranks: int) -> "Shard":
        out = C.c_void_p()
        _check(_lib.pdb_shard_create(m.ptr, ps.ptr, db.ptr if db is not None else None, omega, rank, nranks,
                                     C.byref(out)))
        return cls(out)

    def attach(self, uid: bytes) -> None:
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        _check(_lib.pdb_shard_attach_comm(self._ptr, buf))

    def local_dofs(self) -> np.ndarray:
        out = np.empty(_lib.pdb_shard_local_size(self._ptr), np.int64)
        _check(_lib.pdb_shard_local_dofs(self._ptr, _ip(out)))
        return out

    def owned(self) -> np.ndarray:
        out = np.empty(_lib.pdb_shard_owned_count(self._ptr), np.int64)
        if len(out):
            _check(_lib.pdb_shard_owned(self._ptr, _ip(out)))
        return out

    def relax_device(self, d_b: int, d_x: int, sweeps: int, stream: int = 0) -> None:
        _check(_lib.pdb_shard_relax_device(self._ptr, d_b, d_x, sweeps, stream or None))


_sig("pdb_slab_create", C.c_int, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int64, _P, C.c_double, C.c_char_p,
     C.POINTER(_P))
_sig("pdb_slab_local_ranks", C.c_int, _P)
_sig("pdb_slab_upload_seconds", C.c_double, _P)
_sig("pdb_slab_info", C.c_int, _P, C.c_int, _I64)
_sig("pdb_slab_local_dofs", C.c_int, _P, C.c_int, _I64)
_sig("pdb_slab_owned", C.c_int, _P, C.c_int, _I64)
_sig("pdb_slab_relax_device", C.c_int, _P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int64, C.c_void_p)
_sig("pdb_slab_free", None, _P)
_sig("pdb_slab_create_built", C.c_int, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int64, C.POINTER(CompressOptions),
     C.c_double, C.c_char_p, C.POINTER(_P))
_sig("pdb_slab_database_size", C.c_int64, _P)
_sig("pdb_slab_phi", C.c_int, _P, C.c_int, _I64)
_sig("pdb_slab_creators", C.c_int, _P, _I64)
_sig("pdb_slab_create_subset", C.c_int, C.POINTER(_P), C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int64, _P,
     C.c_double, C.c_char_p, C.POINTER(_P))
_sig("pdb_slab_relax_rank_device", C.c_int, _P, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
_sig("pdb_problem_generate_cells", C.c_int, C.POINTER(GenOptions), C.c_int64, C.c_int64, C.c_int, C.c_int,
     C.POINTER(_P))

SLAB_INFO = ("rank", "nranks", "n_local", "n_rows", "n_patches", "first_patch", "split", "n_owned", "n_up", "n_pin",
             "n_xs", "n_xr")


class Slab(_Handle):
    """Rank-local multi-GPU sweep shards (pdb_slab_*): one rank with an NCCL
    id, or an emulated group of all ranks on one GPU (nccl_id None)."""
    _free = _lib.pdb_slab_free

    @classmethod
    def create(cls, slabs, rank: int, nranks: int, patch_size: int, db: Optional["Database"] = None,
               omega: float = 1.0, nccl_id: Optional[bytes] = None) -> "Slab":
        arr = (C.c_void_p * len(slabs))(*[p.ptr for p in slabs])
        out = C.c_void_p()
        _check(_lib.pdb_slab_create(arr, len(slabs), rank, nranks, patch_size, db.ptr if db is not None else None,
                                    omega, nccl_id, C.byref(out)))
        h = cls(out)
        h._keep = list(slabs)
        return h

    @classmethod
    def create_built(cls, slabs, rank: int, nranks: int, patch_size: int, method: int = 2, eps: float = 1e-7,
                     best_match: bool = False, omega: float = 1.0, nccl_id: Optional[bytes] = None,
                     **kmeans) -> "Slab":
        """Compressed database built from the ranks' own patches (pdb_slab_create_built):
        greedy-l1 (eps, best_match) or entrywise k-means (db_size, seed, max_iters)."""
        arr = (C.c_void_p * len(slabs))(*[p.ptr for p in slabs])
        o = compress_options(method, eps=eps, best_match=int(best_match), **kmeans)
        out = C.c_void_p()
        _check(_lib.pdb_slab_create_built(arr, len(slabs), rank, nranks, patch_size, C.byref(o), omega, nccl_id,
                                          C.byref(out)))
        h = cls(out)
        h._keep = list(slabs)
        return h

    @property
    def database_size(self) -> int:
        return _lib.pdb_slab_database_size(self._ptr)

    def phi(self, i: int = 0) -> np.ndarray:
        out = np.empty(self.info(i)["n_patches"], np.int64)
        _check(_lib.pdb_slab_phi(self._ptr, i, _ip(out)))
        return out

    def creators(self) -> np.ndarray:
        out = np.empty(self.database_size, np.int64)
        _check(_lib.pdb_slab_creators(self._ptr, _ip(out)))
        return out

    @classmethod
    def create_subset(cls, slabs, ranks, rank: int, nranks: int, patch_size: int, omega: float = 1.0) -> "Slab":
        """Emulated group of a subset of the ranks (exact preconditioners)."""
        arr = (C.c_void_p * len(slabs))(*[p.ptr for p in slabs])
        rk = (C.c_int * len(ranks))(*ranks)
        out = C.c_void_p()
        _check(_lib.pdb_slab_create_subset(arr, len(slabs), rk, rank, nranks, patch_size, None, omega, None,
                                           C.byref(out)))
        h = cls(out)
        h._keep = list(slabs)
        return h

    def relax_rank_device(self, i: int, d_b: int, d_x: int, sweeps: int, stream: int = 0) -> None:
        _check(_lib.pdb_slab_relax_rank_device(self._ptr, i, d_b, d_x, sweeps, stream or None))

    @property
    def local_ranks(self) -> int:
        return _lib.pdb_slab_local_ranks(self._ptr)

    @property
    def upload_seconds(self) -> float:
        """Matrix upload + residual storage build inside the setup (pdb_slab_upload_seconds)."""
        return _lib.pdb_slab_upload_seconds(self._ptr)

    def info(self, i: int = 0) -> dict:
        out = np.zeros(12, np.int64)
        _check(_lib.pdb_slab_info(self._ptr, i, _ip(out)))
        return dict(zip(SLAB_INFO, (int(v) for v in out)))

    def local_dofs(self, i: int = 0) -> np.ndarray:
        out = np.empty(self.info(i)["n_local"], np.int64)
        _check(_lib.pdb_slab_local_dofs(self._ptr, i, _ip(out)))
        return out

    def owned(self, i: int = 0) -> np.ndarray:
        out = np.empty(self.info(i)["n_owned"], np.int64)
        _check(_lib.pdb_slab_owned(self._ptr, i, _ip(out)))
        return out

    def relax_device(self, d_b, d_x, sweeps: int, stream: int = 0) -> None:
        """d_b, d_x: one device pointer per local rank (vectors of its local DoFs)."""
        L = self.local_ranks
        bb = (C.c_void_p * L)(*d_b)
        xx = (C.c_void_p * L)(*d_x)
        _check(_lib.pdb_slab_relax_device(self._ptr, bb, xx, sweeps, stream or None))


def compressibility_curve(m: Matrix, ps: "PatchSet", method: int, eps_grid) -> list:
    """Reference compressibility_curve: [(eps, db_size, ratio)] for greedy
    first-match compression over an ascending tolerance grid."""
    g = _f64(eps_grid)
    sizes = np.zeros(len(g), dtype=np.int64)
    ratios = np.zeros(len(g))
    _check(_lib.pdb_compressibility_curve(m.ptr, ps.ptr, int(method), _dp(g), len(g), _ip(sizes), _dp(ratios)))
    return [(float(e), int(n), float(r)) for e, n, r in zip(g, sizes, ratios)]


def debug_mirror_check(csr, x):
    """Test hook (host only, no device): build the half-storage residual
    layout of a CSR matrix and evaluate y = A x through it in the GPU
    kernel's order.  Returns (y or None when the layout does not apply,
    stats dict with the reason)."""
    rp, ci, v = (np.ascontiguousarray(a) for a in csr)
    rp = rp.astype(np.int64)
    ci = ci.astype(np.int64)
    v = _f64(v)
    x = _f64(x)
    n = len(rp) - 1
    y = np.full(n, np.nan)
    out = np.zeros(6, dtype=np.int64)
    _check(_lib.pdb_debug_mirror_check(n, _ip(rp), _ip(ci), _dp(v), _dp(x), _dp(y), _ip(out)))
    stats = {"built": bool(out[0]), "slices": int(out[1]), "values": int(out[2]), "class_offsets": int(out[3]),
             "classes": int(out[4]), "virtual_rows": int(out[5])}
    if not out[0]:
        stats["why"] = _lib.pdb_last_error().decode()
        return None, stats
    return y, stats
