"""ctypes front-end to inputs/libpdbgen.so: the seeded BASELINE input
generator (paper_2306_10025_b200/csrc/generator.cpp) built as a standalone
host library without CUDA and without any pdb_* symbol.  bench.py's
reference arm and the fixture scripts use it, so a process that times the
reference never loads libpatchdb.so.0.  Same seeds, same bytes as
paper_2306_10025_b200.patchdb.Problem.generate (tests/test_generator.py).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpdbgen.so")

_lib = None


def _load():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.pdbgen_last_error.restype = C.c_char_p
        L.pdbgen_generate.argtypes = [C.c_int, C.c_int64, C.POINTER(C.c_void_p)]
        L.pdbgen_n.restype = C.c_int64
        L.pdbgen_n.argtypes = [C.c_void_p]
        L.pdbgen_nnz.restype = C.c_int64
        L.pdbgen_nnz.argtypes = [C.c_void_p]
        L.pdbgen_csr.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.pdbgen_rhs.argtypes = [C.c_void_p, C.c_void_p]
        L.pdbgen_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


class Generated:
    """CSR (int64 row_ptr / col_idx, fp64 values) and right-hand side of one
    BASELINE configuration."""

    def __init__(self, config: int, cells: int = 0):
        L = _load()
        h = C.c_void_p()
        st = L.pdbgen_generate(config, cells, C.byref(h))
        if st != 0:
            raise RuntimeError(f"pdbgen_generate({config}, {cells}): {L.pdbgen_last_error().decode()}")
        try:
            n, nnz = L.pdbgen_n(h), L.pdbgen_nnz(h)
            self.ndofs, self.nnz = n, nnz
            rp, ci, v = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
            L.pdbgen_csr(h, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
            self._csr = (rp, ci, v)
            self._rhs = np.empty(n)
            L.pdbgen_rhs(h, self._rhs.ctypes.data)
        finally:
            L.pdbgen_free(h)

    def csr(self):
        return self._csr

    def rhs(self):
        return self._rhs.copy()
