"""Half-storage ("mirror") residual layout (csrc/sell_mirror.cpp, DESIGN.md
section 3): rows store only their upper entries and read each lower entry
a_ij from row j, where a_ji == a_ij sits bit for bit.

CPU: the layout is built on the host and y = A x is evaluated through it in
the kernel's order (pdb_debug_mirror_check, no device): bitwise the CSR sum
(the reference spmv order, sparse.cpp:50-63) on the BASELINE lattices and on
symmetric band matrices with Dirichlet rows; matrices that break a
precondition keep the plain layout, with the reason.
GPU: residual_mirror_kernel (opt-in, PDB_SELL_MIRROR=1 at matrix creation)
against the oracle and against the default classed SELL copy, bitwise, up to
config 3 at full size.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "inputs"))
from pdbgen import Generated  # noqa: E402


def csr_spmv(csr, x):
    """Sequential CSR-order sum per row (the reference spmv)."""
    import scipy.sparse as sp
    rp, ci, v = csr
    return sp.csr_matrix((v, ci, rp), shape=(len(rp) - 1, len(x))) @ x


def sym_band(seed, n, band, dirichlet=0.05, clip=False):
    """Symmetric band matrix with random values; rows in `dirichlet` (the
    first/last `band` rows unless clip, plus a random fraction) replaced by
    identity rows whose columns stay in the other rows, as the FEM
    generator's Dirichlet rows."""
    rng = np.random.default_rng(seed)
    full = np.zeros((n, 2 * band + 1))
    for d in range(1, band + 1):
        w = rng.uniform(-1, 1, n - d)
        full[d:, band - d] = w      # a_{i, i-d}
        full[:-d, band + d] = w     # a_{i, i+d} (same bits)
    full[:, band] = rng.uniform(4, 5, n)
    dir_rows = set(rng.choice(n, int(dirichlet * n), replace=False).tolist())
    if not clip:
        dir_rows |= set(range(band)) | set(range(n - band, n))
    rp, ci, v = [0], [], []
    for i in range(n):
        if i in dir_rows:
            ci.append(i)
            v.append(1.0)
        else:
            for d in range(-band, band + 1):
                j = i + d
                if 0 <= j < n:
                    ci.append(j)
                    v.append(full[i, band + d])
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int64), np.array(v)


@pytest.mark.parametrize("cfg", [1, 2])
def test_host_layout_bitwise_on_baseline_lattices(P, cfg):
    g = Generated(cfg)
    csr = g.csr()
    x = np.random.default_rng(cfg).uniform(-1, 1, g.ndofs)
    y, st = P.debug_mirror_check(csr, x)
    assert st["built"], st
    assert np.array_equal(y, csr_spmv(csr, x))
    # about half the values are stored (upper entries + identity-row slots)
    assert st["values"] < 0.6 * g.nnz
    assert st["virtual_rows"] > 0


@pytest.mark.parametrize("seed,n,band,clip", [(1, 3000, 4, False), (2, 40000, 17, False), (3, 500, 2, True),
                                               (4, 9000, 9, True)])
def test_host_layout_bitwise_on_symmetric_bands(P, seed, n, band, clip):
    csr = sym_band(seed, n, band, clip=clip)
    x = np.random.default_rng(seed + 7).uniform(-1, 1, n)
    y, st = P.debug_mirror_check(csr, x)
    assert st["built"], st
    assert np.array_equal(y, csr_spmv(csr, x))


def test_host_layout_rejects_non_symmetric(P):
    rp, ci, v = sym_band(5, 2000, 3)
    v = v.copy()
    k = rp[1000] + 1  # a lower entry of an interior row
    v[k] = np.nextafter(v[k], 2.0)
    y, st = P.debug_mirror_check((rp, ci, v), np.ones(2000))
    assert not st["built"] and "symmetric" in st["why"]
    assert y is None


def test_host_layout_rejects_config5_elasticity(P):
    """The elasticity matrix's 3x3 blocks are assembled in an order that is
    not symmetric bit for bit: the plain classed layout stays."""
    g = Generated(5, 4)
    y, st = P.debug_mirror_check(g.csr(), np.ones(g.ndofs))
    assert not st["built"] and "symmetric" in st["why"]


def test_host_layout_rejects_unclassed(P):
    rng = np.random.default_rng(9)
    n = 400
    rows = [np.unique(np.concatenate([[i], rng.choice(n, 5)])) for i in range(n)]
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    csr = (rp, np.concatenate(rows).astype(np.int64), rng.uniform(-1, 1, rp[-1]))
    y, st = P.debug_mirror_check(csr, np.ones(n))
    assert not st["built"] and "pattern" in st["why"]


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("seed,n,band,clip", [(1, 3000, 4, False), (2, 40000, 17, False), (4, 9000, 9, True)])
def test_gpu_mirror_spmv_bitwise(P, orc, monkeypatch, seed, n, band, clip):
    csr = sym_band(seed, n, band, clip=clip)
    monkeypatch.setenv("PDB_SELL_MIRROR", "1")
    A = P.Matrix.from_csr(*csr)
    monkeypatch.delenv("PDB_SELL_MIRROR")
    assert A.mirror_info()["mirror"], A.mirror_info()
    x = np.random.default_rng(seed + 7).uniform(-1, 1, n)
    want = orc.spmv(csr, x)
    assert np.array_equal(A.spmv(x), want)
    B = P.Matrix.from_csr(*csr)
    info = B.mirror_info()
    assert not info["mirror"] and "PDB_SELL_MIRROR=1" in info["why"]
    assert np.array_equal(B.spmv(x), want)


@pytest.mark.gpu
def test_gpu_mirror_not_used_for_config5(P, monkeypatch):
    monkeypatch.setenv("PDB_SELL_MIRROR", "1")
    A = P.Problem.generate(5, 4).matrix()
    info = A.mirror_info()
    assert not info["mirror"] and "symmetric" in info["why"]


@pytest.mark.gpu
def test_gpu_mirror_config3_full(P, orc, monkeypatch):
    """Config 3 at 64^3: the residual through the half storage equals the
    plain classed SELL copy's and the oracle's bit for bit, and 10 sweeps
    (device and host-vector pipelined paths) give the same iterates."""
    prob = P.Problem.generate(3, 0)
    csr = prob.csr()
    monkeypatch.setenv("PDB_SELL_MIRROR", "1")
    A = P.Matrix.from_csr(*csr)
    monkeypatch.delenv("PDB_SELL_MIRROR")
    info = A.mirror_info()
    assert info["mirror"], info
    assert A.sell_info()["val_entries"] < 0.56 * prob.nnz
    x = np.random.default_rng(3).uniform(-1, 1, A.rows)
    y = A.spmv(x)
    assert np.array_equal(y, orc.spmv(csr, x))
    B = prob.matrix()
    assert not B.mirror_info()["mirror"]
    assert np.array_equal(B.spmv(x), y)
    ps = P.PatchSet.detect(A, 27)
    b = prob.rhs()
    pa = P.Preconditioner.create(A, ps, None, omega=1.0)
    pb = P.Preconditioner.create(B, ps, None, omega=1.0)
    xa, ha = pa.relax(A, b, np.zeros_like(b), 10)
    xb, hb = pb.relax(B, b, np.zeros_like(b), 10)
    assert np.array_equal(ha, hb) and np.array_equal(xa, xb)
    # host vectors without a history: the window-pipelined first sweep
    xc, _ = pa.relax(A, b, np.zeros_like(b), 3, history=False)
    xd, _ = pb.relax(B, b, np.zeros_like(b), 3, history=False)
    assert np.array_equal(xc, xd)
