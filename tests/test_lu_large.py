"""Batched LU of large patches (pytest -m gpu): the blocked CTA-per-matrix
kernel (ps > 48, panels of 16 columns) and the unblocked CTA kernel against
the oracle's lu_factor
(dense.cpp:31-75), bitwise, on block-diagonal matrices of random dense
nonsymmetric blocks (every block is one patch, partial pivoting swaps rows
at almost every step).  Also: the explicit inverses the sweep streams
(column-block kernel) against numpy, the singular-block error, and the
ps <= 48 warp kernel forced onto the same inputs (PDB_LU_WARP) for the
sizes both handle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def block_diag_csr(blocks):
    nb, ps, _ = blocks.shape
    n = nb * ps
    rp = np.arange(n + 1, dtype=np.int64) * ps
    ci = np.empty(n * ps, np.int64)
    for b in range(nb):
        cols = np.arange(b * ps, (b + 1) * ps)
        ci[b * ps * ps:(b + 1) * ps * ps] = np.tile(cols, ps)
    return rp, ci, blocks.reshape(-1).copy()


def random_blocks(nb, ps, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, (nb, ps, ps))
    a[:, np.arange(ps), np.arange(ps)] += 0.05  # nonsingular, still pivots
    return a


@pytest.mark.parametrize("ps", [49, 64, 100, 165, 166, 192, 200])
def test_large_lu_bitwise(P, orc, ps):
    nb = 24
    blocks = random_blocks(nb, ps, ps)
    A = P.Matrix.from_csr(*block_diag_csr(blocks))
    pset = P.PatchSet.detect(A, ps)
    assert pset.count == nb
    db = P.Database.build(A, pset, P.EXACT)
    lu, piv = db.factors()
    for b in range(nb):
        lo, po = orc.lu_factor(blocks[b])
        assert np.array_equal(piv[b], po), b
        assert np.array_equal(lu[b].view(np.uint64), lo.view(np.uint64)), b


@pytest.mark.parametrize("ps", [64, 100, 192])
def test_large_lu_kernels_agree(P, monkeypatch, ps):
    """Blocked (default), CTA-unblocked (PDB_LU_CTA) and warp (PDB_LU_WARP)
    kernels: bitwise the same factors and pivots."""
    blocks = random_blocks(6, ps, 3 * ps)
    A = P.Matrix.from_csr(*block_diag_csr(blocks))
    pset = P.PatchSet.detect(A, ps)
    lu_b, piv_b = P.Database.build(A, pset, P.EXACT).factors()
    monkeypatch.setenv("PDB_LU_CTA", "1")
    lu_c, piv_c = P.Database.build(A, pset, P.EXACT).factors()
    monkeypatch.delenv("PDB_LU_CTA")
    monkeypatch.setenv("PDB_LU_WARP", "1")
    lu_w, piv_w = P.Database.build(A, pset, P.EXACT).factors()
    assert np.array_equal(piv_b, piv_w) and np.array_equal(piv_c, piv_w)
    assert np.array_equal(lu_b.view(np.uint64), lu_w.view(np.uint64))
    assert np.array_equal(lu_c.view(np.uint64), lu_w.view(np.uint64))


@pytest.mark.parametrize("ps", [40, 64, 192])
def test_large_inverse_apply(P, ps):
    """Exact preconditioner (explicit column-block inverses): one apply with
    omega = 1 and unit weights is the block solve A_b^{-1} r_b."""
    nb = 8
    blocks = random_blocks(nb, ps, 7 * ps)
    A = P.Matrix.from_csr(*block_diag_csr(blocks))
    pset = P.PatchSet.detect(A, ps)
    pc = P.Preconditioner.create(A, pset, None, omega=1.0)
    r = np.random.default_rng(ps).uniform(-1, 1, nb * ps)
    z = pc.apply(r)
    want = np.concatenate([np.linalg.solve(blocks[b], r[b * ps:(b + 1) * ps]) for b in range(nb)])
    np.testing.assert_allclose(z, want, rtol=1e-9, atol=1e-9 * np.abs(want).max())


def test_large_singular_block(P, orc):
    ps = 192
    blocks = random_blocks(4, ps, 11)
    blocks[2, :, 5] = 0.0  # column 5 of patch 2 is zero
    A = P.Matrix.from_csr(*block_diag_csr(blocks))
    pset = P.PatchSet.detect(A, ps)
    with pytest.raises(P.PatchdbError) as e:
        P.Database.build(A, pset, P.EXACT)
    with pytest.raises(Exception) as eo:
        orc.lu_factor(blocks[2])
    assert e.value.status == P.PDB_ERR_SINGULAR_MATRIX
    assert e.value.message == "patch 2: " + eo.value.message
