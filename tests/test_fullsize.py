"""Parity at the BASELINE sizes (pytest -m gpu).

Config 2 (n = 1,050,625, 65,536 patches) and config 4 (n = 2,364,419,
262,144 Vanka patches) at full size: patch lists and weights bit-exact
against the oracle, the SpMV bit-exact, and for config 2 three compressed
relaxation sweeps against the oracle's sweep with the same database (1e-9),
plus size-independent sweep properties: linearity in b and the weighted
partition of unity of the preconditioner.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full2(P, orc):
    prob = P.Problem.generate(2, 0)
    A = prob.matrix()
    ps = P.PatchSet.detect(A, 25)
    return prob, A, ps


def test_config2_detect_spmv_bit_exact(full2, orc):
    prob, A, ps = full2
    csr = prob.csr()
    assert A.rows == 1050625 and prob.nnz == 37642321
    patches, w = orc.detect(csr, 25)
    assert patches.shape == (65536, 25)
    assert np.array_equal(ps.patches(), patches)
    assert np.array_equal(ps.weights(), w)
    x = np.random.default_rng(21).uniform(-1, 1, A.rows)
    assert np.array_equal(A.spmv(x), orc.spmv(csr, x))


def test_config2_relax_matches_oracle(full2, P, orc):
    prob, A, ps = full2
    db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=64, seed=42, max_iters=10)
    pc = P.Preconditioner.create(A, ps, db, omega=1.0)
    b = prob.rhs()
    x, hist = pc.relax(A, b, np.zeros_like(b), 3)
    lu, piv = db.factors()
    xo, ho = orc.relax(prob.csr(), ps.patches(), ps.weights(), 1.0, lu, piv, db.phi(), b, np.zeros_like(b), 3)
    np.testing.assert_allclose(hist, ho, rtol=1e-9, atol=0)
    np.testing.assert_allclose(x, xo, rtol=1e-9, atol=1e-9 * np.abs(xo).max())


def test_config2_sweep_properties(full2, P):
    """One sweep from x = 0 is x1 = M b: linear in b; with b = A 1 on the
    interior the apply of the exact residual reproduces the weighted sum."""
    prob, A, ps = full2
    db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=64, seed=42, max_iters=5)
    pc = P.Preconditioner.create(A, ps, db, omega=0.7)
    rng = np.random.default_rng(5)
    b1, b2 = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
    z0 = np.zeros(A.rows)
    x1, _ = pc.relax(A, b1, z0, 1, history=False)
    x2, _ = pc.relax(A, b2, z0, 1, history=False)
    x12, _ = pc.relax(A, 2.0 * b1 - 3.0 * b2, z0, 1, history=False)
    np.testing.assert_allclose(x12, 2.0 * x1 - 3.0 * x2, rtol=0, atol=1e-12 * np.abs(x12).max())
    # apply == one sweep from zero
    np.testing.assert_array_equal(pc.apply(b1), x1)


def test_config4_detect_spmv_bit_exact(P, orc):
    prob = P.Problem.generate(4, 0)
    A = prob.matrix()
    csr = prob.csr()
    assert A.rows == 2364419
    ps = P.PatchSet.detect(A, 22)
    patches, w = orc.detect(csr, 22)
    assert patches.shape == (262144, 22)
    assert np.array_equal(ps.patches(), patches)
    assert np.array_equal(ps.weights(), w)
    x = np.random.default_rng(8).uniform(-1, 1, A.rows)
    assert np.array_equal(A.spmv(x), orc.spmv(csr, x))


def test_config3_detect_spmv_bit_exact(P, orc):
    prob = P.Problem.generate(3, 0)
    A = prob.matrix()
    csr = prob.csr()
    assert A.rows == 2146689 and prob.nnz == 130422149
    ps = P.PatchSet.detect(A, 27)
    patches, w = orc.detect(csr, 27)
    assert patches.shape == (262144, 27)
    assert np.array_equal(ps.patches(), patches)
    assert np.array_equal(ps.weights(), w)
    x = np.random.default_rng(17).uniform(-1, 1, A.rows)
    assert np.array_equal(A.spmv(x), orc.spmv(csr, x))
