"""Configs 4 (2D Stokes Q2-Q1, Vanka patches of 22 DoFs, indefinite) and
5 (3D elasticity Q3, 192-DoF cell patches) at reduced meshes.

CPU: generator invariants (sizes, symmetry of the free block, null spaces),
the oracle pinned to the compiled reference on these matrices (detection,
extraction, pivoted LU of indefinite Vanka blocks, 192x192 LU, spectral and
l1 criteria).  GPU (-m gpu): the device path bit-exact against the oracle
(patch lists, weights, extraction, LU + pivots, k-means / greedy decisions,
SpMV) and relaxation histories within 1e-9.
"""
import numpy as np
import pytest

RTOL_HIST = 1e-9


def n_stokes(cells):
    return 2 * (2 * cells + 1) ** 2 + (cells + 1) ** 2


def n_elastic(cells):
    return 3 * (3 * cells + 1) ** 3


class Case:
    def __init__(self, P, orc, config, cells, ps):
        self.prob = P.Problem.generate(config, cells)
        self.csr = self.prob.csr()
        self.b = self.prob.rhs()
        self.ps_size = ps
        self.patches, self.w = orc.detect(self.csr, ps)
        self.mats = orc.extract_all(self.csr, self.patches)


@pytest.fixture(scope="module")
def c4s(P, orc):
    return Case(P, orc, 4, 8, 22)


@pytest.fixture(scope="module")
def c5s(P, orc):
    return Case(P, orc, 5, 4, 192)


# ------------------------------------------------------------------ CPU ---

def test_preset_sizes(P):
    assert P.Problem.generate(4, 8).ndofs == n_stokes(8)
    assert P.Problem.generate(5, 2).ndofs == n_elastic(2)
    # full config 4 size (2,364,419 DoFs)
    assert n_stokes(512) == 2364419
    assert n_elastic(96) == 72412707


def _dense(csr):
    rp, ci, v = csr
    n = len(rp) - 1
    a = np.zeros((n, n))
    for i in range(n):
        a[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    return a


@pytest.mark.parametrize("config,cells", [(4, 3), (5, 2)])
def test_generator_invariants(P, config, cells):
    prob = P.Problem.generate(config, cells, jitter=0.1)
    rp, ci, v = prob.csr()
    a = _dense((rp, ci, v))
    n = a.shape[0]
    free = np.diff(rp) > 1
    fa = a[np.ix_(free, free)]
    np.testing.assert_allclose(fa, fa.T, atol=1e-13 * np.abs(fa).max())
    ncomp = 2 if config == 4 else 3
    nu = ncomp * ((2 * cells + 1) ** 2 if config == 4 else (3 * cells + 1) ** 3)
    for c in range(ncomp):  # rigid translations have zero energy (no column elimination)
        t = np.zeros(n)
        t[c:nu:ncomp] = 1.0
        r = a @ t
        assert np.abs(r[free & (np.arange(n) < nu)]).max() < 1e-12
    if config == 4:  # constant pressure is in the kernel of B^T
        t = np.zeros(n)
        t[nu:] = 1.0
        assert np.abs((a @ t)[free & (np.arange(n) < nu)]).max() < 1e-12
        assert np.all(a[nu:, nu:] == 0.0)  # no pressure-pressure block
    # Dirichlet rows are identity rows
    bnd = np.nonzero(~free)[0]
    assert np.all(a[bnd, bnd] == 1.0)


def test_stokes_vanka_patches(c4s):
    assert c4s.patches.shape == (64, 22)  # one Vanka patch per cell
    # 18 velocity + 4 pressure DoFs
    nu = 2 * (2 * 8 + 1) ** 2
    assert np.all((c4s.patches < nu).sum(axis=1) == 18)
    # indefinite saddle blocks: zero pressure-pressure part
    assert np.all(c4s.mats[:, 18:, 18:] == 0.0)


def test_elastic_patches(c5s):
    assert c5s.patches.shape == (64, 192)


@pytest.mark.parametrize("name", ["c4s", "c5s"])
def test_ref_pins(name, request, ref, orc):
    c = request.getfixturevalue(name)
    rm = ref.matrix(c.csr)
    rps = rm.detect(c.ps_size)
    assert np.array_equal(rps.patches(), c.patches)
    assert np.array_equal(rps.weights(len(c.b)), c.w)
    assert np.array_equal(rps.extract(rm), c.mats)
    for k in range(0, len(c.mats), max(1, len(c.mats) // 8)):
        lr, pr = ref.lu_factor(c.mats[k])
        lo, po = orc.lu_factor(c.mats[k])
        assert np.array_equal(lr, lo) and np.array_equal(pr, po)
    a, b = c.mats[0], c.mats[len(c.mats) // 2]
    assert ref.l1_distance(a, b) == orc.l1_distance(a, b)
    if c.ps_size == 22:
        lb, pb = orc.lu_factor(b)
        assert ref.spectral_distance(a, b) == orc.spectral_distance(a, lb, pb)[0]


def test_vanka_lu_pivots(c4s, orc):
    """The saddle blocks need row exchanges: pivoting must be exercised."""
    swapped = sum(not np.array_equal(orc.lu_factor(m)[1], np.arange(22)) for m in c4s.mats[:16])
    assert swapped > 0


# ------------------------------------------------------------------ GPU ---

@pytest.fixture(scope="module")
def dev4(P, c4s):
    A = c4s.prob.matrix()
    return A, P.PatchSet.detect(A, 22)


@pytest.fixture(scope="module")
def dev5(P, c5s):
    A = c5s.prob.matrix()
    return A, P.PatchSet.detect(A, 192)


@pytest.mark.gpu
@pytest.mark.parametrize("name,dev", [("c4s", "dev4"), ("c5s", "dev5")])
def test_gpu_detect_extract_spmv_lu(name, dev, request, P, orc):
    c = request.getfixturevalue(name)
    A, ps = request.getfixturevalue(dev)
    assert np.array_equal(ps.patches(), c.patches)
    assert np.array_equal(ps.weights(), c.w)
    assert np.array_equal(ps.extract(A), c.mats)
    x = np.random.default_rng(4).uniform(-1, 1, A.rows)
    assert np.array_equal(A.spmv(x), orc.spmv(c.csr, x))
    db = P.Database.build(A, ps, P.EXACT)
    lu, piv = db.factors()
    for k in range(0, len(c.mats), max(1, len(c.mats) // 16)):
        lo, po = orc.lu_factor(c.mats[k])
        assert np.array_equal(lu[k], lo) and np.array_equal(piv[k], po), k


@pytest.mark.gpu
def test_gpu_stokes_kmeans_spectral(c4s, dev4, P, orc):
    A, ps = dev4
    want = orc.partitioned_build(c4s.mats, 12, 1, seed=5, max_iters=6)
    db = P.Database.build(A, ps, P.KMEANS_SPECTRAL, db_size=12, seed=5, max_iters=6)
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])
    assert np.array_equal(db.representatives(), want["reps"])
    lu, piv = db.factors()
    assert np.array_equal(lu, want["lu"]) and np.array_equal(piv, want["piv"])


@pytest.mark.gpu
def test_gpu_elastic_greedy_l1(c5s, dev5, P, orc):
    want = orc.greedy_bisect(c5s.mats, 6, 12, spectral=False)
    db = P.Database.build(dev5[0], dev5[1], P.GREEDY_L1, eps=want["eps"])
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])


@pytest.mark.gpu
def test_gpu_elastic_kmeans_entrywise(c5s, dev5, P, orc):
    """Entrywise k-means at p_s = 192 (the (patch, entry tile) pair path of
    the assignment): phi and representatives bitwise the oracle's."""
    want = orc.partitioned_build(c5s.mats, 40, 0, seed=9, max_iters=8)
    db = P.Database.build(dev5[0], dev5[1], P.KMEANS_ENTRYWISE, db_size=40, seed=9, max_iters=8)
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])
    assert np.array_equal(db.representatives(), want["reps"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,dev,compressed", [("c4s", "dev4", True), ("c5s", "dev5", False)])
def test_gpu_relax_history(name, dev, compressed, request, P, orc):
    c = request.getfixturevalue(name)
    A, ps = request.getfixturevalue(dev)
    omega = 0.6
    if compressed:
        db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=12, seed=1, max_iters=10)
        lu, piv = db.factors()
        phi = db.phi()
    else:
        db = None
        f = [orc.lu_factor(m) for m in c.mats]
        lu, piv, phi = np.stack([a for a, _ in f]), np.stack([p for _, p in f]), None
    pc = P.Preconditioner.create(A, ps, db, omega=omega)
    x, hist = pc.relax(A, c.b, np.zeros_like(c.b), 10)
    xo, ho = orc.relax(c.csr, c.patches, c.w, omega, lu, piv, phi, c.b, np.zeros_like(c.b), 10)
    np.testing.assert_allclose(hist, ho, rtol=RTOL_HIST, atol=0)
    np.testing.assert_allclose(x, xo, rtol=RTOL_HIST, atol=RTOL_HIST * np.abs(xo).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name,dev", [("c4s", "dev4"), ("c5s", "dev5")])
def test_gpu_compressed_apply(name, dev, request, P, orc):
    """Cluster-grouped tensor-core apply (22-DoF tiles; 192-DoF tiles with the
    inverse streamed from L2) against the oracle's apply.  Databases with >= 4
    patches per entry so the grouped path is taken."""
    c = request.getfixturevalue(name)
    A, ps = request.getfixturevalue(dev)
    if c.ps_size == 22:
        db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=12, seed=2, max_iters=6)
    else:  # 27 boundary partitions at 4^3 cells: use the (unpartitioned) greedy instead
        eps = orc.greedy_bisect(c.mats, 6, 12, spectral=False)["eps"]
        db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps)
    assert len(c.patches) >= 4 * db.size
    pc = P.Preconditioner.create(A, ps, db, omega=0.8)
    r = np.random.default_rng(9).uniform(-1, 1, A.rows)
    lu, piv = db.factors()
    want = orc.precond_apply(c.patches, c.w, 0.8, lu, piv, db.phi(), r)
    np.testing.assert_allclose(pc.apply(r), want, rtol=1e-10, atol=1e-12 * np.abs(want).max())


@pytest.mark.gpu
@pytest.mark.parametrize("degree,cells", [(5, 10), (6, 8), (7, 8)])
def test_gpu_tma_staged_apply_ragged_sizes(degree, cells, P, orc):
    """The TMA-staged tile apply (patches above 32 DoFs) at sizes whose k-step
    count is not a multiple of the 8-k-step stage (36, 49 and 64 DoFs: 9, 13
    and 16 k-steps; the box columns past the row are zero-filled by the TMA
    unit) and with ragged last tiles, against the oracle's apply
    (precond.cpp:58-88)."""
    ps_size = (degree + 1) ** 2
    prob = P.Problem.generate(1, cells, degree=degree)
    csr = prob.csr()
    patches, w = orc.detect(csr, ps_size)
    assert patches.shape == (cells * cells, ps_size)
    mats = orc.extract_all(csr, patches)
    A = prob.matrix()
    ps = P.PatchSet.detect(A, ps_size)
    eps = orc.greedy_bisect(mats, 6, 12, spectral=False)["eps"]
    db = P.Database.build(A, ps, P.GREEDY_L1, eps=eps)
    assert len(patches) >= 4 * db.size
    pc = P.Preconditioner.create(A, ps, db, omega=0.7)
    r = np.random.default_rng(degree).uniform(-1, 1, A.rows)
    lu, piv = db.factors()
    want = orc.precond_apply(patches, w, 0.7, lu, piv, db.phi(), r)
    np.testing.assert_allclose(pc.apply(r), want, rtol=1e-10, atol=1e-12 * np.abs(want).max())
