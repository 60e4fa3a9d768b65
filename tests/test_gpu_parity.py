"""GPU-vs-oracle parity through the C-ABI (pytest -m gpu).

The oracle (oracle/pdb_oracle.c) is itself pinned bit-for-bit to the
compiled reference in tests/test_oracle_pins.py.  Bars (BASELINE.json
north_star): patch lists, weights, extraction, LU factors, cluster ids and
representatives bit-exact; residual histories within 1e-9 relative;
Krylov iteration counts identical.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL_HIST = 1e-9  # north_star: residual histories within 1e-9 relative


class Case:
    def __init__(self, P, orc, config, cells, ps):
        self.prob = P.Problem.generate(config, cells)
        self.csr = self.prob.csr()
        self.b = self.prob.rhs()
        self.A = self.prob.matrix()
        self.ps_size = ps
        self.ps = P.PatchSet.detect(self.A, ps)
        self.patches, self.w = orc.detect(self.csr, ps)
        self.mats = orc.extract_all(self.csr, self.patches)


@pytest.fixture(scope="module")
def c1(P, orc):
    return Case(P, orc, 1, 0, 9)


@pytest.fixture(scope="module")
def c2s(P, orc):
    return Case(P, orc, 2, 16, 25)


@pytest.fixture(scope="module")
def c3s(P, orc):
    return Case(P, orc, 3, 6, 27)


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s"])
def test_detect_and_extract_bit_exact(name, request, P):
    c = request.getfixturevalue(name)
    assert c.ps.count == len(c.patches)
    assert np.array_equal(c.ps.patches(), c.patches)
    assert np.array_equal(c.ps.weights(), c.w)
    assert np.array_equal(c.ps.extract(c.A), c.mats)


def test_spmv(c1, orc):
    x = np.random.default_rng(1).uniform(-1, 1, c1.A.rows)
    y = c1.A.spmv(x)
    np.testing.assert_allclose(y, orc.spmv(c1.csr, x), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s"])
def test_spmv_bit_exact(name, request, orc):
    """The default SELL-C-sigma SpMV sums every row sequentially in CSR order
    with unfused multiply/add, as the reference spmv (sparse.cpp:50-63)."""
    c = request.getfixturevalue(name)
    x = np.random.default_rng(11).uniform(-1, 1, c.A.rows)
    assert np.array_equal(c.A.spmv(x), orc.spmv(c.csr, x))


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s"])
def test_exact_database_lu_bit_exact(name, request, P, orc):
    c = request.getfixturevalue(name)
    db = P.Database.build(c.A, c.ps, P.EXACT)
    lu, piv = db.factors()
    for k in range(0, len(c.mats), max(1, len(c.mats) // 64)):
        lo, po = orc.lu_factor(c.mats[k])
        assert np.array_equal(lu[k], lo) and np.array_equal(piv[k], po), k
    assert np.array_equal(db.phi(), np.arange(len(c.mats)))
    assert np.array_equal(db.representatives(), c.mats)


def _eps_for(orc, mats, lo, hi, spectral):
    return orc.greedy_bisect(mats, lo, hi, spectral=spectral)["eps"]


@pytest.mark.parametrize("spectral", [False, True])
@pytest.mark.parametrize("best_match", [False, True])
def test_greedy_bit_exact(c1, P, orc, spectral, best_match):
    eps = _eps_for(orc, c1.mats, 46, 57, spectral)  # 5% of 1024 patches (config 1)
    want = orc.greedy(c1.mats, eps, spectral=spectral, best_match=best_match)
    db = P.Database.build(c1.A, c1.ps, P.GREEDY_SPECTRAL if spectral else P.GREEDY_L1, eps=eps,
                          best_match=int(best_match))
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])
    assert np.array_equal(db.representatives(), want["reps"])
    lu, piv = db.factors()
    assert np.array_equal(lu, want["lu"]) and np.array_equal(piv, want["piv"])


@pytest.mark.parametrize("spectral", [False, True])
def test_greedy_bisect_bit_exact(c1, P, orc, spectral):
    want = orc.greedy_bisect(c1.mats, 46, 57, spectral=spectral)
    db, eps = P.Database.build_to_size(c1.A, c1.ps, 46, 57, P.GREEDY_SPECTRAL if spectral else P.GREEDY_L1)
    assert eps == want["eps"]
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])


def test_greedy_l1_larger(c3s, P, orc):
    want = orc.greedy_bisect(c3s.mats, 9, 13, spectral=False)
    db = P.Database.build(c3s.A, c3s.ps, P.GREEDY_L1, eps=want["eps"])
    assert np.array_equal(db.phi(), want["phi"])


@pytest.mark.parametrize("method,variant", [(3, 0), (4, 1), (5, 2)])
def test_kmeans_partitioned_bit_exact(c1, P, orc, method, variant):
    want = orc.partitioned_build(c1.mats, 51, variant, seed=42, max_iters=50)
    db = P.Database.build(c1.A, c1.ps, method, db_size=51, seed=42, max_iters=50)
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])
    assert np.array_equal(db.representatives(), want["reps"])
    lu, piv = db.factors()
    assert np.array_equal(lu, want["lu"]) and np.array_equal(piv, want["piv"])


@pytest.mark.parametrize("name", ["c2s", "c3s"])
def test_kmeans_spectral_larger_patches(name, request, P, orc):
    """Spectral criterion at p_s = 25 and 27 (the register-tiled kernels)."""
    c = request.getfixturevalue(name)
    budget = 16 if c.ps_size == 25 else 30
    want = orc.partitioned_build(c.mats, budget, 1, seed=3, max_iters=8)
    db = P.Database.build(c.A, c.ps, P.KMEANS_SPECTRAL, db_size=budget, seed=3, max_iters=8)
    assert np.array_equal(db.phi(), want["phi"])
    assert np.array_equal(db.representatives(), want["reps"])


def test_greedy_spectral_c3(c3s, P, orc):
    want = orc.greedy_bisect(c3s.mats, 40, 50, spectral=True)
    db = P.Database.build(c3s.A, c3s.ps, P.GREEDY_SPECTRAL, eps=want["eps"])
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])


def test_kmeans_entrywise_c2(c2s, P, orc):
    want = orc.partitioned_build(c2s.mats, 64, 0, seed=7, max_iters=30)
    db = P.Database.build(c2s.A, c2s.ps, P.KMEANS_ENTRYWISE, db_size=64, seed=7, max_iters=30)
    assert np.array_equal(db.phi(), want["phi"])
    assert np.array_equal(db.representatives(), want["reps"])


def test_bootstrap_bit_exact(P, orc):
    prob = P.Problem.generate(1, 12)
    csr = prob.csr()
    A = prob.matrix()
    ps = P.PatchSet.detect(A, 9)
    patches, _ = orc.detect(csr, 9)
    mats = orc.extract_all(csr, patches)
    eps = orc.greedy_bisect(mats, 10, 14, spectral=True)["eps"]
    want = orc.bootstrapped(mats, eps, 2, 20)
    db = P.Database.build(A, ps, P.BOOTSTRAP, eps=eps, max_iters=20)
    assert db.size == want["m"]
    assert np.array_equal(db.phi(), want["phi"])


def _oracle_pc(orc, c, db=None):
    if db is None:
        f = [orc.lu_factor(m) for m in c.mats]
        return np.stack([a for a, _ in f]), np.stack([p for _, p in f]), None
    lu, piv = db.factors()
    return lu, piv, db.phi()


@pytest.mark.parametrize("compressed", [False, True])
@pytest.mark.parametrize("name", ["c1", "c2s", "c3s"])
def test_precond_apply(name, compressed, request, P, orc):
    c = request.getfixturevalue(name)
    budget = 12 if c.ps_size in (9, 25) else 32  # >= 9 boundary partitions in 2D, 27 in 3D
    db = P.Database.build(c.A, c.ps, P.KMEANS_ENTRYWISE, db_size=budget) if compressed else None
    pc = P.Preconditioner.create(c.A, c.ps, db, omega=0.7)
    r = np.random.default_rng(3).uniform(-1, 1, c.A.rows)
    lu, piv, phi = _oracle_pc(orc, c, db)
    want = orc.precond_apply(c.patches, c.w, 0.7, lu, piv, phi, r)
    np.testing.assert_allclose(pc.apply(r), want, rtol=1e-11, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("compressed", [False, True])
@pytest.mark.parametrize("name", ["c1", "c3s"])
def test_relax_history(name, compressed, request, P, orc):
    """Config 1: damped Richardson, 20 sweeps; history within 1e-9 relative."""
    c = request.getfixturevalue(name)
    omega = 0.8
    if compressed:
        eps = _eps_for(orc, c.mats, max(1, int(0.045 * len(c.mats))), max(2, int(0.055 * len(c.mats)) + 1), False)
        db = P.Database.build(c.A, c.ps, P.GREEDY_L1, eps=eps)
    else:
        db = None
    pc = P.Preconditioner.create(c.A, c.ps, db, omega=omega)
    x, hist = pc.relax(c.A, c.b, np.zeros_like(c.b), 20)
    lu, piv, phi = _oracle_pc(orc, c, db)
    xo, ho = orc.relax(c.csr, c.patches, c.w, omega, lu, piv, phi, c.b, np.zeros_like(c.b), 20)
    np.testing.assert_allclose(hist, ho, rtol=RTOL_HIST, atol=0)
    np.testing.assert_allclose(x, xo, rtol=RTOL_HIST, atol=RTOL_HIST * np.abs(xo).max())


def test_gmres_iterations(c1, P, orc):
    pc = P.Preconditioner.create(c1.A, c1.ps, None, omega=1.0)
    x, rep = P.gmres(c1.A, c1.b, pc)
    lu, piv, _ = _oracle_pc(orc, c1)
    xo, ro = orc.gmres(c1.csr, c1.b, dict(patches=c1.patches, weights=c1.w, omega=1.0, lu=lu, piv=piv, phi=None))
    assert rep.iterations == ro["iterations"] and rep.restarts == ro["restarts"]
    assert rep.converged == ro["converged"]
    np.testing.assert_allclose(rep.residual_history, ro["residual_history"], rtol=1e-7)


def test_pcg_iterations(c2s, P, orc):
    db = P.Database.build(c2s.A, c2s.ps, P.KMEANS_ENTRYWISE, db_size=16)
    pc = P.Preconditioner.create(c2s.A, c2s.ps, db, omega=1.0)
    x, rep = P.pcg(c2s.A, c2s.b, pc, tol=1e-8)
    lu, piv, phi = _oracle_pc(orc, c2s, db)
    xo, ro = orc.pcg(c2s.csr, c2s.b, dict(patches=c2s.patches, weights=c2s.w, omega=1.0, lu=lu, piv=piv, phi=phi),
                     tol=1e-8)
    assert rep.converged and ro["converged"]
    assert rep.iterations == ro["iterations"]  # north_star: identical iteration counts
    # CG amplifies last-bit differences of the dot products over many
    # iterations; the early history must agree tightly.
    np.testing.assert_allclose(rep.residual_history[:10], ro["residual_history"][:10], rtol=1e-9)


@pytest.mark.parametrize("compressed", [False, True])
def test_pcg_reproducible_bitwise(c2s, P, orc, monkeypatch, compressed):
    """pdb_pcg_solve_ex(PDB_PCG_REPRODUCIBLE): the oracle's PCG sequence bit for
    bit -- identical iteration count, residual history and solution."""
    db = P.Database.build(c2s.A, c2s.ps, P.KMEANS_ENTRYWISE, db_size=16) if compressed else None
    monkeypatch.setenv("PDB_APPLY", "lu")
    pc = P.Preconditioner.create(c2s.A, c2s.ps, db, omega=1.0)
    monkeypatch.delenv("PDB_APPLY")
    x, rep = P.pcg(c2s.A, c2s.b, pc, tol=1e-10, reproducible=True)
    if compressed:
        lu, piv, phi = _oracle_pc(orc, c2s, db)
    else:
        lu = np.stack([orc.lu_factor(m)[0] for m in c2s.mats])
        piv = np.stack([orc.lu_factor(m)[1] for m in c2s.mats])
        phi = None
    xo, ro = orc.pcg(c2s.csr, c2s.b, dict(patches=c2s.patches, weights=c2s.w, omega=1.0, lu=lu, piv=piv, phi=phi),
                     tol=1e-10)
    assert rep.iterations == ro["iterations"]
    assert np.array_equal(np.asarray(rep.residual_history), ro["residual_history"])
    assert np.array_equal(x, xo)


def test_singular_patch_error(c1, P, orc):
    rp, ci, v = [a.copy() for a in c1.csr]
    # zero one cell-interior row (its stored entries stay in the pattern)
    k = 37
    row = c1.patches[k][4]
    v[rp[row]:rp[row + 1]] = 0.0
    A = P.Matrix.from_csr(rp, ci, v)
    ps = P.PatchSet.detect(A, 9)
    with pytest.raises(P.PatchdbError) as e:
        P.Database.build(A, ps, P.EXACT)
    assert e.value.status == P.PDB_ERR_SINGULAR_MATRIX
    mats = orc.extract_all((rp, ci, v), c1.patches)
    with pytest.raises(Exception) as eo:
        orc.lu_factor(mats[k])
    assert e.value.message == f"patch {k}: " + eo.value.message
    with pytest.raises(P.PatchdbError) as e2:
        P.Preconditioner.create(A, ps, None)
    assert e2.value.status == P.PDB_ERR_SINGULAR_MATRIX and e2.value.message == e.value.message


def test_error_paths(c1, P):
    with pytest.raises(P.PatchdbError) as e:
        P.PatchSet.detect(c1.A, 7)
    assert e.value.status == P.PDB_ERR_NO_PATCHES_FOUND
    assert e.value.message == "no row has exactly 7 stored entries"
    with pytest.raises(P.PatchdbError) as e:
        P.Database.build(c1.A, c1.ps, P.KMEANS_ENTRYWISE, db_size=5)
    assert e.value.status == P.PDB_ERR_BUDGET_TOO_SMALL
    with pytest.raises(P.PatchdbError) as e:
        P.Database.build(c1.A, c1.ps, P.GREEDY_L1, eps=0.0)
    assert e.value.status == P.PDB_ERR_INVALID_ARGUMENT


def test_identity_phi_compressed_equals_exact(c1, P):
    """SPEC acceptance 3: Exact == Compressed when m_p = n_p with identity phi."""
    db = P.Database.build(c1.A, c1.ps, P.EXACT)
    pe = P.Preconditioner.create(c1.A, c1.ps, None)
    pcmp = P.Preconditioner.create(c1.A, c1.ps, db)
    r = np.random.default_rng(5).uniform(-1, 1, c1.A.rows)
    assert np.array_equal(pe.apply(r), pcmp.apply(r))


@pytest.mark.parametrize("sweeps", [1, 3])
def test_pipelined_host_relax_matches_device_path(P, monkeypatch, sweeps):
    """pdb_relax overlaps the b upload with the chunked residual (8 chunks of
    whole SELL windows at 64x64 cells); the result must be bitwise the
    unpipelined path's (same kernels, same row sums)."""
    prob = P.Problem.generate(2, 64)
    A = prob.matrix()
    ps = P.PatchSet.detect(A, 25)
    db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=16)
    pc = P.Preconditioner.create(A, ps, db, omega=0.9)
    b = prob.rhs()
    x0 = np.random.default_rng(2).uniform(-1, 1, A.rows)
    got, _ = pc.relax(A, b, x0, sweeps, history=False)
    monkeypatch.setenv("PDB_PIPELINE", "0")
    want, _ = pc.relax(A, b, x0, sweeps, history=False)
    assert np.array_equal(got, want)
    assert not np.array_equal(got, x0)


@pytest.mark.parametrize("method", [2, 3, 4])
def test_database_export_import_round_trip(c1, P, tmp_path, method):
    """pdb_database_import(pdb_database_export(db)) == db bit for bit (phi,
    representatives, recomputed factors), and it drives the same sweep."""
    kw = dict(eps=2.0) if method == 2 else dict(db_size=51, seed=42, max_iters=20)
    db = P.Database.build(c1.A, c1.ps, method, **kw)
    js, bn = str(tmp_path / "db.json"), str(tmp_path / "db.bin")
    db.export(js, bn)
    db2 = P.Database.load(js, bn)
    assert db2.size == db.size and db2.n_patches == db.n_patches
    assert np.array_equal(db2.phi(), db.phi())
    assert np.array_equal(db2.representatives(), db.representatives())
    l1, p1 = db.factors()
    l2, p2 = db2.factors()
    assert np.array_equal(l1, l2) and np.array_equal(p1, p2)
    pc1 = P.Preconditioner.create(c1.A, c1.ps, db, omega=0.8)
    pc2 = P.Preconditioner.create(c1.A, c1.ps, db2, omega=0.8)
    x1, h1 = pc1.relax(c1.A, c1.b, np.zeros_like(c1.b), 5)
    x2, h2 = pc2.relax(c1.A, c1.b, np.zeros_like(c1.b), 5)
    assert np.array_equal(x1, x2) and np.array_equal(h1, h2)


def _ragged_csr(seed, n):
    """Random CSR with empty rows, single entries, rows longer than a warp item
    (> 256) and than a SELL step group, unsorted lengths."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.choice([0, 1, 3, 17, 50, 300, 1100], size=n, p=[0.1, 0.2, 0.2, 0.2, 0.2, 0.08, 0.02]), n)
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(n, size=int(k), replace=False)) for k in lens if k > 0]).astype(np.int64)
    v = rng.uniform(-1, 1, rp[-1])
    return rp, ci, v


@pytest.mark.parametrize("seed,n", [(1, 37), (2, 5000), (3, 9001)])
def test_spmv_ragged_rows(P, orc, monkeypatch, seed, n):
    """Empty, single-entry and long rows: the SELL kernel stays bitwise the
    reference sum; the CSR warp-item (v5, long-row path) and row-group (v2)
    kernels agree to rounding."""
    csr = _ragged_csr(seed, n)
    A = P.Matrix.from_csr(*csr)
    x = np.random.default_rng(seed + 10).uniform(-1, 1, n)
    want = orc.spmv(csr, x)
    assert np.array_equal(A.spmv(x), want)
    for ver in ("5", "2"):
        monkeypatch.setenv("PDB_SPMV_VERSION", ver)
        np.testing.assert_allclose(A.spmv(x), want, rtol=1e-12, atol=1e-12)


def _banded_csr(seed, n, band):
    """Band matrix clipped at both ends: a few repeated column patterns
    (row + offsets), i.e. every row in a column-pattern class."""
    rows = [np.arange(max(0, i - band), min(n, i + band + 1)) for i in range(n)]
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    return rp, np.concatenate(rows).astype(np.int64), np.random.default_rng(seed).uniform(-1, 1, rp[-1])


@pytest.mark.parametrize("seed,n,band", [(4, 3000, 7), (5, 20000, 40), (6, 200, 3)])
def test_spmv_pattern_classes(P, orc, monkeypatch, seed, n, band):
    """Rows stored without column indices (every row in a column-pattern
    class): bitwise the reference sum, and equal to the explicit-column copy."""
    csr = _banded_csr(seed, n, band)
    A = P.Matrix.from_csr(*csr)
    info = A.sell_info()
    assert info["classes"] >= 1 and info["col_entries"] == 0
    x = np.random.default_rng(seed + 10).uniform(-1, 1, n)
    want = orc.spmv(csr, x)
    assert np.array_equal(A.spmv(x), want)
    monkeypatch.setenv("PDB_SELL_CLASSES", "0")
    B = P.Matrix.from_csr(*csr)
    assert B.sell_info()["classes"] == 0 and B.sell_info()["col_entries"] >= csr[0][-1]
    assert np.array_equal(B.spmv(x), want)


def test_spmv_unclassed_rows_keep_columns(P, orc):
    """Rows that do not share column patterns (more than n/8 patterns): the
    copy keeps explicit column indices."""
    rp, ci, v = _banded_csr(7, 4000, 5)
    ci = ci.copy()
    for i in range(100, 3900, 4):  # 950 rows: first column moved to a row-dependent place
        ci[rp[i]] = (7 * i) % 90
    A = P.Matrix.from_csr(rp, ci, v)
    assert A.sell_info()["classes"] == 0
    x = np.random.default_rng(8).uniform(-1, 1, 4000)
    assert np.array_equal(A.spmv(x), orc.spmv((rp, ci, v), x))


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s"])
def test_fem_rows_are_classed(name, request):
    """On the structured FEM lattices every row falls into a column-pattern
    class (one per node type, Dirichlet identity rows): the residual streams
    no column indices."""
    c = request.getfixturevalue(name)
    info = c.A.sell_info()
    assert 1 <= info["classes"] <= 64 and info["col_entries"] == 0


@pytest.mark.parametrize("cells", [60, 120, 180, 250, 512])
def test_gmres_fused_mgs_matches_per_vector_launches(P, cells, monkeypatch):
    """The cooperative MGS kernel (vector in registers, one launch per Arnoldi
    step; E = 1..16 elements per thread across these sizes) against the
    per-i dot + axpy launches: same iteration count; the dot products sum in
    another order, so histories agree to rounding (1e-7 relative after 40
    restarted iterations, as against the reference)."""
    p = P.Problem.assemble(dict(cells=cells, degree=2))
    A = p.matrix()
    ps = P.PatchSet.detect(A, 9)
    pc = P.Preconditioner.create(A, ps)
    b = p.rhs()
    x1, r1 = P.gmres(A, b, pc, restart=12, tol=1e-10, max_iters=40)
    monkeypatch.setenv("PDB_MGS", "0")
    x0, r0 = P.gmres(A, b, pc, restart=12, tol=1e-10, max_iters=40)
    assert r1.iterations == r0.iterations
    np.testing.assert_allclose(r1.residual_history, r0.residual_history, rtol=1e-7)
    np.testing.assert_allclose(x1, x0, rtol=0, atol=1e-8 * np.abs(x0).max())


@pytest.mark.parametrize("cfg,cells,ps,k,method", [(2, 48, 25, 24, "KMEANS_SPECTRAL"), (1, 24, 9, 12, "KMEANS_SPECTRAL"),
                                                   (3, 8, 27, 40, "KMEANS_SPECTRAL"), (4, 16, 22, 16, "KMEANS_SPECTRAL"),
                                                   (2, 32, 25, 16, "BOOTSTRAP"), (1, 32, 9, 0, "BOOTSTRAP"),
                                                   (4, 12, 22, 0, "BOOTSTRAP")])
def test_kmeans_assignment_pruning_changes_nothing(P, cfg, cells, ps, k, method, monkeypatch):
    """Cutting losing pairs' power iterations short (their Rayleigh quotient
    already exceeds the patch's distance to its current centroid) leaves the
    whole k-means run bitwise unchanged: phi, representatives, factors."""
    prob = P.Problem.generate(cfg, cells)
    A = prob.matrix()
    pset = P.PatchSet.detect(A, ps)
    kw = dict(db_size=k, seed=7, max_iters=30) if method != "BOOTSTRAP" else dict(eps=1e-3 if k else 0.3, max_iters=10)
    on = P.Database.build(A, pset, getattr(P, method), **kw)
    monkeypatch.setenv("PDB_KMEANS_PRUNE", "0")
    off = P.Database.build(A, pset, getattr(P, method), **kw)
    assert np.array_equal(on.phi(), off.phi())
    assert np.array_equal(on.representatives(), off.representatives())
    for a, b in zip(on.factors(), off.factors()):
        assert np.array_equal(a, b)
    assert on.work()["power_iters"] <= off.work()["power_iters"]  # executed power iterations
    # the bound pass in patch order (in-block refill) instead of the sorted work order
    monkeypatch.setenv("PDB_KMEANS_PRUNE", "1")
    monkeypatch.setenv("PDB_DIAG_SORT", "0")
    plain = P.Database.build(A, pset, getattr(P, method), **kw)
    assert np.array_equal(on.phi(), plain.phi())
    assert np.array_equal(on.representatives(), plain.representatives())
    assert on.work()["power_iters"] == plain.work()["power_iters"]


@pytest.mark.parametrize("best_match", [False, True])
@pytest.mark.parametrize("cfg,cells,ps,eps", [(1, 32, 9, 1e-2), (1, 32, 9, 0.3), (2, 24, 25, 0.05), (3, 6, 27, 0.2)])
def test_greedy_spectral_pruning_changes_nothing(P, cfg, cells, ps, eps, best_match, monkeypatch):
    """Greedy only looks at distances below eps, so pairs cut short once their
    Rayleigh quotient proves d > eps leave the database unchanged."""
    prob = P.Problem.generate(cfg, cells)
    A = prob.matrix()
    pset = P.PatchSet.detect(A, ps)
    on = P.Database.build(A, pset, P.GREEDY_SPECTRAL, eps=eps, best_match=best_match)
    monkeypatch.setenv("PDB_GREEDY_PRUNE", "0")
    off = P.Database.build(A, pset, P.GREEDY_SPECTRAL, eps=eps, best_match=best_match)
    assert on.size == off.size
    assert np.array_equal(on.phi(), off.phi())
    assert np.array_equal(on.representatives(), off.representatives())
    assert on.work()["power_iters"] <= off.work()["power_iters"]


@pytest.mark.parametrize("name", ["c1", "c2s"])
def test_objective_and_compressibility_curve(name, request, P, ref):
    """pdb_database_objective / pdb_compressibility_curve against the
    reference build on the same matrix: the objective bitwise (same distances,
    same summation order), the curve's sizes and ratios exactly."""
    c = request.getfixturevalue(name)
    rm = ref.matrix(c.csr)
    rps = rm.detect(c.ps_size)
    grid = [1e-3, 1e-2, 0.1, 0.5, 2.0]
    for method, spectral in ((P.GREEDY_L1, False), (P.GREEDY_SPECTRAL, True)):
        assert P.compressibility_curve(c.A, c.ps, method, grid) == rps.curve(rm, spectral, grid)
    for method, kw in ((P.GREEDY_SPECTRAL, dict(eps=0.5)), (P.KMEANS_SPECTRAL, dict(db_size=12, seed=3, max_iters=6))):
        db = P.Database.build(c.A, c.ps, method, **kw)
        rdb = rps.build(rm, method, **kw)
        assert db.objective(c.A, c.ps, 0.25) == rps.objective(rm, rdb, 0.25)
    with pytest.raises(P.PatchdbError):
        db.objective(c.A, c.ps, -1.0)
    with pytest.raises(P.PatchdbError):
        P.compressibility_curve(c.A, c.ps, P.GREEDY_L1, [0.1, 0.01])


@pytest.mark.parametrize("name,ps", [("c1", 9), ("c2s", 25), ("c3s", 27)])
def test_l1_tiled_kernels_match_thread_per_patch(name, ps, request, P, monkeypatch):
    """The tiled l1 kernels (64 patches x 32 entries per block, staged k-chunks)
    and the candidate-bit batch resolution give bitwise the databases of the
    thread-per-patch kernels and the one-warp resolution: greedy first / best
    match and entrywise k-means (assignment by argmin and by pairs)."""
    case = request.getfixturevalue(name)
    A, pset = case.A, case.ps
    builds = [dict(method=P.GREEDY_L1, eps=e, best_match=bm) for e in (0.5, 2.0) for bm in (False, True)]
    builds.append(dict(method=P.KMEANS_ENTRYWISE, db_size=max(30, pset.count // 8), seed=3, max_iters=12))
    for kw in builds:
        kw = dict(kw)
        method = kw.pop("method")
        monkeypatch.setenv("PDB_L1_TILED", "1")
        a = P.Database.build(A, pset, method, **kw)
        monkeypatch.setenv("PDB_L1_TILED", "0")
        monkeypatch.setenv("PDB_RESOLVE_BITS", "0")  # and the one-warp batch resolution
        b = P.Database.build(A, pset, method, **kw)
        monkeypatch.delenv("PDB_L1_TILED")
        monkeypatch.delenv("PDB_RESOLVE_BITS")
        assert a.size == b.size, kw
        assert np.array_equal(a.phi(), b.phi()), kw
        assert np.array_equal(a.representatives(), b.representatives()), kw


def _front_csr(seed, groups, per_group, ps):
    """Patches emitted out of front order, some sharing a front.  Row 0..G-1
    are hubs (not candidates: ps + 1 entries); each patch is {hub g} + ps - 1
    private DoFs whose rows hold exactly that set, so the patch is emitted at
    its first private row with front g.  Patches are laid out so emission order
    (ascending first private row) is a shuffled order of the fronts."""
    rng = np.random.default_rng(seed)
    fronts = np.repeat(np.arange(groups), per_group)
    rng.shuffle(fronts)
    n = groups + len(fronts) * (ps - 1)
    rows = [[] for _ in range(n)]
    nxt = groups
    for g in fronts:
        priv = list(range(nxt, nxt + ps - 1))
        nxt += ps - 1
        for r in priv:
            rows[r] = [int(g)] + priv
    for g in range(groups):
        rows[g] = sorted(set([g] + [int(c) for c in rng.choice(np.arange(groups, n), size=ps, replace=False)]))
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate([np.array(r, dtype=np.int64) for r in rows])
    v = rng.uniform(1, 2, rp[-1])
    return rp, ci, v


@pytest.mark.parametrize("seed,groups,per_group,ps", [(1, 40, 1, 3), (2, 30, 3, 4), (3, 7, 40, 3), (4, 200, 2, 5)])
def test_detect_front_order_and_ties(P, ref, seed, groups, per_group, ps):
    """Detection sorts patches by front (std::sort, patch.cpp:82-83).  Distinct
    fronts emitted out of order take the device sort; shared fronts take
    libstdc++'s own unstable std::sort on the host: either way the patch list
    equals the reference library's on the same matrix."""
    csr = _front_csr(seed, groups, per_group, ps)
    A = P.Matrix.from_csr(*csr)
    got = P.PatchSet.detect(A, ps)
    rps = ref.matrix(csr).detect(ps)
    assert got.count == rps.count == groups * per_group
    assert np.array_equal(got.patches(), rps.patches().reshape(got.patches().shape))
    assert np.array_equal(got.weights(), rps.weights(len(csr[0]) - 1))


@pytest.mark.parametrize("kind", ["ragged", "banded", "c1", "c3s", "c4s", "c5s"])
def test_sell_device_build_equals_host_build(P, orc, monkeypatch, kind):
    """The SELL copy built on the device (sell_build.cu) has the host build's
    classes, slices and stored entries, and its residual is bitwise the
    reference sum, on unclassed (ragged), banded and FEM matrices."""
    if kind == "ragged":
        csr = _ragged_csr(5, 7000)
    elif kind == "banded":
        csr = _banded_csr(6, 20000, 7)
    else:
        cfg, cells = {"c1": (1, 0), "c3s": (3, 6), "c4s": (4, 16), "c5s": (5, 3)}[kind]
        csr = P.Problem.generate(cfg, cells).csr()
    n = len(csr[0]) - 1
    x = np.random.default_rng(n).uniform(-1, 1, n)
    want = orc.spmv(csr, x)
    A = P.Matrix.from_csr(*csr)  # device build (default)
    monkeypatch.setenv("PDB_SELL_DEVICE", "0")
    H = P.Matrix.from_csr(*csr)  # host build
    assert A.sell_info() == H.sell_info()
    if kind in ("banded", "c1", "c3s"):
        assert A.sell_info()["classes"] >= 1
    assert np.array_equal(A.spmv(x), want)
    assert np.array_equal(H.spmv(x), want)
