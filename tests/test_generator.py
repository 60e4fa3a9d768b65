"""The seeded input generator (host-only, no GPU): sizes of the BASELINE
configs, agreement with the reference assembler on uniform meshes,
determinism, Dirichlet-row conventions."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_config1_sizes(P):
    p = P.Problem.generate(1)
    assert (p.ndofs, p.nnz) == (4225, 63257)  # SURVEY.md §8d (= reference assembler pattern)


def test_config2_sizes(P):
    p = P.Problem.generate(2)
    assert (p.ndofs, p.nnz) == (1050625, 37642321)


def test_config3_pattern_small(P):
    p = P.Problem.generate(3, 8)
    assert p.ndofs == 17 ** 3


def test_determinism_and_seed(P):
    a = P.Problem.generate(2, 16)
    b = P.Problem.generate(2, 16)
    c = P.Problem.generate(2, 16, seed=7)
    ca, cb, cc = a.csr(), b.csr(), c.csr()
    assert all(np.array_equal(x, y) for x, y in zip(ca, cb))
    assert np.array_equal(a.rhs(), b.rhs())
    assert np.array_equal(ca[1], cc[1]) and not np.array_equal(ca[2], cc[2])


def test_thread_count_invariance(P):
    a = P.Problem.generate(3, 6, threads=1).csr()
    b = P.Problem.generate(3, 6, threads=7).csr()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_dirichlet_rows_and_rhs(P):
    p = P.Problem.generate(1)
    rp, ci, v = p.csr()
    b = p.rhs()
    npa = 65
    for i in range(p.ndofs):
        ix, iy = i % npa, i // npa
        if ix in (0, npa - 1) or iy in (0, npa - 1):
            assert rp[i + 1] - rp[i] == 1 and ci[rp[i]] == i and v[rp[i]] == 1.0 and b[i] == 0.0
    interior = [i for i in range(p.ndofs) if 0 < i % npa < npa - 1 and 0 < i // npa < npa - 1]
    assert np.all(np.abs(b[interior]) <= 1.0)


@pytest.mark.parametrize("dim,cells,degree", [(2, 8, 2), (2, 4, 4), (3, 3, 2)])
def test_uniform_mesh_matches_reference_assembler(P, ref, dim, cells, degree):
    """jitter 0, rho = 1: same pattern and values (to rounding) as fem.cpp:248-346."""
    ours = P.Problem.generate(1 if dim == 2 else 3, cells, jitter=0.0, degree=degree).csr()
    rp, ci, v = ref.assemble(dim, cells, degree, coeff_kind=0, value=1.0)
    assert np.array_equal(ours[0], rp) and np.array_equal(ours[1], ci)
    np.testing.assert_allclose(ours[2], v, rtol=1e-12, atol=1e-12 * np.abs(v).max())


def test_interior_block_symmetric(P):
    rp, ci, v = P.Problem.generate(2, 8).csr()
    n = len(rp) - 1
    d = np.zeros((n, n))
    for i in range(n):
        d[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    bnd = np.array([rp[i + 1] - rp[i] == 1 for i in range(n)])
    inner = d[np.ix_(~bnd, ~bnd)]
    np.testing.assert_allclose(inner, inner.T, rtol=1e-12, atol=1e-12 * np.abs(inner).max())


def test_random_block_coefficient_levels(P):
    p = P.Problem.generate(2, 32)
    v = p.csr()[2]
    # four coefficient levels spanning three decades show up in the diagonal scale
    rp = p.csr()[0]
    diag_scale = np.abs(v[rp[:-1]])
    assert diag_scale.max() / diag_scale[diag_scale > 1.0 + 1e-12].min() > 100


def test_invalid_generator_options(P):
    with pytest.raises(P.PatchdbError) as e:
        P.Problem.generate(1, degree=0)
    assert e.value.status == P.PDB_ERR_INVALID_DEGREE
    with pytest.raises(P.PatchdbError) as e:
        P.Problem.generate(1, jitter=0.6)
    assert e.value.status == P.PDB_ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("cfg,cells", [(1, 0), (2, 16), (3, 6), (4, 8), (5, 3)])
def test_standalone_generator_library_matches(P, cfg, cells):
    """inputs/libpdbgen.so (the generator without libpatchdb, used by the
    reference arm of bench.py) produces the same bytes as pdb_problem_generate."""
    sys.path.insert(0, os.path.join(ROOT, "inputs"))
    import pdbgen
    g = pdbgen.Generated(cfg, cells)
    p = P.Problem.generate(cfg, cells)
    assert all(np.array_equal(x, y) for x, y in zip(g.csr(), p.csr()))
    assert np.array_equal(g.rhs(), p.rhs())


@pytest.mark.parametrize("cfg,cells,ranks", [(1, 8, 2), (1, 9, 4), (2, 8, 3), (3, 6, 2), (3, 7, 3), (4, 8, 2),
                                             (4, 9, 4), (5, 4, 2)])
def test_slab_rows_equal_global_rows(P, cfg, cells, ranks):
    """pdb_problem_generate_slab: each rank's rows are bitwise the same rows of
    the whole problem (global column ids), the right-hand side too, and the
    slabs' rows cover every row (neighbours share their face rows)."""
    g = P.Problem.generate(cfg, cells)
    rp, ci, v = g.csr()
    b = g.rhs()
    seen = np.zeros(g.ndofs, bool)
    for r in range(ranks):
        s = P.Problem.generate_slab(cfg, cells, r, ranks)
        assert s.rows_global == g.ndofs
        rows = s.row_ids()
        srp, sci, sv = s.csr()
        assert len(rows) == s.ndofs
        lens = rp[rows + 1] - rp[rows]
        assert np.array_equal(np.diff(srp), lens)
        take = np.concatenate([np.arange(rp[i], rp[i + 1]) for i in rows])
        assert np.array_equal(sci, ci[take])
        assert np.array_equal(sv.view(np.uint64), v[take].view(np.uint64))
        assert np.array_equal(s.rhs(), b[rows])
        seen[rows] = True
    assert seen.all()


def test_slab_errors(P):
    with pytest.raises(P.PatchdbError):
        P.Problem.generate_slab(3, 6, 0, 4)  # 6 cells over 4 ranks: < 2 layers each
    with pytest.raises(P.PatchdbError):
        P.Problem.generate_slab(3, 6, 2, 2)
    s = P.Problem.generate_slab(3, 6, 0, 2)
    with pytest.raises(P.PatchdbError):
        s.matrix()
