"""Rank-local multi-GPU sweep (csrc/slab.cu) on one GPU as an emulated group
(pytest -m gpu): W ranks, each built only from its own slab rows
(pdb_problem_generate_slab), patches detected locally, weights / ownership /
exchange lists set up with the neighbours, exchanges as device copies.  After
k sweeps the owned DoFs of all ranks must be BITWISE the single-GPU
pdb_relax of the whole problem (the interface partial sums continue in the
reference's ascending patch order, precond.cpp:81-86), for exact and
compressed preconditioners, W = 2, 3, 8, at configs 2 and 3 (full size) and
reduced configs 1-5.  Also: every global DoF is owned by exactly one rank,
the ranks' patch ranges are consecutive, and setup rejects slabs thinner than
two cell layers.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def emulated_relax(P, sl, b, x0, sweeps):
    L = sl.local_ranks
    gids = [sl.local_dofs(i) for i in range(L)]
    bs = [torch.from_numpy(b[g].copy()).cuda() for g in gids]
    xs = [torch.from_numpy(x0[g].copy()).cuda() for g in gids]
    sl.relax_device([t.data_ptr() for t in bs], [t.data_ptr() for t in xs], sweeps)
    torch.cuda.synchronize()
    x = np.full_like(x0, np.nan)
    owner = np.full(len(x0), -1)
    for i in range(L):
        own = sl.owned(i)
        g = gids[i][own]
        assert (owner[g] < 0).all(), "a DoF owned twice"
        owner[g] = i
        x[g] = xs[i].cpu().numpy()[own]
    return x, owner


CASES = [  # config, cells, patch size, ranks, database
    (2, 0, 25, 2, "kmeans"), (2, 0, 25, 8, "exact"), (3, 0, 27, 3, "greedy"), (3, 0, 27, 8, "exact"),
    (1, 0, 9, 3, "greedy"), (2, 16, 25, 2, "exact"), (3, 8, 27, 4, "greedy"), (4, 8, 22, 2, "kmeans"),
    (5, 4, 192, 2, "exact"),
]


@pytest.mark.parametrize("cfg,cells,ps,ranks,method", CASES)
def test_emulated_slabs_match_single_gpu(P, cfg, cells, ps, ranks, method):
    g = P.Problem.generate(cfg, cells)
    A = g.matrix()
    pset = P.PatchSet.detect(A, ps)
    db = None
    if method == "greedy":
        db = P.Database.build(A, pset, P.GREEDY_L1, eps=0.5 if cfg != 3 else 0.137)
    elif method == "kmeans":
        db = P.Database.build(A, pset, P.KMEANS_ENTRYWISE, db_size=64, seed=42, max_iters=5)
    pc = P.Preconditioner.create(A, pset, db, omega=0.9)
    b = g.rhs()
    x0 = np.random.default_rng(cfg).uniform(-1, 1, len(b))
    want, _ = pc.relax(A, b, x0, 3, history=False)
    slabs = [P.Problem.generate_slab(cfg, cells, r, ranks) for r in range(ranks)]
    sl = P.Slab.create(slabs, 0, ranks, ps, db, omega=0.9)
    info = [sl.info(i) for i in range(ranks)]
    assert sum(f["n_patches"] for f in info) == pset.count
    assert [f["first_patch"] for f in info] == list(np.cumsum([0] + [f["n_patches"] for f in info[:-1]]))
    got, owner = emulated_relax(P, sl, b, x0, 3)
    assert (owner >= 0).all(), "a DoF without owner"
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_single_rank_slab_equals_relax(P):
    g = P.Problem.generate(3, 6)
    A = g.matrix()
    pset = P.PatchSet.detect(A, 27)
    pc = P.Preconditioner.create(A, pset, None, omega=1.0)
    b = g.rhs()
    x0 = np.zeros_like(b)
    want, _ = pc.relax(A, b, x0, 4, history=False)
    sl = P.Slab.create([P.Problem.generate_slab(3, 6, 0, 1)], 0, 1, 27)
    got, _ = emulated_relax(P, sl, b, x0, 4)
    assert np.array_equal(got, want)


def test_thin_slabs_rejected(P):
    with pytest.raises(P.PatchdbError):
        [P.Problem.generate_slab(3, 6, r, 4) for r in range(4)]


@pytest.mark.parametrize("cfg,cells,ps,ranks,r", [(3, 12, 27, 4, 1), (5, 8, 192, 4, 2)])
def test_subset_group_one_rank_slice(P, cfg, cells, ps, ranks, r):
    """A slice of a larger job on one GPU: rank r's slab plus one-cell-layer
    neighbours (pdb_problem_generate_cells) as an emulated subset.  After one
    sweep from the same x0, rank r's owned DoFs are bitwise the whole
    problem's single-GPU sweep (exact patches)."""
    g = P.Problem.generate(cfg, cells)
    A = g.matrix()
    pset = P.PatchSet.detect(A, ps)
    pc = P.Preconditioner.create(A, pset, None, omega=1.0)
    b = g.rhs()
    x0 = np.random.default_rng(4).uniform(-1, 1, len(b))
    want, _ = pc.relax(A, b, x0, 1, history=False)
    s0, s1 = cells * r // ranks, cells * (r + 1) // ranks
    probs = [P.Problem.generate_cells(cfg, cells, s0 - 1, s0, r - 1, ranks), P.Problem.generate_slab(cfg, cells, r, ranks),
             P.Problem.generate_cells(cfg, cells, s1, s1 + 1, r + 1, ranks)]
    sl = P.Slab.create_subset(probs, [r - 1, r, r + 1], r, ranks, ps)
    gid = sl.local_dofs(1)
    bl = torch.from_numpy(b[gid].copy()).cuda()
    xl = torch.from_numpy(x0[gid].copy()).cuda()
    bs = [torch.from_numpy(b[sl.local_dofs(i)].copy()).cuda() for i in range(3)]
    xs = [torch.from_numpy(x0[sl.local_dofs(i)].copy()).cuda() for i in range(3)]
    sl.relax_device([t.data_ptr() for t in bs], [t.data_ptr() for t in xs], 1)
    own = sl.owned(1)
    got = xs[1].cpu().numpy()[own]
    assert np.array_equal(got, want[gid[own]])
    # the rank-alone timing path runs (values not a sweep: exchanges skipped)
    sl.relax_rank_device(1, bl.data_ptr(), xl.data_ptr(), 2)
    torch.cuda.synchronize()


@pytest.mark.parametrize("cfg,cells,ps,ranks,eps,best", [(3, 0, 27, 3, 0.13699942677165544, False),
                                                          (3, 0, 27, 8, 0.13699942677165544, False),
                                                          (1, 0, 9, 2, 2.0, False), (1, 0, 9, 4, 2.0, True),
                                                          (2, 16, 25, 2, 0.5, True), (3, 8, 27, 4, 0.3, False)])
def test_rank_local_greedy_equals_single_gpu(P, cfg, cells, ps, ranks, eps, best):
    """pdb_slab_create_built: the greedy-l1 database built from the ranks' own
    patches (batches broadcast by their owners, each rank scanning only its
    patches) is bitwise the single-GPU build -- size, creators, phi -- and the
    sweeps with it are bitwise pdb_relax's."""
    g = P.Problem.generate(cfg, cells)
    A = g.matrix()
    pset = P.PatchSet.detect(A, ps)
    db = P.Database.build(A, pset, P.GREEDY_L1, eps=eps, best_match=int(best))
    slabs = [P.Problem.generate_slab(cfg, cells, r, ranks) for r in range(ranks)]
    sl = P.Slab.create_built(slabs, 0, ranks, ps, P.GREEDY_L1, eps=eps, best_match=best, omega=0.9)
    assert sl.database_size == db.size
    phi = db.phi()
    assert np.array_equal(np.concatenate([sl.phi(i) for i in range(ranks)]), phi)
    _, first = np.unique(phi, return_index=True)
    assert np.array_equal(sl.creators(), first[np.argsort(phi[first])])
    pc = P.Preconditioner.create(A, pset, db, omega=0.9)
    b = g.rhs()
    x0 = np.zeros_like(b)
    want, _ = pc.relax(A, b, x0, 3, history=False)
    got, _ = emulated_relax(P, sl, b, x0, 3)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("cfg,cells,ps,ranks,k,iters", [(2, 16, 25, 2, 30, 20), (3, 8, 27, 4, 40, 20),
                                                         (4, 8, 22, 2, 24, 20), (5, 4, 192, 2, 40, 8),
                                                         (2, 0, 25, 8, 64, 50), (4, 0, 22, 4, 128, 10)])
def test_rank_local_kmeans_equals_single_gpu(P, cfg, cells, ps, ranks, k, iters):
    """pdb_slab_create_built with KMEANS_ENTRYWISE: boundary partitions in
    global first-occurrence order, local assignment, gathered reseed, means
    chain-folded along the ranks -- bitwise the single-GPU partitioned build
    (phi and sweeps)."""
    g = P.Problem.generate(cfg, cells)
    A = g.matrix()
    pset = P.PatchSet.detect(A, ps)
    db = P.Database.build(A, pset, P.KMEANS_ENTRYWISE, db_size=k, seed=42, max_iters=iters)
    slabs = [P.Problem.generate_slab(cfg, cells, r, ranks) for r in range(ranks)]
    sl = P.Slab.create_built(slabs, 0, ranks, ps, P.KMEANS_ENTRYWISE, omega=0.9, db_size=k, seed=42, max_iters=iters)
    assert sl.database_size == db.size
    assert np.array_equal(np.concatenate([sl.phi(i) for i in range(ranks)]), db.phi())
    pc = P.Preconditioner.create(A, pset, db, omega=0.9)
    b = g.rhs()
    want, _ = pc.relax(A, b, np.zeros_like(b), 3, history=False)
    got, _ = emulated_relax(P, sl, b, np.zeros_like(b), 3)
    assert np.array_equal(got, want)
