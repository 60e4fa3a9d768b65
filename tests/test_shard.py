"""Multi-rank sweep: the slab partition and its exchange schedule.

CPU (world_size 2 and 3 over gloo): every rank builds its plan with the
library's host planner (pdb_shard_plan_create), runs the sweep on its shard
with the oracle's kernels (sequential SpMV, LU solves), exchanges interface
partial sums and x halos exactly as the device shard does over NCCL, and the
assembled result must equal the serial reference sweep BIT FOR BIT -- the
ordered interface sums reproduce the reference's ascending-patch scatter.
GPU: a 1-rank device shard equals pdb_relax.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(cfg, cells, ps):
    import oracle as O
    from paper_2306_10025_b200 import patchdb as P
    orc = O.Oracle()
    prob = P.Problem.generate(cfg, cells)
    csr = prob.csr()
    patches, w = orc.detect(csr, ps)
    return orc, P, csr, prob.rhs(), patches, w


def _exchange(send_idx, send_peer, vals, recv_idx, recv_peer, nlocal_recv):
    """Grouped point-to-point exchange following the plan's (peer-sorted) lists."""
    reqs, bufs = [], {}
    for peer in sorted(set(recv_peer.tolist())):
        sel = np.nonzero(recv_peer == peer)[0]
        bufs[peer] = (sel, torch.empty(len(sel), dtype=torch.float64))
        reqs.append(dist.irecv(bufs[peer][1], src=int(peer)))
    for peer in sorted(set(send_peer.tolist())):
        sel = np.nonzero(send_peer == peer)[0]
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(vals[sel])), dst=int(peer)))
    for r in reqs:
        r.wait()
    out = np.zeros(nlocal_recv)
    for sel, t in bufs.values():
        out[sel] = t.numpy()
    return out


def _rank_main(rank, world, port, cfg, cells, ps, sweeps, omega, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    orc, P, csr, b, patches, w = _problem(cfg, cells, ps)
    plan = P.shard_plan(csr, patches, w, rank, world)
    dofs = plan["dofs"]
    nl = len(dofs)
    lcsr = (plan["row_ptr"], plan["cols"], plan["values"])
    lp = plan["patches"].reshape(-1, ps)
    mats = orc.extract_all(lcsr, lp)
    fac = [orc.lu_factor(m) for m in mats]
    inv = [[] for _ in range(nl)]
    for k in range(len(lp)):
        for slot, d in enumerate(lp[k]):
            inv[d].append((k, slot))
    ow = omega * plan["weights"]
    x = np.zeros(nl)
    bl = b[dofs]
    for _ in range(sweeps):
        r = bl - orc.spmv(lcsr, x)
        sols = [orc.lu_solve(f[0], f[1], r[lp[k]]) for k, f in enumerate(fac)]

        def zsum(d, init=0.0):
            z = init
            for k, slot in inv[d]:
                z += sols[k][slot]
            return z
        zup = np.array([zsum(d) for d in plan["up"]])
        zin = _exchange(plan["up"], plan["up_peer"], zup, plan["pin"], plan["pin_peer"], len(plan["pin"]))
        init = np.zeros(nl)
        init[plan["pin"]] = zin
        for d in plan["owned"]:
            z = zsum(d, init[d])
            x[d] = z * ow[d] + x[d]
        xin = _exchange(plan["xs"], plan["xs_peer"], x[plan["xs"]], plan["xr"], plan["xr_peer"], len(plan["xr"]))
        x[plan["xr"]] = xin
    owned_g = dofs[plan["owned"]]
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), ids=owned_g, x=x[plan["owned"]])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,cells,ps", [(2, 1, 12, 9), (3, 1, 12, 9), (2, 3, 4, 27)])
def test_sharded_sweep_matches_serial_bitwise(world, cfg, cells, ps):
    sweeps, omega = 4, 0.8
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_rank_main, args=(world, _free_port(), cfg, cells, ps, sweeps, omega, td), nprocs=world, join=True)
        orc, P, csr, b, patches, w = _problem(cfg, cells, ps)
        mats = orc.extract_all(csr, patches)
        fac = [orc.lu_factor(m) for m in mats]
        lu, piv = np.stack([a for a, _ in fac]), np.stack([p for _, p in fac])
        want, _ = orc.relax(csr, patches, w, omega, lu, piv, None, b, np.zeros_like(b), sweeps)
        got = np.full_like(want, np.nan)
        seen = np.zeros(len(want), int)
        for r in range(world):
            d = np.load(os.path.join(td, f"rank{r}.npz"))
            got[d["ids"]] = d["x"]
            seen[d["ids"]] += 1
    assert np.all(seen == 1), "every DoF must be owned by exactly one rank"
    assert np.array_equal(got, want)


@pytest.mark.parametrize("world", [2, 4])
def test_plan_lists_are_consistent(P, orc, world):
    prob = P.Problem.generate(1, 16)
    csr = prob.csr()
    patches, w = orc.detect(csr, 9)
    plans = [P.shard_plan(csr, patches, w, r, world) for r in range(world)]
    owned = np.concatenate([p["dofs"][p["owned"]] for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(prob.ndofs))
    for r, p in enumerate(plans):
        for q, o in enumerate(plans):
            if q == r:
                continue
            sent = p["dofs"][p["up"][p["up_peer"] == q]]
            recv = o["dofs"][o["pin"][o["pin_peer"] == r]]
            assert np.array_equal(sent, recv)
            xs = p["dofs"][p["xs"][p["xs_peer"] == q]]
            xr = o["dofs"][o["xr"][o["xr_peer"] == r]]
            assert np.array_equal(xs, xr)
        lo, hi = p["patch_range"]
        assert hi - lo in (len(patches) // world, len(patches) // world + 1)


def test_plan_rejects_too_thin_slabs(P, orc):
    prob = P.Problem.generate(1, 4)
    csr = prob.csr()
    patches, w = orc.detect(csr, 9)
    with pytest.raises(P.PatchdbError) as e:
        P.shard_plan(csr, patches, w, 0, 16)
    assert "too thin" in e.value.message


@pytest.mark.gpu
def test_single_rank_device_shard_equals_relax(P):
    prob = P.Problem.generate(2, 32)
    A = prob.matrix()
    ps = P.PatchSet.detect(A, 25)
    db = P.Database.build(A, ps, P.KMEANS_ENTRYWISE, db_size=16)
    pc = P.Preconditioner.create(A, ps, db, omega=0.9)
    b = prob.rhs()
    x_ref, _ = pc.relax(A, b, np.zeros_like(b), 6, history=False)
    sh = P.Shard.create(A, ps, db, 0.9, 0, 1)
    dofs = sh.local_dofs()
    bd = torch.from_numpy(b[dofs]).cuda()
    xd = torch.zeros_like(bd)
    sh.relax_device(bd.data_ptr(), xd.data_ptr(), 6)
    torch.cuda.synchronize()
    got = np.zeros_like(b)
    got[dofs] = xd.cpu().numpy()
    np.testing.assert_allclose(got, x_ref, rtol=1e-12, atol=1e-14 * np.abs(x_ref).max())


# --------------------------------------------------------- sharded setup ---

def _sharded_case(P, method, best_match=0):
    prob = P.Problem.generate(2, 16)
    A = prob.matrix()
    ps = P.PatchSet.detect(A, 25)
    if method in (1, 2):  # greedy: a tolerance giving ~16 entries
        want, eps = P.Database.build_to_size(A, ps, 12, 20, method, best_match=best_match)
        kw = dict(eps=eps, best_match=best_match)
    else:
        kw = dict(db_size=16, seed=3, max_iters=8)
    want = P.Database.build(A, ps, method, **kw)
    return A, ps, kw, want


@pytest.mark.gpu
@pytest.mark.parametrize("method,best", [(1, 0), (2, 0), (2, 1), (3, 0), (4, 0)])
def test_sharded_build_matches_single_gpu(P, orc, method, best):
    """pdb_database_build_sharded over a 1-rank NCCL communicator (the
    all-gather / all-reduce paths) returns the single-GPU database bit for bit."""
    A, ps, kw, want = _sharded_case(P, method, best)
    comm = P.Comm.create(P.comm_unique_id(), 0, 1)
    got = P.Database.build(A, ps, method, comm=comm, **kw)
    assert np.array_equal(got.phi(), want.phi())
    assert np.array_equal(got.representatives(), want.representatives())
    lu, piv = got.factors()
    lw, pw = want.factors()
    assert np.array_equal(lu, lw) and np.array_equal(piv, pw)
    assert got.work()["power_iters"] == want.work()["power_iters"]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("method,best", [(1, 0), (2, 0), (2, 1), (3, 0), (4, 0)])
def test_emulated_shard_chunks_match_single_gpu(P, monkeypatch, world, method, best):
    """PDB_SHARD_EMULATE=W evaluates the W rank chunks (k-means assignment,
    greedy scan) one after another on this GPU: same decomposition as W
    ranks, bitwise result."""
    A, ps, kw, want = _sharded_case(P, method, best)
    monkeypatch.setenv("PDB_SHARD_EMULATE", str(world))
    got = P.Database.build(A, ps, method, **kw)
    assert np.array_equal(got.phi(), want.phi())
    assert np.array_equal(got.representatives(), want.representatives())


@pytest.mark.gpu
def test_sharded_bisection_matches_single_gpu(P):
    prob = P.Problem.generate(2, 16)
    A = prob.matrix()
    ps = P.PatchSet.detect(A, 25)
    want, we = P.Database.build_to_size(A, ps, 12, 20, 2)
    comm = P.Comm.create(P.comm_unique_id(), 0, 1)
    got, ge = P.Database.build_to_size(A, ps, 12, 20, 2, comm=comm)
    assert ge == we and np.array_equal(got.phi(), want.phi())


@pytest.mark.gpu
def test_shard_create_rejects_mismatched_inputs(P):
    """pdb_shard_create checks the patch set and the database against the
    matrix (dimension_mismatch), as the reference's preconditioner does."""
    small = P.Problem.generate(1, 8)
    big = P.Problem.generate(1, 12)
    As, Ab = small.matrix(), big.matrix()
    pss, psb = P.PatchSet.detect(As, 9), P.PatchSet.detect(Ab, 9)
    with pytest.raises(P.PatchdbError) as e:
        P.Shard.create(As, psb, None, 1.0, 0, 1)
    assert e.value.status == P.PDB_ERR_DIMENSION_MISMATCH
    dbb = P.Database.build(Ab, psb, P.GREEDY_L1, eps=2.0)
    with pytest.raises(P.PatchdbError) as e:
        P.Shard.create(As, pss, dbb, 1.0, 0, 1)
    assert e.value.status == P.PDB_ERR_DIMENSION_MISMATCH
