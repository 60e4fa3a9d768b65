#!/usr/bin/env python
"""Benchmark: compressed patch-relaxation sweeps on B200 (BASELINE.json config 2).

Step = one relaxation sweep x <- x + M~^{-1}(b - A x) (reference smooth(),
precond.cpp:90-101) over the whole config-2 problem: 2D Q4 on 256x256 cells
(n = 1,050,625 DoFs, 37.6M nonzeros, 65,536 patches of 25 DoFs), coefficient
on random 8x8-cell blocks from {1,10,100,1000}, jitter 0.05h, compressed to
k = 64 representatives by partitioned spectral k-means.  Inputs are seeded
synthetic data from the repo's generator (the reference ships no datasets).

value = DoF-updates/s of the sweep (n * steps / device time), inputs resident
in HBM.  e2e = the same metric through the C-ABI call pdb_relax with pinned
host buffers (b and x copied in, x copied out every step).  Setup
(detect + extract + k-means + LU + sweep structures) is reported as
setup_patches_per_s.  `--impl reference` times the reference's own CPU
implementation (oracle/_ref, compiled from the unmodified sources) with all
host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sweep DOF-updates/s + setup patches/s at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "DOF-updates/s"
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback

METHODS = {"exact": 0, "greedy-spectral": 1, "greedy-l1": 2, "kmeans-entrywise": 3, "kmeans-spectral": 4,
           "kmeans-varmin": 5, "bootstrap": 6}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--cells", type=int, default=0)
    ap.add_argument("--method", default="kmeans-spectral", choices=list(METHODS))
    ap.add_argument("--db-size", type=int, default=64)
    ap.add_argument("--omega", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    return ap.parse_args()


def patch_size(cfg_id):
    return {1: 9, 2: 25, 3: 27}[cfg_id]


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def sweep_bytes(n, nnz, np_, ps, nf):
    """SURVEY.md §8d algorithmic bytes of one fused compressed sweep."""
    rp = 8 if nnz >= 2 ** 31 else 4
    return 12 * nnz + rp * (n + 1) + 32 * n + 4 * np_ * ps + 4 * np_ + 8 * nf * ps * ps


def residual_bytes(n, nnz):
    """Algorithmic bytes of the residual SpMV launch: CSR values+cols, row_ptr, x, b read, r written."""
    rp = 8 if nnz >= 2 ** 31 else 4
    return 12 * nnz + rp * (n + 1) + 24 * n


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.seek(0)
        rows = []
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6], float(parts[6])))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        busy = [r for r in rows if r[3] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in busy), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(busy)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2306_10025_b200 import patchdb as P

    ps_size = patch_size(args.config)
    t_gen = time.perf_counter()
    prob = P.Problem.generate(args.config, args.cells)
    t_gen = time.perf_counter() - t_gen
    n, nnz = prob.ndofs, prob.nnz
    A = prob.matrix()  # CSR resident in HBM before any timing

    # ---- setup: detect + extract + compress + LU + sweep structures (synchronous calls)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ps = P.PatchSet.detect(A, ps_size)
    t1 = time.perf_counter()
    db = P.Database.build(A, ps, METHODS[args.method], db_size=args.db_size, seed=42, max_iters=50)
    t2 = time.perf_counter()
    pc = P.Preconditioner.create(A, ps, db, omega=args.omega)
    t3 = time.perf_counter()
    np_ = ps.count
    m_p = db.size
    work = db.work()
    setup_s = t3 - t0

    # ---- sweeps on device-resident inputs
    rhs = prob.rhs()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    shard = None
    if world > 1:
        # slab partition: rank r sweeps patches [np r/N, np (r+1)/N) and exchanges
        # interface partial sums + x halos with NCCL inside the library
        shard = P.Shard.create(A, ps, db, args.omega, rank, world)
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.tensor(list(P.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        shard.attach(bytes(uid.cpu().tolist()))
        ldofs = shard.local_dofs()
        b = torch.from_numpy(rhs[ldofs]).cuda()
    else:
        b = torch.from_numpy(rhs).cuda()
    x = torch.zeros_like(b)

    def sweeps(k):
        if shard is not None:
            shard.relax_device(b.data_ptr(), x.data_ptr(), k, stream=sptr)
        else:
            pc.relax_device(A, b.data_ptr(), x.data_ptr(), k, stream=sptr)

    sweeps(args.warmup)
    torch.cuda.synchronize()

    def timed():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sweeps(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    reps_ms = []
    with Clocks(local) as clk:
        t_begin = time.perf_counter()
        while len(reps_ms) < 3 or (time.perf_counter() - t_begin < 1.5 and len(reps_ms) < 200):
            reps_ms.append(timed())
    clocks = clk.summary()
    ms = statistics.median(reps_ms)
    value = n * args.steps / (ms / 1e3)  # whole-job DoF-updates/s (the mesh is split across ranks)

    # ---- per-kernel split (CUDA events around each launch, same stream)
    phase = P.relax_profile(pc, A, b.data_ptr(), x.data_ptr(), args.steps, stream=sptr) if shard is None else \
        P.relax_profile(pc, A, torch.from_numpy(rhs).cuda().data_ptr(),
                        torch.zeros(n, dtype=torch.float64, device="cuda").data_ptr(), args.steps, stream=sptr)

    # ---- e2e through the C-ABI with pinned host buffers
    lib = P.lib
    import ctypes as C
    dp = C.POINTER(C.c_double)
    e2e_steps = max(5, min(args.steps, 200))
    if shard is None:
        bh = torch.from_numpy(rhs).pin_memory()
        xh = torch.zeros(n, dtype=torch.float64).pin_memory()
        bptr = C.cast(bh.data_ptr(), dp)
        xptr = C.cast(xh.data_ptr(), dp)

        def e2e_step():
            P._check(lib.pdb_relax(A.ptr, pc.ptr, bptr, xptr, 1, None))
        h2d, d2h = 16 * n, 8 * n
    else:
        bh = torch.from_numpy(rhs[ldofs]).pin_memory()
        xh = torch.zeros(len(ldofs), dtype=torch.float64).pin_memory()

        def e2e_step():
            b.copy_(bh, non_blocking=True)
            x.copy_(xh, non_blocking=True)
            shard.relax_device(b.data_ptr(), x.data_ptr(), 1, stream=sptr)
            xh.copy_(x, non_blocking=True)
            torch.cuda.synchronize()
        h2d, d2h = 16 * len(ldofs) * world, 8 * len(ldofs) * world
    for _ in range(3):
        e2e_step()
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    te = time.perf_counter() - te
    if world > 1:
        t = torch.tensor([te], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    # host-link floor: the same bytes as plain pinned copies (no compute)
    hb = torch.empty(h2d // 8 // max(world, 1), dtype=torch.float64).pin_memory()
    db_ = torch.empty_like(hb, device="cuda")
    ob = torch.empty(d2h // 8 // max(world, 1), dtype=torch.float64).pin_memory()
    od = torch.empty_like(ob, device="cuda")
    for _ in range(3):
        db_.copy_(hb, non_blocking=True)
        ob.copy_(od, non_blocking=True)
    torch.cuda.synchronize()
    tl = time.perf_counter()
    for _ in range(20):
        db_.copy_(hb, non_blocking=True)
        ob.copy_(od, non_blocking=True)
        torch.cuda.synchronize()
    tl = (time.perf_counter() - tl) / 20
    e2e = {"value": n * e2e_steps / te, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "steps": e2e_steps, "host_link_floor": {"value": n / tl, "ms_per_step": tl * 1e3,
                                                   "note": "same H2D+D2H bytes as bare pinned copies, no compute"},
           "call": "pdb_relax (1 sweep, pinned host b/x)" if shard is None else
                   "pdb_shard_relax_device (1 sweep) with pinned host b/x copies per rank"}

    hbm, peak_src = peaks()
    rb = residual_bytes(n, nnz)
    achieved = rb / (phase[0] * 1e-3) / 1e9
    sb = sweep_bytes(n, nnz, np_, ps_size, m_p)
    sweep_gbs = sb / (ms / args.steps * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(f"config{args.config}", {}).get("residual")
        except Exception:
            traffic = None

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, BASELINE config %d)" % args.config,
        "config": {"workload": f"config{args.config}: 2D Q4 256x256, 65,536 x 25-DoF patches, k=64 "
                               f"{args.method} compressed sweep" if args.config == 2 else f"config{args.config}",
                   "n_dofs": n, "nnz": nnz, "n_patches": np_, "patch_size": ps_size, "m_p": m_p,
                   "method": args.method, "omega": args.omega, "cells": args.cells or None,
                   "l2": "inputs larger than L2 (CSR alone %.0f MB > 126 MB)" % (12 * nnz / 1e6),
                   "parallelism": f"slab{world}: patch slabs + NCCL halo/interface exchange" if world > 1
                   else "single GPU"},
        "setup_patches_per_s": np_ / setup_s,
        "setup": {"seconds": setup_s, "detect_s": t1 - t0, "compress_s": t2 - t1, "precond_s": t3 - t2,
                  "pair_evals": work["pair_evals"], "power_iters": work["power_iters"], "lu": work["lu_count"],
                  "generator_s": t_gen},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": "residual_sell_kernel<8> (r = b - A x over the SELL-C-sigma copy)",
                     "algorithmic_bytes_per_launch": rb, "ms_per_launch": phase[0], "peak_source": peak_src},
        "sweep_roofline": {"bytes_per_sweep": sb, "achieved_gbs": sweep_gbs, "frac": sweep_gbs / hbm,
                           "kernel_ms": {"residual": phase[0], "patch_apply_dmma": phase[1], "scatter_update": phase[2]}},
        "e2e": e2e,
        "gpu_launches": 3 * args.steps,
        "clocks": clocks,
        "timing": {"repeats": len(reps_ms), "ms_all": [round(v, 4) for v in reps_ms]},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(prob, ps, db, args)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(prob, ps, db, args):
    """Reference smooth() (oracle/_ref, unmodified sources) on the same config-2
    problem and the same database, all host threads, bounded sample."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.have_ref():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "oracle/_ref not built"}
    ref = O.RefLib()
    threads = os.cpu_count() or 1
    csr = prob.csr()
    rm = ref.matrix(csr)
    rps = rm.patchset(prob.ndofs, ps.patches())
    lu, piv = db.factors()
    rdb = ref.database(db.representatives(), lu, piv, db.phi())
    pc = rps.precond(rm, rdb, args.omega, threads)
    b = prob.rhs()
    x = np.zeros_like(b)
    x = pc.smooth(x, b, 1, threads)  # warm-up
    t = time.perf_counter()
    sweeps = 0
    while sweeps < 3 or time.perf_counter() - t < args.cpu_seconds * 0.5:
        x = pc.smooth(x, b, 1, threads)
        sweeps += 1
        if sweeps >= 500:
            break
    dt = time.perf_counter() - t
    return {"value": prob.ndofs * sweeps / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{sweeps} reference smooth() sweeps on the full config-{args.config} problem with the same "
                      f"database (threads={threads}), {dt:.1f} s"}


# ---------------------------------------------------------------------- reference
def run_reference(args):
    world, rank, local = dist_init()
    if rank != 0:
        return
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpdbref.so was not built"}))
        return
    from paper_2306_10025_b200 import patchdb as P  # generator only (host code), no GPU use
    ref = O.RefLib()
    threads = os.cpu_count() or 1
    ps_size = patch_size(args.config)
    prob = P.Problem.generate(args.config, args.cells)
    csr = prob.csr()
    b = prob.rhs()
    n = prob.ndofs
    rm = ref.matrix(csr)
    t0 = time.perf_counter()
    rps = rm.detect(ps_size)
    t_detect = time.perf_counter() - t0
    # The sweep cost depends only on n, nnz, n_p, p_s and m_p; the reference
    # builds its k=64 database with partitioned entrywise k-means (spectral
    # k-means at this size runs for hours on the CPU).
    t0 = time.perf_counter()
    rdb = rps.build(rm, 3, db_size=args.db_size, seed=42, max_iters=10, threads=threads)
    t_db = time.perf_counter() - t0
    pc = rps.precond(rm, rdb, args.omega, threads)
    x = np.zeros_like(b)
    for _ in range(max(1, min(args.warmup, 3))):
        x = pc.smooth(x, b, 1, threads)
    budget = 90.0
    t = time.perf_counter()
    done = 0
    while done < args.steps:
        x = pc.smooth(x, b, 1, threads)
        done += 1
        if time.perf_counter() - t > budget:
            break
    dt = time.perf_counter() - t
    value = n * done / dt
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / done * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, BASELINE config %d)" % args.config,
        "config": {"workload": f"config{args.config} compressed sweep, reference smooth() on host cores",
                   "n_dofs": n, "m_p": rdb.size},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{done} of {args.steps} steps timed (budget {budget:.0f} s), threads={threads}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_patches_per_s": rps.count / (t_detect + t_db),
        "setup": {"detect_s": t_detect, "compress_s": t_db, "method": "kmeans-entrywise (max_iters 10)"},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
