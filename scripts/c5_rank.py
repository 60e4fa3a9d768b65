"""Config 5 at its BASELINE size (3D elasticity Q3, 96^3 cells, 884,736 x
192-DoF patches, ~26.5G nonzeros) does not fit one GPU: all-patch factors are
261 GB and the CSR 318 GB.  This runs ONE rank's share of the W-rank job on
the single GPU: rank r's slab (pdb_problem_generate_slab: only its rows are
ever generated) and one-cell-layer slices of its neighbours
(pdb_problem_generate_cells), set up as an emulated subset group through the
multi-rank API (pdb_slab_create_subset: local patches, weights / ownership /
halo lists with the neighbours, exact factors of the local patches only,
streamed), then times rank r's sweep phases alone (CUDA events).  Prints one
JSON line with the per-rank HBM budget, setup time, sweep time, bytes and
exchange volume.

    python scripts/c5_rank.py [--ranks 8] [--rank 3] [--cells 96] [--sweeps 10]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10025_b200 import patchdb as P  # noqa: E402


def gib(x):
    return round(x / 2 ** 30, 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--rank", type=int, default=3)
    ap.add_argument("--cells", type=int, default=96)
    ap.add_argument("--sweeps", type=int, default=10)
    a = ap.parse_args()
    W, r, C = a.ranks, a.rank, a.cells
    torch.cuda.init()
    free0, total = torch.cuda.mem_get_info()
    s0, s1 = C * r // W, C * (r + 1) // W
    t = time.perf_counter()
    probs, ranks = [], []
    if r > 0:
        probs.append(P.Problem.generate_cells(5, C, s0 - 1, s0, r - 1, W))
        ranks.append(r - 1)
    mine = P.Problem.generate_slab(5, C, r, W)
    probs.append(mine)
    ranks.append(r)
    if r < W - 1:
        probs.append(P.Problem.generate_cells(5, C, s1, s1 + 1, r + 1, W))
        ranks.append(r + 1)
    t_gen = time.perf_counter() - t
    me = ranks.index(r)
    t = time.perf_counter()
    sl = P.Slab.create_subset(probs, ranks, r, W, 192)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t
    free1, _ = torch.cuda.mem_get_info()
    info = sl.info(me)
    gid = sl.local_dofs(me)
    rows = mine.row_ids()
    b = torch.zeros(len(gid), dtype=torch.float64, device="cuda")
    b[torch.from_numpy(np.searchsorted(gid, rows)).cuda()] = torch.from_numpy(mine.rhs()).cuda()
    x = torch.zeros_like(b)
    stream = torch.cuda.current_stream()
    sl.relax_rank_device(me, b.data_ptr(), x.data_ptr(), 2, stream.cuda_stream)
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sl.relax_rank_device(me, b.data_ptr(), x.data_ptr(), a.sweeps, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1) / a.sweeps)
    msw = sorted(ms)[1]
    nnz_rows = mine.nnz
    n_rows = info["n_rows"]
    npl = info["n_patches"]
    # algorithmic bytes of the rank's exact sweep: values (SELL, no column
    # stream) + row descriptors, x/b/r, patch lists, the per-patch inverses
    # streamed once, x read/write in the scatter
    sweep_bytes = 8 * nnz_rows + 8 * n_rows + 24 * info["n_local"] + 4 * npl * 192 + 8 * npl * 192 * 192 + 16 * n_rows
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    ex = 8 * (info["n_up"] + info["n_pin"] + info["n_xs"] + info["n_xr"])
    out = {
        "config": f"config5 at {C}^3 (3D elasticity Q3, {C ** 3:,} x 192-DoF patches), rank {r} of {W}",
        "group": {"ranks": ranks, "note": "rank r's slab + one-cell-layer neighbour slices, emulated subset"},
        "rank_info": info,
        "rank_rows": n_rows, "rank_nnz": nnz_rows, "rank_patches": npl,
        "generate_s": t_gen, "setup_s": t_setup,
        "hbm": {"total_gib": gib(total), "free_before_gib": gib(free0), "used_by_group_gib": gib(free0 - free1),
                "rank_factor_gib": gib(8 * npl * 192 * 192), "rank_sell_values_gib": gib(8 * nnz_rows)},
        "sweep_ms_per_rank": msw, "sweep_ms_all": ms,
        "rank_sweep_bytes": sweep_bytes, "rank_sweep_gbs": sweep_bytes / (msw * 1e-3) / 1e9,
        "rank_sweep_frac_hbm": sweep_bytes / (msw * 1e-3) / 1e9 / hbm,
        "exchange_bytes_per_sweep": ex,
        "exchange_us_at_900GBs": ex / 900e9 * 1e6,
        "job_dof_updates_per_s_if_balanced": mine.rows_global / (msw * 1e-3),
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
