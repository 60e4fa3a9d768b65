"""Combo preconditioner timing (paper Experiment 1 sizes and larger).

Per case: device apply of the plain patch preconditioner and of the combo
(CUDA events on torch's stream, 50 applies after warm-up), the coarse term
alone (difference), and a whole GMRES(20) solve through the C-ABI (host
vectors) beside the reference's (oracle/_ref, one thread, as its experiment
driver runs it).  Prints one JSON line per case.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from paper_2306_10025_b200 import patchdb as P  # noqa: E402
import oracle as O  # noqa: E402


def dev_time(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ref = O.RefLib() if O.have_ref() else None
    cases = [(60, 2), (60, 3), (120, 2), (250, 2), (256, 4)]
    if len(sys.argv) > 1:
        cases = [tuple(int(v) for v in c.split(",")) for c in sys.argv[1:]]
    for cells, deg in cases:
        cfg = json.dumps(dict(cells=cells, degree=deg, coefficient=dict(kind="smooth")))
        p = P.Problem.assemble(cfg)
        A = p.matrix()
        ps = P.PatchSet.detect(A, (deg + 1) ** 2)
        plain = P.Preconditioner.create(A, ps)
        n = p.ndofs
        r = torch.rand(n, dtype=torch.float64, device="cuda")
        z = torch.empty_like(r)
        s = torch.cuda.current_stream().cuda_stream
        ms_plain = dev_time(lambda: plain.apply_device(r.data_ptr(), z.data_ptr(), s))
        b = p.rhs()
        row = dict(cells=cells, degree=deg, n=n, apply_plain_us=round(1e3 * ms_plain, 2))
        for path in ("dense", "blocked", "band"):
            nc = (cells + 1) ** 2
            if path == "dense" and nc > 16384:
                continue
            if path == "band" and nc > 20000:
                continue
            os.environ["PDB_COARSE"] = path
            t = time.time()
            combo = P.Preconditioner.create_combo(p, ps)
            t_setup = time.time() - t
            ms_combo = dev_time(lambda: combo.apply_device(r.data_ptr(), z.data_ptr(), s))
            t_gmres = 1e30
            for _ in range(2):  # the first solve also pays lazy module loading
                t = time.time()
                x, rep = P.gmres(A, b, combo)
                t_gmres = min(t_gmres, time.time() - t)
            row.update({"nc": combo.coarse_size()[0], "band": combo.coarse_size()[1:],
                        f"{path}_setup_s": round(t_setup, 4), f"{path}_apply_us": round(1e3 * ms_combo, 2),
                        f"{path}_coarse_us": round(1e3 * (ms_combo - ms_plain), 2),
                        f"{path}_gmres_iters": rep.iterations, f"{path}_gmres_s": round(t_gmres, 4),
                        f"{path}_l2_error": p.l2_error(x)})
            del combo
        os.environ.pop("PDB_COARSE", None)
        if ref is not None and cells <= 120:
            rp = ref.problem(cfg)
            rA = rp.matrix()
            rps = rA.detect((deg + 1) ** 2)
            t = time.time()
            rpc = rp.combo(rA, rps, None)
            row["ref_setup_s"] = round(time.time() - t, 4)
            t = time.time()
            for _ in range(5):
                rpc.apply(b)
            row["ref_apply_us"] = round(1e6 * (time.time() - t) / 5, 1)
            t = time.time()
            _, rr = rpc.gmres(b)
            row["ref_gmres_s"] = round(time.time() - t, 4)
            row["ref_iters"] = rr["iterations"]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
