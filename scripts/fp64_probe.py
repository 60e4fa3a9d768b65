"""Measure FP64 peaks on this GPU and write profiles/fp64_peaks.json.

  python scripts/fp64_probe.py        (builds scripts/fp64_probe.so with nvcc if missing)

dfma: 2 flop per DFMA; dmuladd: 2 flop per (DMUL, DADD) pair, i.e. the rate
of the unfused arithmetic the bit-exact criterion kernels must use; dmma:
2*8*8*4 flop per mma.sync.m8n8k4.f64.
"""
import ctypes as C
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "fp64_probe.so")


def main():
    if not os.path.exists(SO):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                               "-fPIC", "-o", SO, os.path.join(HERE, "fp64_probe.cu")])
    lib = C.CDLL(SO)
    lib.fp64_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {"gpu": torch.cuda.get_device_name(0), "sms": sms}
    iters = 20000
    for which, name, flop_per_thread_iter in ((0, "dfma", 2 * 8), (1, "dmuladd", 2 * 8), (2, "dmma", 0)):
        best = 0.0
        for blocks_per_sm in (2, 4, 8):
            for threads in (128, 256):
                ms = C.c_float()
                rc = lib.fp64_probe(which, sms * blocks_per_sm, threads, iters, C.byref(ms))
                if rc != 0:
                    raise SystemExit(f"probe {name} failed: {rc}")
                nthreads = sms * blocks_per_sm * threads
                if which == 2:
                    flops = (nthreads // 32) * iters * 4 * 2 * 8 * 8 * 4
                else:
                    flops = nthreads * iters * flop_per_thread_iter
                best = max(best, flops / (ms.value * 1e-3) / 1e12)
        out[f"{name}_tflops"] = best
    out["note"] = ("dfma/dmuladd: 8 independent chains per thread; dmuladd counts 2 flop per DMUL+DADD pair "
                   "(the unfused rate the bit-exact spectral/LU kernels are bound by); dmma: mma.sync m8n8k4 f64")
    path = os.path.join(os.path.dirname(HERE), "profiles", "fp64_peaks.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
