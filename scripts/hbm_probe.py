"""Achievable HBM read bandwidth on this box (torch reductions and copies)
for context next to the SpMV numbers."""
import torch

def bench(fn, nbytes, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return nbytes / ms / 1e6

n = 37_642_321
v = torch.rand(n, dtype=torch.float64, device="cuda")
c = torch.randint(0, 1 << 20, (n,), dtype=torch.int32, device="cuda")
big = torch.rand(1 << 28, dtype=torch.float64, device="cuda")  # 2 GiB
out = torch.empty_like(big)
print("sum f64 301MB read  GB/s", round(bench(lambda: v.sum(), 8 * n)))
print("sum i32 150MB read  GB/s", round(bench(lambda: c.sum(), 4 * n)))
print("sum f64 2GiB read   GB/s", round(bench(lambda: big.sum(), 8 * big.numel())))
print("copy 2GiB (r+w)     GB/s", round(bench(lambda: out.copy_(big), 16 * big.numel())))
