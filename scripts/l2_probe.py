"""L2 read-bandwidth probe: a grid-stride kernel reads a buffer that fits in
L2 (and one that does not) many times; reports GB/s.  Sizes the mirror-SELL
residual's L2 budget."""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
__global__ void rd(const double2* __restrict__ a, long n, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
      double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 1.2345) out[0] = s;
}
void run(torch::Tensor a, int reps, int blocks, torch::Tensor out) {
  rd<<<blocks, 512>>>((const double2*)a.data_ptr<double>(), a.numel() / 2, reps, out.data_ptr<double>());
}
"""
m = load_inline("l2probe", cpp_sources="void run(torch::Tensor a, int reps, int blocks, torch::Tensor out);",
                cuda_sources=src, functions=["run"], extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"])
out = torch.zeros(1, dtype=torch.float64, device="cuda")
for mb in (8, 24, 48, 96, 1024):
    a = torch.ones(mb * (1 << 20) // 8, dtype=torch.float64, device="cuda")
    reps = max(1, 2048 // mb)
    for blocks in (148 * 4, 148 * 8):
        m.run(a, reps, blocks, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.run(a, reps, blocks, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{mb:5d} MB x{reps:4d} blocks {blocks}: {mb * (1 << 20) * reps / ms / 1e6:8.0f} GB/s", flush=True)
