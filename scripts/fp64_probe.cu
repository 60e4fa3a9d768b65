// FP64 peak probes for the setup roofline (MEASURED_PEAKS.json has HBM and
// bf16 only; SURVEY.md §8d asks the builder to measure FP64 on the box).
//   dfma : independent DFMA chains            -> FMA issue rate (2 flop each)
//   dmuladd : __dmul_rn then __dadd_rn chains -> the unfused rate the bit-exact
//             criterion kernels are limited to (1 flop per instruction)
//   dmma : mma.sync.m8n8k4.f64 loop           -> FP64 tensor-core rate
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o scripts/fp64_probe.so scripts/fp64_probe.cu   (scripts/fp64_probe.py does it)
#include <cuda_runtime.h>
#include <cstdint>

constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmuladd_kernel(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __dadd_rn(__dmul_rn(x[c], a), b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c0[k]), "+d"(c1[k])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c0[k] + c1[k];
  if (s == 1.2345) out[0] = s;
}

extern "C" int fp64_probe(int which, int blocks, int threads, int iters, float* ms) {
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    if (which == 0) dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    else if (which == 1) dmuladd_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    else dmma_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(ms, e0, e1);
  cudaFree(d);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}
