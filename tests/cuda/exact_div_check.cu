// Test harness (not product code): compares the product's div_rn_recip
// (csrc/kernels/exact_div.cuh) with __ddiv_rn bit for bit on random operands.
#include <cstdint>
#include "exact_div.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {  // splitmix64
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ double operand(uint64_t r, int regime) {
  const uint64_t mant = r & ((1ull << 52) - 1);
  const uint64_t sign = (r >> 63) << 63;
  int64_t ex;
  switch (regime) {
    case 0: ex = 1023 + (int64_t)((r >> 52) % 24) - 12; break;          // |x| in [2^-12, 2^12)
    case 1: ex = 1023 + (int64_t)((r >> 52) % 1800) - 900; break;       // wide, incl. the guard bands
    case 2: ex = 1 + (int64_t)((r >> 52) % 2046); break;                // every normal exponent
    default: {                                                          // significand all ones / all zeros
      const uint64_t m2 = (r & 1) ? ((1ull << 52) - 1) : 0;
      ex = 1023 + (int64_t)((r >> 52) % 40) - 20;
      return __longlong_as_double((long long)(sign | ((uint64_t)ex << 52) | m2));
    }
  }
  return __longlong_as_double((long long)(sign | ((uint64_t)ex << 52) | mant));
}

__global__ void check_kernel(uint64_t n, uint64_t seed, int regime, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double a = operand(mix(seed ^ (2 * i)), regime);
    const double b = operand(mix(seed ^ (2 * i + 1)), regime == 3 ? 3 : regime);
    const double y = __ddiv_rn(1.0, b);
    const double q1 = pdb::k::div_rn_recip(a, b, y);
    const double q2 = __ddiv_rn(a, b);
    if (__double_as_longlong(q1) != __double_as_longlong(q2)) atomicAdd(bad, 1ull);
  }
}

extern "C" unsigned long long exact_div_check(unsigned long long n, unsigned long long seed, int regime) {
  unsigned long long* d = nullptr;
  cudaMalloc(&d, sizeof(*d));
  cudaMemset(d, 0, sizeof(*d));
  check_kernel<<<148 * 8, 256>>>(n, seed, regime, d);
  unsigned long long h = ~0ull;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}
