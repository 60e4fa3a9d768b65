// Bit-exact batched LU with partial pivoting (reference lu_factor,
// dense.cpp:31-75).  Compiled with --fmad=false and written with explicit
// round-to-nearest intrinsics, so every element sees the reference's exact
// operation sequence: a_ij <- a_ij - l_ik * u_kj for k = 0,1,... (mul then
// sub, never fused), l_ik = a_ik / pivot by IEEE division.
//
// One warp per matrix; lane t owns rows t, t+32, ...  The pivot is the
// FIRST row holding the column maximum (strict >, dense.cpp:49-58): each
// lane scans its rows in ascending order with strict >, and the warp
// reduction keeps the larger value, ties to the smaller row.  Singular when
// best == 0 or best < 1e-14 * (largest initial |.| of the column)
// (dense.cpp:59-61).  The working matrix lives in shared memory with an odd
// leading dimension (conflict-free 8-byte lane-strided accesses) when it
// fits, else in the output buffer itself.
#include "../kernels.hpp"

namespace pdb::k {

namespace {

constexpr int kWarps = 4;
constexpr int kSmemMaxPs = 48;  // 4 warps * 48*49*8 B = 75 KB

__device__ __forceinline__ void warp_pivot(double& best, int& p) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int op = __shfl_xor_sync(0xffffffffu, p, off);
    if (ob > best || (ob == best && op < p)) {
      best = ob;
      p = op;
    }
  }
}

template <bool kSmem>
__global__ void __launch_bounds__(kWarps * 32) lu_kernel(int64_t count, int ps, const double* __restrict__ mats,
                                                         const int32_t* __restrict__ src, double* __restrict__ lu,
                                                         int32_t* __restrict__ piv, int32_t* __restrict__ status,
                                                         double* __restrict__ fail_best) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kWarps + warp;
  if (t >= count) return;
  const int64_t len = (int64_t)ps * ps;
  const int ld = kSmem ? (ps | 1) : ps;
  double* colmax = smem + (size_t)warp * (kSmem ? (ps * ld + ps) : ps);
  double* W = kSmem ? colmax + ps : lu + t * len;
  const double* A = mats + (src ? (int64_t)src[t] : t) * len;
  int32_t* P = piv + t * ps;

  for (int64_t e = lane; e < len; e += 32) W[(e / ps) * ld + e % ps] = A[e];
  for (int i = lane; i < ps; i += 32) P[i] = i;
  for (int j = lane; j < ps; j += 32) {
    double m = 0.0;
    for (int i = 0; i < ps; ++i) m = fmax(m, fabs(A[(int64_t)i * ps + j]));
    colmax[j] = m;
  }
  __syncwarp();

  for (int k = 0; k < ps; ++k) {
    double best = -1.0;
    int p = ps;
    for (int i = k + lane; i < ps; i += 32) {
      const double v = fabs(W[(int64_t)i * ld + k]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    warp_pivot(best, p);
    if (best == 0.0 || best < __dmul_rn(1e-14, colmax[k])) {
      if (lane == 0) {
        status[t] = k + 1;
        fail_best[t] = best;
      }
      return;
    }
    if (p != k) {
      for (int j = lane; j < ps; j += 32) {
        const double a = W[(int64_t)k * ld + j];
        W[(int64_t)k * ld + j] = W[(int64_t)p * ld + j];
        W[(int64_t)p * ld + j] = a;
      }
      if (lane == 0) {
        const int32_t tmp = P[k];
        P[k] = P[p];
        P[p] = tmp;
      }
    }
    __syncwarp();
    const double pv = W[(int64_t)k * ld + k];
    for (int i = k + 1 + lane; i < ps; i += 32) {
      double* Wi = W + (int64_t)i * ld;
      const double lik = __ddiv_rn(Wi[k], pv);
      Wi[k] = lik;
      if (lik == 0.0) continue;
      const double* Wk = W + (int64_t)k * ld;
      for (int j = k + 1; j < ps; ++j) Wi[j] = __dsub_rn(Wi[j], __dmul_rn(lik, Wk[j]));
    }
    __syncwarp();
  }
  if (kSmem)
    for (int64_t e = lane; e < len; e += 32) lu[t * len + e] = W[(e / ps) * ld + e % ps];
  if (lane == 0) status[t] = 0;
}

}  // namespace

void lu_batched(int64_t count, int ps, const double* mats, const int32_t* src, double* lu, int32_t* piv,
                int32_t* status, double* fail_best, cudaStream_t s) {
  if (count <= 0) return;
  const unsigned grid = (unsigned)((count + kWarps - 1) / kWarps);
  if (ps <= kSmemMaxPs) {
    const size_t smem = (size_t)kWarps * ((size_t)ps * (ps | 1) + ps) * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(lu_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lu_kernel<true><<<grid, kWarps * 32, smem, s>>>(count, ps, mats, src, lu, piv, status, fail_best);
  } else {
    const size_t smem = (size_t)kWarps * ps * sizeof(double);
    lu_kernel<false><<<grid, kWarps * 32, smem, s>>>(count, ps, mats, src, lu, piv, status, fail_best);
  }
}

}  // namespace pdb::k
