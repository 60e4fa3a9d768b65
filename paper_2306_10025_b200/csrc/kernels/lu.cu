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
#include <cstdlib>

#include "../common.hpp"
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

// ---------------------------------------------------------------------------
// CTA per matrix (ps > kSmemMaxPs; config 5's 192-DoF elasticity patches).
//
// A 192 x 192 fp64 matrix (295 KB) does not fit the 227 KB of shared memory,
// but after step k of the right-looking elimination rows < k are final (the
// pivot search and every later swap only involve rows >= k), so only the
// trailing block has to stay on chip.  Steps k < k0 run on the output buffer
// in global memory (L2-resident: one matrix per SM), with coalesced row-wise
// swaps and updates (warp per row, lane per column); at k0 the trailing
// (ps-k0) x (ps-k0) block moves to shared memory (odd leading dimension) and
// the remaining steps run there; the columns < k0 of rows >= k0 (the L part
// from the global phase) stay in global memory and are swapped there.  k0 is
// the smallest step whose trailing block fits (k0 = 32 at ps = 192; 0 for
// ps <= 165).  Every element still sees a_ij <- a_ij - l_ik * u_kj for
// k = 0, 1, ... in order, unfused, with l_ik by IEEE division and the skip
// at l_ik == 0 (dense.cpp:66-72), so factors and pivots are bitwise the
// reference's.
constexpr int kCtaThreads = 512;
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr size_t kCtaSmemCap = 220 * 1024;

__host__ __device__ inline size_t cta_smem_bytes(int ps, int k0) {
  const int t = ps - k0;
  return ((size_t)t * (t | 1) + 2 * (size_t)ps + 2 * kCtaWarps) * sizeof(double) + (size_t)ps * sizeof(int32_t);
}

inline int cta_k0(int ps) {
  int k0 = 0;
  while (k0 < ps && cta_smem_bytes(ps, k0) > kCtaSmemCap) ++k0;
  return k0;
}

// pivot of column k over rows [k, ps): the first row holding the maximum |.|
// (dense.cpp:49-58); `at(i)` gives the element; warp-level, result in lane 0..31.
template <typename At>
__device__ __forceinline__ void column_pivot(int k, int ps, At at, double& best, int& p) {
  const int lane = threadIdx.x & 31;
  best = -1.0;
  p = ps;
  for (int i = k + lane; i < ps; i += 32) {
    const double v = fabs(at(i));
    if (v > best) {
      best = v;
      p = i;
    }
  }
  warp_pivot(best, p);
}

__global__ void __launch_bounds__(kCtaThreads, 1)
    lu_cta_kernel(int64_t count, int ps, int k0, const double* __restrict__ mats, const int32_t* __restrict__ src,
                  double* __restrict__ lu, int32_t* __restrict__ piv, int32_t* __restrict__ status,
                  double* __restrict__ fail_best) {
  extern __shared__ double smem[];
  const int tn = ps - k0, ldt = tn | 1;
  double* T = smem;                                 // trailing block [tn][ldt]
  double* colmax = T + (size_t)tn * ldt;            // [ps]
  double* lcol = colmax + ps;                       // [ps] multipliers of the current step
  double* red = lcol + ps;                          // [2 * warps] scratch
  int32_t* perm = reinterpret_cast<int32_t*>(red + 2 * kCtaWarps);  // [ps]
  __shared__ double s_best;
  __shared__ int s_p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t len = (int64_t)ps * ps;

  for (int64_t t = blockIdx.x; t < count; t += gridDim.x) {
    const double* A = mats + (src ? (int64_t)src[t] : t) * len;
    double* W = lu + t * len;
    // column maxima of the input (order-free: max is exact), the input copied
    // to W (global phase) or straight into T (k0 == 0)
    for (int j = threadIdx.x; j < ps; j += kCtaThreads) {
      double m = 0.0;
      for (int i = 0; i < ps; ++i) m = fmax(m, fabs(A[(int64_t)i * ps + j]));
      colmax[j] = m;
      perm[j] = j;
    }
    if (k0 > 0)
      for (int64_t e = threadIdx.x; e < len; e += kCtaThreads) W[e] = A[e];
    else
      for (int64_t e = threadIdx.x; e < len; e += kCtaThreads) T[(e / ps) * ldt + e % ps] = A[e];
    __syncthreads();

    bool failed = false;
    for (int k = 0; k < ps; ++k) {
      const bool on_chip = k >= k0;
      if (k == k0 && k0 > 0) {  // move the trailing block on chip
        for (int64_t e = threadIdx.x; e < (int64_t)tn * tn; e += kCtaThreads) {
          const int r = (int)(e / tn), c = (int)(e % tn);
          T[(size_t)r * ldt + c] = W[(int64_t)(k0 + r) * ps + k0 + c];
        }
        __syncthreads();
      }
      auto elem = [&](int i, int j) -> double& {
        return on_chip && j >= k0 ? T[(size_t)(i - k0) * ldt + (j - k0)] : W[(int64_t)i * ps + j];
      };
      if (warp == 0) {
        double best;
        int p;
        column_pivot(k, ps, [&](int i) { return elem(i, k); }, best, p);
        if (lane == 0) {
          s_best = best;
          s_p = p;
        }
      }
      __syncthreads();
      const double best = s_best;
      const int p = s_p;
      if (best == 0.0 || best < __dmul_rn(1e-14, colmax[k])) {
        if (threadIdx.x == 0) {
          status[t] = k + 1;
          fail_best[t] = best;
        }
        failed = true;
        break;
      }
      if (p != k) {  // full row swap (dense.cpp:62-65)
        for (int j = threadIdx.x; j < ps; j += kCtaThreads) {
          double& a = elem(k, j);
          double& b = elem(p, j);
          const double x = a;
          a = b;
          b = x;
        }
        if (threadIdx.x == 0) {
          const int32_t x = perm[k];
          perm[k] = perm[p];
          perm[p] = x;
        }
        __syncthreads();
      }
      const double pv = elem(k, k);
      for (int i = k + 1 + (int)threadIdx.x; i < ps; i += kCtaThreads) {
        double& a = elem(i, k);
        const double l = __ddiv_rn(a, pv);
        a = l;
        lcol[i] = l;
      }
      __syncthreads();
      // trailing update: warp per row, lane per column (coalesced in either memory)
      if (on_chip) {
        const double* Uk = T + (size_t)(k - k0) * ldt - k0;
        for (int i = k + 1 + warp; i < ps; i += kCtaWarps) {
          const double l = lcol[i];
          if (l == 0.0) continue;
          double* Ti = T + (size_t)(i - k0) * ldt - k0;
          for (int j = k + 1 + lane; j < ps; j += 32) Ti[j] = __dsub_rn(Ti[j], __dmul_rn(l, Uk[j]));
        }
      } else {
        const double* Uk = W + (int64_t)k * ps;
        for (int i = k + 1 + warp; i < ps; i += kCtaWarps) {
          const double l = lcol[i];
          if (l == 0.0) continue;
          double* Wi = W + (int64_t)i * ps;
          for (int j = k + 1 + lane; j < ps; j += 32) Wi[j] = __dsub_rn(Wi[j], __dmul_rn(l, Uk[j]));
        }
      }
      __syncthreads();
    }
    if (!failed) {
      for (int64_t e = threadIdx.x; e < (int64_t)tn * tn; e += kCtaThreads) {
        const int r = (int)(e / tn), c = (int)(e % tn);
        W[(int64_t)(k0 + r) * ps + k0 + c] = T[(size_t)r * ldt + c];
      }
      for (int j = threadIdx.x; j < ps; j += kCtaThreads) piv[t * ps + j] = perm[j];
      if (threadIdx.x == 0) status[t] = 0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Blocked right-looking LU, CTA per matrix (default for ps > kSmemMaxPs).
// The matrix is factored in a per-CTA scratch copy (L2-resident) with its
// rows addressed through a row map: a row swap exchanges two map entries
// (and the two rows of the shared-memory panel), never moves data in global
// memory; the factor is written out in the pivoted order at the end.  Panels
// of kNb columns: (1) the panel (rows k0.., nb columns) is factored in
// shared memory with partial pivoting; (2) U12 by forward substitution with
// the unit L11, thread per column, rows in order; (3) the trailing block
// A22 -= L21 U12 with each element held in a register through its nb
// updates (warp per row, a lane holding kCols columns so the dependent
// mul/sub chains interleave).  Every element still sees
// a_ij <- a_ij - l_ik u_kj for k = 0, 1, ... in order, unfused, skipped where
// l_ik == 0, and the pivot of column k is chosen after all updates 0..k-1 --
// the unblocked algorithm's per-element sequence (dense.cpp:31-75), so
// factors and pivots are bitwise identical (tests/test_lu_large.py).
constexpr int kNb = 16;
constexpr int kCols = 6;  // trailing-update columns per lane (6 x 32 >= 192 - 16)
constexpr int kBlkThreads = 256;
constexpr int kBlkWarps = kBlkThreads / 32;

inline size_t blk_smem_bytes(int ps) {
  // panel [ps][kNb+1], U12 [kNb][ps], colmax [ps], perm [ps] (int), row map [ps] (int)
  return ((size_t)ps * (kNb + 1) + (size_t)kNb * ps + ps) * sizeof(double) + 2 * (size_t)ps * sizeof(int32_t);
}

__global__ void __launch_bounds__(kBlkThreads)
    lu_blocked_kernel(int64_t count, int ps, const double* __restrict__ mats, const int32_t* __restrict__ src,
                      double* __restrict__ lu, int32_t* __restrict__ piv, int32_t* __restrict__ status,
                      double* __restrict__ fail_best, double* __restrict__ scratch) {
  extern __shared__ double smem[];
  constexpr int LP = kNb + 1;
  double* Pn = smem;                       // panel rows [ps][LP] (row r = logical row k0 + r)
  double* Us = Pn + (size_t)ps * LP;       // U12 [kNb][ps]
  double* colmax = Us + (size_t)kNb * ps;  // [ps]
  int32_t* perm = reinterpret_cast<int32_t*>(colmax + ps);
  int32_t* rmap = perm + ps;  // logical row -> row of the scratch copy
  __shared__ double s_best;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t len = (int64_t)ps * ps;
  double* S = scratch + (int64_t)blockIdx.x * len;
  for (int64_t t = blockIdx.x; t < count; t += gridDim.x) {
    const double* A = mats + (src ? (int64_t)src[t] : t) * len;
    for (int64_t e = threadIdx.x; e < len; e += kBlkThreads) S[e] = A[e];
    for (int j = threadIdx.x; j < ps; j += kBlkThreads) {  // column maxima, 8 loads in flight
      double m = 0.0;
      for (int i0 = 0; i0 < ps; i0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i0 + u < ps ? A[(int64_t)(i0 + u) * ps + j] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) m = fmax(m, fabs(v[u]));
      }
      colmax[j] = m;
      perm[j] = j;
      rmap[j] = j;
    }
    __syncthreads();
    bool failed = false;
    for (int k0 = 0; k0 < ps && !failed; k0 += kNb) {
      const int nb = min(kNb, ps - k0), nr = ps - k0;
      // (1) panel into shared memory (logical row order) and its factorisation
      for (int e = threadIdx.x; e < nr * nb; e += kBlkThreads) {
        const int r = e / nb, c = e - r * nb;
        Pn[r * LP + c] = S[(int64_t)rmap[k0 + r] * ps + k0 + c];
      }
      __syncthreads();
      for (int kk = 0; kk < nb; ++kk) {
        const int k = k0 + kk;
        if (warp == 0) {
          double best = -1.0;
          int p = ps;
          for (int r = kk + lane; r < nr; r += 32) {
            const double v = fabs(Pn[r * LP + kk]);
            if (v > best) {
              best = v;
              p = k0 + r;
            }
          }
          warp_pivot(best, p);  // every lane holds the result
          const bool ok = !(best == 0.0 || best < __dmul_rn(1e-14, colmax[k]));
          if (lane == 0) {
            s_best = best;
            if (ok && p != k) {  // full row swap (dense.cpp:62-65): the map, the permutation
              int32_t x = perm[k];
              perm[k] = perm[p];
              perm[p] = x;
              x = rmap[k];
              rmap[k] = rmap[p];
              rmap[p] = x;
            }
          }
          if (ok && p != k && lane < nb) {  // and the two panel rows (lanes over the nb columns)
            const double x = Pn[kk * LP + lane];
            Pn[kk * LP + lane] = Pn[(p - k0) * LP + lane];
            Pn[(p - k0) * LP + lane] = x;
          }
        }
        __syncthreads();
        const double best = s_best;
        if (best == 0.0 || best < __dmul_rn(1e-14, colmax[k])) {
          if (threadIdx.x == 0) {
            status[t] = k + 1;
            fail_best[t] = best;
          }
          failed = true;
          break;
        }
        const double pv = Pn[kk * LP + kk];
        for (int r = kk + 1 + threadIdx.x; r < nr; r += kBlkThreads) Pn[r * LP + kk] = __ddiv_rn(Pn[r * LP + kk], pv);
        __syncthreads();
        const int w = nb - kk - 1;  // panel columns right of kk
        if (w > 0)
          for (int e = threadIdx.x; e < (nr - kk - 1) * w; e += kBlkThreads) {
            const int r = kk + 1 + e / w, c = kk + 1 + e % w;
            const double l = Pn[r * LP + kk];
            if (l != 0.0) Pn[r * LP + c] = __dsub_rn(Pn[r * LP + c], __dmul_rn(l, Pn[kk * LP + c]));
          }
        __syncthreads();
      }
      if (failed) break;
      for (int e = threadIdx.x; e < nr * nb; e += kBlkThreads) {  // panel back (logical rows via the map)
        const int r = e / nb, c = e - r * nb;
        S[(int64_t)rmap[k0 + r] * ps + k0 + c] = Pn[r * LP + c];
      }
      const int j0 = k0 + nb, nc = ps - j0;
      if (nc <= 0) {
        __syncthreads();
        break;
      }
      // (2) U12 = L11^{-1} A12, thread per column, rows in order
      for (int j = threadIdx.x; j < nc; j += kBlkThreads) {
        double u[kNb];
#pragma unroll
        for (int kk = 0; kk < kNb; ++kk) {
          if (kk >= nb) break;
          double* sp = S + (int64_t)rmap[k0 + kk] * ps + j0 + j;
          double a = *sp;
#pragma unroll
          for (int mm = 0; mm < kk; ++mm) {
            const double l = Pn[kk * LP + mm];
            if (l != 0.0) a = __dsub_rn(a, __dmul_rn(l, u[mm]));
          }
          u[kk] = a;
          *sp = a;
          Us[kk * ps + j] = a;
        }
      }
      __syncthreads();
      // (3) A22 -= L21 U12
      for (int i = j0 + warp; i < ps; i += kBlkWarps) {
        const double* Li = Pn + (i - k0) * LP;
        double* Wi = S + (int64_t)rmap[i] * ps + j0;
        for (int jb = 0; jb < nc; jb += 32 * kCols) {
          double a[kCols];
#pragma unroll
          for (int c = 0; c < kCols; ++c) {
            const int j = jb + lane + 32 * c;
            a[c] = j < nc ? Wi[j] : 0.0;
          }
          for (int kk = 0; kk < nb; ++kk) {
            const double l = Li[kk];
            if (l == 0.0) continue;  // warp-uniform (dense.cpp:70)
            const double* Uk = Us + kk * ps + jb + lane;
#pragma unroll
            for (int c = 0; c < kCols; ++c)
              if (jb + lane + 32 * c < nc) a[c] = __dsub_rn(a[c], __dmul_rn(l, Uk[32 * c]));
          }
#pragma unroll
          for (int c = 0; c < kCols; ++c) {
            const int j = jb + lane + 32 * c;
            if (j < nc) Wi[j] = a[c];
          }
        }
      }
      __syncthreads();
    }
    if (!failed) {
      double* W = lu + t * len;
      for (int64_t e = threadIdx.x; e < len; e += kBlkThreads) {
        const int i = (int)(e / ps), j = (int)(e - (int64_t)i * ps);
        W[e] = S[(int64_t)rmap[i] * ps + j];
      }
      for (int j = threadIdx.x; j < ps; j += kBlkThreads) piv[t * ps + j] = perm[j];
      if (threadIdx.x == 0) status[t] = 0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Reproducible PCG pieces (the oracle's orc_pcg order, oracle/pdb_oracle.c):
// the patch solve of lu_solve_into (dense.cpp:77-94) in the reference's
// order -- permutation, forward and backward substitution both row-oriented
// with ascending j -- on the column-major LU (F[j * ps + i] = LU(i, j)), one
// thread per patch; chunk sums of the blocked inner product; unfused axpys.
__global__ void patch_solve_ref_kernel(int64_t np, int ps, const int32_t* __restrict__ patches,
                                       const double* __restrict__ F, const int32_t* __restrict__ piv,
                                       const int32_t* __restrict__ phi, const double* __restrict__ r,
                                       const double* __restrict__ in_scale, double* __restrict__ sols) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int64_t f = phi ? (int64_t)phi[k] : k;
  const double* Fk = F + f * (int64_t)ps * ps;
  const int32_t* P = piv + f * ps;
  double* y = sols + k * ps;
  for (int i = 0; i < ps; ++i) {
    const int32_t g = patches[k * ps + P[i]];
    y[i] = in_scale ? __dmul_rn(r[g], in_scale[g]) : r[g];
  }
  for (int i = 1; i < ps; ++i) {
    double s = y[i];
    for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(Fk[(int64_t)j * ps + i], y[j]));
    y[i] = s;
  }
  for (int i = ps - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < ps; ++j) s = __dsub_rn(s, __dmul_rn(Fk[(int64_t)j * ps + i], y[j]));
    y[i] = __ddiv_rn(s, Fk[(int64_t)i * ps + i]);
  }
}

__global__ void dot_chunks_kernel(int64_t n, int chunk, const double* __restrict__ a, const double* __restrict__ b,
                                  double* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = c * chunk;
  if (i0 >= n) return;
  const int64_t i1 = i0 + chunk < n ? i0 + chunk : n;
  double s = 0.0;
  for (int64_t i = i0; i < i1; ++i) s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
  out[c] = s;
}

__global__ void axpy_ref_kernel(int64_t n, double alpha, const double* __restrict__ x, double* __restrict__ y,
                                int mode) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (mode == 0)
    y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i]));  // y += alpha x
  else if (mode == 1)
    y[i] = __dsub_rn(y[i], __dmul_rn(alpha, x[i]));  // y -= alpha x
  else
    y[i] = __dadd_rn(x[i], __dmul_rn(alpha, y[i]));  // y = x + alpha y
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
  } else if (std::getenv("PDB_LU_WARP") == nullptr && std::getenv("PDB_LU_CTA") == nullptr &&
             blk_smem_bytes(ps) <= 200 * 1024) {
    const size_t smem = blk_smem_bytes(ps);
    static int configured[64] = {};
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    if (smem > 48 * 1024 && dev < 64 && !configured[dev]) {
      PDB_CUDA(cudaFuncSetAttribute(lu_blocked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      configured[dev] = 1;
    }
    int sms = 148, per = 1;
    PDB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PDB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lu_blocked_kernel, kBlkThreads, smem));
    const unsigned g = (unsigned)std::min<int64_t>(count, (int64_t)sms * std::max(per, 1));
    Scratch<double> work(static_cast<size_t>(g) * ps * ps, s);  // one pivoting copy per CTA
    lu_blocked_kernel<<<g, kBlkThreads, smem, s>>>(count, ps, mats, src, lu, piv, status, fail_best, work.get());
  } else if (cta_smem_bytes(ps, cta_k0(ps)) <= kCtaSmemCap && std::getenv("PDB_LU_WARP") == nullptr) {
    const int k0 = cta_k0(ps);
    const size_t smem = cta_smem_bytes(ps, k0);
    static int configured[64] = {};
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && !configured[dev]) {
      PDB_CUDA(cudaFuncSetAttribute(lu_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCtaSmemCap + 4096));
      configured[dev] = 1;
    }
    int sms = 148;
    PDB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned g = (unsigned)std::min<int64_t>(count, (int64_t)sms);
    lu_cta_kernel<<<g, kCtaThreads, smem, s>>>(count, ps, k0, mats, src, lu, piv, status, fail_best);
  } else {
    const size_t smem = (size_t)kWarps * ps * sizeof(double);
    lu_kernel<false><<<grid, kWarps * 32, smem, s>>>(count, ps, mats, src, lu, piv, status, fail_best);
  }
}

void patch_solve_ref(int64_t np, int ps, const int32_t* patches, const double* F, const int32_t* piv,
                     const int32_t* phi, const double* r, const double* in_scale, double* sols, cudaStream_t s) {
  if (np > 0) patch_solve_ref_kernel<<<(unsigned)((np + 127) / 128), 128, 0, s>>>(np, ps, patches, F, piv, phi, r,
                                                                                 in_scale, sols);
}

void dot_chunks(int64_t n, int chunk, const double* a, const double* b, double* out, cudaStream_t s) {
  const int64_t nch = (n + chunk - 1) / chunk;
  if (nch > 0) dot_chunks_kernel<<<(unsigned)((nch + 127) / 128), 128, 0, s>>>(n, chunk, a, b, out);
}

void axpy_ref(int64_t n, double alpha, const double* x, double* y, int mode, cudaStream_t s) {
  if (n > 0) axpy_ref_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, alpha, x, y, mode);
}

}  // namespace pdb::k
