// Coarse correction of the combo preconditioner on the device (reference
// ComboPreconditioner::apply precond.cpp:115-121, band_factor /
// BandedFactor::solve_into banded.cpp:11-84):
//
//   z += P0 (R0 A P0)^{-1} R0 r
//
// Setup factors R0 A P0 once on the device on a cooperative grid (one
// barrier per column): the LAPACK-style partial-pivoting band LU (pivot =
// first maximum |.|, full row swap inside the band, multipliers by true
// division, a -= m*b updates unfused), so band, pivots and multipliers are
// bitwise the reference's.  Each apply is three launches:
//   restrict   rc = R0 r, one thread per coarse vertex summing its fine DoFs
//              in ascending order from 0.0 (= the reference's scatter order,
//              fem.cpp:373-382), bitwise;
//   solve      one of three coarse solvers (PDB_COARSE=dense|blocked|band):
//              dense    n_c <= 16384: the explicit inverse (its columns are
//                       the reference's solves of unit vectors, bitwise),
//                       one HBM-bound matrix-vector product per apply;
//              blocked  larger n_c: 2 n_c / Bk dense block maps, one
//                       cooperative kernel with a grid barrier per block;
//              band     one warp walks the 2 n_c steps (forward in the
//                       reference's order, backward column oriented);
//              the product / reordered sums give parity 1e-12 relative
//              (tests/test_combo.py), not bitwise;
//   prolong    z_i += sum_q p0_iq xc_q (<= 4 terms, in order), bitwise.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "host.hpp"

namespace pdb {

namespace {

// ---------------------------------------------------------------------------
// Band LU on a cooperative grid.  B is column-major band storage:
// B[j*ldab + r] holds the reference's ab[r*n + j] (band row r of column j).
// Step j: every CTA reads column j and finds the pivot itself (first maximum
// of |a(j+t, j)| -- the same deterministic (value, index) reduction in every
// CTA, so no broadcast is needed), applies the swap to its copy and forms the
// multipliers by true division; CTA 0 writes column j back.  Columns
// j+1..j+kv are dealt round-robin to the CTAs, each swapping rows j and p in
// its columns and applying a -= m*b (unfused) in ascending t.  One grid
// barrier per column.  Every element sees the reference's operations in the
// reference's order, so band and pivots are bitwise banded.cpp:11-60's.

constexpr int kFactorThreads = 512;

struct FactorSync {
  unsigned count;
  unsigned gen;
};

__device__ __forceinline__ void factor_barrier(FactorSync* sy) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = &sy->gen;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(&sy->count, 1u) == gridDim.x - 1) {
      sy->count = 0;
      __threadfence();
      atomicAdd(&sy->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kFactorThreads) band_factor_kernel(int n, int kl, int ku, int ldab, double* B,
                                                                     int32_t* ipiv, double* rdiag, int* bad_col,
                                                                     FactorSync* sy) {
  extern __shared__ double mult[];  // column j after the swap: [0] pivot, [t] multiplier t
  __shared__ double red_v[kFactorThreads / 32];
  __shared__ int red_t[kFactorThreads / 32];
  __shared__ double s_best;
  __shared__ int s_jp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kv = kl + ku;
  for (int j = 0; j < n; ++j) {
    const int km = min(kl, n - 1 - j);
    double* col = B + static_cast<int64_t>(j) * ldab;
    double bv = -1.0;
    int bt = 0;
    for (int t = tid; t <= km; t += kFactorThreads) {
      const double v = __ldcg(col + kv + t);
      mult[t] = v;
      const double a = fabs(v);
      if (a > bv) {
        bv = a;
        bt = t;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int ot = __shfl_xor_sync(0xffffffffu, bt, off);
      if (ov > bv || (ov == bv && ot < bt)) {
        bv = ov;
        bt = ot;
      }
    }
    if (lane == 0) {
      red_v[warp] = bv;
      red_t[warp] = bt;
    }
    __syncthreads();
    if (tid == 0) {
      double v = red_v[0];
      int t = red_t[0];
      for (int w = 1; w < kFactorThreads / 32; ++w)
        if (red_v[w] > v || (red_v[w] == v && red_t[w] < t)) {
          v = red_v[w];
          t = red_t[w];
        }
      s_best = v;
      s_jp = t;
      if (t != 0) {
        const double a = mult[0];
        mult[0] = mult[t];
        mult[t] = a;
      }
      if (v == 0.0 && blockIdx.x == 0) *bad_col = j;
    }
    __syncthreads();
    if (s_best == 0.0) return;  // every CTA sees the same column: all stop here
    const int jp = s_jp;
    const double piv = mult[0];
    __syncthreads();
    for (int t = 1 + tid; t <= km; t += kFactorThreads) mult[t] = __ddiv_rn(mult[t], piv);
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) {
      ipiv[j] = j + jp;
      rdiag[j] = __ddiv_rn(1.0, piv);
    }
    // columns j+1..jend, round-robin over the CTAs: swap rows j, j+jp, then
    // a(j+t, jj) -= m_t a(j, jj)
    const int jend = min(j + kv, n - 1);
    for (int jj = j + 1 + static_cast<int>(blockIdx.x); jj <= jend; jj += gridDim.x) {
      double* c = B + static_cast<int64_t>(jj) * ldab;
      const int r0 = kv + j - jj;  // band row of matrix row j in column jj
      double u = __ldcg(c + r0);
      if (jp != 0) {
        const double w = __ldcg(c + r0 + jp);
        __syncthreads();  // every thread has read u and w before they are overwritten
        if (tid == 0) {
          c[r0] = w;
          c[r0 + jp] = u;
        }
        u = w;
        __syncthreads();
      }
      for (int t = 1 + tid; t <= km; t += kFactorThreads) {
        const double m = mult[t];
        if (m == 0.0) continue;
        c[r0 + t] = __dsub_rn(__ldcg(c + r0 + t), __dmul_rn(m, u));
      }
    }
    factor_barrier(sy);
    // column j is written back only now: every CTA has finished reading it
    if (blockIdx.x == 0) {
      for (int t = tid; t <= km; t += kFactorThreads) col[kv + t] = mult[t];
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Band solve, one warp.  w (shared memory, or global scratch for large n)
// holds the working vector.  R = entries per lane of one band column
// (ceil(kv / 32)), D = steps whose band columns are prefetched at a time.

template <int R, int D, bool SMEM>
__global__ void __launch_bounds__(32) band_solve_kernel(int n, int kl, int ku, int ldab, const double* __restrict__ B,
                                                        const int32_t* __restrict__ ipiv,
                                                        const double* __restrict__ rdiag, const double* __restrict__ rhs,
                                                        double* __restrict__ x, double* gwork) {
  extern __shared__ double sw[];
  double* w = SMEM ? sw : gwork;  // a compile-time choice keeps shared accesses LDS/STS
  const int lane = threadIdx.x;
  const int kv = kl + ku;
  for (int i = lane; i < n; i += 32) w[i] = rhs[i];
  __syncwarp();

  // forward: for j ascending, swap (j, ipiv[j]) then out[j+t] -= l(t, j) out[j]
  double Lc[D][R], Ln[D][R];
  int pc[D], pn[D];
  auto load_fwd = [&](int j0, double (&L)[D][R], int (&pv)[D]) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int j = j0 + d;
      pv[d] = j < n ? ipiv[j] : j;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = 1 + lane + 32 * r;
        L[d][r] = (j < n && t <= kl && j + t < n) ? B[static_cast<int64_t>(j) * ldab + kv + t] : 0.0;
      }
    }
  };
  load_fwd(0, Lc, pc);
  double prev = 0.0;  // x_{j-1}: lane 0 stores it one step late (w[j-1] is not read in step j)
  for (int j0 = 0; j0 < n; j0 += D) {
    load_fwd(j0 + D, Ln, pn);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int j = j0 + d;
      if (j < n) {
        const int km = min(kl, n - 1 - j);
        const int p = pc[d];
        const double oj = w[j], op = w[p];
        double base[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int t = 1 + lane + 32 * r;
          base[r] = t <= km ? w[j + t] : 0.0;
        }
        const double xj = p != j ? op : oj;
        if (lane == 0 && j > 0) w[j - 1] = prev;
        prev = xj;
        const bool nz = xj != 0.0;  // the reference skips the column when x_j == 0
#pragma unroll
        for (int r = 0; r < R; ++r) {  // branch-free: selects and a predicated store
          const int t = 1 + lane + 32 * r;
          const double b = j + t == p ? oj : base[r];
          const double u = __dsub_rn(b, __dmul_rn(Lc[d][r], xj));
          const double v = nz ? u : b;
          if (t <= km) w[j + t] = v;
        }
        __syncwarp();
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      pc[d] = pn[d];
#pragma unroll
      for (int r = 0; r < R; ++r) Lc[d][r] = Ln[d][r];
    }
  }
  if (lane == 0 && n > 0) w[n - 1] = prev;
  __syncwarp();

  // backward, column oriented: x_i = out_i / u_ii; out[i-e] -= u(i-e, i) x_i
  double Uc[D][R], Un[D][R], rc[D], rn[D];
  auto load_bwd = [&](int i0, double (&U)[D][R], double (&rd)[D]) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int i = i0 - d;
      rd[d] = i >= 0 ? rdiag[i] : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int e = 1 + lane + 32 * r;
        U[d][r] = (i >= 0 && e <= kv && e <= i) ? B[static_cast<int64_t>(i) * ldab + kv - e] : 0.0;
      }
    }
  };
  load_bwd(n - 1, Uc, rc);
  for (int i0 = n - 1; i0 >= 0; i0 -= D) {
    load_bwd(i0 - D, Un, rn);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int i = i0 - d;
      if (i >= 0) {
        const int cnt = min(kv, i);
        const double xi = __dmul_rn(w[i], rc[d]);
        double base[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = 1 + lane + 32 * r;
          base[r] = e <= cnt ? w[i - e] : 0.0;
        }
        if (lane == 0) x[i] = xi;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = 1 + lane + 32 * r;
          const double v = __dsub_rn(base[r], __dmul_rn(Uc[d][r], xi));
          if (e <= cnt) w[i - e] = v;
        }
        __syncwarp();
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      rc[d] = rn[d];
#pragma unroll
      for (int r = 0; r < R; ++r) Uc[d][r] = Un[d][r];
    }
  }
}

// rc_c = sum over R0 row c (ascending fine DoF) of r0 * r, from 0.0
__global__ void restrict_kernel(int nc, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                const double* __restrict__ val, const double* __restrict__ r, double* __restrict__ rc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double s = 0.0;
  for (int q = ptr[c]; q < ptr[c + 1]; ++q) s = __dadd_rn(s, __dmul_rn(val[q], r[col[q]]));
  rc[c] = s;
}

// z_i += sum over P0 row i of p0 * xc, from 0.0
__global__ void prolong_add_kernel(int64_t n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                   const double* __restrict__ val, const double* __restrict__ xc,
                                   double* __restrict__ z) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q) s = __dadd_rn(s, __dmul_rn(val[q], xc[col[q]]));
  z[i] = __dadd_rn(z[i], s);
}

// ---------------------------------------------------------------------------
// Dense inverse (n_c <= kDenseMax): setup solves the n_c unit vectors, one
// thread per column, each exactly as BandedFactor::solve_into (forward with
// swaps and zero skips, backward row sums in ascending column order, true
// division), so column c of Z is bitwise the reference's solve of e_c.
// Z is row-major [n_c][ld] (ld = n_c rounded up to 64, zero padded): the 32
// threads of a warp touch 256 contiguous bytes of one row per access.  Each
// apply is then one bandwidth-bound dense matrix-vector product over all SMs
// instead of 2 n_c dependent steps.

__global__ void __launch_bounds__(128) band_inverse_kernel(int n, int kl, int ku, int ldab, int ld,
                                                           const double* __restrict__ B,
                                                           const int32_t* __restrict__ ipiv, double* __restrict__ Z) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int kv = kl + ku;
  auto z = [&](int i) -> double& { return Z[static_cast<int64_t>(i) * ld + c]; };
  z(c) = 1.0;
  // steps j < c - kl only see zeros (a swap partner p <= j + kl < c)
  for (int j = max(0, c - kl); j < n; ++j) {
    const int p = ipiv[j];
    if (p != j) {
      const double a = z(j);
      z(j) = z(p);
      z(p) = a;
    }
    const double xj = z(j);
    if (xj == 0.0) continue;
    const int km = min(kl, n - 1 - j);
    const double* col = B + static_cast<int64_t>(j) * ldab + kv;
    // batches of 8 independent loads in flight, then the updates
    for (int t0 = 1; t0 <= km; t0 += 8) {
      double zv[8], lv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int t = t0 + q;
        zv[q] = t <= km ? z(j + t) : 0.0;
        lv[q] = t <= km ? col[t] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (t0 + q <= km) z(j + t0 + q) = __dsub_rn(zv[q], __dmul_rn(lv[q], xj));
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double sum = z(i);
    const int jend = min(i + kv, n - 1);
    for (int j0 = i + 1; j0 <= jend; j0 += 8) {
      double zv[8], uv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int jj = j0 + q;
        zv[q] = jj <= jend ? z(jj) : 0.0;
        uv[q] = jj <= jend ? B[static_cast<int64_t>(jj) * ldab + kv + i - jj] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (j0 + q <= jend) sum = __dsub_rn(sum, __dmul_rn(uv[q], zv[q]));  // ascending jj, as the reference
    }
    z(i) = __ddiv_rn(sum, B[static_cast<int64_t>(i) * ldab + kv]);
  }
}

constexpr int kGemvWarps = 16;
constexpr Index kDenseMax = 16384;  // 2 GB inverse, ~0.1 s setup

// xc = Z rc: one warp per row, 16-byte loads, rc staged in shared memory.
__global__ void __launch_bounds__(kGemvWarps * 32) dense_apply_kernel(int nc, int ld, const double* __restrict__ Z,
                                                                      const double* __restrict__ rc,
                                                                      double* __restrict__ xc) {
  extern __shared__ double s_rc[];
  for (int i = threadIdx.x; i < ld; i += blockDim.x) s_rc[i] = i < nc ? rc[i] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = ld / 2;
  const double2* sv = reinterpret_cast<const double2*>(s_rc);
  for (int row = blockIdx.x * kGemvWarps + warp; row < nc; row += gridDim.x * kGemvWarps) {
    const double2* a = reinterpret_cast<const double2*>(Z + static_cast<int64_t>(row) * ld);
    double s0 = 0.0, s1 = 0.0;
    int k = lane;
    for (; k + 96 < half; k += 128) {
      const double2 v0 = __ldcs(a + k), v1 = __ldcs(a + k + 32), v2 = __ldcs(a + k + 64), v3 = __ldcs(a + k + 96);
      const double2 r0 = sv[k], r1 = sv[k + 32], r2 = sv[k + 64], r3 = sv[k + 96];
      s0 = fma(v0.x, r0.x, s0);
      s1 = fma(v0.y, r0.y, s1);
      s0 = fma(v1.x, r1.x, s0);
      s1 = fma(v1.y, r1.y, s1);
      s0 = fma(v2.x, r2.x, s0);
      s1 = fma(v2.y, r2.y, s1);
      s0 = fma(v3.x, r3.x, s0);
      s1 = fma(v3.y, r3.y, s1);
    }
    for (; k < half; k += 32) {
      const double2 v = __ldcs(a + k), r = sv[k];
      s0 = fma(v.x, r.x, s0);
      s1 = fma(v.y, r.y, s1);
    }
    double sum = s0 + s1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) xc[row] = sum;
  }
}

// ---------------------------------------------------------------------------
// Blocked solve (n_c > kDenseMax): the 2 n_c dependent steps become
// 2 n_c / Bk dense matrix-vector products over all SMs.
//   forward  block k (steps J..J+Bk-1 of the pivoted elimination) touches
//            only rows [J, J+Bk+kl): it is the dense map F_k of that segment
//            (the Bk swaps and rank-1 updates applied to the identity);
//   backward x_J = U_JJ^{-1} (y_J - U_JR x_R), R = the next kv rows:
//            G_k = [U_JJ^{-1} | -U_JJ^{-1} U_JR].
// Setup builds every F_k / G_k column in parallel (one thread per column,
// the band factor's own steps); each apply is one cooperative kernel with a
// grid barrier per block.  Rows [J, J+Bk) leave a forward block final; the
// kl rows after them are carried (ping-pong) into the next block.

__global__ void fwd_block_kernel(int n, int kl, int ku, int ldab, int bk, int nblk, const double* __restrict__ B,
                                 const int32_t* __restrict__ ipiv, const int64_t* __restrict__ off,
                                 double* __restrict__ F) {
  const int k = blockIdx.y;
  const int J = k * bk;
  const int bj = min(bk, n - J), m = min(n, J + bk + kl) - J;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nblk || c >= m) return;
  const int kv = kl + ku;
  double* col = F + off[k] + c;  // element (r, c) at col[r * m]
  for (int r = 0; r < m; ++r) col[static_cast<int64_t>(r) * m] = r == c ? 1.0 : 0.0;
  for (int j = J; j < J + bj; ++j) {
    const int lj = j - J, lp = ipiv[j] - J;
    if (lp != lj) {
      const double a = col[static_cast<int64_t>(lj) * m];
      col[static_cast<int64_t>(lj) * m] = col[static_cast<int64_t>(lp) * m];
      col[static_cast<int64_t>(lp) * m] = a;
    }
    const double xj = col[static_cast<int64_t>(lj) * m];
    if (xj == 0.0) continue;
    const int km = min(kl, n - 1 - j);
    const double* l = B + static_cast<int64_t>(j) * ldab + kv;
    for (int t = 1; t <= km; ++t) {
      double& y = col[static_cast<int64_t>(lj + t) * m];
      y = __dsub_rn(y, __dmul_rn(l[t], xj));
    }
  }
}

__global__ void bwd_block_kernel(int n, int kl, int ku, int ldab, int bk, int nblk, const double* __restrict__ B,
                                 const int64_t* __restrict__ off, double* __restrict__ G) {
  const int k = blockIdx.y;
  const int J = k * bk;
  const int bj = min(bk, n - J), nr = min(kl + ku, n - J - bj), w = bj + nr;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nblk || c >= w) return;
  const int kv = kl + ku;
  auto U = [&](int i, int col) -> double {  // U(i, col) of the band factor, 0 outside the band
    return (col >= i && col - i <= kv) ? B[static_cast<int64_t>(col) * ldab + kv + i - col] : 0.0;
  };
  double* z = G + off[k] + c;  // element (r, c) at z[r * w]
  for (int r = 0; r < bj; ++r) z[static_cast<int64_t>(r) * w] = c < bj ? (r == c ? 1.0 : 0.0) : U(J + r, J + c);
  for (int i = bj - 1; i >= 0; --i) {
    double sum = z[static_cast<int64_t>(i) * w];
    const int kend = min(bj - 1, i + kv);
    for (int q = i + 1; q <= kend; ++q) sum = __dsub_rn(sum, __dmul_rn(U(J + i, J + q), z[static_cast<int64_t>(q) * w]));
    z[static_cast<int64_t>(i) * w] = __ddiv_rn(sum, U(J + i, J + i));
  }
  if (c >= bj)
    for (int r = 0; r < bj; ++r) z[static_cast<int64_t>(r) * w] = -z[static_cast<int64_t>(r) * w];
}

struct BlockSync {
  unsigned count;
  unsigned gen;
};

__device__ __forceinline__ void coarse_grid_barrier(BlockSync* sy) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = &sy->gen;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(&sy->count, 1u) == gridDim.x - 1) {
      sy->count = 0;
      __threadfence();
      atomicAdd(&sy->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kBlkThreads = 256;

// Row r of a dense (rows x w) block times the staged vector v (shared).
__device__ __forceinline__ double row_dot(const double* __restrict__ row, int w, const double* v, int lane) {
  double s0 = 0.0, s1 = 0.0;
  int c = lane;
  for (; c + 32 < w; c += 64) {
    s0 = fma(__ldcs(row + c), v[c], s0);
    s1 = fma(__ldcs(row + c + 32), v[c + 32], s1);
  }
  if (c < w) s0 = fma(__ldcs(row + c), v[c], s0);
  double sum = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  return sum;
}

__global__ void __launch_bounds__(kBlkThreads) blocked_solve_kernel(int n, int kl, int kv, int bk, int nblk,
                                                                    const int64_t* __restrict__ foff,
                                                                    const int64_t* __restrict__ goff,
                                                                    const double* __restrict__ F,
                                                                    const double* __restrict__ G,
                                                                    const double* __restrict__ rhs, double* yf,
                                                                    double* carry, double* x, BlockSync* sy) {
  extern __shared__ double sv[];
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (kBlkThreads / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (kBlkThreads / 32);
  for (int k = 0; k < nblk; ++k) {
    const int J = k * bk, bj = min(bk, n - J), m = min(n, J + bk + kl) - J;
    const int cin = k == 0 ? 0 : min(kl, m);
    const double* cur = carry + (k & 1) * kl;
    double* nxt = carry + ((k + 1) & 1) * kl;
    for (int i = threadIdx.x; i < m; i += kBlkThreads) sv[i] = i < cin ? __ldcg(cur + i) : rhs[J + i];
    __syncthreads();
    const double* Fk = F + foff[k];
    for (int r = gw; r < m; r += nw) {
      const double v = row_dot(Fk + static_cast<int64_t>(r) * m, m, sv, lane);
      if (lane == 0) {
        if (r < bj) yf[J + r] = v;
        else nxt[r - bj] = v;
      }
    }
    coarse_grid_barrier(sy);
  }
  for (int k = nblk - 1; k >= 0; --k) {
    const int J = k * bk, bj = min(bk, n - J), nr = min(kv, n - J - bj), w = bj + nr;
    for (int i = threadIdx.x; i < w; i += kBlkThreads) sv[i] = i < bj ? __ldcg(yf + J + i) : __ldcg(x + J + i);
    __syncthreads();
    const double* Gk = G + goff[k];
    for (int r = gw; r < bj; r += nw) {
      const double v = row_dot(Gk + static_cast<int64_t>(r) * w, w, sv, lane);
      if (lane == 0) x[J + r] = v;
    }
    coarse_grid_barrier(sy);
  }
}

// Same solve with the next block's matrix row prefetched into registers
// before each grid barrier (the HBM latency of the 2-5 MB block hides behind
// the barrier); one row per warp, so it needs rows <= warps and width <= 32 R.
template <int R>
__global__ void __launch_bounds__(kBlkThreads) blocked_solve_pf_kernel(int n, int kl, int kv, int bk, int nblk,
                                                                       const int64_t* __restrict__ foff,
                                                                       const int64_t* __restrict__ goff,
                                                                       const double* __restrict__ F,
                                                                       const double* __restrict__ G,
                                                                       const double* __restrict__ rhs, double* yf,
                                                                       double* carry, double* x, BlockSync* sy) {
  extern __shared__ double sv[];  // 32 R entries, zero past the block width
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (kBlkThreads / 32) + (threadIdx.x >> 5);
  const int nsteps = 2 * nblk;
  double fr[R];
  auto prefetch = [&](int st) {
    const bool fwd = st < nblk;
    const int k = fwd ? st : nsteps - 1 - st;
    const int J = k * bk, bj = min(bk, n - J);
    const int width = fwd ? min(n, J + bk + kl) - J : bj + min(kv, n - J - bj);
    const int rows = fwd ? width : bj;
    const double* row = (fwd ? F + foff[k] : G + goff[k]) + static_cast<int64_t>(gw) * width;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = lane + 32 * i;
      fr[i] = (gw < rows && c < width) ? __ldcs(row + c) : 0.0;
    }
  };
  prefetch(0);
  for (int st = 0; st < nsteps; ++st) {
    const bool fwd = st < nblk;
    const int k = fwd ? st : nsteps - 1 - st;
    const int J = k * bk, bj = min(bk, n - J);
    int width, rows;
    if (fwd) {
      width = min(n, J + bk + kl) - J;
      rows = width;
      const int cin = k == 0 ? 0 : min(kl, width);
      const double* cur = carry + (k & 1) * kl;
      for (int i = threadIdx.x; i < 32 * R; i += kBlkThreads)
        sv[i] = i < cin ? __ldcg(cur + i) : (i < width ? rhs[J + i] : 0.0);
    } else {
      width = bj + min(kv, n - J - bj);
      rows = bj;
      for (int i = threadIdx.x; i < 32 * R; i += kBlkThreads)
        sv[i] = i < bj ? __ldcg(yf + J + i) : (i < width ? __ldcg(x + J + i) : 0.0);
    }
    __syncthreads();
    if (gw < rows) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int i = 0; i < R; i += 4) {
        a0 = fma(fr[i], sv[lane + 32 * i], a0);
        if (i + 1 < R) a1 = fma(fr[i + 1], sv[lane + 32 * (i + 1)], a1);
        if (i + 2 < R) a2 = fma(fr[i + 2], sv[lane + 32 * (i + 2)], a2);
        if (i + 3 < R) a3 = fma(fr[i + 3], sv[lane + 32 * (i + 3)], a3);
      }
      double v = (a0 + a1) + (a2 + a3);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) {
        if (!fwd) x[J + gw] = v;
        else if (gw < bj) yf[J + gw] = v;
        else carry[((k + 1) & 1) * kl + gw - bj] = v;
      }
    }
    if (st + 1 < nsteps) prefetch(st + 1);
    coarse_grid_barrier(sy);
  }
}

constexpr size_t kSolveSmem = 200 * 1024;

template <int R, int D>
void launch_solve(const CoarseDev& c, const double* rhs, double* x, double* gwork, cudaStream_t s) {
  const size_t smem = gwork ? 0 : static_cast<size_t>(c.nc) * sizeof(double);
  auto kern = gwork ? band_solve_kernel<R, D, false> : band_solve_kernel<R, D, true>;
  if (smem > 48 * 1024) PDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<1, 32, smem, s>>>(static_cast<int>(c.nc), static_cast<int>(c.kl), static_cast<int>(c.ku),
                           static_cast<int>(c.ldab), c.band.get(), c.ipiv.get(), c.rdiag.get(), rhs, x, gwork);
}

template <typename T>
void upload_vec(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  d.alloc(std::max<size_t>(h.size(), 1));
  if (!h.empty()) d.upload(h.data(), h.size(), s);
}

void upload_op(const CoarseOp& op, DevBuf<int32_t>& ptr, DevBuf<int32_t>& col, DevBuf<double>& val, cudaStream_t s) {
  require(op.ptr.back() < (int64_t{1} << 31), Errc::invalid_argument, "coarse transfer operator too large");
  std::vector<int32_t> p32(op.ptr.begin(), op.ptr.end());
  upload_vec(ptr, p32, s);
  upload_vec(col, op.col, s);
  upload_vec(val, op.val, s);
}

}  // namespace

void coarse_setup(const CoarseSpaceHost& cs, CoarseDev& out, cudaStream_t s) {
  require_device();
  const CoarseOp& A = cs.coarse;
  require(A.rows >= 1, Errc::invalid_argument, "band_factor needs a nonempty matrix");
  require(A.rows < (Index{1} << 31), Errc::invalid_argument, "coarse space too large");
  Index kl = 0, ku = 0;
  for (Index i = 0; i < A.rows; ++i)
    for (int64_t q = A.ptr[static_cast<size_t>(i)]; q < A.ptr[static_cast<size_t>(i) + 1]; ++q) {
      kl = std::max<Index>(kl, i - A.col[static_cast<size_t>(q)]);
      ku = std::max<Index>(ku, A.col[static_cast<size_t>(q)] - i);
    }
  const Index n = A.rows, kv = kl + ku, ldab = 2 * kl + ku + 1;
  std::vector<double> band(static_cast<size_t>(n * ldab), 0.0);
  for (Index i = 0; i < n; ++i)
    for (int64_t q = A.ptr[static_cast<size_t>(i)]; q < A.ptr[static_cast<size_t>(i) + 1]; ++q) {
      const Index c = A.col[static_cast<size_t>(q)];
      band[static_cast<size_t>(c * ldab + kv + i - c)] = A.val[static_cast<size_t>(q)];
    }
  out.fine_n = cs.p0.rows;
  out.nc = n;
  out.kl = kl;
  out.ku = ku;
  out.ldab = ldab;
  upload_vec(out.band, band, s);
  out.ipiv.alloc(static_cast<size_t>(n));
  out.rdiag.alloc(static_cast<size_t>(n));
  Scratch<int> bad(1, s);
  PDB_CUDA(cudaMemsetAsync(bad.get(), 0xff, sizeof(int), s));
  const size_t smem = static_cast<size_t>(kl + 1) * sizeof(double);
  require(smem <= 200 * 1024, Errc::invalid_argument, "coarse band too wide");
  if (smem > 48 * 1024)
    PDB_CUDA(cudaFuncSetAttribute(band_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  {
    Scratch<FactorSync> fsync(1, s);
    PDB_CUDA(cudaMemsetAsync(fsync.get(), 0, sizeof(FactorSync), s));
    int per_sm = 0;
    PDB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, band_factor_kernel, kFactorThreads, smem));
    // about 4 trailing columns per CTA per step, at most one CTA per SM
    const int grid = static_cast<int>(std::max<Index>(1, std::min<Index>((kv + 3) / 4, static_cast<Index>(num_sms()) *
                                                                                       std::max(per_sm, 1))));
    int n_ = static_cast<int>(n), kl_ = static_cast<int>(kl), ku_ = static_cast<int>(ku), ld_ = static_cast<int>(ldab);
    double* bp = out.band.get();
    int32_t* ip = out.ipiv.get();
    double* rd = out.rdiag.get();
    int* bc = bad.get();
    FactorSync* fs = fsync.get();
    void* args[] = {&n_, &kl_, &ku_, &ld_, &bp, &ip, &rd, &bc, &fs};
    PDB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(band_factor_kernel), dim3(grid),
                                         dim3(kFactorThreads), args, smem, s));
    PDB_LAUNCH_CHECK();
    sync(s);
  }
  upload_op(cs.p0, out.p0_ptr, out.p0_col, out.p0_val, s);
  upload_op(cs.r0, out.r0_ptr, out.r0_col, out.r0_val, s);
  int bad_h = -1;
  PDB_CUDA(cudaMemcpyAsync(&bad_h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  sync(s);
  if (bad_h >= 0)
    fail(Errc::singular_matrix, "banded factorization hit a zero pivot in column " + std::to_string(bad_h));
  // dense inverse for small coarse spaces (PDB_COARSE=band / dense forces a path)
  const char* e = getenv("PDB_COARSE");
  const bool dense = e ? std::string(e) == "dense" : n <= kDenseMax;
  out.ld = 0;
  if (dense) {
    const Index ld = (n + 63) / 64 * 64;
    require(static_cast<size_t>(ld) * sizeof(double) <= kSolveSmem, Errc::invalid_argument,
            "coarse space too large for the dense inverse (PDB_COARSE=dense)");
    out.inv.alloc(static_cast<size_t>(n * ld));
    PDB_CUDA(cudaMemsetAsync(out.inv.get(), 0, static_cast<size_t>(n * ld) * sizeof(double), s));
    band_inverse_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(
        static_cast<int>(n), static_cast<int>(kl), static_cast<int>(ku), static_cast<int>(ldab), static_cast<int>(ld),
        out.band.get(), out.ipiv.get(), out.inv.get());
    PDB_LAUNCH_CHECK();
    sync(s);
    out.ld = ld;
    return;
  }
  const bool blocked = e ? std::string(e) == "blocked" : true;
  if (!blocked) return;
  // blocked solve: Bk = 2 kl steps per block (>= 32), trimmed so that a
  // backward row (Bk + kv wide) fits the 1024-column register row when that
  // costs less than a quarter of the block
  Index bk = std::max<Index>(32, 2 * kl);
  if (bk + kv > 1024 && 1024 - kv >= (3 * bk) / 4) bk = 1024 - kv;
  const Index nblk = (n + bk - 1) / bk;
  std::vector<int64_t> foff(static_cast<size_t>(nblk)), goff(static_cast<size_t>(nblk));
  int64_t fo = 0, go = 0;
  Index fmax = 0, gmax = 0;
  for (Index k = 0; k < nblk; ++k) {
    const Index J = k * bk, bj = std::min(bk, n - J), m = std::min(n, J + bk + kl) - J;
    const Index w = bj + std::min(kv, n - J - bj);
    foff[static_cast<size_t>(k)] = fo;
    goff[static_cast<size_t>(k)] = go;
    fo += m * m;
    go += bj * w;
    fmax = std::max(fmax, m);
    gmax = std::max(gmax, w);
  }
  out.bk = bk;
  out.nblk = nblk;
  out.vmax = std::max(fmax, gmax);
  upload_vec(out.foff, foff, s);
  upload_vec(out.goff, goff, s);
  out.fblk.alloc(static_cast<size_t>(fo));
  out.gblk.alloc(static_cast<size_t>(go));
  fwd_block_kernel<<<dim3(static_cast<unsigned>((fmax + 127) / 128), static_cast<unsigned>(nblk)), 128, 0, s>>>(
      static_cast<int>(n), static_cast<int>(kl), static_cast<int>(ku), static_cast<int>(ldab), static_cast<int>(bk),
      static_cast<int>(nblk), out.band.get(), out.ipiv.get(), out.foff.get(), out.fblk.get());
  bwd_block_kernel<<<dim3(static_cast<unsigned>((gmax + 127) / 128), static_cast<unsigned>(nblk)), 128, 0, s>>>(
      static_cast<int>(n), static_cast<int>(kl), static_cast<int>(ku), static_cast<int>(ldab), static_cast<int>(bk),
      static_cast<int>(nblk), out.band.get(), out.goff.get(), out.gblk.get());
  PDB_LAUNCH_CHECK();
  sync(s);
}

void coarse_correct(const CoarseDev& c, const double* r, double* z, cudaStream_t s) {
  const size_t nc = static_cast<size_t>(c.nc);
  Scratch<double> rc(nc, s), xc(nc, s);
  const bool in_smem = nc * sizeof(double) <= kSolveSmem;
  Scratch<double> work(in_smem ? 1 : nc, s);
  double* gwork = in_smem ? nullptr : work.get();
  restrict_kernel<<<static_cast<unsigned>((nc + 255) / 256), 256, 0, s>>>(
      static_cast<int>(nc), c.r0_ptr.get(), c.r0_col.get(), c.r0_val.get(), r, rc.get());
  if (c.ld > 0) {
    const size_t smem = static_cast<size_t>(c.ld) * sizeof(double);
    if (smem > 48 * 1024)
      PDB_CUDA(cudaFuncSetAttribute(dense_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int rows_per = kGemvWarps;
    const unsigned grid = static_cast<unsigned>(std::min<Index>((c.nc + rows_per - 1) / rows_per, 148 * 2));
    dense_apply_kernel<<<grid, kGemvWarps * 32, smem, s>>>(static_cast<int>(c.nc), static_cast<int>(c.ld), c.inv.get(),
                                                          rc.get(), xc.get());
    prolong_add_kernel<<<static_cast<unsigned>((c.fine_n + 255) / 256), 256, 0, s>>>(
        c.fine_n, c.p0_ptr.get(), c.p0_col.get(), c.p0_val.get(), xc.get(), z);
    PDB_LAUNCH_CHECK();
    return;
  }
  if (c.nblk > 0) {
    const size_t smem = static_cast<size_t>(c.vmax) * sizeof(double);
    require(smem <= kSolveSmem, Errc::invalid_argument, "coarse band too wide for the blocked solve");
    if (smem > 48 * 1024)
      PDB_CUDA(cudaFuncSetAttribute(blocked_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    Scratch<BlockSync> bsync(1, s);  // per call: concurrent applies on one handle stay independent
    PDB_CUDA(cudaMemsetAsync(bsync.get(), 0, sizeof(BlockSync), s));
    BlockSync* sy = bsync.get();
    Scratch<double> yf(nc, s), carry(static_cast<size_t>(2 * std::max<Index>(c.kl, 1)), s);
    int n_ = static_cast<int>(c.nc), kl_ = static_cast<int>(c.kl), kv_ = static_cast<int>(c.kl + c.ku),
        bk_ = static_cast<int>(c.bk), nb_ = static_cast<int>(c.nblk);
    const int64_t* fo = c.foff.get();
    const int64_t* go = c.goff.get();
    const double* F = c.fblk.get();
    const double* G = c.gblk.get();
    const double* rhs = rc.get();
    double* yfp = yf.get();
    double* cp = carry.get();
    double* xp = xc.get();
    void* args[] = {&n_, &kl_, &kv_, &bk_, &nb_, &fo, &go, &F, &G, &rhs, &yfp, &cp, &xp, &sy};
    // register-prefetched variant when one row per warp suffices
    const Index rows_max = c.bk + c.kl;  // forward block height
    const char* pe = getenv("PDB_COARSE_PF");
    const bool pf_ok = !(pe && pe[0] == '0') && c.vmax <= 32 * 48 && rows_max <= num_sms() * (kBlkThreads / 32);
    void* kern = reinterpret_cast<void*>(blocked_solve_kernel);
    size_t ksmem = smem;
    if (pf_ok) {
      const int R = c.vmax <= 256 ? 8 : c.vmax <= 512 ? 16 : c.vmax <= 1024 ? 32 : 48;
      kern = R == 8 ? reinterpret_cast<void*>(blocked_solve_pf_kernel<8>)
             : R == 16 ? reinterpret_cast<void*>(blocked_solve_pf_kernel<16>)
             : R == 32 ? reinterpret_cast<void*>(blocked_solve_pf_kernel<32>)
                       : reinterpret_cast<void*>(blocked_solve_pf_kernel<48>);
      ksmem = static_cast<size_t>(32 * R) * sizeof(double);
    }
    int per_sm = 0;
    PDB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlkThreads, ksmem));
    // the prefetch variant needs rows_max warps: one CTA per SM is enough and
    // keeps the barrier cheap
    const int grid = pf_ok ? num_sms() : std::max(1, std::min(per_sm, 2) * num_sms());
    require(per_sm >= 1, Errc::internal, "coarse solve kernel cannot be resident");
    PDB_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kBlkThreads), args, ksmem, s));
    prolong_add_kernel<<<static_cast<unsigned>((c.fine_n + 255) / 256), 256, 0, s>>>(
        c.fine_n, c.p0_ptr.get(), c.p0_col.get(), c.p0_val.get(), xc.get(), z);
    PDB_LAUNCH_CHECK();
    return;
  }
  const Index kv = c.kl + c.ku;
  if (kv <= 32)
    launch_solve<1, 16>(c, rc.get(), xc.get(), gwork, s);
  else if (kv <= 64)
    launch_solve<2, 16>(c, rc.get(), xc.get(), gwork, s);
  else if (kv <= 128)
    launch_solve<4, 8>(c, rc.get(), xc.get(), gwork, s);
  else if (kv <= 256)
    launch_solve<8, 4>(c, rc.get(), xc.get(), gwork, s);
  else if (kv <= 512)
    launch_solve<16, 2>(c, rc.get(), xc.get(), gwork, s);
  else
    fail(Errc::invalid_argument, "coarse band wider than 512 (more than ~254 cells per axis)");
  prolong_add_kernel<<<static_cast<unsigned>((c.fine_n + 255) / 256), 256, 0, s>>>(
      c.fine_n, c.p0_ptr.get(), c.p0_col.get(), c.p0_val.get(), xc.get(), z);
  PDB_LAUNCH_CHECK();
}

}  // namespace pdb
