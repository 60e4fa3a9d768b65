// Coarse correction of the combo preconditioner on the device (reference
// ComboPreconditioner::apply precond.cpp:115-121, band_factor /
// BandedFactor::solve_into banded.cpp:11-84):
//
//   z += P0 (R0 A P0)^{-1} R0 r
//
// Setup factors R0 A P0 once on the device with one CTA per factorization:
// the LAPACK-style partial-pivoting band LU runs column by column (pivot =
// first maximum |.|, full row swap inside the band, multipliers by true
// division, a -= m*b updates unfused), so band, pivots and multipliers are
// bitwise the reference's.  Each apply is three launches:
//   restrict   rc = R0 r, one thread per coarse vertex summing its fine DoFs
//              in ascending order from 0.0 (= the reference's scatter order,
//              fem.cpp:373-382), bitwise;
//   band solve one warp walks the n_c columns: the forward sweep (swap, then
//              out[j+t] -= l_tj x_j, skipped when x_j == 0) is the
//              reference's order exactly; the backward sweep is column
//              oriented (x_i = out_i * (1/u_ii), then out[i-d] -= u x_i),
//              which reorders the reference's row sums (parity 1e-12
//              relative, tests/test_combo.py).  The band columns of the next
//              D steps are loaded into registers while the current ones are
//              applied, so the sweep runs at shared-memory latency;
//   prolong    z_i += sum_q p0_iq xc_q (<= 4 terms, in order), bitwise.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "host.hpp"

namespace pdb {

namespace {

// ---------------------------------------------------------------------------
// Band LU, one CTA.  B is column-major band storage: B[j*ldab + r] holds the
// reference's ab[r*n + j] (band row r of column j).

constexpr int kFactorThreads = 1024;

__global__ void __launch_bounds__(kFactorThreads) band_factor_kernel(int n, int kl, int ku, int ldab, double* B,
                                                                     int32_t* ipiv, double* rdiag, int* bad_col) {
  extern __shared__ double smem[];
  double* mult = smem;  // kl multipliers of the current column
  __shared__ double red_v[kFactorThreads / 32];
  __shared__ int red_t[kFactorThreads / 32];
  __shared__ double s_best;
  __shared__ int s_jp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kv = kl + ku;
  for (int j = 0; j < n; ++j) {
    const int km = min(kl, n - 1 - j);
    double* col = B + static_cast<int64_t>(j) * ldab;
    // pivot: first maximum of |a(j+t, j)|, t = 0..km (strict > in ascending t)
    double bv = -1.0;
    int bt = 0;
    for (int t = tid; t <= km; t += kFactorThreads) {
      const double v = fabs(col[kv + t]);
      if (v > bv) {
        bv = v;
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
      if (v == 0.0) *bad_col = j;
    }
    __syncthreads();
    if (s_best == 0.0) return;
    const int jp = s_jp;
    const int jend = min(j + kv, n - 1);
    if (jp != 0)
      for (int jj = j + tid; jj <= jend; jj += kFactorThreads) {
        double* c = B + static_cast<int64_t>(jj) * ldab;
        const double a = c[kv + j - jj], b = c[kv + j + jp - jj];
        c[kv + j - jj] = b;
        c[kv + j + jp - jj] = a;
      }
    __syncthreads();
    const double piv = col[kv];
    for (int t = 1 + tid; t <= km; t += kFactorThreads) {
      const double m = __ddiv_rn(col[kv + t], piv);
      col[kv + t] = m;
      mult[t] = m;
    }
    if (tid == 0) {
      ipiv[j] = j + jp;
      rdiag[j] = __ddiv_rn(1.0, piv);
    }
    __syncthreads();
    // a(j+t, jj) -= m_t * a(j, jj) for t = 1..km, jj = j+1..jend
    if (km > 0) {
      const int total = km * (jend - j);
      for (int idx = tid; idx < total; idx += kFactorThreads) {
        const int t = 1 + idx % km, jj = j + 1 + idx / km;
        const double m = mult[t];
        if (m == 0.0) continue;
        double* c = B + static_cast<int64_t>(jj) * ldab;
        c[kv + t + j - jj] = __dsub_rn(c[kv + t + j - jj], __dmul_rn(m, c[kv + j - jj]));
      }
    }
    __syncthreads();
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
  band_factor_kernel<<<1, kFactorThreads, smem, s>>>(static_cast<int>(n), static_cast<int>(kl), static_cast<int>(ku),
                                                    static_cast<int>(ldab), out.band.get(), out.ipiv.get(),
                                                    out.rdiag.get(), bad.get());
  PDB_LAUNCH_CHECK();
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
  }
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
