// The relaxation sweep x <- x + omega W sum_k V_k^T B_phi(k)^{-1} V_k (b - A x)
// (reference: smooth precond.cpp:90-101, PatchPreconditioner::apply
// precond.cpp:58-88, spmv sparse.cpp:50-63).
//
// Three kernels per sweep, each HBM- or L2-bound:
//   residual      r = b - A x           sub-warp per row, coalesced CSR streams,
//                                       optional deterministic per-block sum r^2
//   patch_solve   sols_k = B^{-1} r|_k  sub-warp per patch, lane i owns local row i,
//                                       column-major factors -> lane-contiguous loads,
//                                       compressed factors stay L2-resident
//   scatter_update x += omega W sum sols owner-computes gather through the
//                                       DoF -> (patch, slot) inverse map in ascending
//                                       patch order: the reference's serial scatter
//                                       order (precond.cpp:81-86), no atomics
// r (8n B) and sols (8 np ps B) are produced and consumed back to back, so
// they are L2 hits on the 126 MB L2 for c1-c4 sizes.
#include <cub/cub.cuh>

#include "../kernels.hpp"

namespace pdb::k {

namespace {

constexpr int kBlock = 256;

template <int G>
__global__ void __launch_bounds__(kBlock) residual_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ x, const double* __restrict__ b,
                                                          double* __restrict__ r, double* __restrict__ block_sumsq,
                                                          bool negate_b_absent) {
  const int lane = threadIdx.x % G;
  const int64_t row = (int64_t)blockIdx.x * (kBlock / G) + threadIdx.x / G;
  double acc = 0.0;
  if (row < n) {
    const int64_t lo = rp[row], hi = rp[row + 1];
    for (int64_t p = lo + lane; p < hi; p += G) acc += __ldg(val + p) * __ldg(x + __ldg(col + p));
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off, G);
  double rv = 0.0;
  if (row < n) {
    rv = b ? b[row] - acc : (negate_b_absent ? -acc : acc);
    if (lane == 0) r[row] = rv;
  }
  if (block_sumsq) {
    __shared__ double red[kBlock / 32];
    double sq = (lane == 0 && row < n) ? rv * rv : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kBlock / 32; ++w) t += red[w];
      block_sumsq[blockIdx.x] = t;
    }
  }
}

__global__ void finish_sum_kernel(const double* __restrict__ partials, int count, double* out, bool take_sqrt) {
  __shared__ double red[1024];
  double t = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) t += partials[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = take_sqrt ? sqrt(red[0]) : red[0];
}

// Sub-warp of W lanes per patch (ps <= W <= 32).  Lane i holds local row i.
template <int W>
__global__ void __launch_bounds__(kBlock) patch_solve_kernel(int64_t np, int ps, const int32_t* __restrict__ patches,
                                                             const double* __restrict__ F,
                                                             const int32_t* __restrict__ piv,
                                                             const int32_t* __restrict__ phi,
                                                             const double* __restrict__ r,
                                                             const double* __restrict__ in_scale,
                                                             double* __restrict__ sols) {
  const int i = threadIdx.x % W;
  const int64_t k = (int64_t)blockIdx.x * (kBlock / W) + threadIdx.x / W;
  const bool live = k < np;
  const int64_t kk = live ? k : np - 1;  // keep dead lanes in the shuffles
  const int64_t f = phi ? (int64_t)phi[kk] : kk;
  const double* Fk = F + f * (int64_t)ps * ps;
  const bool row = i < ps;
  // out[i] = rhs[piv[i]] with rhs = r gathered on the patch (precond.cpp:72-73, dense.cpp:83)
  double s = 0.0;
  if (row) {
    const int32_t g = __ldg(patches + kk * ps + __ldg(piv + f * ps + i));
    s = __ldg(r + g);
    if (in_scale) s *= __ldg(in_scale + g);
  }
  // forward substitution, unit lower triangle, column j broadcast by shuffle
  for (int j = 0; j < ps - 1; ++j) {
    const double yj = __shfl_sync(0xffffffffu, s, j, W);
    if (row && i > j) s -= __ldg(Fk + (int64_t)j * ps + i) * yj;
  }
  // back substitution
  for (int j = ps - 1; j >= 0; --j) {
    if (i == j) s = s / __ldg(Fk + (int64_t)j * ps + j);
    const double yj = __shfl_sync(0xffffffffu, s, j, W);
    if (row && i < j) s -= __ldg(Fk + (int64_t)j * ps + i) * yj;
  }
  if (live && row) sols[k * ps + i] = s;
}

// Generic path for ps > 32: one block per patch, thread per local row,
// column-oriented substitutions through shared memory.
__global__ void patch_solve_block_kernel(int64_t np, int ps, const int32_t* __restrict__ patches,
                                         const double* __restrict__ F, const int32_t* __restrict__ piv,
                                         const int32_t* __restrict__ phi, const double* __restrict__ r,
                                         const double* __restrict__ in_scale, double* __restrict__ sols) {
  extern __shared__ double y[];
  const int64_t k = blockIdx.x;
  const int64_t f = phi ? (int64_t)phi[k] : k;
  const double* Fk = F + f * (int64_t)ps * ps;
  for (int i = threadIdx.x; i < ps; i += blockDim.x) {
    const int32_t g = patches[k * ps + piv[f * ps + i]];
    y[i] = in_scale ? r[g] * in_scale[g] : r[g];
  }
  __syncthreads();
  for (int j = 0; j < ps - 1; ++j) {
    const double yj = y[j];
    for (int i = j + 1 + threadIdx.x; i < ps; i += blockDim.x) y[i] -= Fk[(int64_t)j * ps + i] * yj;
    __syncthreads();
  }
  for (int j = ps - 1; j >= 0; --j) {
    if (threadIdx.x == 0) y[j] = y[j] / Fk[(int64_t)j * ps + j];
    __syncthreads();
    const double yj = y[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) y[i] -= Fk[(int64_t)j * ps + i] * yj;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < ps; i += blockDim.x) sols[k * ps + i] = y[i];
}

__global__ void scatter_update_kernel(int64_t n, const int32_t* __restrict__ inv_ptr, const int32_t* __restrict__ inv,
                                      const double* __restrict__ sols, const double* __restrict__ omega_w,
                                      const double* __restrict__ x_in, double* __restrict__ z_out,
                                      double* __restrict__ x_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double z = 0.0;
  const int32_t lo = inv_ptr[i], hi = inv_ptr[i + 1];
  for (int32_t q = lo; q < hi; ++q) z += __ldg(sols + __ldg(inv + q));
  z *= omega_w[i];
  if (z_out) z_out[i] = z;
  if (x_out) x_out[i] = z + x_in[i];
}

__global__ void inverse_count_kernel(int64_t total, const int32_t* __restrict__ patches, int32_t* counts) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < total) atomicAdd(counts + patches[t], 1);
}

__global__ void inverse_fill_kernel(int64_t total, const int32_t* __restrict__ patches,
                                    const int32_t* __restrict__ inv_ptr, int32_t* cursor, int32_t* inv) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int32_t d = patches[t];
  const int32_t pos = atomicAdd(cursor + d, 1);
  inv[inv_ptr[d] + pos] = (int32_t)t;  // t = k*ps + l
}

__global__ void inverse_sort_kernel(int64_t n, const int32_t* __restrict__ inv_ptr, int32_t* inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t lo = inv_ptr[i], hi = inv_ptr[i + 1];
  for (int32_t a = lo + 1; a < hi; ++a) {  // segments are tiny (<= 2^dim entries for cell patches)
    const int32_t key = inv[a];
    int32_t b = a - 1;
    while (b >= lo && inv[b] > key) {
      inv[b + 1] = inv[b];
      --b;
    }
    inv[b + 1] = key;
  }
}

__global__ void transpose_factors_kernel(int64_t nf, int ps, const double* __restrict__ rm, double* __restrict__ cm) {
  const int64_t len = (int64_t)ps * ps;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nf * len) return;
  const int64_t f = t / len, e = t % len;
  const int64_t i = e / ps, j = e % ps;
  cm[f * len + j * ps + i] = rm[t];
}

__global__ void scale_weights_kernel(int64_t n, double omega, const double* __restrict__ w, double* __restrict__ ow) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ow[i] = omega * w[i];
}

__global__ void sqrt_weights_kernel(int64_t n, double omega, const double* __restrict__ w, double* __restrict__ sw,
                                    double* __restrict__ osw) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r = sqrt(w[i]);
  sw[i] = r;
  osw[i] = omega * r;
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

}  // namespace

SpmvPlan spmv_plan(int64_t n, int64_t nnz) {
  SpmvPlan p;
  const double avg = n > 0 ? (double)nnz / (double)n : 1.0;
  int g = 1;
  while (g < 32 && g * 2 <= avg * 0.75 + 1) g *= 2;
  if (avg > 24) g = g < 16 ? 16 : g;
  p.group = g;
  p.rows_per_block = kBlock / g;
  p.blocks = (int)((n + p.rows_per_block - 1) / p.rows_per_block);
  return p;
}

template <int G>
static void launch_residual(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                            const double* x, const double* b, double* r, double* sumsq, bool negate,
                            cudaStream_t s) {
  residual_kernel<G><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate);
}

static void dispatch_residual(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                              const double* x, const double* b, double* r, double* sumsq, bool negate,
                              cudaStream_t s) {
  if (n <= 0) return;
  switch (p.group) {
    case 1: launch_residual<1>(p, n, rp, col, val, x, b, r, sumsq, negate, s); break;
    case 2: launch_residual<2>(p, n, rp, col, val, x, b, r, sumsq, negate, s); break;
    case 4: launch_residual<4>(p, n, rp, col, val, x, b, r, sumsq, negate, s); break;
    case 8: launch_residual<8>(p, n, rp, col, val, x, b, r, sumsq, negate, s); break;
    case 16: launch_residual<16>(p, n, rp, col, val, x, b, r, sumsq, negate, s); break;
    default: launch_residual<32>(p, n, rp, col, val, x, b, r, sumsq, negate, s); break;
  }
}

void residual(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x,
              const double* b, double* r, double* block_sumsq, cudaStream_t s) {
  dispatch_residual(p, n, rp, col, val, x, b, r, block_sumsq, true, s);
}

void spmv(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x,
          double* y, cudaStream_t s) {
  dispatch_residual(p, n, rp, col, val, x, nullptr, y, nullptr, false, s);
}

void finish_sum(const double* partials, int count, double* out, bool sqrt_result, cudaStream_t s) {
  finish_sum_kernel<<<1, 1024, 0, s>>>(partials, count, out, sqrt_result);
}

void patch_solve(int64_t np, int ps, const int32_t* patches, const double* F, const int32_t* piv, const int32_t* phi,
                 const double* r, const double* in_scale, double* sols, cudaStream_t s) {
  if (np <= 0) return;
  if (ps > 32) {
    const int threads = ps >= 128 ? 128 : 64;
    patch_solve_block_kernel<<<(unsigned)np, threads, ps * sizeof(double), s>>>(np, ps, patches, F, piv, phi, r, in_scale, sols);
    return;
  }
  int W = 1;
  while (W < ps) W *= 2;
  const unsigned blocks = grid_for(np, kBlock / W);
  switch (W) {
    case 1:
    case 2: patch_solve_kernel<2><<<grid_for(np, kBlock / 2), kBlock, 0, s>>>(np, ps, patches, F, piv, phi, r, in_scale, sols); break;
    case 4: patch_solve_kernel<4><<<blocks, kBlock, 0, s>>>(np, ps, patches, F, piv, phi, r, in_scale, sols); break;
    case 8: patch_solve_kernel<8><<<blocks, kBlock, 0, s>>>(np, ps, patches, F, piv, phi, r, in_scale, sols); break;
    case 16: patch_solve_kernel<16><<<blocks, kBlock, 0, s>>>(np, ps, patches, F, piv, phi, r, in_scale, sols); break;
    default: patch_solve_kernel<32><<<blocks, kBlock, 0, s>>>(np, ps, patches, F, piv, phi, r, in_scale, sols); break;
  }
}

void scatter_update(int64_t n, const int32_t* inv_ptr, const int32_t* inv, const double* sols, const double* omega_w,
                    const double* x_in, double* z_out, double* x_out, cudaStream_t s) {
  if (n <= 0) return;
  scatter_update_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, inv_ptr, inv, sols, omega_w, x_in, z_out, x_out);
}

void build_inverse_count(int64_t np, int ps, const int32_t* patches, int32_t* counts, cudaStream_t s) {
  const int64_t total = np * ps;
  if (total > 0) inverse_count_kernel<<<grid_for(total, kBlock), kBlock, 0, s>>>(total, patches, counts);
}

void build_inverse_fill(int64_t np, int ps, const int32_t* patches, const int32_t* inv_ptr, int32_t* cursor,
                        int32_t* inv, cudaStream_t s) {
  const int64_t total = np * ps;
  if (total > 0) inverse_fill_kernel<<<grid_for(total, kBlock), kBlock, 0, s>>>(total, patches, inv_ptr, cursor, inv);
}

void sort_inverse_segments(int64_t n, const int32_t* inv_ptr, int32_t* inv, cudaStream_t s) {
  if (n > 0) inverse_sort_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, inv_ptr, inv);
}

void transpose_factors(int64_t nf, int ps, const double* lu_rm, double* lu_cm, cudaStream_t s) {
  const int64_t total = nf * ps * ps;
  if (total > 0) transpose_factors_kernel<<<grid_for(total, kBlock), kBlock, 0, s>>>(nf, ps, lu_rm, lu_cm);
}

void scale_weights(int64_t n, double omega, const double* w, double* omega_w, cudaStream_t s) {
  if (n > 0) scale_weights_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, omega, w, omega_w);
}

void sqrt_weights(int64_t n, double omega, const double* w, double* sw, double* omega_sw, cudaStream_t s) {
  if (n > 0) sqrt_weights_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, omega, w, sw, omega_sw);
}

}  // namespace pdb::k
