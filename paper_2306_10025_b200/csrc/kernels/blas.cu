// Deterministic level-1 kernels for the device Krylov drivers (GMRES,
// PCG).  Reductions use a fixed grid and a fixed two-level tree, so results
// are run-to-run identical for a given length (not order-identical to the
// reference's sequential loops; histories agree to ~1e-15 relative).
#include <algorithm>
#include <cstdlib>

#include "../common.hpp"
#include "../kernels.hpp"

namespace pdb::k {

namespace {

constexpr int kDotBlocks = 592;  // 4 x 148 SMs
constexpr int kDotThreads = 256;

__global__ void __launch_bounds__(kDotThreads) dot_kernel(int64_t n, const double* __restrict__ a,
                                                          const double* __restrict__ b, double* __restrict__ partials) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDotThreads)
    s += a[i] * b[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kDotThreads / 32; ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ partials, int count, double* out) {
  __shared__ double red[1024];
  double t = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) t += partials[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

__global__ void axpy_kernel(int64_t n, const double* __restrict__ alpha, bool negate, const double* __restrict__ x,
                            double* __restrict__ y) {
  const double a = negate ? -alpha[0] : alpha[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

__global__ void xpay_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ beta,
                            double* __restrict__ y) {
  const double bt = beta[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] + bt * y[i];
}

__global__ void axpy_val_kernel(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

__global__ void div_kernel(int64_t n, const double* __restrict__ x, double sc, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / sc;
}

__global__ void sub_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a[i] - b[i];
}

__global__ void scalar_div_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
  out[0] = a[0] / b[0];
}

// CG update fused with its residual norm: x_out = x_in + a p, r -= a q
// (unfused, as the oracle's loops), partials[block] = sum of r^2 over the
// block's fixed grid-stride share (kDotBlocks blocks: deterministic).
__global__ void __launch_bounds__(kDotThreads) cg_update_kernel(int64_t n, const double* __restrict__ alpha,
                                                                const double* __restrict__ p,
                                                                const double* __restrict__ q,
                                                                const double* __restrict__ x_in,
                                                                double* __restrict__ x_out, double* __restrict__ r,
                                                                double* __restrict__ partials) {
  __shared__ double red[kDotThreads / 32];
  const double a = alpha[0];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDotThreads) {
    x_out[i] = __dadd_rn(x_in[i], __dmul_rn(a, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(a, q[i]));
    r[i] = ri;
    s += ri * ri;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kDotThreads / 32; ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

// mode 0: out[0] = num[0] / sum (alpha);  mode 1: out[0] = sum / num[0], num[0] = sum (beta, rz <- rz_new)
__global__ void finish_ratio_kernel(const double* __restrict__ partials, int count, double* num, double* out,
                                    int mode) {
  __shared__ double red[1024];
  double t = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) t += partials[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double sum = red[0];
    if (mode == 0) {
      out[0] = num[0] / sum;
    } else {
      out[0] = sum / num[0];
      num[0] = sum;
    }
  }
}

inline unsigned ew_grid(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (unsigned)(g < 4 * 148 * 8 ? (g > 0 ? g : 1) : 4 * 148 * 8);
}

// ---------------------------------------------------------------------------
// Fused MGS (Arnoldi) with a software grid barrier; co-residency of every CTA
// is guaranteed by the cooperative launch.

constexpr int kMgsThreads = 256;
constexpr int kMgsMaxBlocks = 1184;  // 8 per SM

struct MgsSync {
  unsigned count;
  unsigned gen;
  double partial[2][kMgsMaxBlocks];
};

__device__ __forceinline__ void grid_barrier(MgsSync* sy) {
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

// Block sum in a fixed tree; every thread gets the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kMgsThreads / 32; ++w) t += red[w];
  return t;
}

// Grid-wide sum of each CTA's `v` (same fixed order in every CTA).
__device__ __forceinline__ double grid_sum(double v, MgsSync* sy, int buf, double* red) {
  const double bs = block_sum(v, red);
  if (threadIdx.x == 0) sy->partial[buf][blockIdx.x] = bs;
  grid_barrier(sy);
  double t = 0.0;
  for (int b = threadIdx.x; b < gridDim.x; b += kMgsThreads) t += __ldcg(&sy->partial[buf][b]);
  return block_sum(t, red);
}

template <int E>
__global__ void __launch_bounds__(kMgsThreads) mgs_kernel(int64_t n, int j, const double* __restrict__ V, int64_t ldv,
                                                          double* __restrict__ w, double* __restrict__ h,
                                                          MgsSync* sy) {
  __shared__ double red[kMgsThreads / 32];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kMgsThreads;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kMgsThreads + threadIdx.x;
  double x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t i = base + e * stride;
    x[e] = i < n ? w[i] : 0.0;
  }
  int buf = 0;
  for (int i = 0; i <= j; ++i) {
    const double* v = V + static_cast<int64_t>(i) * ldv;
    double vv[E];
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t q = base + e * stride;
      vv[e] = q < n ? v[q] : 0.0;
      s = fma(x[e], vv[e], s);
    }
    const double hij = grid_sum(s, sy, buf, red);
    buf ^= 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = hij;
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = fma(-hij, vv[e], x[e]);
  }
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) s = fma(x[e], x[e], s);
  const double nn = grid_sum(s, sy, buf, red);
  if (blockIdx.x == 0 && threadIdx.x == 0) h[j + 1] = nn;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t q = base + e * stride;
    if (q < n) w[q] = x[e];
  }
}

template <int E>
bool launch_mgs(int64_t n, int j, const double* V, int64_t ldv, double* w, double* h, cudaStream_t s) {
  // per device: the barrier struct lives in that device's memory
  constexpr int kMaxDev = 64;
  int dev = 0;
  PDB_CUDA(cudaGetDevice(&dev));
  require(dev < kMaxDev, Errc::internal, "device ordinal beyond the per-device caches");
  static thread_local MgsSync* sy_of[kMaxDev] = {};
  MgsSync*& sy = sy_of[dev];
  if (!sy) {
    PDB_CUDA(cudaMalloc(&sy, sizeof(MgsSync)));
    PDB_CUDA(cudaMemset(sy, 0, sizeof(MgsSync)));
  }
  static int per_sm_of[kMaxDev];
  static bool have_of[kMaxDev] = {};
  if (!have_of[dev]) {
    PDB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_of[dev], mgs_kernel<E>, kMgsThreads, 0));
    have_of[dev] = true;
  }
  const int per_sm = per_sm_of[dev];
  const int64_t need = (n + static_cast<int64_t>(kMgsThreads) * E - 1) / (static_cast<int64_t>(kMgsThreads) * E);
  const int64_t cap = std::min<int64_t>(kMgsMaxBlocks, static_cast<int64_t>(per_sm) * num_sms());
  if (need > cap) return false;
  // small vectors: fewer CTAs make the barriers cheaper
  const int grid = static_cast<int>(std::max<int64_t>(1, need));
  void* args[] = {&n, &j, &V, &ldv, &w, &h, &sy};
  PDB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(mgs_kernel<E>), dim3(grid), dim3(kMgsThreads), args, 0, s));
  return true;
}

}  // namespace

bool mgs_fused(int64_t n, int j, const double* V, int64_t ldv, double* w, double* h, cudaStream_t s) {
  const char* e = getenv("PDB_MGS");
  if (e && e[0] == '0') return false;
  const int64_t per = static_cast<int64_t>(kMgsThreads) * 4 * 148;  // elements at 4 CTAs/SM... per E
  if (n <= per * 1 / 4) return launch_mgs<1>(n, j, V, ldv, w, h, s);
  if (n <= per * 2 / 4) return launch_mgs<2>(n, j, V, ldv, w, h, s);
  if (n <= per) return launch_mgs<4>(n, j, V, ldv, w, h, s);
  if (n <= per * 2) return launch_mgs<8>(n, j, V, ldv, w, h, s);
  return launch_mgs<16>(n, j, V, ldv, w, h, s);
}

int dot_partials() { return kDotBlocks; }

void dot_partial(int64_t n, const double* a, const double* b, double* partials, cudaStream_t s) {
  dot_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, b, partials);
}

void cg_update(int64_t n, const double* alpha, const double* p, const double* q, const double* x_in, double* x_out,
               double* r, double* partials, cudaStream_t s) {
  cg_update_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, alpha, p, q, x_in, x_out, r, partials);
}

void finish_ratio(const double* partials, int count, double* num, double* out, bool beta, cudaStream_t s) {
  finish_ratio_kernel<<<1, 1024, 0, s>>>(partials, count, num, out, beta ? 1 : 0);
}

void dot(int64_t n, const double* a, const double* b, double* partials, double* out, cudaStream_t s) {
  dot_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, b, partials);
  sum_partials_kernel<<<1, 1024, 0, s>>>(partials, kDotBlocks, out);
}

void axpy(int64_t n, const double* alpha, bool negate, const double* x, double* y, cudaStream_t s) {
  axpy_kernel<<<ew_grid(n), 256, 0, s>>>(n, alpha, negate, x, y);
}

void xpay(int64_t n, const double* x, const double* beta, double* y, cudaStream_t s) {
  xpay_kernel<<<ew_grid(n), 256, 0, s>>>(n, x, beta, y);
}

void axpy_val(int64_t n, double a, const double* x, double* y, cudaStream_t s) {
  axpy_val_kernel<<<ew_grid(n), 256, 0, s>>>(n, a, x, y);
}

void div_scalar(int64_t n, const double* x, double sc, double* y, cudaStream_t s) {
  div_kernel<<<ew_grid(n), 256, 0, s>>>(n, x, sc, y);
}

void scalar_div(const double* a, const double* b, double* out, cudaStream_t s) {
  scalar_div_kernel<<<1, 1, 0, s>>>(a, b, out);
}

void sub(int64_t n, const double* a, const double* b, double* y, cudaStream_t s) {
  sub_kernel<<<ew_grid(n), 256, 0, s>>>(n, a, b, y);
}

}  // namespace pdb::k
