// Deterministic level-1 kernels for the device Krylov drivers (GMRES,
// PCG).  Reductions use a fixed grid and a fixed two-level tree, so results
// are run-to-run identical for a given length (not order-identical to the
// reference's sequential loops; histories agree to ~1e-15 relative).
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

inline unsigned ew_grid(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (unsigned)(g < 4 * 148 * 8 ? (g > 0 ? g : 1) : 4 * 148 * 8);
}

}  // namespace

int dot_partials() { return kDotBlocks; }

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
