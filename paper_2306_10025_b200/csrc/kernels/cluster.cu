// Data movement for the clustering setup: boundary-pattern masks
// (boundary_pattern patch.cpp:101-111: a local row is a Dirichlet row when
// it holds exactly one value != 0.0) and batched matrix gathers.
#include "../kernels.hpp"

namespace pdb::k {

namespace {

// Warp per patch; bit i of masks[k*words + i/64] set when row i has exactly one nonzero.
__global__ void boundary_masks_kernel(int64_t np, int ps, const double* __restrict__ mats, int words,
                                      unsigned long long* __restrict__ masks) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (k >= np) return;
  const double* A = mats + k * (int64_t)ps * ps;
  for (int w = 0; w < words; ++w) {
    unsigned long long bits = 0ull;
    for (int r = w * 64; r < min(ps, (w + 1) * 64); ++r) {
      int nz = 0;
      for (int j = lane; j < ps; j += 32) nz += A[(int64_t)r * ps + j] != 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, off);
      if (nz == 1) bits |= 1ull << (r - w * 64);
    }
    if (lane == 0) masks[k * words + w] = bits;
  }
}

__global__ void gather_mats_kernel(int64_t count, const int32_t* __restrict__ ids, int64_t len,
                                   const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t t = blockIdx.y;
  if (t >= count) return;
  const double* a = src + (int64_t)ids[t] * len;
  double* b = dst + t * len;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < len; q += (int64_t)gridDim.x * blockDim.x)
    b[q] = a[q];
}

__global__ void gather_i32_kernel(int64_t count, const int32_t* __restrict__ ids, int64_t len,
                                  const int32_t* __restrict__ src, int32_t* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * len) return;
  const int64_t r = t / len, q = t % len;
  dst[t] = src[(int64_t)ids[r] * len + q];
}

}  // namespace

void boundary_masks(int64_t np, int ps, const double* mats, int words, unsigned long long* masks, cudaStream_t s) {
  if (np > 0) boundary_masks_kernel<<<(unsigned)((np + 7) / 8), 256, 0, s>>>(np, ps, mats, words, masks);
}

void gather_mats(int64_t count, const int32_t* ids, int64_t len, const double* src, double* dst, cudaStream_t s) {
  if (count <= 0) return;
  int bx = (int)((len + 255) / 256);
  if (bx > 16) bx = 16;
  for (int64_t t0 = 0; t0 < count; t0 += 65535) {
    const int64_t c = count - t0 < 65535 ? count - t0 : 65535;
    gather_mats_kernel<<<dim3(bx, (unsigned)c), 256, 0, s>>>(c, ids + t0, len, src, dst + t0 * len);
  }
}

void gather_i32(int64_t count, const int32_t* ids, int64_t len, const int32_t* src, int32_t* dst, cudaStream_t s) {
  const int64_t total = count * len;
  if (total > 0) gather_i32_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(count, ids, len, src, dst);
}

}  // namespace pdb::k
