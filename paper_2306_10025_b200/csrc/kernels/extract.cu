// Batched extraction of the dense cell-patch matrices A_k = V_k A V_k^T
// (reference extract_submatrix sparse.cpp:71-103 via extract_all
// patch.cpp:92-99).  A pure copy, so bit-exact by construction.
//
// One warp per patch.  For local row r the warp stages the CSR row of
// global DoF idx[r] (columns) in shared memory with coalesced loads; lane q
// then binary-searches idx[q] in it and writes out[r][q] (the value, or 0.0
// when absent).  Every output element is written exactly once and each warp
// store covers a contiguous run of the row-major patch matrix.
#include "../kernels.hpp"

namespace pdb::k {

namespace {

constexpr int kWarps = 4;
constexpr int kRowCap = 1024;  // staged CSR row length; longer rows search global memory

__global__ void __launch_bounds__(kWarps * 32) extract_kernel(int64_t count, const int32_t* __restrict__ ids, int ps,
                                                              const int32_t* __restrict__ patches,
                                                              const int64_t* __restrict__ rp,
                                                              const int32_t* __restrict__ col,
                                                              const double* __restrict__ val, double* __restrict__ out) {
  __shared__ int32_t rowbuf[kWarps][kRowCap];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kWarps + warp;
  if (t >= count) return;
  const int64_t k = ids ? ids[t] : t;
  const int32_t* idx = patches + k * ps;
  double* o = out + t * (int64_t)ps * ps;
  int32_t* buf = rowbuf[warp];
  for (int r = 0; r < ps; ++r) {
    const int32_t gi = idx[r];
    const int64_t lo = rp[gi];
    const int len = (int)(rp[gi + 1] - lo);
    const bool staged = len <= kRowCap;
    if (staged)
      for (int p = lane; p < len; p += 32) buf[p] = col[lo + p];
    __syncwarp();
    const int32_t* cols = staged ? buf : col + lo;
    for (int q = lane; q < ps; q += 32) {
      const int32_t key = idx[q];
      int a = 0, b = len;  // lower_bound
      while (a < b) {
        const int m = (a + b) >> 1;
        if (cols[m] < key) a = m + 1;
        else b = m;
      }
      o[(int64_t)r * ps + q] = (a < len && cols[a] == key) ? val[lo + a] : 0.0;
    }
    __syncwarp();
  }
}

}  // namespace

void extract(int64_t count, const int32_t* ids, int ps, const int32_t* patches, const int64_t* rp, const int32_t* col,
             const double* val, double* out, cudaStream_t s) {
  if (count <= 0) return;
  extract_kernel<<<(unsigned)((count + kWarps - 1) / kWarps), kWarps * 32, 0, s>>>(count, ids, ps, patches, rp, col,
                                                                                  val, out);
}

}  // namespace pdb::k
