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

// ps <= 32: the warp streams the patch's ps CSR rows as one flat list of
// entries (lane e of every 32), so all rows' loads are in flight together
// instead of one staged row at a time.  Entry (r, p) holds column c of row
// idx[r]; c is searched in the patch's own (sorted) DoF list, and a hit at
// position q writes out[r][q] = val.  A per-row bit mask records the written
// positions; the holes (columns of the patch absent from the row) get 0.0
// afterwards, so every output element is still written once with the
// reference's value.
constexpr int kFlatWarps = 8;

__global__ void __launch_bounds__(kFlatWarps * 32) extract_flat_kernel(
    int64_t count, const int32_t* __restrict__ ids, int ps, const int32_t* __restrict__ patches,
    const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
    double* __restrict__ out) {
  __shared__ int32_t sidx[kFlatWarps][32];
  __shared__ int32_t soff[kFlatWarps][33];
  __shared__ int64_t sbeg[kFlatWarps][32];
  __shared__ uint32_t smask[kFlatWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kFlatWarps + warp;
  if (t >= count) return;
  const int64_t k = ids ? ids[t] : t;
  const int32_t* idx = patches + k * ps;
  double* o = out + t * (int64_t)ps * ps;
  int len = 0;
  if (lane < ps) {
    const int32_t gi = idx[lane];
    const int64_t lo = rp[gi];
    len = (int)(rp[gi + 1] - lo);
    sidx[warp][lane] = gi;
    sbeg[warp][lane] = lo;
  }
  smask[warp][lane] = 0u;
  // inclusive warp scan of the row lengths -> row offsets
  int incl = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  soff[warp][lane + 1] = incl;
  if (lane == 0) soff[warp][0] = 0;
  __syncwarp();
  const int total = soff[warp][ps];
  const int32_t* si = sidx[warp];
  const int32_t* so = soff[warp];
  for (int e = lane; e < total; e += 32) {
    int a = 0, b = ps - 1;  // row r: so[r] <= e < so[r + 1]
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (so[m] <= e) a = m;
      else b = m - 1;
    }
    const int r = a;
    const int64_t g = sbeg[warp][r] + (e - so[r]);
    const int32_t c = __ldg(col + g);
    const double v = __ldg(val + g);
    int lo = 0, hi = ps;  // lower_bound of c in the patch's DoF list
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (si[m] < c) lo = m + 1;
      else hi = m;
    }
    if (lo < ps && si[lo] == c) {
      o[(int64_t)r * ps + lo] = v;
      atomicOr(&smask[warp][r], 1u << lo);
    }
  }
  __syncwarp();
  for (int q = lane; q < ps * ps; q += 32) {
    const int r = q / ps, c = q - r * ps;
    if (!((smask[warp][r] >> c) & 1u)) o[q] = 0.0;
  }
}

}  // namespace

void extract(int64_t count, const int32_t* ids, int ps, const int32_t* patches, const int64_t* rp, const int32_t* col,
             const double* val, double* out, cudaStream_t s) {
  if (count <= 0) return;
  if (ps <= 32) {
    extract_flat_kernel<<<(unsigned)((count + kFlatWarps - 1) / kFlatWarps), kFlatWarps * 32, 0, s>>>(
        count, ids, ps, patches, rp, col, val, out);
    return;
  }
  extract_kernel<<<(unsigned)((count + kWarps - 1) / kWarps), kWarps * 32, 0, s>>>(count, ids, ps, patches, rp, col,
                                                                                  val, out);
}

}  // namespace pdb::k
