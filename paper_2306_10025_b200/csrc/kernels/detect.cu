// Matrix-only cell-patch detection (reference detect_patches, patch.cpp:37-90).
//
//   candidates   rows with exactly ps stored entries (patch.cpp:43)
//   consistency  warp per candidate row i: every candidate j in cols(i)
//                must have the same candidate-restricted footprint
//                (patch.cpp:66-76); also the FNV-1a hash of cols(i)
//                (the reference's IndexVectorHash, patch.cpp:24-33)
//   dedupe       rows sorted by (hash, row); a row is dropped when an
//                earlier row of its hash run has the identical column set,
//                which is exactly "first occurrence wins" (patch.cpp:64)
// Integer work only; the host finishes with std::sort by front, the
// reference's own comparator and algorithm (patch.cpp:82-83).
#include "../kernels.hpp"

namespace pdb::k {

namespace {

constexpr int kWarps = 8;

__global__ void candidates_kernel(int64_t n, const int64_t* __restrict__ rp, int64_t ps, uint8_t* cand, int32_t* any) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool c = rp[i + 1] - rp[i] == ps;
  cand[i] = c ? 1 : 0;
  if (c) atomicOr(any, 1);
}

// dynamic smem: kWarps * ps int32 (footprint of row i)
__global__ void __launch_bounds__(kWarps * 32) consistency_kernel(int64_t nrows, const int32_t* __restrict__ rows,
                                                                  const int64_t* __restrict__ rp,
                                                                  const int32_t* __restrict__ col,
                                                                  const uint8_t* __restrict__ cand, int ps,
                                                                  uint8_t* consistent, uint64_t* hash) {
  extern __shared__ int32_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* fi = smem + warp * ps;
  const int64_t t = (int64_t)blockIdx.x * kWarps + warp;
  if (t >= nrows) return;
  const int32_t i = rows[t];
  const int32_t* ci = col + rp[i];
  // footprint of i, compacted in order
  int nfi = 0;
  for (int base = 0; base < ps; base += 32) {
    const int q = base + lane;
    const bool in = q < ps && cand[ci[q]];
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if (in) fi[nfi + __popc(m & ((1u << lane) - 1))] = ci[q];
    nfi += __popc(m);
  }
  __syncwarp();
  bool ok = true;
  for (int q = 0; q < ps && ok; ++q) {
    const int32_t j = ci[q];
    if (!cand[j] || j == i) continue;
    const int32_t* cj = col + rp[j];  // candidate: exactly ps entries
    int nfj = 0;
    bool same = true;
    for (int base = 0; base < ps; base += 32) {
      const int qq = base + lane;
      const bool in = qq < ps && cand[cj[qq]];
      const unsigned m = __ballot_sync(0xffffffffu, in);
      const int pos = nfj + __popc(m & ((1u << lane) - 1));
      bool mine = true;
      if (in) mine = pos < nfi && fi[pos] == cj[qq];
      same = same && __all_sync(0xffffffffu, mine);
      nfj += __popc(m);
    }
    ok = same && nfj == nfi;
  }
  if (lane == 0) {
    consistent[t] = ok ? 1 : 0;
    uint64_t h = 1469598103934665603ull;
    for (int q = 0; q < ps; ++q) {
      h ^= (uint64_t)(int64_t)ci[q];
      h *= 1099511628211ull;
    }
    hash[t] = h;
  }
}

// Positions are sorted by (hash, position); position order is ascending row
// order, so "an earlier element of my run" means "a smaller row".
__global__ void dedupe_kernel(int64_t nrows, const uint64_t* __restrict__ hs, const int32_t* __restrict__ pos,
                              const int32_t* __restrict__ rows, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ col, int ps, uint8_t* keep_by_pos) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int32_t* a = col + rp[rows[pos[t]]];
  bool d = false;
  for (int64_t u = t - 1; u >= 0 && hs[u] == hs[t] && !d; --u) {
    const int32_t* b = col + rp[rows[pos[u]]];
    bool eq = true;
    for (int q = 0; q < ps && eq; ++q) eq = a[q] == b[q];
    d = eq;
  }
  keep_by_pos[pos[t]] = d ? 0 : 1;
}

__global__ void iota_kernel(int64_t n, int32_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)i;
}

__global__ void gather_patches_kernel(int64_t np, const int32_t* __restrict__ rows, const int32_t* __restrict__ order,
                                      const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int ps,
                                      int32_t* __restrict__ patches) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= np * ps) return;
  const int64_t k = t / ps, q = t % ps;
  const int32_t row = rows[order[k]];
  patches[t] = col[rp[row] + q];
}

__global__ void cover_count_kernel(int64_t total, const int32_t* __restrict__ patches, int32_t* cover) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < total) atomicAdd(cover + patches[t], 1);
}

// compute_weights, patch.cpp:12-20: 1/cover or 0.
__global__ void weights_kernel(int64_t n, const int32_t* __restrict__ cover, double* w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = cover[i] > 0 ? 1.0 / (double)cover[i] : 0.0;
}

// fronts[e] = patches[e * ps] (the first, smallest column of patch e)
__global__ void fronts_kernel(int64_t np, int ps, const int32_t* __restrict__ patches, int32_t* __restrict__ fronts) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < np) fronts[e] = patches[e * ps];
}

// Over the (front, e) pairs sorted by front: flags[0] |= 1 if two patches share
// a front (the sort order is then the comparator's, not a unique one),
// flags[1] |= 1 if the order is not the identity.
__global__ void front_order_kernel(int64_t np, const int32_t* __restrict__ key_sorted,
                                   const int32_t* __restrict__ order, int32_t* flags) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= np) return;
  if (e + 1 < np && key_sorted[e] == key_sorted[e + 1]) atomicOr(flags, 1);
  if (order[e] != e) atomicOr(flags + 1, 1);
}

inline unsigned grid_for(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

void detect_candidates(int64_t n, const int64_t* rp, int64_t ps, uint8_t* cand, int32_t* any, cudaStream_t s) {
  if (n > 0) candidates_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ps, cand, any);
}

void detect_consistency(int64_t nrows, const int32_t* rows, const int64_t* rp, const int32_t* col,
                        const uint8_t* cand, int ps, uint8_t* consistent, uint64_t* hash, cudaStream_t s) {
  if (nrows <= 0) return;
  const size_t smem = (size_t)kWarps * ps * sizeof(int32_t);
  consistency_kernel<<<grid_for(nrows, kWarps), kWarps * 32, smem, s>>>(nrows, rows, rp, col, cand, ps, consistent,
                                                                        hash);
}

void detect_dedupe(int64_t nrows, const uint64_t* hash_sorted, const int32_t* pos_sorted, const int32_t* rows,
                   const int64_t* rp, const int32_t* col, int ps, uint8_t* keep_by_pos, cudaStream_t s) {
  if (nrows > 0)
    dedupe_kernel<<<grid_for(nrows, 256), 256, 0, s>>>(nrows, hash_sorted, pos_sorted, rows, rp, col, ps, keep_by_pos);
}

void iota(int64_t n, int32_t* out, cudaStream_t s) {
  if (n > 0) iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, out);
}

void gather_patches(int64_t np, const int32_t* rows, const int32_t* order, const int64_t* rp, const int32_t* col,
                    int ps, int32_t* patches, cudaStream_t s) {
  const int64_t total = np * ps;
  if (total > 0) gather_patches_kernel<<<grid_for(total, 256), 256, 0, s>>>(np, rows, order, rp, col, ps, patches);
}

void patch_fronts(int64_t np, int ps, const int32_t* patches, int32_t* fronts, cudaStream_t s) {
  if (np > 0) fronts_kernel<<<grid_for(np, 256), 256, 0, s>>>(np, ps, patches, fronts);
}

void front_order(int64_t np, const int32_t* key_sorted, const int32_t* order, int32_t* flags, cudaStream_t s) {
  if (np > 0) front_order_kernel<<<grid_for(np, 256), 256, 0, s>>>(np, key_sorted, order, flags);
}

void cover_weights(int64_t n, int64_t np, int ps, const int32_t* patches, int32_t* cover, double* w, cudaStream_t s) {
  const int64_t total = np * ps;
  if (total > 0) cover_count_kernel<<<grid_for(total, 256), 256, 0, s>>>(total, patches, cover);
  if (n > 0) weights_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, cover, w);
}

}  // namespace pdb::k
