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

// Programmatic dependent launch (sm_90+).  The three sweep kernels are
// launched with programmatic stream serialization: each one issues the loads
// that do not depend on its predecessor (matrix values/columns, tile indices,
// inverse-map slots, x) before griddepcontrol.wait, which returns once the
// predecessor grid has completed and its writes are visible.  Each kernel
// lets its dependent launch only after its own wait (so completion stays
// transitive along the stream); the dependent's CTAs then occupy SMs freed by
// the primary's last wave.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled() {
  const char* e = getenv("PDB_PDL");
  return !(e && e[0] == '0');
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Streaming loads that bypass L1 allocation (the CSR arrays are read once per
// sweep), keeping L1 for the reused x gathers.
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

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
    // Four independent (col, val, x) streams in flight per lane: the col -> x
    // gather is a dependent load, so memory-level parallelism comes from
    // issuing several entries before consuming any.
    int64_t p = lo + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (; p + 3 * G < hi; p += 4 * G) {
      const int32_t c0 = __ldg(col + p), c1 = __ldg(col + p + G), c2 = __ldg(col + p + 2 * G),
                    c3 = __ldg(col + p + 3 * G);
      const double v0 = __ldg(val + p), v1 = __ldg(val + p + G), v2 = __ldg(val + p + 2 * G),
                   v3 = __ldg(val + p + 3 * G);
      a0 += v0 * __ldg(x + c0);
      a1 += v1 * __ldg(x + c1);
      a2 += v2 * __ldg(x + c2);
      a3 += v3 * __ldg(x + c3);
    }
    for (; p < hi; p += G) a0 += __ldg(val + p) * __ldg(x + __ldg(col + p));
    acc = (a0 + a1) + (a2 + a3);
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

// Residual v2: a G-lane group per row loads up to E entries per lane in three
// batched steps (all columns, then all values with streaming cache hints,
// then all x gathers through L1) before any arithmetic, so a row costs three
// memory latencies instead of one per entry batch.  Longer rows loop.
template <int G, int E, int H = 0>
__global__ void __launch_bounds__(kBlock) residual_v2_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                             const int32_t* __restrict__ col,
                                                             const double* __restrict__ val,
                                                             const double* __restrict__ x,
                                                             const double* __restrict__ b, double* __restrict__ r,
                                                             double* __restrict__ block_sumsq, bool negate_b_absent) {
  const int lane = threadIdx.x % G;
  const int64_t row = (int64_t)blockIdx.x * (kBlock / G) + threadIdx.x / G;
  double acc = 0.0;
  if (row < n) {
    const int64_t lo = rp[row], hi = rp[row + 1];
    for (int64_t base = lo; base < hi; base += G * E) {
      int32_t c[E];
      double v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int64_t p = base + lane + e * G;
        c[e] = p < hi ? (H ? ld_stream(col + p) : __ldcs(col + p)) : -1;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int64_t p = base + lane + e * G;
        v[e] = p < hi ? (H ? ld_stream(val + p) : __ldcs(val + p)) : 0.0;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) acc += c[e] >= 0 ? v[e] * (H ? ld_keep(x + c[e]) : __ldg(x + c[e])) : 0.0;
    }
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

// Residual v3 ("CSR stream"): each block owns a contiguous row range whose
// nonzeros (<= kStreamNnz) it streams with fully coalesced loads -- all
// column indices, then all values, then the x gathers, kStreamPer
// independent loads in flight per thread -- into shared-memory products;
// 8-lane groups then reduce the rows out of shared memory.  Row ranges come
// from a per-matrix partition (DeviceCsr::blk_start, built at upload); a row
// longer than kStreamNnz gets a block to itself and is reduced block-wide.
constexpr int kStreamThreads = 256;
constexpr int kStreamPer = 8;   // base partition: 2048 nonzeros / 512 rows per block
constexpr int kStreamNnz = kStreamThreads * kStreamPer;
constexpr int kStreamRows = 512;

template <int PER>
__global__ void __launch_bounds__(kStreamThreads) residual_v3_kernel(
    int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r,
    const int32_t* __restrict__ blk_start, const int64_t* __restrict__ blk_base, double* __restrict__ block_sumsq,
    bool negate_b_absent) {
  constexpr int NNZ = kStreamThreads * PER;
  constexpr int ROWS = kStreamRows;
  __shared__ double prod[NNZ];
  __shared__ int64_t rps[ROWS + 1];
  __shared__ double bs[ROWS];
  __shared__ double red[kStreamThreads / 32];
  const int tid = threadIdx.x;
  // block descriptors are independent loads: the CSR streams can start
  // immediately instead of waiting for row_ptr
  const int64_t r0 = __ldg(blk_start + blockIdx.x), r1 = __ldg(blk_start + blockIdx.x + 1);
  const int64_t base = __ldg(blk_base + blockIdx.x), end = __ldg(blk_base + blockIdx.x + 1);
  const int nrows = (int)(r1 - r0);
  double sq = 0.0;
  if (end - base <= NNZ) {
    const int m = (int)(end - base) - tid;  // entries this thread may touch: k*T < m
    const int32_t* cp = col + base + tid;
    const double* vp = val + base + tid;
    int32_t c[PER];
    double v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) c[k] = k * kStreamThreads < m ? __ldcs(cp + k * kStreamThreads) : 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = k * kStreamThreads < m ? __ldcs(vp + k * kStreamThreads) : 0.0;
    for (int t = tid; t <= nrows; t += kStreamThreads) rps[t] = __ldg(rp + r0 + t);
    if (b)
      for (int t = tid; t < nrows; t += kStreamThreads) bs[t] = __ldcs(b + r0 + t);
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (k * kStreamThreads < m) prod[tid + k * kStreamThreads] = v[k] * __ldg(x + c[k]);
    __syncthreads();
    const int lane8 = tid & 7;
    // warp-uniform trip count: every lane reaches the shuffles
    for (int rr0 = (tid >> 5) * 4; rr0 < nrows; rr0 += kStreamThreads / 8) {
      const int rr = rr0 + ((tid >> 3) & 3);
      const bool has = rr < nrows;
      const int lo = has ? (int)(rps[rr] - base) : 0, hi = has ? (int)(rps[rr + 1] - base) : 0;
      double a = 0.0;
      for (int e = lo + lane8; e < hi; e += 8) a += prod[e];
      a += __shfl_xor_sync(0xffffffffu, a, 4);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      if (has && lane8 == 0) {
        const double rv = b ? bs[rr] - a : (negate_b_absent ? -a : a);
        r[r0 + rr] = rv;
        sq += rv * rv;
      }
    }
  } else {  // one long row (nrows == 1)
    double a = 0.0;
    for (int64_t e = base + tid; e < end; e += kStreamThreads) a += __ldcs(val + e) * __ldg(x + __ldcs(col + e));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if ((tid & 31) == 0) red[tid >> 5] = a;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kStreamThreads / 32; ++w) t += red[w];
      const double rv = b ? b[r0] - t : (negate_b_absent ? -t : t);
      r[r0] = rv;
      sq = rv * rv;
    }
    __syncthreads();
  }
  if (block_sumsq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if ((tid & 31) == 0) red[tid >> 5] = sq;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kStreamThreads / 32; ++w) t += red[w];
      block_sumsq[blockIdx.x] = t;
    }
  }
}

// Residual v4: the v3 chunk structure run by a persistent grid with a
// two-stage software pipeline -- while a block reduces chunk k out of shared
// memory, the column/value/row_ptr/b loads of its next chunk are already in
// flight in registers, so HBM never waits for the reduction phase.
constexpr int kV4Threads = 256;
constexpr int kV4Per = 8;
constexpr int kV4Rows = kStreamRows;                 // partition row cap (shared with v3)
constexpr int kV4RowRegs = (kV4Rows + 1 + kV4Threads - 1) / kV4Threads;  // 3

struct V4Chunk {
  int64_t r0, base;
  int nrows, nnz;
  int32_t c[kV4Per];
  double v[kV4Per];
  int64_t rpv[kV4RowRegs];
  double bv[kV4RowRegs];
};

__device__ __forceinline__ void v4_load(V4Chunk& ck, int ch, const int32_t* __restrict__ blk_start,
                                        const int64_t* __restrict__ blk_base, const int64_t* __restrict__ rp,
                                        const int32_t* __restrict__ col, const double* __restrict__ val,
                                        const double* __restrict__ b, int tid) {
  ck.r0 = __ldg(blk_start + ch);
  const int64_t r1 = __ldg(blk_start + ch + 1);
  ck.base = __ldg(blk_base + ch);
  const int64_t end = __ldg(blk_base + ch + 1);
  ck.nrows = (int)(r1 - ck.r0);
  ck.nnz = (int)(end - ck.base);
  if (ck.nnz <= kV4Threads * kV4Per) {
    const int m = ck.nnz - tid;
    const int32_t* cp = col + ck.base + tid;
    const double* vp = val + ck.base + tid;
#pragma unroll
    for (int k = 0; k < kV4Per; ++k) ck.c[k] = k * kV4Threads < m ? __ldcs(cp + k * kV4Threads) : 0;
#pragma unroll
    for (int k = 0; k < kV4Per; ++k) ck.v[k] = k * kV4Threads < m ? __ldcs(vp + k * kV4Threads) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < kV4RowRegs; ++q) {
    const int t = tid + q * kV4Threads;
    ck.rpv[q] = t <= ck.nrows ? __ldg(rp + ck.r0 + t) : 0;
    ck.bv[q] = (b && t < ck.nrows) ? __ldcs(b + ck.r0 + t) : 0.0;
  }
}

__global__ void __launch_bounds__(kV4Threads, 3) residual_v4_kernel(
    int nblk, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r,
    const int32_t* __restrict__ blk_start, const int64_t* __restrict__ blk_base, double* __restrict__ block_sumsq,
    bool negate_b_absent) {
  __shared__ double prod[kV4Threads * kV4Per];
  __shared__ int64_t rps[kV4Rows + 1];
  __shared__ double bs[kV4Rows];
  __shared__ double red[kV4Threads / 32];
  const int tid = threadIdx.x;
  double sq = 0.0;
  int ch = blockIdx.x;
  V4Chunk cur, nxt;
  if (ch < nblk) v4_load(cur, ch, blk_start, blk_base, rp, col, val, b, tid);
  while (ch < nblk) {
    const int nch = ch + gridDim.x;
    if (nch < nblk) v4_load(nxt, nch, blk_start, blk_base, rp, col, val, b, tid);  // in flight during the work below
#pragma unroll
    for (int q = 0; q < kV4RowRegs; ++q) {
      const int t = tid + q * kV4Threads;
      if (t <= cur.nrows) rps[t] = cur.rpv[q];
      if (t < cur.nrows) bs[t] = cur.bv[q];
    }
    if (cur.nnz <= kV4Threads * kV4Per) {
      const int m = cur.nnz - tid;
#pragma unroll
      for (int k = 0; k < kV4Per; ++k)
        if (k * kV4Threads < m) prod[tid + k * kV4Threads] = cur.v[k] * __ldg(x + cur.c[k]);
      __syncthreads();
      const int lane8 = tid & 7;
      for (int rr0 = (tid >> 5) * 4; rr0 < cur.nrows; rr0 += kV4Threads / 8) {
        const int rr = rr0 + ((tid >> 3) & 3);
        const bool has = rr < cur.nrows;
        const int lo = has ? (int)(rps[rr] - cur.base) : 0, hi = has ? (int)(rps[rr + 1] - cur.base) : 0;
        double a = 0.0;
        for (int e = lo + lane8; e < hi; e += 8) a += prod[e];
        a += __shfl_xor_sync(0xffffffffu, a, 4);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        if (has && lane8 == 0) {
          const double rv = b ? bs[rr] - a : (negate_b_absent ? -a : a);
          r[cur.r0 + rr] = rv;
          sq += rv * rv;
        }
      }
    } else {  // one long row
      double a = 0.0;
      const int64_t end = cur.base + cur.nnz;
      for (int64_t e = cur.base + tid; e < end; e += kV4Threads) a += __ldcs(val + e) * __ldg(x + __ldcs(col + e));
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if ((tid & 31) == 0) red[tid >> 5] = a;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kV4Threads / 32; ++w) t += red[w];
        const double rv = b ? b[cur.r0] - t : (negate_b_absent ? -t : t);
        r[cur.r0] = rv;
        sq += rv * rv;
      }
    }
    __syncthreads();
    cur = nxt;
    ch = nch;
  }
  if (block_sumsq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if ((tid & 31) == 0) red[tid >> 5] = sq;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kV4Threads / 32; ++w) t += red[w];
      block_sumsq[blockIdx.x] = t;
    }
  }
}

// Residual v5: warp-granular CSR streaming.  A precomputed partition gives
// every warp a run of <= 31 consecutive rows holding <= 256 nonzeros.  The
// warp loads that contiguous span with fully coalesced 32-lane loads (one
// 128-byte line per column load, two per value load: ~8x fewer L1 wavefronts
// than a group-per-row layout), gathers x, stages the products in a per-warp
// shared-memory slice (no block barrier), then 4-lane groups reduce the rows.
// A row longer than 256 nonzeros gets a warp to itself and loops.
constexpr int kV5Warps = 8;
constexpr int kV5Per = 8;
constexpr int kV5Rows = 31;

// CHUNK selects the row reduction.  false: 4-lane groups stride through each
// row's products (8 rows at a time; rows of unequal length leave lanes idle
// and the 8 row offsets collide in smem banks).  true (v6): lane l sums its
// own PER consecutive products, cutting at row starts (a 32*PER-bit boundary
// mask), and writes each segment sum at the segment's first position; lane
// rho then adds the segment sums of row rho in ascending position.  Products
// live at i + i/PER so both the slot-interleaved stores and the lane-chunk
// reads are bank-conflict free; ~3x fewer shared-memory wavefronts.
template <int PER, bool CHUNK>
__global__ void __launch_bounds__(kV5Warps * 32) residual_v5_kernel(
    int nwarps, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r,
    const int32_t* __restrict__ wstart, const int64_t* __restrict__ wbase, double* __restrict__ block_sumsq,
    bool negate_b_absent, int prefetch_dist) {
  constexpr int kSlots = CHUNK ? 32 * PER + 32 : 32 * PER;
  constexpr int kMaskWords = PER;  // 32*PER bits
  __shared__ double prod[kV5Warps][kSlots];
  __shared__ uint32_t bmask[kV5Warps][CHUNK ? kMaskWords : 1];
  __shared__ double red[kV5Warps];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * kV5Warps + wib;
  double sq = 0.0;
  if (w < nwarps) {
    // Bulk L2 prefetch (cp.async.bulk.prefetch, one instruction per stream)
    // of the CSR span a warp one prefetch distance ahead will read, so that
    // warp finds its columns/values in L2 instead of waiting on HBM.
    if (prefetch_dist > 0 && lane < 2) {
      const int wf = w + prefetch_dist;
      if (wf < nwarps) {
        const int64_t fb = __ldg(wbase + wf), fe = __ldg(wbase + wf + 1);
        const char* p0 = lane == 0 ? reinterpret_cast<const char*>(val + fb) : reinterpret_cast<const char*>(col + fb);
        const char* p1 = lane == 0 ? reinterpret_cast<const char*>(val + fe) : reinterpret_cast<const char*>(col + fe);
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(p0) & ~uintptr_t(15);
        const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p1) + 15) & ~uintptr_t(15);
        if (a1 > a0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
      }
    }
    const int64_t r0 = __ldg(wstart + w), base = __ldg(wbase + w), end = __ldg(wbase + w + 1);
    const int nrows = __ldg(wstart + w + 1) - (int)r0;
    const int nnz = (int)(end - base);
    const int64_t rpl = lane <= nrows ? __ldg(rp + r0 + lane) : end;
    const double bl = (b && lane < nrows) ? __ldcs(b + r0 + lane) : 0.0;
    if (nnz <= (32 * PER)) {
      int32_t c[PER];
      double v[PER];
      const int32_t* cp = col + base + lane;
      const double* vp = val + base + lane;
#pragma unroll
      for (int e = 0; e < PER; ++e) c[e] = e * 32 + lane < nnz ? __ldcs(cp + e * 32) : 0;
#pragma unroll
      for (int e = 0; e < PER; ++e) v[e] = e * 32 + lane < nnz ? __ldcs(vp + e * 32) : 0.0;
      double* pw = prod[wib];
      if constexpr (CHUNK) {
        uint32_t* mk = bmask[wib];
        if (lane < kMaskWords) mk[lane] = 0u;
        // products at padded position i + i/PER
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int i = e * 32 + lane;
          if (i < nnz) pw[i + i / PER] = v[e] * __ldg(x + c[e]);
        }
        __syncwarp();
        const int o = (int)(rpl - base);  // start of row `lane` (lanes 1..nrows-1 mark a cut)
        if (lane >= 1 && lane < nrows && o < nnz) atomicOr(mk + (o >> 5), 1u << (o & 31));
        __syncwarp();
        const int cb = lane * PER;
        const uint32_t fl = (mk[cb >> 5] >> (cb & 31)) & (PER == 32 ? 0xffffffffu : ((1u << PER) - 1u));
        double* pc = pw + cb + lane;  // = padded position of cb
        double pr[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) pr[j] = cb + j < nnz ? pc[j] : 0.0;
        double acc = 0.0;
        int seg = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const double pj = pr[j];
          if (j > 0 && ((fl >> j) & 1u)) {
            pc[seg] = acc;
            acc = 0.0;
            seg = j;
          }
          acc += pj;
        }
        if (cb < nnz) pc[seg] = acc;
        __syncwarp();
        const int hi = (int)(__shfl_down_sync(0xffffffffu, rpl, 1) - base);
        if (lane < nrows) {
          double a = 0.0;
          if (o < hi) {
            a = pw[o + o / PER];
            for (int q = o / PER + 1; q * PER < hi; ++q) a += pw[q * (PER + 1)];
          }
          const double rv = b ? bl - a : (negate_b_absent ? -a : a);
          r[r0 + lane] = rv;
          sq += rv * rv;
        }
      } else {
#pragma unroll
      for (int e = 0; e < PER; ++e)
        if (e * 32 + lane < nnz) pw[e * 32 + lane] = v[e] * __ldg(x + c[e]);
      __syncwarp();
      const int g4 = lane & 3, grp = lane >> 2;
      for (int rr0 = 0; rr0 < nrows; rr0 += 8) {  // warp-uniform trip count
        const int rr = rr0 + grp;
        const int lo = (int)(__shfl_sync(0xffffffffu, rpl, rr & 31) - base);
        const int hi = (int)(__shfl_sync(0xffffffffu, rpl, (rr + 1) & 31) - base);
        const double brr = __shfl_sync(0xffffffffu, bl, rr & 31);
        double a = 0.0;
        if (rr < nrows)
          for (int e = lo + g4; e < hi; e += 4) a += pw[e];
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        if (rr < nrows && g4 == 0) {
          const double rv = b ? brr - a : (negate_b_absent ? -a : a);
          r[r0 + rr] = rv;
          sq += rv * rv;
        }
      }
      }
    } else {  // one long row
      double a = 0.0;
      for (int64_t e = base + lane; e < end; e += 32) a += __ldcs(val + e) * __ldg(x + __ldcs(col + e));
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if (lane == 0) {
        const double rv = b ? b[r0] - a : (negate_b_absent ? -a : a);
        r[r0] = rv;
        sq += rv * rv;
      }
    }
  }
  if (block_sumsq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[wib] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < kV5Warps; ++q) t += red[q];
      block_sumsq[blockIdx.x] = t;
    }
  }
}

// Residual v7: v5's warp items fed by the bulk-copy (TMA) engine.  A
// persistent grid; warp gw processes items gw, gw + TW, ... (TW = all warps,
// so the GPU sweeps a window of consecutive rows and x stays L2-hot).  Each
// warp owns an S-stage ring in shared memory; lane 0 arms stage s's mbarrier
// with the byte count and issues cp.async.bulk copies of the item's values
// and columns S items ahead, so a warp always has S items of CSR bytes in
// flight without holding them in registers (v5 keeps ~3 KB per warp in
// flight only during its load phase, which left DRAM at ~50 % busy).  The
// consumer then gathers x, forms the products in place and reduces rows as
// v5.  Copies are 16-byte aligned: the span is widened to aligned bounds
// (the device CSR arrays carry 32 elements of zero padding) and the data
// sits at offset base & 1 (values) / base & 3 (columns) in the stage.
constexpr int kV7Vals = 32 * kV5Per + 4;  // 256 + alignment slack, doubles
constexpr int kV7Cols = 32 * kV5Per + 8;  // ints
constexpr int kV7StageBytes = kV7Vals * 8 + kV7Cols * 4;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

template <int S>
__global__ void __launch_bounds__(kV5Warps * 32) residual_v7_kernel(
    int nitems, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r,
    const int32_t* __restrict__ wstart, const int64_t* __restrict__ wbase, double* __restrict__ block_sumsq,
    bool negate_b_absent) {
  extern __shared__ __align__(128) unsigned char v7_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int TW = gridDim.x * kV5Warps;
  const int gw = blockIdx.x * kV5Warps + wib;
  uint64_t* bars = reinterpret_cast<uint64_t*>(v7_smem) + wib * S;
  unsigned char* ring = v7_smem + 128 * ((kV5Warps * S * 8 + 127) / 128) + (size_t)wib * S * kV7StageBytes;
  __shared__ double red[kV5Warps];
  if (lane < S) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bars + lane)) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // issue item j into stage st (lane 0 only)
  auto issue = [&](int j, int st) {
    unsigned char* sg = ring + (size_t)st * kV7StageBytes;
    const int64_t base = __ldg(wbase + j), end = __ldg(wbase + j + 1);
    const uint32_t bar = smem_addr(bars + st);
    if (end - base <= 32 * kV5Per) {
      const int64_t vb = base & ~int64_t(1), cb = base & ~int64_t(3);
      const uint32_t vbytes = (uint32_t)(((end - vb) * 8 + 15) & ~int64_t(15));
      const uint32_t cbytes = (uint32_t)(((end - cb) * 4 + 15) & ~int64_t(15));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(vbytes + cbytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(sg)),
          "l"(val + vb), "r"(vbytes), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(sg + kV7Vals * 8)),
          "l"(col + cb), "r"(cbytes), "r"(bar)
          : "memory");
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    }
  };
  if (lane == 0)
    for (int q = 0; q < S; ++q)
      if (gw + q * TW < nitems) issue(gw + q * TW, q);
  __syncwarp();
  double sq = 0.0;
  int it = 0;
  for (int j = gw; j < nitems; j += TW, ++it) {
    const int st = it % S;
    unsigned char* sg = ring + (size_t)st * kV7StageBytes;
    // independent of the staged bytes: row pointers and b for this item
    const int64_t r0 = __ldg(wstart + j);
    const int nrows = __ldg(wstart + j + 1) - (int)r0;
    const int64_t base = __ldg(wbase + j), end = __ldg(wbase + j + 1);
    const int64_t rpl = lane <= nrows ? __ldg(rp + r0 + lane) : end;
    const double bl = (b && lane < nrows) ? __ldcs(b + r0 + lane) : 0.0;
    const int nnz = (int)(end - base);
    mbar_wait(smem_addr(bars + st), (uint32_t)((it / S) & 1));
    if (nnz <= 32 * kV5Per) {
      double* vs = reinterpret_cast<double*>(sg) + (base & 1);
      const int32_t* cs = reinterpret_cast<const int32_t*>(sg + kV7Vals * 8) + (base & 3);
      int32_t c[kV5Per];
#pragma unroll
      for (int e = 0; e < kV5Per; ++e) c[e] = e * 32 + lane < nnz ? cs[e * 32 + lane] : 0;
      double xv[kV5Per];
#pragma unroll
      for (int e = 0; e < kV5Per; ++e) xv[e] = e * 32 + lane < nnz ? __ldg(x + c[e]) : 0.0;
#pragma unroll
      for (int e = 0; e < kV5Per; ++e)
        if (e * 32 + lane < nnz) vs[e * 32 + lane] *= xv[e];
      __syncwarp();
      const int g4 = lane & 3, grp = lane >> 2;
      for (int rr0 = 0; rr0 < nrows; rr0 += 8) {  // warp-uniform trip count
        const int rr = rr0 + grp;
        const int lo = (int)(__shfl_sync(0xffffffffu, rpl, rr & 31) - base);
        const int hi = (int)(__shfl_sync(0xffffffffu, rpl, (rr + 1) & 31) - base);
        const double brr = __shfl_sync(0xffffffffu, bl, rr & 31);
        double a = 0.0;
        if (rr < nrows)
          for (int e = lo + g4; e < hi; e += 4) a += vs[e];
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        if (rr < nrows && g4 == 0) {
          const double rv = b ? brr - a : (negate_b_absent ? -a : a);
          r[r0 + rr] = rv;
          sq += rv * rv;
        }
      }
    } else {  // one long row, straight from global memory
      double a = 0.0;
      for (int64_t e = base + lane; e < end; e += 32) a += __ldcs(val + e) * __ldg(x + __ldcs(col + e));
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if (lane == 0) {
        const double rv = b ? b[r0] - a : (negate_b_absent ? -a : a);
        r[r0] = rv;
        sq += rv * rv;
      }
    }
    __syncwarp();
    const int jn = j + S * TW;
    if (lane == 0 && jn < nitems) issue(jn, st);
  }
  if (block_sumsq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[wib] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < kV5Warps; ++q) t += red[q];
      block_sumsq[blockIdx.x] = t;
    }
  }
}

// Residual v8: v5's warp items with block-local column windows (built by
// build_windows, matrix.cpp).  The block first stages x over its window --
// runs of consecutive columns, one warp per run, coalesced -- while every
// warp already has its item's values and 16-bit local columns in flight;
// after one block barrier the x gathers read shared memory.  Per nonzero the
// kernel streams 10 bytes (value + local column) instead of 12, and the L1
// no longer replays x gathers over ~6 cache lines per warp load.
static_assert(kItemNnz == 32 * kV5Per, "v8 item capacity");
static_assert(kWindowItems == kV5Warps, "v8 block = one window");

template <int MINB>
__global__ void __launch_bounds__(kV5Warps * 32, MINB) residual_v8_kernel(
    int nitems, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
    const uint16_t* __restrict__ lcol, const int32_t* __restrict__ win_ptr, const int2* __restrict__ win_runs,
    const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r,
    const int32_t* __restrict__ wstart, const int64_t* __restrict__ wbase, double* __restrict__ block_sumsq,
    bool negate_b_absent) {
  extern __shared__ double xs[];
  __shared__ double prod[kV5Warps][32 * kV5Per];
  __shared__ double red[kV5Warps];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * kV5Warps + wib;
  const bool has = w < nitems;
  int64_t r0 = 0, base = 0, end = 0;
  int nrows = 0;
  if (has) {
    r0 = __ldg(wstart + w);
    nrows = __ldg(wstart + w + 1) - (int)r0;
    base = __ldg(wbase + w);
    end = __ldg(wbase + w + 1);
  }
  const int nnz = (int)(end - base);
  const bool shortitem = has && nnz <= 32 * kV5Per;
  // item bytes in flight before the window staging
  uint16_t lc[kV5Per];
  double v[kV5Per];
  if (shortitem) {
#pragma unroll
    for (int e = 0; e < kV5Per; ++e) lc[e] = e * 32 + lane < nnz ? __ldcs(lcol + base + e * 32 + lane) : 0;
#pragma unroll
    for (int e = 0; e < kV5Per; ++e) v[e] = e * 32 + lane < nnz ? __ldcs(val + base + e * 32 + lane) : 0.0;
  }
  const int64_t rpl = (has && lane <= nrows) ? __ldg(rp + r0 + lane) : end;
  const double bl = (has && b && lane < nrows) ? __ldcs(b + r0 + lane) : 0.0;
  {
    const int q0 = __ldg(win_ptr + blockIdx.x), q1 = __ldg(win_ptr + blockIdx.x + 1) - 1;  // last: sentinel
    for (int q = q0 + wib; q < q1; q += kV5Warps) {
      const int2 a = __ldg(win_runs + q);
      const int len = __ldg(win_runs + q + 1).y - a.y;
      for (int j = lane; j < len; j += 32) xs[a.y + j] = __ldg(x + a.x + j);
    }
  }
  __syncthreads();
  double sq = 0.0;
  if (shortitem) {
    double* pw = prod[wib];
#pragma unroll
    for (int e = 0; e < kV5Per; ++e)
      if (e * 32 + lane < nnz) pw[e * 32 + lane] = v[e] * xs[lc[e]];
    __syncwarp();
    const int g4 = lane & 3, grp = lane >> 2;
    for (int rr0 = 0; rr0 < nrows; rr0 += 8) {  // warp-uniform trip count
      const int rr = rr0 + grp;
      const int lo = (int)(__shfl_sync(0xffffffffu, rpl, rr & 31) - base);
      const int hi = (int)(__shfl_sync(0xffffffffu, rpl, (rr + 1) & 31) - base);
      const double brr = __shfl_sync(0xffffffffu, bl, rr & 31);
      double a = 0.0;
      if (rr < nrows)
        for (int e = lo + g4; e < hi; e += 4) a += pw[e];
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      if (rr < nrows && g4 == 0) {
        const double rv = b ? brr - a : (negate_b_absent ? -a : a);
        r[r0 + rr] = rv;
        sq += rv * rv;
      }
    }
  } else if (has) {  // one long row, global columns
    double a = 0.0;
    for (int64_t e = base + lane; e < end; e += 32) a += __ldcs(val + e) * __ldg(x + __ldcs(col + e));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if (lane == 0) {
      const double rv = b ? b[r0] - a : (negate_b_absent ? -a : a);
      r[r0] = rv;
      sq += rv * rv;
    }
  }
  if (block_sumsq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[wib] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < kV5Warps; ++q) t += red[q];
      block_sumsq[blockIdx.x] = t;
    }
  }
}

// Residual v9 over the SELL-C-sigma copy (build_sell, matrix.cpp): warp per
// slice of 32 rows, lane l owns slice row l.  Step j loads entry j of all 32
// rows -- one 256-byte value span and one 128-byte column span, fully
// coalesced -- and the x gathers of 32 similar rows hit a few lines.  U steps
// are loaded before any is consumed (memory-level parallelism without a
// shared-memory stage), lanes past their row's end are predicated off, and
// each lane accumulates its row in CSR order with unfused multiply/add:
// r = b - s bit for bit as the reference spmv + smooth (sparse.cpp:50-63,
// precond.cpp:95-97).
template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) residual_sell_kernel(int64_t nslices, const int64_t* __restrict__ soff,
                                                            const int2* __restrict__ srow,
                                                            const double* __restrict__ sval,
                                                            const int32_t* __restrict__ scol,
                                                            const double* __restrict__ x, const double* __restrict__ b,
                                                            double* __restrict__ r, double* __restrict__ block_sumsq,
                                                            bool negate_b_absent, int pf) {
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t sl = (int64_t)blockIdx.x * 8 + wib;
  double sq = 0.0;
  if (sl >= nslices) {
    grid_dep_wait();
    grid_dep_trigger();
  }
  if (sl < nslices) {
    const int2 rl = __ldg(srow + sl * 32 + lane);
    const int len = rl.y;
    const int L = __reduce_max_sync(0xffffffffu, (unsigned)len);
    const int64_t o = __ldg(soff + sl);
    const double* vp = sval + o + lane;
    const int32_t* cp = scol + o + lane;
    const double bl = (rl.x >= 0 && b) ? __ldcs(b + rl.x) : 0.0;
    double acc = 0.0;
    int32_t c[U];
    double v[U];
    // first step group: independent of the predecessor (the scatter writing x)
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = u < len ? __ldcs(cp + (int64_t)u * 32) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = u < len ? __ldcs(vp + (int64_t)u * 32) : 0.0;
    grid_dep_wait();
    grid_dep_trigger();
    for (int j = 0; j < L; j += U) {
      // pull the slice's next columns/values towards L2 (bulk prefetch, no
      // registers held) so the loads pf iterations ahead find them there
      if (pf > 0 && lane == 0) {
        const int jn = j + pf * U;
        if (jn < L) {
          const int cnt = (L - jn < U ? L - jn : U) * 32;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sval + o + (int64_t)jn * 32),
                       "r"((unsigned)(cnt * 8)));
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(scol + o + (int64_t)jn * 32),
                       "r"((unsigned)(cnt * 4)));
        }
      }
      if (j > 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = j + u < len ? __ldcs(cp + (int64_t)(j + u) * 32) : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = j + u < len ? __ldcs(vp + (int64_t)(j + u) * 32) : 0.0;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = j + u < len ? __ldg(x + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    if (rl.x >= 0) {
      const double rv = b ? __dsub_rn(bl, acc) : (negate_b_absent ? -acc : acc);
      r[rl.x] = rv;
      sq += rv * rv;
    }
  }
  if (block_sumsq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[wib] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += red[q];
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

// Patch apply with explicit inverses (the default sweep path).  A block
// holds PPB patches x ps threads; the gathered residual of each patch is
// staged in shared memory once, then thread (patch, i) forms row i of
// B^{-1} r_k from the column-major inverse (threads of a patch read
// consecutive addresses; compressed inverses are L2-resident).  Every
// product is independent -- no dependent shuffle chain as in a triangular
// solve -- so the kernel runs at memory speed.
__global__ void patch_apply_inv_kernel(int64_t np, int ps, int ppb, const int32_t* __restrict__ patches,
                                       const double* __restrict__ Binv, const int32_t* __restrict__ phi,
                                       const double* __restrict__ r, const double* __restrict__ in_scale,
                                       double* __restrict__ sols) {
  extern __shared__ double rk[];  // ppb * ps
  const int pl = threadIdx.x / ps, i = threadIdx.x % ps;
  const int64_t k = (int64_t)blockIdx.x * ppb + pl;
  const bool live = pl < ppb && k < np;
  if (live) {
    const int32_t g = __ldg(patches + k * ps + i);
    double v = __ldg(r + g);
    if (in_scale) v *= __ldg(in_scale + g);
    rk[pl * ps + i] = v;
  }
  __syncthreads();
  if (!live) return;
  const int64_t f = phi ? (int64_t)__ldg(phi + k) : k;
  const double* B = Binv + f * (int64_t)ps * ps + i;
  const double* x = rk + pl * ps;
  // same summation order as the grouped kernel (one accumulator, ascending
  // j), so exact and identity-phi compressed applies agree bit for bit
  double a = 0.0;
  for (int j = 0; j < ps; ++j) a += __ldg(B + (int64_t)j * ps) * x[j];
  sols[k * ps + i] = a;
}

// Cluster-grouped apply (compressed mode): patches are pre-sorted by their
// database entry; a block takes one tile of up to TP patches sharing entry
// f, stages B_f^{-1} (ps^2 doubles) and the tile's gathered residuals in
// shared memory, then forms the dense product B_f^{-1} [r_k1 .. r_kTP].
// Each inverse is read once per tile instead of once per patch (the 64
// config-2 inverses would otherwise cost 328 MB of L2 traffic per sweep).
// Patch DoF lists and solutions are stored in tile order (tile_idx / sols
// position s = rank of the patch in the entry-sorted order), so a tile reads
// and writes contiguous runs; the scatter's inverse map points at the same
// tile-order slots.
__global__ void patch_apply_grouped_kernel(int ps, const int32_t* __restrict__ tile_entry,
                                           const int32_t* __restrict__ tile_start,
                                           const int32_t* __restrict__ tile_idx, const int32_t* __restrict__ order,
                                           const double* __restrict__ Binv,
                                           const double* __restrict__ r, const double* __restrict__ in_scale,
                                           double* __restrict__ sols) {
  extern __shared__ double sm[];
  const int t = blockIdx.x;
  const int64_t f = __ldg(tile_entry + t);
  const int s0 = __ldg(tile_start + t), cnt = __ldg(tile_start + t + 1) - s0;
  const int len = ps * ps;
  double* B = sm;          // column-major inverse
  double* rk = sm + len;   // cnt x ps gathered residuals
  const double* Bg = Binv + f * (int64_t)len;
  const int NG = blockDim.x / ps;
  const int i = threadIdx.x % ps, g = threadIdx.x / ps;
  for (int e = threadIdx.x; e < len; e += blockDim.x) B[e] = __ldg(Bg + e);
  if (g < NG)
    for (int p = g; p < cnt; p += NG) {
      const int32_t gi = __ldg(tile_idx + (int64_t)(s0 + p) * ps + i);
      double v = __ldg(r + gi);
      if (in_scale) v *= __ldg(in_scale + gi);
      rk[p * ps + i] = v;
    }
  __syncthreads();
  // Register tiling: thread (g, i) owns row i of patches g, g+NG, g+2NG,
  // g+3NG, so each B element read from shared memory feeds four products.
  if (g >= NG) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < ps; ++j) {
    const double bij = B[j * ps + i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = g + q * NG;
      if (p < cnt) acc[q] += bij * rk[p * ps + j];
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int p = g + q * NG;
    if (p < cnt) sols[(int64_t)__ldg(order + s0 + p) * ps + i] = acc[q];
  }
}

// Tensor-core grouped apply.  A tile of up to 32 patches sharing entry f is
// the dense product S (ps x 32) = B_f^{-1} (ps x ps) R (ps x 32), done with
// FP64 mma.sync.m8n8k4: warp w owns rows [8w, 8w+8) of B_f^{-1} (MT = ps/8
// warps), keeps its KS = ps/4 A-fragments in registers (loaded coalesced from
// the fragment-ordered copy, L2-resident), and sweeps the four 8-patch column
// blocks of R from shared memory.  Per tile: 4 x MT x KS DMMAs and MT x KS x 4
// fragment loads, against ps x 32 x 5 shared loads for the CUDA-core version.
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): A row-major, lane (g = lane/4,
// t = lane%4) holds A[g][t]; B column-major, B[t][g]; C/D: C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int kDmmaTile = 32;  // patches per tile (4 column blocks of 8)

constexpr int32_t kDofMask = (1 << 28) - 1;  // zfwd = (slot rank << 28) | dof

// Z = false: solutions to sols in tile order (idx = tile_idx).  Z = true:
// idx = zfwd, each solution value goes to out[(f >> 28) * n + (f & mask)].
// R is staged unpadded (patch p, local row k at p * ps + k), so the copy is a
// flat, division-free loop; the A fragments are zero for k >= ps, which
// cancels the neighbouring patch's values a B fragment reads there, and the
// stage is zero-filled past the tile's cnt * ps live values (no NaN garbage).
template <int MT, int KS, bool Z>
__global__ void __launch_bounds__(MT * 32) patch_apply_dmma_kernel(int ps, int64_t n,
                                                                   const int32_t* __restrict__ tile_entry,
                                                                   const int32_t* __restrict__ tile_start,
                                                                   const int32_t* __restrict__ idx,
                                                                   const int32_t* __restrict__ order,
                                                                   const double* __restrict__ frag,
                                                                   const double* __restrict__ r,
                                                                   const double* __restrict__ in_scale,
                                                                   double* __restrict__ out) {
  constexpr int NTH = MT * 32;
  constexpr int TOT = kDmmaTile * KS * 4;  // >= 31 * ps + 4 * KS: every B-fragment read
  constexpr int ITER = (TOT + NTH - 1) / NTH;
  __shared__ double rk[TOT];
  __shared__ int32_t fk[Z ? TOT : 1];
  __shared__ int32_t ko[kDmmaTile];  // patch index of each tile column (output in patch order)
  const int t = blockIdx.x;
  const int f = __ldg(tile_entry + t);
  const int s0 = __ldg(tile_start + t), cnt = __ldg(tile_start + t + 1) - s0;
  if (!Z && threadIdx.x < cnt) ko[threadIdx.x] = __ldg(order + s0 + threadIdx.x);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a[KS];
  const double* fa = frag + ((int64_t)f * MT + w) * (KS * 32) + lane;
#pragma unroll
  for (int q = 0; q < KS; ++q) a[q] = __ldg(fa + q * 32);
  const int live = cnt * ps;
  const int32_t* ti = idx + (int64_t)s0 * ps;
  int32_t gi[ITER];
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int e = threadIdx.x + it * NTH;
    gi[it] = e < live ? __ldg(ti + e) : -1;
  }
  grid_dep_wait();  // r is the residual kernel's output
  grid_dep_trigger();
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int e = threadIdx.x + it * NTH;
    double v = 0.0;
    if (gi[it] >= 0) {
      const int32_t d = Z ? (gi[it] & kDofMask) : gi[it];
      v = __ldg(r + d);
      if (in_scale) v *= __ldg(in_scale + d);
      if constexpr (Z) fk[e] = gi[it];
    }
    if (e < TOT) rk[e] = v;
  }
  __syncthreads();
  const int g = lane >> 2, tg = lane & 3;
  const int row = w * 8 + g;
#pragma unroll
  for (int nt = 0; nt < kDmmaTile / 8; ++nt) {
    if (nt * 8 < cnt) {  // block-uniform
      double c0 = 0.0, c1 = 0.0;
      const double* bp = rk + (nt * 8 + g) * ps + tg;
#pragma unroll
      for (int q = 0; q < KS; ++q) dmma_m8n8k4(c0, c1, a[q], bp[q * 4]);
      const int p0 = nt * 8 + 2 * tg;
      if (row < ps) {
        if constexpr (Z) {
          if (p0 < cnt) {
            const int32_t z0 = fk[p0 * ps + row];
            out[(int64_t)(z0 >> 28) * n + (z0 & kDofMask)] = c0;
          }
          if (p0 + 1 < cnt) {
            const int32_t z1 = fk[(p0 + 1) * ps + row];
            out[(int64_t)(z1 >> 28) * n + (z1 & kDofMask)] = c1;
          }
        } else {
          if (p0 < cnt) out[(int64_t)ko[p0] * ps + row] = c0;
          if (p0 + 1 < cnt) out[(int64_t)ko[p0 + 1] * ps + row] = c1;
        }
      }
    }
  }
}

// Large patches (32 < ps <= 256, e.g. the 192-DoF elasticity patches): the
// same tile product with run-time shapes.  MT = ps/8 warps (<= 32), the
// inverse's A fragments streamed from L2 in chunks of 8 k-steps (a 192x192
// entry is 295 KB -- it cannot stay in registers or shared memory), R staged
// with a row stride padded to avoid bank conflicts.  Each tile reads its
// entry once instead of once per patch.
__global__ void __launch_bounds__(1024) patch_apply_dmma_large_kernel(
    int ps, int mt, int ks, int kstr, const int32_t* __restrict__ tile_entry, const int32_t* __restrict__ tile_start,
    const int32_t* __restrict__ tile_idx, const int32_t* __restrict__ order, const double* __restrict__ frag,
    const double* __restrict__ r, const double* __restrict__ in_scale, double* __restrict__ sols) {
  extern __shared__ double rk[];  // kDmmaTile * kstr
  __shared__ int32_t ko[kDmmaTile];
  const int t = blockIdx.x;
  const int f = __ldg(tile_entry + t);
  const int s0 = __ldg(tile_start + t), cnt = __ldg(tile_start + t + 1) - s0;
  const int nth = blockDim.x;
  if ((int)threadIdx.x < cnt) ko[threadIdx.x] = __ldg(order + s0 + threadIdx.x);
  const int32_t* ti = tile_idx + (int64_t)s0 * ps;
  grid_dep_wait();
  grid_dep_trigger();
  const int tot = kDmmaTile * kstr;
  for (int e = threadIdx.x; e < tot; e += nth) {
    const int p = e / kstr, k = e - p * kstr;
    double v = 0.0;
    if (p < cnt && k < ps) {
      const int32_t g = __ldg(ti + p * ps + k);
      v = __ldg(r + g);
      if (in_scale) v *= __ldg(in_scale + g);
    }
    rk[e] = v;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tg = lane & 3;
  double c[kDmmaTile / 8][2];
#pragma unroll
  for (int nt = 0; nt < kDmmaTile / 8; ++nt) c[nt][0] = c[nt][1] = 0.0;
  const double* fa = frag + ((int64_t)f * mt + w) * ks * 32 + lane;
  for (int kc = 0; kc < ks; kc += 8) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = kc + q < ks ? __ldg(fa + (int64_t)(kc + q) * 32) : 0.0;
#pragma unroll
    for (int nt = 0; nt < kDmmaTile / 8; ++nt) {
      if (nt * 8 < cnt) {
        const double* bp = rk + (nt * 8 + g) * kstr + kc * 4 + tg;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (kc + q < ks) dmma_m8n8k4(c[nt][0], c[nt][1], a[q], bp[q * 4]);
      }
    }
  }
  const int row = w * 8 + g;
  if (row < ps) {
#pragma unroll
    for (int nt = 0; nt < kDmmaTile / 8; ++nt) {
      const int p0 = nt * 8 + 2 * tg;
      if (p0 < cnt) sols[(int64_t)ko[p0] * ps + row] = c[nt][0];
      if (p0 + 1 < cnt) sols[(int64_t)ko[p0 + 1] * ps + row] = c[nt][1];
    }
  }
}

__global__ void build_zmap_kernel(int64_t n, int ps, const int32_t* __restrict__ inv_ptr,
                                  const int32_t* __restrict__ inv, const int32_t* __restrict__ slot_of,
                                  int32_t* __restrict__ zfwd, uint8_t* __restrict__ zcnt) {
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int32_t lo = inv_ptr[d], hi = inv_ptr[d + 1];
  zcnt[d] = (uint8_t)(hi - lo);
  for (int32_t q = lo; q < hi; ++q) {
    const int32_t e = inv[q];  // k * ps + l
    zfwd[(int64_t)slot_of[e / ps] * ps + e % ps] = ((q - lo) << 28) | (int32_t)d;
  }
}

// Scatter over DoF-major slots: loads only the zcnt[i] live slots of DoF i
// (ascending patch order), weight recomputed as scatter_update_pad_kernel.
template <int MAXC>
__global__ void scatter_z_kernel(int64_t n, const uint8_t* __restrict__ zcnt, const double* __restrict__ Z,
                                 double omega, bool sym, const double* __restrict__ x_in,
                                 double* __restrict__ z_out, double* __restrict__ x_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cnt = zcnt[i];
  double v[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) v[c] = c < cnt ? __ldcs(Z + (int64_t)c * n + i) : 0.0;
  const double xi = x_out ? __ldcs(x_in + i) : 0.0;
  double z = 0.0;
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
    if (c < cnt) z += v[c];
  double w = cnt > 0 ? 1.0 / (double)cnt : 0.0;
  if (sym) w = sqrt(w);
  z *= omega * w;
  if (z_out) z_out[i] = z;
  if (x_out) x_out[i] = z + xi;
}

// frag[f][w][q][lane] = B_f^{-1}[8w + lane/4][4q + lane%4] (0 outside ps x ps)
__global__ void build_frag_kernel(int64_t total, int ps, int mt, int ks, const double* __restrict__ inv_cm,
                                  double* __restrict__ frag) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int lane = (int)(e & 31);
  const int64_t rest = e >> 5;
  const int q = (int)(rest % ks);
  const int w = (int)((rest / ks) % mt);
  const int64_t f = rest / ((int64_t)ks * mt);
  const int row = w * 8 + (lane >> 2), c = q * 4 + (lane & 3);
  frag[e] = (row < ps && c < ps) ? inv_cm[f * ps * ps + (int64_t)c * ps + row] : 0.0;
}

// Shard scatter over a DoF list: z = init[d] (or 0) + sum of the DoF's
// solution slots in ascending patch order; optionally z_out[t] = z, and/or
// x[d] += z * omega_w[d] (the smooth() update for owned DoFs).
__global__ void shard_scatter_kernel(int64_t count, const int32_t* __restrict__ list,
                                     const int32_t* __restrict__ inv_ptr, const int32_t* __restrict__ inv,
                                     const double* __restrict__ sols, const double* __restrict__ init,
                                     const double* __restrict__ omega_w, double* __restrict__ z_out,
                                     double* __restrict__ x) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int32_t d = list[t];
  double z = init ? init[d] : 0.0;
  for (int32_t q = inv_ptr[d]; q < inv_ptr[d + 1]; ++q) z += __ldg(sols + __ldg(inv + q));
  if (z_out) z_out[t] = z;
  if (x) x[d] = z * omega_w[d] + x[d];
}

__global__ void gather_vals_kernel(int64_t count, const int32_t* __restrict__ idx, const double* __restrict__ src,
                                   double* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) dst[t] = src[idx[t]];
}

__global__ void scatter_vals_kernel(int64_t count, const int32_t* __restrict__ idx, const double* __restrict__ src,
                                    double* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) dst[idx[t]] = src[t];
}

// inverse-map entries k*ps + l -> slot_of[k]*ps + l (tile-order solution slots)
__global__ void remap_inverse_kernel(int64_t count, int ps, const int32_t* __restrict__ slot_of, int32_t* inv) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const int32_t t = inv[q];
  inv[q] = slot_of[t / ps] * ps + t % ps;
}

// Scatter/update with the padded slot-major inverse map: slot c of DoF i is
// inv_pad[c*n + i] (ascending patch order, -1 = empty), so all slot loads of
// a DoF are independent and coalesced.  The overlap weight is recomputed
// from the slot count exactly as compute_weights does (patch.cpp:12-20):
// scale = omega * (1.0 / count) (or omega * sqrt(1.0 / count) for the
// symmetric PCG weighting).
constexpr int kScatterU = 2;

template <int MAXC>
__global__ void scatter_update_pad_kernel(int64_t n, const int32_t* __restrict__ inv_pad,
                                          const double* __restrict__ sols, double omega, bool sym,
                                          const double* __restrict__ x_in, double* __restrict__ z_out,
                                          double* __restrict__ x_out) {
  // kScatterU DoFs per thread (blockDim apart, so every load stays
  // coalesced): all index loads, then all solution / x loads are in flight
  // together -- the kernel is latency-bound on the idx -> sols chain.
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x * kScatterU + threadIdx.x;
  int32_t e[kScatterU][MAXC];
  double v[kScatterU][MAXC], xi[kScatterU];
#pragma unroll
  for (int u = 0; u < kScatterU; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) e[u][c] = i < n ? __ldcs(inv_pad + (int64_t)c * n + i) : -1;
    xi[u] = (x_out && i < n) ? __ldcs(x_in + i) : 0.0;
  }
  grid_dep_wait();  // sols is the apply kernel's output
  grid_dep_trigger();
#pragma unroll
  for (int u = 0; u < kScatterU; ++u) {
#pragma unroll
    for (int c = 0; c < MAXC; ++c) v[u][c] = e[u][c] >= 0 ? __ldg(sols + e[u][c]) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kScatterU; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    if (i >= n) break;
    double z = 0.0;
    int cnt = 0;
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (e[u][c] >= 0) {
        z += v[u][c];
        ++cnt;
      }
    double w = cnt > 0 ? 1.0 / (double)cnt : 0.0;
    if (sym) w = sqrt(w);
    z *= omega * w;
    if (z_out) z_out[i] = z;
    if (x_out) x_out[i] = z + xi[u];
  }
}

__global__ void build_inverse_pad_kernel(int64_t n, int maxc, const int32_t* __restrict__ inv_ptr,
                                         const int32_t* __restrict__ inv, int32_t* __restrict__ pad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t lo = inv_ptr[i], hi = inv_ptr[i + 1];
  for (int c = 0; c < maxc; ++c) pad[(int64_t)c * n + i] = lo + c < hi ? inv[lo + c] : -1;
}

// Column c of B^{-1} = lu_solve(LU, e_c) (dense.cpp:77-94 applied to unit
// vectors).  Warp per factor, lanes over columns; the per-lane work vector
// lives in the (column-major) output itself.
__global__ void invert_factors_kernel(int64_t nf, int ps, const double* __restrict__ lu,
                                      const int32_t* __restrict__ piv, double* __restrict__ inv) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (f >= nf) return;
  const int64_t len = (int64_t)ps * ps;
  const double* L = lu + f * len;
  const int32_t* P = piv + f * ps;
  for (int c = lane; c < ps; c += 32) {
    double* o = inv + f * len + (int64_t)c * ps;  // column c, contiguous
    for (int i = 0; i < ps; ++i) o[i] = P[i] == c ? 1.0 : 0.0;
    for (int i = 1; i < ps; ++i) {
      double s = o[i];
      for (int j = 0; j < i; ++j) s -= L[(int64_t)i * ps + j] * o[j];
      o[i] = s;
    }
    for (int i = ps - 1; i >= 0; --i) {
      double s = o[i];
      for (int j = i + 1; j < ps; ++j) s -= L[(int64_t)i * ps + j] * o[j];
      o[i] = s / L[(int64_t)i * ps + i];
    }
  }
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

int stream_nnz() { return kStreamNnz; }

std::vector<int32_t> stream_partition(int64_t n, const int64_t* rp, int per) {
  if (per < 0) return row_partition(n, rp, 32 * (int64_t)(-per), kV5Rows);  // v5 warp partition
  return row_partition(n, rp, (int64_t)kStreamThreads * per, kStreamRows);
}

std::vector<int32_t> row_partition(int64_t n, const int64_t* rp, int64_t cap_nnz, int64_t cap_rows) {
  std::vector<int32_t> starts;
  starts.push_back(0);
  int64_t row = 0;
  while (row < n) {
    const int64_t b0 = rp[row];
    int64_t end = row + 1;  // a block always takes at least one row
    while (end < n && end - row < cap_rows && rp[end + 1] - b0 <= cap_nnz) ++end;
    if (rp[row + 1] - b0 > cap_nnz) end = row + 1;  // long row alone
    starts.push_back((int32_t)end);
    row = end;
  }
  return starts;
}

int v7_stages();
template <int S>
int v7_grid(int nitems);

SpmvPlan spmv_plan_stream(int64_t n, int64_t nnz, const int32_t* blk_start, const int64_t* blk_base, int nblk,
                          int per) {
  SpmvPlan p = spmv_plan(n, nnz);
  const char* e = getenv("PDB_SPMV_VERSION");
  // Default: v5 (measured fastest on config 2: 117 us vs v2 127, v3 150, the
  // pipelined v4 176; L2 bulk prefetch made v5 slower), see DESIGN.md §3.
  const int want = e ? atoi(e) : 5;
  if (blk_start && blk_base && nblk > 0 && want == 7 && per == -kV5Per) {
    // v7 reuses the v5 item partition; `entries` carries the stage count and
    // `blocks` the persistent grid
    p.version = 7;
    p.entries = v7_stages();
    p.blk_start = blk_start;
    p.blk_base = blk_base;
    p.nblk = nblk;
    p.blocks = p.entries == 2 ? v7_grid<2>(nblk) : p.entries == 4 ? v7_grid<4>(nblk) : v7_grid<3>(nblk);
    return p;
  }
  if (blk_start && blk_base && nblk > 0 && (want == 5 || want == 6) && per < 0) {
    p.version = want;
    p.entries = -per;
    p.blk_start = blk_start;
    p.blk_base = blk_base;
    p.nblk = nblk;  // warps
    p.blocks = (nblk + kV5Warps - 1) / kV5Warps;
    return p;
  }
  if (blk_start && blk_base && nblk > 0 && (want == 3 || want == 4) && per > 0) {
    p.version = want;
    p.blk_start = blk_start;
    p.blk_base = blk_base;
    p.nblk = nblk;
    p.blocks = nblk;
    p.entries = per;
    if (want == 4) {
      int dev = 0, sms = 148, per_sm = 2;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, residual_v4_kernel, kV4Threads, 0);
      if (per_sm < 1) per_sm = 1;
      p.blocks = nblk < sms * per_sm ? nblk : sms * per_sm;  // persistent grid: one wave
    }
  }
  return p;
}

SpmvPlan spmv_plan(int64_t n, int64_t nnz) {
  SpmvPlan p;
  const double avg = n > 0 ? (double)nnz / (double)n : 1.0;
  // ~one 4-deep unrolled pass per row: G ~ avg/8 (power of two, 2..32)
  int g = 2;
  while (g < 32 && g * 8 < avg) g *= 2;
  p.group = g;
  p.version = 2;
  p.entries = 4;
  // v2: G*E ~ the typical row length (config 2, avg 36: G=4,E=8 measured best;
  // config 3, avg 61: G=8,E=8)
  if (avg <= 16) p.group = 2, p.entries = 8;
  else if (avg <= 48) p.group = 4, p.entries = 8;
  else p.group = 8, p.entries = 8;
  if (const char* e = getenv("PDB_SPMV_VERSION")) p.version = atoi(e) == 1 ? 1 : 2;
  if (p.version == 1) p.group = g;
  if (const char* e = getenv("PDB_SPMV_GROUP")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32) p.group = v;
  }
  if (const char* e = getenv("PDB_SPMV_ENTRIES")) {
    const int v = atoi(e);
    if (v == 2 || v == 4 || v == 8 || v == 5 || v == 9) p.entries = v;  // 5/9: E=4/8 with L1-bypass hints
  }
  p.rows_per_block = kBlock / p.group;
  p.blocks = (int)((n + p.rows_per_block - 1) / p.rows_per_block);
  return p;
}

template <int G>
static void launch_residual(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                            const double* x, const double* b, double* r, double* sumsq, bool negate,
                            cudaStream_t s) {
  if (p.version == 1) {
    residual_kernel<G><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate);
    return;
  }
  switch (p.entries) {
    case 2: residual_v2_kernel<G, 2><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate); break;
    case 8: residual_v2_kernel<G, 8><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate); break;
    case 9: residual_v2_kernel<G, 8, 1><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate); break;
    case 5: residual_v2_kernel<G, 4, 1><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate); break;
    default: residual_v2_kernel<G, 4><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate); break;
  }
}

int v7_stages() {
  const char* e = getenv("PDB_SPMV_STAGES");
  const int v = e ? atoi(e) : 3;
  return v == 2 || v == 4 ? v : 3;
}

size_t v7_smem(int stages) {
  return 128 * ((kV5Warps * stages * 8 + 127) / 128) + (size_t)kV5Warps * stages * kV7StageBytes;
}

template <int S>
int v7_grid(int nitems) {
  static int per_sm[5] = {0, 0, 0, 0, 0};
  if (!per_sm[S]) {
    const size_t smem = v7_smem(S);
    cudaFuncSetAttribute(residual_v7_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, residual_v7_kernel<S>, kV5Warps * 32, smem);
    per_sm[S] = occ > 0 ? occ : 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int need = (nitems + kV5Warps - 1) / kV5Warps;
  return need < sms * per_sm[S] ? need : sms * per_sm[S];
}

template <int S>
static void launch_v7_s(const SpmvPlan& p, const int64_t* rp, const int32_t* col, const double* val, const double* x,
                        const double* b, double* r, double* sumsq, bool negate, cudaStream_t s) {
  residual_v7_kernel<S><<<p.blocks, kV5Warps * 32, v7_smem(S), s>>>(p.nblk, rp, col, val, x, b, r, p.blk_start,
                                                                    p.blk_base, sumsq, negate);
}

static void launch_v7(const SpmvPlan& p, const int64_t* rp, const int32_t* col, const double* val, const double* x,
                      const double* b, double* r, double* sumsq, bool negate, cudaStream_t s) {
  if (p.entries == 2)
    launch_v7_s<2>(p, rp, col, val, x, b, r, sumsq, negate, s);
  else if (p.entries == 4)
    launch_v7_s<4>(p, rp, col, val, x, b, r, sumsq, negate, s);
  else
    launch_v7_s<3>(p, rp, col, val, x, b, r, sumsq, negate, s);
}

template <bool CHUNK>
static void launch_v5(const SpmvPlan& p, const int64_t* rp, const int32_t* col, const double* val, const double* x,
                      const double* b, double* r, double* sumsq, bool negate, int pf, cudaStream_t s) {
  const unsigned th = kV5Warps * 32;
  if (p.entries == 16)
    residual_v5_kernel<16, CHUNK><<<p.blocks, th, 0, s>>>(p.nblk, rp, col, val, x, b, r, p.blk_start, p.blk_base,
                                                          sumsq, negate, pf);
  else if (p.entries == 4)
    residual_v5_kernel<4, CHUNK><<<p.blocks, th, 0, s>>>(p.nblk, rp, col, val, x, b, r, p.blk_start, p.blk_base,
                                                         sumsq, negate, pf);
  else
    residual_v5_kernel<8, CHUNK><<<p.blocks, th, 0, s>>>(p.nblk, rp, col, val, x, b, r, p.blk_start, p.blk_base,
                                                         sumsq, negate, pf);
}

static void dispatch_residual(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                              const double* x, const double* b, double* r, double* sumsq, bool negate,
                              cudaStream_t s) {
  if (n <= 0) return;
  if (p.version == 9 && p.sell_off) {
    const unsigned g = (unsigned)p.blocks;
    const int2* sr = reinterpret_cast<const int2*>(p.sell_row);
    // L2 bulk prefetch one step group ahead (measured: pf 1 best, 90.5 us vs
    // 96.7 without on config 2; 263 vs 301 us on config 3)
    const char* pfe = getenv("PDB_SELL_PF");
    const int pf = pfe ? atoi(pfe) : 1;
    const char* mbe = getenv("PDB_SELL_MINB");
    const int minb = mbe ? atoi(mbe) : 0;
#define PDB_SELL(U, M)                                                                                             \
  launch_pdl(residual_sell_kernel<U, M>, dim3(g), dim3(256), 0, s, p.nslices, p.sell_off, sr, p.sell_val, p.sell_col, \
             x, b, r, sumsq, negate, pf)
    if (p.entries == 2) PDB_SELL(2, 1);
    else if (p.entries == 4) PDB_SELL(4, 1);
    else if (p.entries == 16) PDB_SELL(16, 1);
    else if (minb == 5) PDB_SELL(8, 5);
    else if (minb == 6) PDB_SELL(8, 6);
    else PDB_SELL(8, 1);
#undef PDB_SELL
    return;
  }
  if (p.version == 8 && p.blk_start && p.lcol) {
    const size_t smem = (size_t)p.win_max * sizeof(double);
    const char* mb = getenv("PDB_V8_MINB");
    const bool capped = mb && atoi(mb) == 5;
    static size_t opted[2] = {48 * 1024, 48 * 1024};
    if (smem > opted[capped]) {
      if (capped)
        cudaFuncSetAttribute(residual_v8_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      else
        cudaFuncSetAttribute(residual_v8_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      opted[capped] = smem;
    }
    if (capped)
      residual_v8_kernel<5><<<p.blocks, kV5Warps * 32, smem, s>>>(p.nblk, rp, col, val, p.lcol, p.win_ptr,
                                                                  reinterpret_cast<const int2*>(p.win_runs), x, b, r,
                                                                  p.blk_start, p.blk_base, sumsq, negate);
    else
      residual_v8_kernel<1><<<p.blocks, kV5Warps * 32, smem, s>>>(p.nblk, rp, col, val, p.lcol, p.win_ptr,
                                                                  reinterpret_cast<const int2*>(p.win_runs), x, b, r,
                                                                  p.blk_start, p.blk_base, sumsq, negate);
    return;
  }
  if (p.version == 7 && p.blk_start) {
    launch_v7(p, rp, col, val, x, b, r, sumsq, negate, s);
    return;
  }
  if ((p.version == 5 || p.version == 6) && p.blk_start) {
    // prefetch distance in warps (PDB_SPMV_PREFETCH; 0 disables)
    const char* pfe = getenv("PDB_SPMV_PREFETCH");
    const int pf = pfe ? atoi(pfe) : 0;
    if (p.version == 6)
      launch_v5<true>(p, rp, col, val, x, b, r, sumsq, negate, pf, s);
    else
      launch_v5<false>(p, rp, col, val, x, b, r, sumsq, negate, pf, s);
    return;
  }
  if (p.version == 4 && p.blk_start) {
    residual_v4_kernel<<<p.blocks, kV4Threads, 0, s>>>(p.nblk, rp, col, val, x, b, r, p.blk_start, p.blk_base, sumsq,
                                                       negate);
    return;
  }
  if (p.version == 3 && p.blk_start) {
    if (p.entries == 16)
      residual_v3_kernel<16><<<p.blocks, kStreamThreads, 0, s>>>(n, rp, col, val, x, b, r, p.blk_start, p.blk_base,
                                                                 sumsq, negate);
    else
      residual_v3_kernel<8><<<p.blocks, kStreamThreads, 0, s>>>(n, rp, col, val, x, b, r, p.blk_start, p.blk_base,
                                                                sumsq, negate);
    return;
  }
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

void residual_slices(const SpmvPlan& p, int64_t s0, int64_t s1, const double* x, const double* b, double* r,
                     cudaStream_t s) {
  if (s1 <= s0 || p.version != 9) return;
  const int2* sr = reinterpret_cast<const int2*>(p.sell_row) + s0 * 32;
  const unsigned g = (unsigned)((s1 - s0 + 7) / 8);
  residual_sell_kernel<8, 1><<<g, 256, 0, s>>>(s1 - s0, p.sell_off + s0, sr, p.sell_val, p.sell_col, x, b, r, nullptr,
                                               true, 1);
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

void patch_apply_inv(int64_t np, int ps, const int32_t* patches, const double* Binv, const int32_t* phi,
                     const double* r, const double* in_scale, double* sols, cudaStream_t s) {
  if (np <= 0) return;
  const int ppb = ps >= 256 ? 1 : 256 / ps;
  const int threads = ppb * ps;
  const unsigned blocks = (unsigned)((np + ppb - 1) / ppb);
  patch_apply_inv_kernel<<<blocks, threads, (size_t)ppb * ps * sizeof(double), s>>>(np, ps, ppb, patches, Binv, phi,
                                                                                     r, in_scale, sols);
}

int grouped_tile(int ps) {
  const int ng = ps >= 256 ? 1 : 256 / ps;
  return 4 * ng < 32 ? 4 * ng : 32;
}

void patch_apply_grouped(int ntiles, int ps, const int32_t* tile_entry, const int32_t* tile_start,
                         const int32_t* tile_idx, const int32_t* order, const double* Binv, const double* r,
                         const double* in_scale, double* sols, int max_tile, cudaStream_t s) {
  if (ntiles <= 0) return;
  const size_t smem = ((size_t)ps * ps + (size_t)max_tile * ps) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(patch_apply_grouped_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = ps >= 256 ? ps : (256 / ps) * ps;
  patch_apply_grouped_kernel<<<(unsigned)ntiles, threads, smem, s>>>(ps, tile_entry, tile_start, tile_idx, order,
                                                                     Binv, r, in_scale, sols);
}

bool dmma_apply_supported(int ps) { return ps >= 1 && ps <= 256; }

int apply_tile(int ps) { return dmma_apply_supported(ps) ? kDmmaTile : grouped_tile(ps); }

int64_t frag_len(int ps) { return (int64_t)((ps + 7) / 8) * ((ps + 3) / 4) * 32; }

void build_frag_inverses(int64_t nf, int ps, const double* inv_cm, double* frag, cudaStream_t s) {
  const int64_t total = nf * frag_len(ps);
  if (total > 0)
    build_frag_kernel<<<grid_for(total, kBlock), kBlock, 0, s>>>(total, ps, (ps + 7) / 8, (ps + 3) / 4, inv_cm, frag);
}

template <bool Z>
static void launch_dmma(int ntiles, int ps, int64_t n, const int32_t* tile_entry, const int32_t* tile_start,
                        const int32_t* idx, const int32_t* order, const double* frag, const double* r, const double* in_scale, double* out,
                        cudaStream_t s) {
  if (ntiles <= 0) return;
  const int mt = (ps + 7) / 8, ks = (ps + 3) / 4;
  if (ps > 32) {  // run-time shapes, inverse streamed from L2
    int kstr = ks * 4;
    if (kstr % 8 == 0) kstr += 4;
    const size_t smem = (size_t)kDmmaTile * kstr * sizeof(double);
    static size_t opted = 48 * 1024;
    if (smem > opted) {
      cudaFuncSetAttribute(patch_apply_dmma_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      opted = smem;
    }
    if (!Z)
      launch_pdl(patch_apply_dmma_large_kernel, dim3((unsigned)ntiles), dim3(mt * 32), smem, s, ps, mt, ks, kstr,
                 tile_entry, tile_start, idx, order, frag, r, in_scale, out);
    return;
  }
#define PDB_DMMA_CASE(M, K)                                                                                    \
  if (mt == M && ks == K) {                                                                                    \
    launch_pdl(patch_apply_dmma_kernel<M, K, Z>, dim3((unsigned)ntiles), dim3(M * 32), 0, s, ps, n, tile_entry, \
               tile_start, idx, order, frag, r, in_scale, out);                                               \
    return;                                                                                                    \
  }
  PDB_DMMA_CASE(1, 1)
  PDB_DMMA_CASE(1, 2)
  PDB_DMMA_CASE(2, 3)
  PDB_DMMA_CASE(2, 4)
  PDB_DMMA_CASE(3, 5)
  PDB_DMMA_CASE(3, 6)
  PDB_DMMA_CASE(4, 7)
  PDB_DMMA_CASE(4, 8)
#undef PDB_DMMA_CASE
}

void patch_apply_dmma(int ntiles, int ps, const int32_t* tile_entry, const int32_t* tile_start,
                      const int32_t* tile_idx, const int32_t* order, const double* frag, const double* r,
                      const double* in_scale, double* sols, cudaStream_t s) {
  launch_dmma<false>(ntiles, ps, 0, tile_entry, tile_start, tile_idx, order, frag, r, in_scale, sols, s);
}

void patch_apply_dmma_z(int ntiles, int ps, int64_t n, const int32_t* tile_entry, const int32_t* tile_start,
                        const int32_t* zfwd, const double* frag, const double* r, const double* in_scale, double* Z,
                        cudaStream_t s) {
  launch_dmma<true>(ntiles, ps, n, tile_entry, tile_start, zfwd, nullptr, frag, r, in_scale, Z, s);
}

void build_zmap(int64_t n, int ps, const int32_t* inv_ptr, const int32_t* inv, const int32_t* slot_of, int32_t* zfwd,
                uint8_t* zcnt, cudaStream_t s) {
  if (n > 0) build_zmap_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, ps, inv_ptr, inv, slot_of, zfwd, zcnt);
}

void scatter_z(int64_t n, int maxc, const uint8_t* zcnt, const double* Z, double omega, bool sym, const double* x_in,
               double* z_out, double* x_out, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned g = grid_for(n, kBlock);
  switch (maxc) {
    case 1: scatter_z_kernel<1><<<g, kBlock, 0, s>>>(n, zcnt, Z, omega, sym, x_in, z_out, x_out); break;
    case 2: scatter_z_kernel<2><<<g, kBlock, 0, s>>>(n, zcnt, Z, omega, sym, x_in, z_out, x_out); break;
    case 3:
    case 4: scatter_z_kernel<4><<<g, kBlock, 0, s>>>(n, zcnt, Z, omega, sym, x_in, z_out, x_out); break;
    default: scatter_z_kernel<8><<<g, kBlock, 0, s>>>(n, zcnt, Z, omega, sym, x_in, z_out, x_out); break;
  }
}

void shard_scatter(int64_t count, const int32_t* list, const int32_t* inv_ptr, const int32_t* inv, const double* sols,
                   const double* init, const double* omega_w, double* z_out, double* x, cudaStream_t s) {
  if (count > 0)
    shard_scatter_kernel<<<grid_for(count, kBlock), kBlock, 0, s>>>(count, list, inv_ptr, inv, sols, init, omega_w,
                                                                    z_out, x);
}

void gather_vals(int64_t count, const int32_t* idx, const double* src, double* dst, cudaStream_t s) {
  if (count > 0) gather_vals_kernel<<<grid_for(count, kBlock), kBlock, 0, s>>>(count, idx, src, dst);
}

void scatter_vals(int64_t count, const int32_t* idx, const double* src, double* dst, cudaStream_t s) {
  if (count > 0) scatter_vals_kernel<<<grid_for(count, kBlock), kBlock, 0, s>>>(count, idx, src, dst);
}

void remap_inverse(int64_t count, int ps, const int32_t* slot_of, int32_t* inv, cudaStream_t s) {
  if (count > 0) remap_inverse_kernel<<<grid_for(count, kBlock), kBlock, 0, s>>>(count, ps, slot_of, inv);
}

void build_inverse_pad(int64_t n, int maxc, const int32_t* inv_ptr, const int32_t* inv, int32_t* pad,
                       cudaStream_t s) {
  if (n > 0) build_inverse_pad_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, maxc, inv_ptr, inv, pad);
}

void scatter_update_pad(int64_t n, int maxc, const int32_t* inv_pad, const double* sols, double omega, bool sym,
                        const double* x_in, double* z_out, double* x_out, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned g = grid_for(n, kBlock * kScatterU);
  switch (maxc) {
    case 1: launch_pdl(scatter_update_pad_kernel<1>, dim3(g), dim3(kBlock), 0, s, n, inv_pad, sols, omega, sym, x_in, z_out, x_out); break;
    case 2: launch_pdl(scatter_update_pad_kernel<2>, dim3(g), dim3(kBlock), 0, s, n, inv_pad, sols, omega, sym, x_in, z_out, x_out); break;
    case 3:
    case 4: launch_pdl(scatter_update_pad_kernel<4>, dim3(g), dim3(kBlock), 0, s, n, inv_pad, sols, omega, sym, x_in, z_out, x_out); break;
    default: launch_pdl(scatter_update_pad_kernel<8>, dim3(g), dim3(kBlock), 0, s, n, inv_pad, sols, omega, sym, x_in, z_out, x_out); break;
  }
}

void invert_factors(int64_t nf, int ps, const double* lu, const int32_t* piv, double* inv, cudaStream_t s) {
  if (nf > 0) invert_factors_kernel<<<(unsigned)((nf + 3) / 4), 128, 0, s>>>(nf, ps, lu, piv, inv);
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
