// Residual r = b - A x and SpMV y = A x (reference spmv sparse.cpp:50-63,
// the residual of smooth precond.cpp:95-97).
//
// Three kernels, chosen by plan_of (matrix.cpp):
//   residual_sell_kernel (default)  the SELL-C-sigma copy built at upload:
//       warp per 32-row slice, lane per row, coalesced column-major steps,
//       each row summed in CSR order with unfused multiply/add -> bitwise the
//       reference's residual;
//   residual_v5_kernel              CSR warp items (<= 31 rows / 256 nonzeros),
//       coalesced item loads, products reduced per row through shared memory
//       (PDB_SPMV_VERSION=5, or when no SELL copy exists);
//   residual_v2_kernel              G lanes per row, for plans without a row
//       partition (PDB_SPMV_VERSION=2).
// With block_sumsq the kernels also write one sum of r^2 per block (residual
// histories, finished by finish_sum in a fixed order: deterministic).
#include "../kernels.hpp"
#include "pdl.cuh"

namespace pdb::k {

namespace {

constexpr int kBlock = 256;

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// -- v2: G lanes per row, E entries per lane loaded before use -------------
template <int G, int E>
__global__ void __launch_bounds__(kBlock) residual_v2_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                             const int32_t* __restrict__ col,
                                                             const double* __restrict__ val,
                                                             const double* __restrict__ x,
                                                             const double* __restrict__ b, double* __restrict__ r,
                                                             double* __restrict__ block_sumsq, bool negate_b_absent,
                                                             const double* __restrict__ dotv) {
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
        c[e] = p < hi ? __ldcs(col + p) : -1;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int64_t p = base + lane + e * G;
        v[e] = p < hi ? __ldcs(val + p) : 0.0;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) acc += c[e] >= 0 ? v[e] * __ldg(x + c[e]) : 0.0;
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
    double sq = (lane == 0 && row < n) ? rv * (dotv ? dotv[row] : rv) : 0.0;
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

// -- v5: warp items ---------------------------------------------------------
// A precomputed partition gives every warp a run of <= 31 consecutive rows
// holding <= 256 nonzeros.  The warp loads that contiguous span with fully
// coalesced 32-lane loads, gathers x, stages the products in a per-warp
// shared-memory slice (no block barrier), then 4-lane groups reduce the rows.
// A row longer than 256 nonzeros gets a warp to itself and loops.
constexpr int kV5Warps = 8;
constexpr int kV5Per = 8;
constexpr int kV5Rows = 31;

__global__ void __launch_bounds__(kV5Warps * 32) residual_v5_kernel(
    int nwarps, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r,
    const int32_t* __restrict__ wstart, const int64_t* __restrict__ wbase, double* __restrict__ block_sumsq,
    bool negate_b_absent, const double* __restrict__ dotv) {
  constexpr int PER = kV5Per;
  __shared__ double prod[kV5Warps][32 * PER];
  __shared__ double red[kV5Warps];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * kV5Warps + wib;
  double sq = 0.0;
  if (w < nwarps) {
    const int64_t r0 = __ldg(wstart + w), base = __ldg(wbase + w), end = __ldg(wbase + w + 1);
    const int nrows = __ldg(wstart + w + 1) - (int)r0;
    const int nnz = (int)(end - base);
    const int64_t rpl = lane <= nrows ? __ldg(rp + r0 + lane) : end;
    const double bl = (b && lane < nrows) ? __ldcs(b + r0 + lane) : 0.0;
    if (nnz <= 32 * PER) {
      int32_t c[PER];
      double v[PER];
      const int32_t* cp = col + base + lane;
      const double* vp = val + base + lane;
#pragma unroll
      for (int e = 0; e < PER; ++e) c[e] = e * 32 + lane < nnz ? __ldcs(cp + e * 32) : 0;
#pragma unroll
      for (int e = 0; e < PER; ++e) v[e] = e * 32 + lane < nnz ? __ldcs(vp + e * 32) : 0.0;
      double* pw = prod[wib];
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
          sq += rv * (dotv ? dotv[r0 + rr] : rv);
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
        sq += rv * (dotv ? dotv[r0] : rv);
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

// -- SELL-C-sigma (default) -------------------------------------------------
// Warp per slice of 32 rows, lane l owns slice row l.  Step j loads entry j
// of all 32 rows -- one 256-byte value span and one 128-byte column span,
// fully coalesced -- and the x gathers of 32 similar rows hit a few lines.  U
// steps are loaded before any is consumed (the first group before the
// programmatic-launch wait: matrix bytes do not depend on the predecessor),
// an L2 bulk prefetch runs pf step groups ahead, lanes past their row's end
// are predicated off, and each lane accumulates its row in CSR order with
// unfused multiply/add: r = b - s bit for bit as the reference spmv + smooth
// (sparse.cpp:50-63, precond.cpp:95-97).  The explicit minimum of 1 block
// per SM lets ptxas keep the next step group's loads in flight (72 registers
// at U = 8; without it the allocation drops to 48 and the kernel loses ~4 %).
// CLS: every row of the matrix is in a column-pattern class (build_sell):
// srow.y = length | (class + 1) << 16 and the columns of a row are
// row + tab[tstart[class] + j] -- no column stream (8 instead of 12 bytes per
// nonzero); same per-row summation order, so still bitwise.
template <int U, bool CLS = false>
__global__ void __launch_bounds__(256, 1) residual_sell_kernel(int64_t nslices, const int64_t* __restrict__ soff,
                                                            const int2* __restrict__ srow,
                                                            const double* __restrict__ sval,
                                                            const int32_t* __restrict__ scol,
                                                            const double* __restrict__ x, const double* __restrict__ b,
                                                            double* __restrict__ r, double* __restrict__ block_sumsq,
                                                            bool negate_b_absent, int pf,
                                                            const double* __restrict__ dotv,
                                                            const int32_t* __restrict__ tab = nullptr,
                                                            const int32_t* __restrict__ tstart = nullptr) {
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
    const int len = CLS ? (rl.y & 0xFFFF) : rl.y;
    const int L = __reduce_max_sync(0xffffffffu, (unsigned)len);
    const int64_t o = __ldg(soff + sl);
    const double* vp = sval + o + lane;
    const int32_t* cp = CLS ? tab + (rl.x >= 0 ? __ldg(tstart + (rl.y >> 16) - 1) : 0) : scol + o + lane;
    const double bl = (rl.x >= 0 && b) ? __ldcs(b + rl.x) : 0.0;
    double acc = 0.0;
    int32_t c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = u < len ? (CLS ? rl.x + __ldg(cp + u) : __ldcs(cp + (int64_t)u * 32)) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = u < len ? __ldcs(vp + (int64_t)u * 32) : 0.0;
    grid_dep_wait();  // x is the predecessor's (the scatter's) output
    grid_dep_trigger();
    for (int j = 0; j < L; j += U) {
      if (pf > 0 && lane == 0) {
        const int jn = j + pf * U;
        if (jn < L) {
          const int cnt = (L - jn < U ? L - jn : U) * 32;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sval + o + (int64_t)jn * 32),
                       "r"((unsigned)(cnt * 8)));
          if (!CLS)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(scol + o + (int64_t)jn * 32),
                         "r"((unsigned)(cnt * 4)));
        }
      }
      if (j > 0) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          c[u] = j + u < len ? (CLS ? rl.x + __ldg(cp + j + u) : __ldcs(cp + (int64_t)(j + u) * 32)) : 0;
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
      sq += rv * (dotv ? dotv[rl.x] : rv);
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

// -- half ("mirror") storage (sell_mirror.cpp) -------------------------------
// Same warp-per-slice, lane-per-row scheme and the same per-row CSR-order
// summation as residual_sell_kernel over the half-storage layout.  The class
// tables (column offsets, and per lower entry 32 * the slot of the mirrored
// value in the target row's storage) sit in shared memory.  Lower entries
// first (CSR order): the target row j = i + offset gives both x[j] and
// rbase[j] (same gather index), the value is sval[rbase[j] + kslot] -- a_ji,
// stored once in row j, an L2 hit when j's warp streamed it shortly before.
// Then the row's own upper entries stream from its slice block (slot t at
// soff + 32 t + lane), prefetched into L2 in one bulk request at the start.
// Bitwise the CSR residual.
__device__ __forceinline__ double ld_na(const double* p) {  // no L1 allocation
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int U>
__global__ void __launch_bounds__(256, 1) residual_mirror_kernel(
    int64_t nslices, const int64_t* __restrict__ soff, const int2* __restrict__ srow,
    const double* __restrict__ sval, const int32_t* __restrict__ tab, const int32_t* __restrict__ kslot,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ clo, int ntab, int ncls,
    const int32_t* __restrict__ rbase, const double* __restrict__ x, const double* __restrict__ b,
    double* __restrict__ r, double* __restrict__ block_sumsq, bool negate_b_absent, int pf,
    const double* __restrict__ dotv, int64_t ahead, int64_t nval) {
  extern __shared__ int32_t mirror_tab[];  // int2 {offset, 32 slot} [ntab], lower counts [ncls], starts [ncls + 1]
  __shared__ double red[8];
  int2* s_k = reinterpret_cast<int2*>(mirror_tab);
  int32_t* s_lo = mirror_tab + 2 * ntab;
  int32_t* s_ts = s_lo + ncls;
  for (int q = threadIdx.x; q < ntab; q += blockDim.x) s_k[q] = make_int2(__ldg(tab + q), __ldg(kslot + q));
  for (int q = threadIdx.x; q < ncls; q += blockDim.x) s_lo[q] = __ldg(clo + q);
  for (int q = threadIdx.x; q <= ncls; q += blockDim.x) s_ts[q] = __ldg(tstart + q);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t sl = (int64_t)blockIdx.x * 8 + wib;
  double sq = 0.0;
  if (sl >= nslices) {
    grid_dep_wait();
    grid_dep_trigger();
  }
  if (sl < nslices) {
    const int2 rl = __ldg(srow + sl * 32 + lane);
    const bool live = rl.x >= 0;
    const int len = live ? (rl.y & 0xFFFF) : 0;
    const int c = live ? (rl.y >> 16) - 1 : 0;
    const int lo = live ? s_lo[c] : 0;
    const int own = len - lo;
    const int M = (int)__reduce_max_sync(0xffffffffu, (unsigned)lo);
    const int W = (int)__reduce_max_sync(0xffffffffu, (unsigned)own);
    const int64_t o = __ldg(soff + sl);
    // L2 prefetch: this slice's own block, and the block of slice sl + ahead
    // (beyond the slices in flight) so that rows read as mirror targets
    // later are L2-resident before their readers run
    if (pf > 0 && lane == 0) {
      if (W > 0 && sl < ahead)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sval + o), "r"((unsigned)W * 256u));
      if (ahead > 0 && sl + ahead < nslices) {
        const int64_t oa = __ldg(soff + sl + ahead);
        const int64_t ob = sl + ahead + 1 < nslices ? __ldg(soff + sl + ahead + 1) : nval;
        if (ob > oa) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sval + oa), "r"((unsigned)((ob - oa) * 8)));
      }
    }
    const int2* kp = s_k + (live ? s_ts[c] : 0);
    const int row = live ? rl.x : 0;
    const int Mmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)(live ? lo : 0));
    const double* vo = sval + o + lane;
    const double bl = (live && b) ? __ldcs(b + rl.x) : 0.0;
    // full step groups for the lanes' common counts (no predicates: a
    // uniform slice runs only these), predicated single steps after
    const int Wmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)(live ? own : 0));
    grid_dep_wait();  // x is the predecessor's (the scatter's) output
    grid_dep_trigger();
    double acc = 0.0;
    // lower entries, CSR order: the target row j = i + offset gives x[j]
    // and rbase[j] (same gather index); the value is sval[rbase[j] + kslot]
    int m = 0;
    for (; m + U <= Mmin; m += U) {
      int j[U], ks[U], rb[U];
      double xv[U], v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int2 k = kp[m + u];
        j[u] = row + k.x;
        ks[u] = k.y;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        rb[u] = __ldg(rbase + j[u]);
        xv[u] = __ldg(x + j[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_na(sval + (rb[u] + ks[u]));
#pragma unroll
      for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    for (; m < M; m += U) {  // remainder: predicated (inactive steps add +0 * +0, acc unchanged)
      int j[U], ks[U], rb[U];
      double xv[U], v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int2 k = m + u < lo ? kp[m + u] : make_int2(0, 0);
        j[u] = row + k.x;
        ks[u] = k.y;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        rb[u] = m + u < lo ? __ldg(rbase + j[u]) : 0;
        xv[u] = m + u < lo ? __ldg(x + j[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = m + u < lo ? ld_na(sval + (rb[u] + ks[u])) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    const int2* ku = kp + lo;
    int t = 0;
    for (; t + U <= Wmin; t += U) {
      double xv[U], v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = ld_na(vo + 32 * (t + u));
        xv[u] = __ldg(x + (row + ku[t + u].x));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    for (; t < W; t += U) {
      double xv[U], v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = t + u < own ? ld_na(vo + 32 * (t + u)) : 0.0;
        xv[u] = t + u < own ? __ldg(x + (row + ku[t + u].x)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    if (live) {
      const double rv = b ? __dsub_rn(bl, acc) : (negate_b_absent ? -acc : acc);
      r[rl.x] = rv;
      sq += rv * (dotv ? dotv[rl.x] : rv);
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

inline size_t mirror_smem(int ntab, int ncls) { return (size_t)(2 * ntab + 2 * ncls + 1) * sizeof(int32_t); }

// opt the mirror kernels into dynamic shared memory above 48 KB when the
// class tables need it (once per device and instance)
template <class K>
void mirror_smem_attr(K kern, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  struct Done {
    const void* f;
    int dev;
    size_t bytes;
  };
  static thread_local Done done[16];
  static thread_local int ndone = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* f = reinterpret_cast<const void*>(kern);
  for (int i = 0; i < ndone; ++i)
    if (done[i].f == f && done[i].dev == dev) {
      if (done[i].bytes >= bytes) return;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      done[i].bytes = bytes;
      return;
    }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (ndone < 16) done[ndone++] = {f, dev, bytes};
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

template <int G>
void launch_v2(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x,
               const double* b, double* r, double* sumsq, bool negate, const double* dotv, cudaStream_t s) {
  if (p.entries == 4)
    residual_v2_kernel<G, 4><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate, dotv);
  else
    residual_v2_kernel<G, 8><<<p.blocks, kBlock, 0, s>>>(n, rp, col, val, x, b, r, sumsq, negate, dotv);
}

// The residual gathers x through L1; it asks for the largest L1 carve-out so
// that its blocks never run under the shared-memory-heavy split a preceding
// kernel left on an SM (with programmatic dependent launch the SMs are never
// idle between kernels, so the split of the 192-DoF tile apply -- 197 KB of
// shared memory -- otherwise sticks: config-5 sweep 1.68 vs 1.51 ms).
// PDB_RES_CARVEOUT=<percent> overrides the hint, -1 leaves the default.
template <typename K>
void prefer_l1(K kern) {
  static const int carve = [] {
    const char* e = getenv("PDB_RES_CARVEOUT");
    return e ? atoi(e) : 0;
  }();
  static bool done[64] = {};
  int dev = 0;
  PDB_CUDA(cudaGetDevice(&dev));
  if (carve < 0 || dev >= 64 || done[dev]) return;
  PDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  done[dev] = true;
}

void dispatch_residual(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                       const double* x, const double* b, double* r, double* sumsq, bool negate, cudaStream_t s,
                       const double* dotv = nullptr) {
  if (n <= 0) return;
  if (p.version == 9 && p.sell_off) {
    const int2* sr = reinterpret_cast<const int2*>(p.sell_row);
    // L2 bulk prefetch one step group ahead (PDB_SELL_PF; measured best at 1)
    const char* pfe = getenv("PDB_SELL_PF");
    const int pf = pfe ? atoi(pfe) : 1;
    if (p.mir_rbase) {
      // PDB_MIRROR_U (A/B): steps in flight per lane, 4 (default: 4 blocks
      // per SM at 64 registers, measured best) or 8
      const char* ue = getenv("PDB_MIRROR_U");
      auto kern = ue && atoi(ue) == 8 ? residual_mirror_kernel<8> : residual_mirror_kernel<4>;
      const size_t sm = mirror_smem(p.mir_ntab, p.mir_ncls);
      mirror_smem_attr(kern, sm);
      // PDB_MIRROR_AHEAD: slices between a warp's slice and the one whose
      // block it prefetches (0: only its own block)
      const char* ae = getenv("PDB_MIRROR_AHEAD");
      const int64_t ahead = ae ? atoll(ae) : 2048;
      launch_pdl(kern, dim3((unsigned)p.blocks), dim3(256), sm, s, p.nslices, p.sell_off, sr, p.sell_val, p.sell_tab,
                 p.mir_kslot, p.sell_tstart, p.mir_clo, p.mir_ntab, p.mir_ncls, p.mir_rbase, x, b, r, sumsq, negate, pf,
                 dotv, ahead, p.mir_nval);
      return;
    }
    if (p.sell_tab) {
      const char* ue = getenv("PDB_SELL_CLS_U");
      if (ue && atoi(ue) == 16) {
        prefer_l1(residual_sell_kernel<16, true>);
        launch_pdl(residual_sell_kernel<16, true>, dim3((unsigned)p.blocks), dim3(256), 0, s, p.nslices, p.sell_off,
                   sr, p.sell_val, p.sell_col, x, b, r, sumsq, negate, pf, dotv, p.sell_tab, p.sell_tstart);
      } else {
        prefer_l1(residual_sell_kernel<8, true>);
        launch_pdl(residual_sell_kernel<8, true>, dim3((unsigned)p.blocks), dim3(256), 0, s, p.nslices, p.sell_off,
                   sr, p.sell_val, p.sell_col, x, b, r, sumsq, negate, pf, dotv, p.sell_tab, p.sell_tstart);
      }
    } else if (p.entries == 4) {
      prefer_l1(residual_sell_kernel<4>);
      launch_pdl(residual_sell_kernel<4>, dim3((unsigned)p.blocks), dim3(256), 0, s, p.nslices, p.sell_off, sr,
                 p.sell_val, p.sell_col, x, b, r, sumsq, negate, pf, dotv, nullptr, nullptr);
    } else {
      prefer_l1(residual_sell_kernel<8>);
      launch_pdl(residual_sell_kernel<8>, dim3((unsigned)p.blocks), dim3(256), 0, s, p.nslices, p.sell_off, sr,
                 p.sell_val, p.sell_col, x, b, r, sumsq, negate, pf, dotv, nullptr, nullptr);
    }
    return;
  }
  if (p.version == 5 && p.blk_start) {
    residual_v5_kernel<<<p.blocks, kV5Warps * 32, 0, s>>>(p.nblk, rp, col, val, x, b, r, p.blk_start, p.blk_base,
                                                          sumsq, negate, dotv);
    return;
  }
  switch (p.group) {
    case 2: launch_v2<2>(p, n, rp, col, val, x, b, r, sumsq, negate, dotv, s); break;
    case 4: launch_v2<4>(p, n, rp, col, val, x, b, r, sumsq, negate, dotv, s); break;
    case 8: launch_v2<8>(p, n, rp, col, val, x, b, r, sumsq, negate, dotv, s); break;
    case 16: launch_v2<16>(p, n, rp, col, val, x, b, r, sumsq, negate, dotv, s); break;
    default: launch_v2<32>(p, n, rp, col, val, x, b, r, sumsq, negate, dotv, s); break;
  }
}

}  // namespace

std::vector<int32_t> item_partition(int64_t n, const int64_t* rp) {
  // warp items: consecutive rows, <= kV5Rows rows and <= 32*kV5Per nonzeros;
  // a longer row forms an item alone
  const int64_t cap_nnz = 32 * (int64_t)kV5Per;
  std::vector<int32_t> starts;
  starts.push_back(0);
  int64_t row = 0;
  while (row < n) {
    const int64_t b0 = rp[row];
    int64_t end = row + 1;
    while (end < n && end - row < kV5Rows && rp[end + 1] - b0 <= cap_nnz) ++end;
    if (rp[row + 1] - b0 > cap_nnz) end = row + 1;
    starts.push_back((int32_t)end);
    row = end;
  }
  return starts;
}

SpmvPlan spmv_plan(int64_t n, int64_t nnz) {
  SpmvPlan p;
  const double avg = n > 0 ? (double)nnz / (double)n : 1.0;
  // G * E ~ the typical row length (config 2, avg 36: G=4, E=8; config 3, avg 61: G=8, E=8)
  p.version = 2;
  p.entries = 8;
  p.group = avg <= 16 ? 2 : avg <= 48 ? 4 : 8;
  p.rows_per_block = kBlock / p.group;
  p.blocks = (int)((n + p.rows_per_block - 1) / p.rows_per_block);
  return p;
}

SpmvPlan spmv_plan_items(int64_t n, int64_t nnz, const int32_t* item_start, const int64_t* item_base, int nitems) {
  SpmvPlan p = spmv_plan(n, nnz);
  if (!item_start || !item_base || nitems <= 0) return p;
  p.version = 5;
  p.entries = kV5Per;
  p.blk_start = item_start;
  p.blk_base = item_base;
  p.nblk = nitems;
  p.blocks = (nitems + kV5Warps - 1) / kV5Warps;
  return p;
}

void residual(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x,
              const double* b, double* r, double* block_sumsq, cudaStream_t s) {
  dispatch_residual(p, n, rp, col, val, x, b, r, block_sumsq, true, s);
}

void residual_slices(const SpmvPlan& p, int64_t s0, int64_t s1, const double* x, const double* b, double* r,
                     cudaStream_t s) {
  if (s1 <= s0 || p.version != 9) return;
  const int2* sr = reinterpret_cast<const int2*>(p.sell_row) + s0 * 32;
  if (p.mir_rbase) {
    const size_t sm = mirror_smem(p.mir_ntab, p.mir_ncls);
    mirror_smem_attr(residual_mirror_kernel<4>, sm);
    residual_mirror_kernel<4><<<grid_for(s1 - s0, 8), 256, sm, s>>>(
        s1 - s0, p.sell_off + s0, sr, p.sell_val, p.sell_tab, p.mir_kslot, p.sell_tstart, p.mir_clo, p.mir_ntab,
        p.mir_ncls, p.mir_rbase, x, b, r, nullptr, true, 1, nullptr, int64_t{2048}, p.mir_nval);
  } else if (p.sell_tab) {
    prefer_l1(residual_sell_kernel<8, true>);
    residual_sell_kernel<8, true><<<grid_for(s1 - s0, 8), 256, 0, s>>>(
        s1 - s0, p.sell_off + s0, sr, p.sell_val, p.sell_col, x, b, r, nullptr, true, 1, nullptr, p.sell_tab,
        p.sell_tstart);
  } else {
    prefer_l1(residual_sell_kernel<8>);
    residual_sell_kernel<8><<<grid_for(s1 - s0, 8), 256, 0, s>>>(s1 - s0, p.sell_off + s0, sr, p.sell_val, p.sell_col,
                                                                 x, b, r, nullptr, true, 1, nullptr);
  }
}

void spmv(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x,
          double* y, cudaStream_t s) {
  dispatch_residual(p, n, rp, col, val, x, nullptr, y, nullptr, false, s);
}

void finish_sum(const double* partials, int count, double* out, bool sqrt_result, cudaStream_t s) {
  finish_sum_kernel<<<1, 1024, 0, s>>>(partials, count, out, sqrt_result);
}

void spmv_dot(const SpmvPlan& p, int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x,
              double* y, double* partials, cudaStream_t s) {
  dispatch_residual(p, n, rp, col, val, x, nullptr, y, partials, false, s, x);
}

}  // namespace pdb::k
