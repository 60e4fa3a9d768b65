// Bit-exact compression criteria and clustering steps (reference
// compress.cpp / dense.cpp).  Compiled with --fmad=false and written with
// explicit _rn intrinsics: every distance is computed by ONE thread in the
// reference's sequential operation order, so the values -- and therefore
// the greedy and k-means decisions built on strict < comparisons -- are
// bitwise those of the reference.
//
//   l1 distances        entrywise_l1_distance dense.cpp:192-197
//   spectral distance   spectral_distance dense.cpp:154-190 with
//                       lu_solve_into :77-94, lu_solve_transpose_into :102-120,
//                       mat_vec :122-131, mat_tvec :133-142, norm2 :146-150
//   greedy resolution   greedy_impl compress.cpp:40-95 (round-batched, exact)
//   k-means steps       kmeans_loop compress.cpp:150-166 (assignment),
//                       entrywise_mean_indexed dense.cpp:211-223 (update)
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include <math_constants.h>

#include "../common.hpp"
#include "../kernels.hpp"

namespace pdb::k {

namespace {

inline unsigned grid_for(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// ---------------------------------------------------------------- L1 ----
constexpr int kL1Threads = 128;
constexpr int kL1Ent = 4;    // entries per tile (register accumulators)
constexpr int kL1Chunk = 512;  // elements per staged chunk

// d[t*ne + e] for a tile of kL1Ent entries; entries staged chunk-wise in smem,
// each thread streams its own patch matrix once per tile.
__global__ void __launch_bounds__(kL1Threads) l1_pairs_kernel(int64_t npat, const int32_t* __restrict__ pid, int64_t ne,
                                                              int len, const double* __restrict__ mats,
                                                              const int32_t* __restrict__ rep_src,
                                                              const double* __restrict__ reps, double* __restrict__ d) {
  __shared__ double R[kL1Ent][kL1Chunk];
  const int64_t t = (int64_t)blockIdx.x * kL1Threads + threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.y * kL1Ent;
  const bool live = t < npat;
  const double* A = mats + (live ? (int64_t)(pid ? pid[t] : t) : 0) * len;
  double acc[kL1Ent];
#pragma unroll
  for (int c = 0; c < kL1Ent; ++c) acc[c] = 0.0;
  for (int q0 = 0; q0 < len; q0 += kL1Chunk) {
    const int qn = min(kL1Chunk, len - q0);
    __syncthreads();
    for (int c = 0; c < kL1Ent; ++c) {
      const int64_t e = e0 + c;
      if (e >= ne) break;
      const double* Re = rep_src ? mats + (int64_t)rep_src[e] * len : reps + e * len;
      for (int q = threadIdx.x; q < qn; q += kL1Threads) R[c][q] = Re[q0 + q];
    }
    __syncthreads();
    if (live)
      for (int q = 0; q < qn; ++q) {
        const double a = A[q0 + q];
#pragma unroll
        for (int c = 0; c < kL1Ent; ++c) acc[c] = __dadd_rn(acc[c], fabs(__dsub_rn(a, R[c][q])));
      }
  }
  if (live)
    for (int c = 0; c < kL1Ent; ++c)
      if (e0 + c < ne) d[t * ne + e0 + c] = acc[c];
}

// ------------------------------------------------------- tiled L1 ----
// One block = 64 patches x tiles of TE entries (TE = 32, 64 or 128); thread
// (tp, te) keeps the 4 x JB running sums of patches tp + 16 i and entries
// te + (TE / JB) j (i < 4, j < JB) in registers.  The patch tile is staged
// once per entry tile, so its traffic (the patch matrices exceed L2 at
// config 3) falls as 1 / TE.  The patch and entry matrices are staged k-chunk by k-chunk
// (32 entries of each matrix, 8-byte cp.async, double-buffered) into shared
// memory rows of odd stride, so every load of the inner loop is a
// bank-conflict-free broadcast and each staged value feeds 4 (patch) or 8
// (entry) pairs.  Each pair is still summed by one thread in ascending k
// from 0.0 with |a - b| (dense.cpp:192-197), so distances are bitwise the
// sequential kernel's.  Modes: all pair distances, the greedy first-/best-
// match scan (compress.cpp:63-83), the k-means argmin (compress.cpp:154-160).
constexpr int kTP = 64, kTK = 32, kTL = kTK + 1;
template <int TE>
struct L1Tile {
  static constexpr int JB = TE == 32 ? 4 : 8;      // entries per thread
  static constexpr int EL = TE / JB;               // entry lanes
  static constexpr int NT = 16 * EL;               // threads: 16 patch lanes x EL
  static constexpr size_t STAGE = (size_t)(kTP + TE) * kTL;  // doubles per stage
  static constexpr size_t SMEM = 2 * STAGE * sizeof(double);
  static_assert(2 * STAGE >= (size_t)kTP * (TE + 1), "epilogue tile must fit stage memory");
};
enum L1Mode { kL1Pairs = 0, kL1Scan = 1, kL1Argmin = 2 };

struct L1Args {
  int64_t npat;
  const int32_t* pid;  // patch rows (null: 0..npat-1)
  int len;
  const double* mats;
  int64_t e0, e1;         // entries [e0, e1)
  const int32_t* rep_src;  // entry e -> patch id in mats, else reps + e*len
  const double* reps;
  double* d;  // pairs: d[t * (e1 - e0) + (e - e0)]
  double eps;
  int best_match;
  int32_t* phi;  // scan: match (phi[me]); argmin: previous assignment (read)
  double* best_d;
  int32_t* new_phi;
  double* min_dist;
  int32_t* changed;
  // scan, best match: creator id of entry e (default rep_src) and the id of
  // patch row t = pid[t] + id_offset (distributed greedy: global ids)
  const int32_t* creator;
  int64_t id_offset;
  // scan split over entries (few patch tiles, many entries): block y scans
  // entries [e0 + y chunk, e0 + (y+1) chunk) and records its first / best
  // match in part_j / part_d [y][t]; l1_scan_reduce merges the chunks in order
  int64_t chunk;
  int32_t* part_j;
  double* part_d;
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

template <int Mode, int TE>
__global__ void __launch_bounds__(L1Tile<TE>::NT) l1_tile_kernel(L1Args a) {
  constexpr int kTE = TE, JB = L1Tile<TE>::JB, EL = L1Tile<TE>::EL, kTThreads = L1Tile<TE>::NT;
  constexpr size_t kTStage = L1Tile<TE>::STAGE;
  extern __shared__ double sm[];  // 2 stages [kTP + kTE][kTL]; the epilogue tile aliases stage 0
  __shared__ const double* psrc[kTP];
  __shared__ const double* esrc[kTE];
  __shared__ int32_t pme[kTP];
  const int t = threadIdx.x, tp = t / EL, te = t % EL;
  const int64_t p0 = (int64_t)blockIdx.x * kTP;
  const int len = a.len;
  if (t < kTP) {
    const int64_t g = p0 + t;
    const int32_t id = g < a.npat ? (a.pid ? a.pid[g] : (int32_t)g) : -1;
    pme[t] = id;
    psrc[t] = id >= 0 ? a.mats + (int64_t)id * len : nullptr;
  }
  // per-patch state, owned by thread t < kTP
  bool done = true;
  double cur = CUDART_INF;
  int32_t cur_j = -1;
  if (t < kTP && p0 + t < a.npat) {
    done = false;
    if (Mode == kL1Scan) {
      cur = a.eps;
      if (a.best_match) {
        const int32_t me = a.pid[p0 + t];  // phi / best_d are indexed by the row id
        cur = a.best_d[me];
        cur_j = a.phi[me];
      }
    } else if (Mode == kL1Argmin) {
      cur_j = 0;
    }
  }
  const int nchunk = (len + kTK - 1) / kTK;
  // pairs: entry tiles split over gridDim.y; scan / argmin keep one block per patch tile (ordered state),
  // or (scan, a.chunk > 0) one block per (patch tile, entry chunk), merged afterwards
  const int64_t ebeg = a.chunk ? a.e0 + (int64_t)blockIdx.y * a.chunk : a.e0 + (int64_t)blockIdx.y * kTE;
  const int64_t eend = a.chunk ? (a.e1 < ebeg + a.chunk ? a.e1 : ebeg + a.chunk) : a.e1;
  const int64_t estep = a.chunk ? kTE : (int64_t)gridDim.y * kTE;
  for (int64_t et0 = ebeg; et0 < eend; et0 += estep) {
    if (Mode == kL1Scan && !a.best_match) {
      if (__syncthreads_and(done)) break;
    } else {
      __syncthreads();
    }
    const int ne = eend - et0 < kTE ? (int)(eend - et0) : kTE;
    if (t < kTE) {
      const int64_t e = et0 + t;
      esrc[t] = t < ne ? (a.rep_src ? a.mats + (int64_t)a.rep_src[e] * len : a.reps + e * len) : nullptr;
    }
    __syncthreads();
    auto issue = [&](int c) {
      double* st = sm + (size_t)(c & 1) * kTStage;
      const int k0 = c * kTK;
      const int qn = min(kTK, len - k0);
      for (int idx = t; idx < (kTP + kTE) * kTK; idx += kTThreads) {
        const int r = idx / kTK, k = idx % kTK;
        const double* src = r < kTP ? psrc[r] : esrc[r - kTP];
        if (k < qn && src) cp_async8(st + r * kTL + k, src + k0 + k);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[4][JB];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < JB; ++j) acc[i][j] = 0.0;
    issue(0);
    for (int c = 0; c < nchunk; ++c) {
      if (c + 1 < nchunk) {
        issue(c + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double* A = sm + (size_t)(c & 1) * kTStage;
      const double* B = A + kTP * kTL;
      const int qn = min(kTK, len - c * kTK);
#pragma unroll 4
      for (int k = 0; k < qn; ++k) {
        double av[4], bv[JB];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = A[(tp + 16 * i) * kTL + k];
#pragma unroll
        for (int j = 0; j < JB; ++j) bv[j] = B[(te + EL * j) * kTL + k];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < JB; ++j) acc[i][j] = __dadd_rn(acc[i][j], fabs(__dsub_rn(av[i], bv[j])));
      }
      __syncthreads();  // the stage is refilled by issue(c + 2)
    }
    if (Mode == kL1Pairs) {
      const int64_t ld = a.e1 - a.e0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t g = p0 + tp + 16 * i;
        if (g >= a.npat) continue;
#pragma unroll
        for (int j = 0; j < JB; ++j) {
          const int e = te + EL * j;
          if (e < ne) a.d[g * ld + (et0 - a.e0) + e] = acc[i][j];
        }
      }
      continue;
    }
    // scan / argmin: the tile's distances through shared memory, then each
    // patch walks its entries in ascending order
    double* D = sm;  // [kTP][kTE + 1], aliases stage 0 (all reads of it are done)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < JB; ++j) D[(tp + 16 * i) * (kTE + 1) + te + EL * j] = acc[i][j];
    __syncthreads();
    if (t < kTP && !done) {
      const double* Dr = D + t * (kTE + 1);
      if (Mode == kL1Argmin) {
        for (int e = 0; e < ne; ++e)
          if (Dr[e] < cur) {  // strict <: lowest index wins ties (compress.cpp:154-160)
            cur = Dr[e];
            cur_j = (int32_t)(et0 + e);
          }
      } else if (a.best_match) {
        const int64_t me = pme[t] + a.id_offset;
        const int32_t* cr = a.creator ? a.creator : a.rep_src;
        for (int e = 0; e < ne; ++e) {
          const int64_t j = et0 + e;
          if (cr[j] < me && Dr[e] < cur) {
            cur = Dr[e];
            cur_j = (int32_t)j;
          }
        }
      } else {
        for (int e = 0; e < ne; ++e)
          if (Dr[e] < a.eps) {  // first match (compress.cpp:77-80)
            cur_j = (int32_t)(et0 + e);
            done = true;
            break;
          }
      }
    }
  }
  if (t >= kTP || p0 + t >= a.npat) return;
  if (Mode == kL1Scan && a.chunk) {
    const int64_t q = (int64_t)blockIdx.y * a.npat + p0 + t;
    a.part_j[q] = cur_j;
    if (a.best_match) a.part_d[q] = cur;
    return;
  }
  if (Mode == kL1Scan) {
    const int32_t me = pme[t];
    if (a.best_match) {
      a.best_d[me] = cur;
      a.phi[me] = cur_j;
    } else if (cur_j >= 0) {
      a.phi[me] = cur_j;
    }
  } else if (Mode == kL1Argmin) {
    const int64_t g = p0 + t;
    a.new_phi[g] = cur_j;
    a.min_dist[g] = cur;
    if (cur_j != a.phi[g]) atomicOr(a.changed, 1);
  }
}

// merge of the entry chunks of a split scan, in chunk (= entry) order
__global__ void l1_scan_reduce_kernel(int64_t npat, int gy, const int32_t* __restrict__ pid, int best_match,
                                      const int32_t* __restrict__ part_j, const double* __restrict__ part_d,
                                      int32_t* __restrict__ phi, double* __restrict__ best_d) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npat) return;
  const int32_t me = pid[g];
  if (!best_match) {
    for (int y = 0; y < gy; ++y) {
      const int32_t j = part_j[(int64_t)y * npat + g];
      if (j >= 0) {  // the first chunk holding a match has the first match
        phi[me] = j;
        return;
      }
    }
    return;
  }
  double cur = best_d[me];
  int32_t cj = phi[me];
  for (int y = 0; y < gy; ++y) {
    const double d = part_d[(int64_t)y * npat + g];
    if (d < cur) {  // strict: the earlier chunk keeps ties
      cur = d;
      cj = part_j[(int64_t)y * npat + g];
    }
  }
  best_d[me] = cur;
  phi[me] = cj;
}

template <int Mode, int TE>
void l1_tile_launch_te(const L1Args& a, cudaStream_t s) {
  constexpr int kTE = TE, NT = L1Tile<TE>::NT;
  constexpr size_t smem = L1Tile<TE>::SMEM;
  if (smem > 48 * 1024) cudaFuncSetAttribute(l1_tile_kernel<Mode, TE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned gy = 1;
  if (Mode == kL1Pairs) {
    // enough blocks to fill the GPU when the patch count is small (greedy batches: 1024 x 1024)
    const int64_t tiles = (a.e1 - a.e0 + kTE - 1) / kTE;
    const int64_t px = (a.npat + kTP - 1) / kTP;
    gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (4 * 148 + px - 1) / px));
  }
  if (Mode == kL1Scan) {
    const int64_t px = (a.npat + kTP - 1) / kTP, ne = a.e1 - a.e0;
    const char* sp = getenv("PDB_L1_SPLIT");
    if (px < 2 * 148 && ne > 2 * kTE && !(sp && sp[0] == '0')) {
      const int64_t want = std::min<int64_t>((ne + kTE - 1) / kTE, (4 * 148 + px - 1) / px);
      int64_t chunk = (ne + want - 1) / want;
      chunk = (chunk + kTE - 1) / kTE * kTE;
      const int gys = (int)((ne + chunk - 1) / chunk);
      if (gys > 1) {
        L1Args b = a;
        b.chunk = chunk;
        PDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&b.part_j), (size_t)gys * a.npat * sizeof(int32_t), s));
        PDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&b.part_d), (size_t)gys * a.npat * sizeof(double), s));
        l1_tile_kernel<Mode, TE><<<dim3(grid_for(a.npat, kTP), (unsigned)gys), NT, smem, s>>>(b);
        l1_scan_reduce_kernel<<<grid_for(a.npat, 256), 256, 0, s>>>(a.npat, gys, a.pid, a.best_match, b.part_j,
                                                                     b.part_d, a.phi, a.best_d);
        PDB_CUDA(cudaFreeAsync(b.part_j, s));
        PDB_CUDA(cudaFreeAsync(b.part_d, s));
        return;
      }
    }
  }
  l1_tile_kernel<Mode, TE><<<dim3(grid_for(a.npat, kTP), gy), NT, smem, s>>>(a);
}

// Entry-tile width: PDB_L1_TE = 32 / 64 / 128 (A/B runs); 64 by default (config-3 1 % greedy
// build: 22.5 / 20.1 / 20.9 ms; the scan is FP64-pipe bound at 59 % with TE = 32, ncu).
template <int Mode>
void l1_tile_launch(const L1Args& a, cudaStream_t s) {
  static const int te = [] {
    const char* e = getenv("PDB_L1_TE");
    return e ? atoi(e) : 64;
  }();
  if (te == 128)
    l1_tile_launch_te<Mode, 128>(a, s);
  else if (te == 64)
    l1_tile_launch_te<Mode, 64>(a, s);
  else
    l1_tile_launch_te<Mode, 32>(a, s);
}

bool l1_tiled_enabled() {  // PDB_L1_TILED=0: the thread-per-patch kernels below (A/B runs, tests)
  const char* e = getenv("PDB_L1_TILED");
  return !(e && e[0] == '0');
}

// First-/best-match scan of unresolved patches over entries [e0, e1)
// (greedy_impl compress.cpp:51-84).  Entries are patch matrices of their
// creators.  Block-uniform early exit once every thread has matched.
__global__ void __launch_bounds__(kL1Threads) l1_scan_kernel(int64_t nu, const int32_t* __restrict__ pid, int64_t e0,
                                                             int64_t e1, int len, const double* __restrict__ mats,
                                                             const int32_t* __restrict__ creators, double eps,
                                                             int best_match, int32_t* __restrict__ phi,
                                                             double* __restrict__ best_d) {
  __shared__ double R[kL1Ent][kL1Chunk];
  const int64_t t = (int64_t)blockIdx.x * kL1Threads + threadIdx.x;
  const bool live = t < nu;
  const int32_t me = live ? pid[t] : 0;
  const double* A = mats + (int64_t)me * len;
  bool done = !live;
  double cur = eps;
  int32_t cur_j = -1;
  if (live && best_match) {
    cur = best_d[me];
    cur_j = phi[me];
  }
  for (int64_t tile = e0; tile < e1; tile += kL1Ent) {
    if (__syncthreads_and(done)) break;
    double acc[kL1Ent];
#pragma unroll
    for (int c = 0; c < kL1Ent; ++c) acc[c] = 0.0;
    for (int q0 = 0; q0 < len; q0 += kL1Chunk) {
      const int qn = min(kL1Chunk, len - q0);
      __syncthreads();
      for (int c = 0; c < kL1Ent; ++c) {
        const int64_t e = tile + c;
        if (e >= e1) break;
        const double* Re = mats + (int64_t)creators[e] * len;
        for (int q = threadIdx.x; q < qn; q += kL1Threads) R[c][q] = Re[q0 + q];
      }
      __syncthreads();
      if (!done)
        for (int q = 0; q < qn; ++q) {
          const double a = A[q0 + q];
#pragma unroll
          for (int c = 0; c < kL1Ent; ++c) acc[c] = __dadd_rn(acc[c], fabs(__dsub_rn(a, R[c][q])));
        }
    }
    if (!done)
      for (int c = 0; c < kL1Ent; ++c) {
        const int64_t j = tile + c;
        if (j >= e1) break;
        if (best_match) {
          if (creators[j] < me && acc[c] < cur) {
            cur = acc[c];
            cur_j = (int32_t)j;
          }
        } else if (acc[c] < eps) {
          cur_j = (int32_t)j;
          done = true;
          break;
        }
      }
  }
  if (live) {
    if (best_match) {
      best_d[me] = cur;
      phi[me] = cur_j;
    } else if (cur_j >= 0) {
      phi[me] = cur_j;
    }
  }
}

// Match-state update from a precomputed distance block (spectral flavour).
__global__ void apply_scan_kernel(int64_t nu, const int32_t* __restrict__ pid, int64_t e0, int64_t ne,
                                  const double* __restrict__ d, const int32_t* __restrict__ creators, double eps,
                                  int best_match, int32_t* __restrict__ phi, double* __restrict__ best_d) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nu) return;
  const int32_t me = pid[t];
  if (best_match) {
    double cur = best_d[me];
    int32_t cj = phi[me];
    for (int64_t e = 0; e < ne; ++e)
      if (creators[e0 + e] < me && d[t * ne + e] < cur) {
        cur = d[t * ne + e];
        cj = (int32_t)(e0 + e);
      }
    best_d[me] = cur;
    phi[me] = cj;
  } else {
    if (phi[me] >= 0) return;
    for (int64_t e = 0; e < ne; ++e)
      if (d[t * ne + e] < eps) {
        phi[me] = (int32_t)(e0 + e);
        return;
      }
  }
}

// Sequential resolution of a batch S against the entries it creates itself.
// One warp: for each a in order, the candidate entries are the batch members
// b < a that became entries; first-match takes the lowest such b with
// D[a][b] < eps, best-match the smallest D < eps (ties: lowest b).  Batch
// members were unmatched against every earlier entry, so this reproduces the
// sequential pass exactly.
// Batch resolution, two phases (one block of 1024 threads).  Whether b < a
// is a candidate for a (D[a][b] < eps) does not depend on the sequential
// state, so all candidate bits are computed first in parallel (one ballot
// per 32 columns) into shared memory; the sequential pass over a then only
// intersects a's candidate words with the bit set of batch members that
// became entries (lane l holds word l): first match = the lowest set bit;
// best match = the smallest D among the set bits, ties to the lowest b --
// exactly the scan of the one-warp kernel below (compress.cpp:63-92).
constexpr int kResolveMax = 1024;

// phase 1 over the whole GPU: cand[a][w] = bits of b in [32w, 32w+32), b < a, D[a][b] < eps
__global__ void greedy_cand_bits_kernel(int B, const double* __restrict__ D, double eps, uint32_t* __restrict__ cand) {
  const int words = (B + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // global warp = (a, w) item
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t item = gw; item < (int64_t)B * words; item += nwarps) {
    const int a = (int)(item / words), w = (int)(item % words);
    const int b = w * 32 + lane;
    const bool c = b < a && D[(int64_t)a * B + b] < eps;
    const uint32_t bits = __ballot_sync(0xffffffffu, c);
    if (lane == 0) cand[a * 32 + w] = bits;
  }
}

// The sequential pass touches shared memory only: the batch ids and LU
// statuses are staged first, each step's outcome is recorded per batch member
// (res[a] = the entry it created or matched), and phi / creators / entry_of
// are written by the whole block afterwards -- a global load or store inside
// the pass would put its latency on every one of the B dependent steps.
__global__ void __launch_bounds__(1024) greedy_resolve_bits_kernel(
    int B, const int32_t* __restrict__ S, const double* __restrict__ D, double eps, int best_match,
    int64_t abort_above, const int32_t* __restrict__ lu_status, int32_t* __restrict__ phi,
    int32_t* __restrict__ creators, int32_t* __restrict__ entry_of, int64_t* state,
    const uint32_t* __restrict__ cand_g) {
  extern __shared__ uint32_t cand[];  // [B][32]
  __shared__ int32_t ent_s[kResolveMax];
  __shared__ int32_t S_s[kResolveMax];
  __shared__ int32_t res[kResolveMax];  // >= 0: entry created (new) or matched (old); filled for a < a_end
  __shared__ uint8_t is_new[kResolveMax];
  __shared__ uint8_t bad_lu[kResolveMax];
  __shared__ int a_end_s;
  __shared__ long long m0_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int words = (B + 31) / 32;
  for (int e = threadIdx.x; e < B * 32; e += blockDim.x) cand[e] = cand_g[e];
  for (int e = threadIdx.x; e < B; e += blockDim.x) {
    S_s[e] = S[e];
    bad_lu[e] = lu_status && lu_status[e] != 0;
  }
  if (threadIdx.x == 0) m0_s = state[0];
  __syncthreads();
  if (warp == 0) {
    uint32_t ent = 0;  // word `lane` of the entry bit set
    int64_t m = m0_s;
    int a = 0;
    for (; a < B; ++a) {
      const uint32_t w = lane < words ? cand[a * 32 + lane] & ent : 0u;
      int bb = B;
      if (!best_match) {
        const uint32_t any = __ballot_sync(0xffffffffu, w != 0);
        if (any) {
          const int L = __ffs(any) - 1;
          const uint32_t wl = __shfl_sync(0xffffffffu, w, L);
          bb = L * 32 + __ffs(wl) - 1;
        }
      } else {
        double bd = eps;
        uint32_t r = w;
        while (r) {
          const int b = lane * 32 + __ffs(r) - 1;
          r &= r - 1;
          const double dv = D[(int64_t)a * B + b];
          if (dv < bd) {
            bd = dv;
            bb = b;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, bd, off);
          const int ob = __shfl_xor_sync(0xffffffffu, bb, off);
          if (od < bd || (od == bd && ob < bb)) {
            bd = od;
            bb = ob;
          }
        }
      }
      if (bb < B) {
        if (lane == 0) {
          res[a] = ent_s[bb];
          is_new[a] = 0;
        }
        __syncwarp();
        continue;
      }
      if (abort_above > 0 && m + 1 > abort_above) {
        if (lane == 0) state[1] = 1;
        break;
      }
      if (bad_lu[a]) {
        if (lane == 0) state[2] = a;
        break;
      }
      if (lane == 0) {
        res[a] = (int32_t)m;
        is_new[a] = 1;
        ent_s[a] = (int32_t)m;
      }
      if (lane == (a >> 5)) ent |= 1u << (a & 31);
      ++m;
      __syncwarp();
    }
    if (lane == 0) {
      state[0] = m;
      a_end_s = a;
    }
  }
  __syncthreads();
  const int a_end = a_end_s;
  for (int a = threadIdx.x; a < a_end; a += blockDim.x) {
    const int32_t v = res[a];
    phi[S_s[a]] = v;
    if (is_new[a]) {
      creators[v] = S_s[a];
      entry_of[a] = v;
    } else {
      entry_of[a] = -1;
    }
  }
}

__global__ void greedy_resolve_kernel(int B, const int32_t* __restrict__ S, const double* __restrict__ D, double eps,
                                      int best_match, int64_t abort_above, const int32_t* __restrict__ lu_status,
                                      int32_t* __restrict__ phi, int32_t* __restrict__ creators,
                                      int32_t* __restrict__ entry_of, int64_t* state) {
  const int lane = threadIdx.x;
  int64_t m = state[0];
  for (int a = 0; a < B; ++a) {
    double bd = eps;
    int bb = B;
    for (int b = lane; b < a; b += 32) {
      const int ent = entry_of[b];
      if (ent < 0) continue;
      const double dv = D[(int64_t)a * B + b];
      if (best_match) {
        if (dv < bd) {  // lanes scan their b ascending: keeps the lowest b on ties
          bd = dv;
          bb = b;
        }
      } else if (dv < eps && b < bb) {
        bb = b;
        bd = dv;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, off);
      const int ob = __shfl_xor_sync(0xffffffffu, bb, off);
      if (best_match) {
        if (od < bd || (od == bd && ob < bb)) {
          bd = od;
          bb = ob;
        }
      } else if (ob < bb) {
        bb = ob;
        bd = od;
      }
    }
    if (bb < B) {
      if (lane == 0) {
        phi[S[a]] = entry_of[bb];
        entry_of[a] = -1;
      }
      __syncwarp();
      continue;
    }
    if (abort_above > 0 && m + 1 > abort_above) {
      if (lane == 0) state[1] = 1;
      break;
    }
    if (lu_status && lu_status[a] != 0) {
      if (lane == 0) state[2] = a;
      break;
    }
    if (lane == 0) {
      creators[m] = S[a];
      phi[S[a]] = (int32_t)m;
      entry_of[a] = (int32_t)m;
    }
    ++m;
    __syncwarp();
  }
  if (lane == 0) state[0] = m;
}

// ----------------------------------------------------------- spectral ----
// Per-thread vectors live in shared memory at [q * BD + tid] (lane-contiguous).
struct Vec {
  double* p;
  int stride;
  __device__ double& operator[](int q) const { return p[q * stride]; }
};

// lu_solve_into (dense.cpp:77-94): out = B^{-1} rhs.
__device__ void lu_solve_dev(int n, const double* __restrict__ LU, const int32_t* __restrict__ P, Vec rhs, Vec out) {
  for (int i = 0; i < n; ++i) out[i] = rhs[P[i]];
  for (int i = 1; i < n; ++i) {
    double s = out[i];
    for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(LU[i * n + j], out[j]));
    out[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = out[i];
    for (int j = i + 1; j < n; ++j) s = __dsub_rn(s, __dmul_rn(LU[i * n + j], out[j]));
    out[i] = __ddiv_rn(s, LU[i * n + i]);
  }
}

// lu_solve_transpose_into (dense.cpp:102-120); w is consumed (it holds the
// reference's internal copy of rhs), out[P[i]] = w[i].
__device__ void lu_solve_t_dev(int n, const double* __restrict__ LU, const int32_t* __restrict__ P, Vec w, Vec out) {
  for (int i = 0; i < n; ++i) {
    double s = w[i];
    for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(LU[j * n + i], w[j]));
    w[i] = __ddiv_rn(s, LU[i * n + i]);
  }
  for (int i = n - 2; i >= 0; --i) {
    double s = w[i];
    for (int j = i + 1; j < n; ++j) s = __dsub_rn(s, __dmul_rn(LU[j * n + i], w[j]));
    w[i] = s;
  }
  for (int i = 0; i < n; ++i) out[P[i]] = w[i];
}

__device__ double norm2_dev(int n, Vec v) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(v[i], v[i]));
  return __dsqrt_rn(s);
}

// spectral_distance (dense.cpp:154-190).  A: patch matrix (row-major,
// per-thread), LU/P: factor (shared), v,t,w,s: per-thread vectors.
__device__ double spectral_dev(int n, const double* __restrict__ A, const double* __restrict__ LU,
                               const int32_t* __restrict__ P, Vec v, Vec t, Vec w, Vec s, int* iters) {
  for (int i = 0; i < n; ++i) v[i] = __dadd_rn(1.0, __dmul_rn(1e-6, (double)i));
  const double vn = norm2_dev(n, v);
  for (int i = 0; i < n; ++i) v[i] = __ddiv_rn(v[i], vn);
  double lambda = 0.0;
  for (int it = 0; it < 200; ++it) {
    *iters = it + 1;
    lu_solve_dev(n, LU, P, v, t);  // t = B^{-1} v
    for (int i = 0; i < n; ++i) {  // w = v - A t   (mat_vec, then subtract)
      double acc = 0.0;
      const double* Ai = A + (int64_t)i * n;
      for (int j = 0; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(Ai[j], t[j]));
      w[i] = __dsub_rn(v[i], acc);
    }
    for (int j = 0; j < n; ++j) s[j] = 0.0;  // s = A^T w  (mat_tvec loop order)
    for (int i = 0; i < n; ++i) {
      const double xi = w[i];
      const double* Ai = A + (int64_t)i * n;
      for (int j = 0; j < n; ++j) s[j] = __dadd_rn(s[j], __dmul_rn(Ai[j], xi));
    }
    lu_solve_t_dev(n, LU, P, s, t);  // t = B^{-T} s
    double rq = 0.0;
    for (int i = 0; i < n; ++i) {  // u = w - t (stored in t); rq = v.u
      const double u = __dsub_rn(w[i], t[i]);
      t[i] = u;
      rq = __dadd_rn(rq, __dmul_rn(v[i], u));
    }
    rq = rq > 0.0 ? rq : 0.0;
    if (rq <= 1e-28) return __dsqrt_rn(rq);
    if (it > 0 && fabs(__dsub_rn(rq, lambda)) < __dmul_rn(1e-8, rq)) return __dsqrt_rn(rq);
    lambda = rq;
    const double un2 = norm2_dev(n, t);
    if (un2 == 0.0) return 0.0;
    for (int i = 0; i < n; ++i) v[i] = __ddiv_rn(t[i], un2);
  }
  return __dsqrt_rn(lambda);
}

// Block = BD patches x one factor (grid.y); factor staged in shared memory
// and broadcast, patch matrices streamed per thread.
// stage = false (large patches whose factor does not fit next to the vectors):
// the factor is read from global memory (L2-resident, shared by the block).
__global__ void spectral_pairs_kernel(int64_t npat, const int32_t* __restrict__ pid, int64_t ne, int ps,
                                      const double* __restrict__ mats, const double* __restrict__ lu,
                                      const int32_t* __restrict__ piv, double* __restrict__ d,
                                      unsigned long long* iters_total, bool stage) {
  extern __shared__ double sm[];
  const int BD = blockDim.x;
  const int64_t len = (int64_t)ps * ps;
  const int64_t e = blockIdx.y;
  const double* LU = lu + e * len;
  const int32_t* P = piv + e * ps;
  double* vec = sm;
  if (stage) {
    double* LUs = sm;
    int32_t* Ps = reinterpret_cast<int32_t*>(LUs + len);
    vec = LUs + len + (ps + 1) / 2;
    for (int64_t q = threadIdx.x; q < len; q += BD) LUs[q] = lu[e * len + q];
    for (int q = threadIdx.x; q < ps; q += BD) Ps[q] = piv[e * ps + q];
    LU = LUs;
    P = Ps;
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * BD + threadIdx.x;
  if (t >= npat) return;
  const double* A = mats + (int64_t)(pid ? pid[t] : t) * len;
  Vec v{vec + threadIdx.x, BD}, tv{vec + ps * BD + threadIdx.x, BD}, w{vec + 2 * ps * BD + threadIdx.x, BD},
      s{vec + 3 * ps * BD + threadIdx.x, BD};
  int it = 0;
  d[t * ne + e] = spectral_dev(ps, A, LU, P, v, tv, w, s, &it);
  if (iters_total) atomicAdd(iters_total, (unsigned long long)it);
}

// Listed pairs: thread per pair, factor read from global (L2).
__global__ void spectral_list_kernel(int64_t npairs, const int32_t* __restrict__ pa, const int32_t* __restrict__ fb,
                                     int ps, const double* __restrict__ mats, const double* __restrict__ lu,
                                     const int32_t* __restrict__ piv, double* __restrict__ d,
                                     unsigned long long* iters_total) {
  extern __shared__ double sm[];
  const int BD = blockDim.x;
  const int64_t len = (int64_t)ps * ps;
  const int64_t t = (int64_t)blockIdx.x * BD + threadIdx.x;
  if (t >= npairs) return;
  const double* A = mats + (int64_t)pa[t] * len;
  const double* LU = lu + (int64_t)fb[t] * len;
  const int32_t* P = piv + (int64_t)fb[t] * ps;
  Vec v{sm + threadIdx.x, BD}, tv{sm + ps * BD + threadIdx.x, BD}, w{sm + 2 * ps * BD + threadIdx.x, BD},
      s{sm + 3 * ps * BD + threadIdx.x, BD};
  int it = 0;
  d[t] = spectral_dev(ps, A, LU, P, v, tv, w, s, &it);
  if (iters_total) atomicAdd(iters_total, (unsigned long long)it);
}

// ----------------------------------------------- spectral, tiled (fast) ----
// Compile-time patch size: the per-thread vectors t (B^{-1} v) and s (A^T w)
// live in registers, so the two matrix-vector products share one pass over
// A (each A(i,j) is loaded once and used for w_i and s_j -- the same
// per-element operation order as mat_vec then mat_tvec), the triangular
// solves run on register arrays with immediate indices, and only v, w and
// the permuted t go through shared memory.  A block owns a tile of TA
// patches x TE factors; its factors sit in shared memory, its patches stay
// L1-resident, and every thread keeps pulling (patch, factor) pairs from the
// tile until it is exhausted, so a lane that converges early starts a new
// pair instead of idling until the slowest lane of its warp finishes.
constexpr int kTileA = 32;  // patches per tile (L1-resident)
constexpr int kTileE = 8;   // factors per tile (L1-resident, read by broadcast)
constexpr int kTileThreads = 64;

// IL = true: patches and factors come pre-interleaved (interleave_mats):
// element q of the tile's patch a at A[q * 32 + a], of factor e at
// L[q * 8 + e], pivot i at P[i * 8 + e].  Lanes of a warp work on different
// (patch, factor) pairs of one tile, so each load of the interleaved copy is
// one contiguous 256-byte (patches) / 64-byte (factors) span instead of up to
// 32 separate cache lines.
// DIAG (with IL): one pair per patch, (patch, its centroid diag_phi[patch]),
// the factors in the plain layout (d[patch] is written) -- the pruning bound.
// KmeansReuse (k-means assignment, all pointers may be null): ub = per-patch
// bound, chg = per-entry "centroid changed since the previous assignment",
// lbq = per-pair Rayleigh quotient at which a pair was pruned, dprev (DIAG) =
// the previous distance matrix with mfull columns.  A pair whose centroid is
// unchanged keeps its previous exact distance, or stays +inf when its stored
// quotient already exceeds the bound; only pairs of changed centroids run.
template <int PS, bool IL, bool DIAG = false>
__global__ void __launch_bounds__(kTileThreads) spectral_tile_kernel(int64_t npat, const int32_t* __restrict__ pid,
                                                                     int64_t ne, const double* __restrict__ mats,
                                                                     const double* __restrict__ lu,
                                                                     const int32_t* __restrict__ piv,
                                                                     double* __restrict__ d,
                                                                     unsigned long long* iters_total,
                                                                     KmeansReuse ru,
                                                                     const int32_t* __restrict__ diag_phi = nullptr) {
  const double* __restrict__ ub = ru.ub;
  constexpr int LEN = PS * PS;
  constexpr int BD = kTileThreads;
  constexpr int SA = IL ? kTileA : 1;             // element stride of a patch matrix
  constexpr int SL = (IL && !DIAG) ? kTileE : 1;  // element stride of a factor / pivot vector
  extern __shared__ double sm[];
  double* vec = sm;  // 3 * PS * BD: v, w, t
  __shared__ int counter;
  const int tid = threadIdx.x;
  // DIAG: 128 patches pulled by 64 threads; sorted DIAG (pid): 64, one per thread
  const int TA = DIAG ? (pid ? kTileThreads : 2 * kTileThreads) : kTileA;
  // pruned assignment with ru.tile_order: blocks take their tiles longest
  // first (the previous Lloyd iteration's power iterations per tile)
  const int64_t tile = (!DIAG && ru.tile_order) ? (int64_t)ru.tile_order[blockIdx.x] : (int64_t)blockIdx.x;
  const int64_t a0 = tile * TA, e0 = (int64_t)blockIdx.y * kTileE;
  const int na = (int)(npat - a0 < TA ? npat - a0 : TA);
  // pruned k-means assignment (IL, bound given): one block takes every factor
  // of its patches, so the few pairs that run to convergence overlap with
  // many that are cut after an iteration or two
  const bool all_e = IL && !DIAG && ru.ub != nullptr;
  const int nev = all_e ? (int)ne : (int)(ne - e0 < kTileE ? ne - e0 : kTileE);
  const double* LUs = IL ? lu + (int64_t)blockIdx.y * LEN * kTileE : lu + e0 * LEN;
  const int32_t* Ps = IL ? piv + (int64_t)blockIdx.y * PS * kTileE : piv + e0 * PS;
  if (tid == 0) counter = 0;
  __syncthreads();
  double* V = vec + tid;
  double* W = vec + PS * BD + tid;
  double* Tv = vec + 2 * PS * BD + tid;
  const int npairs = DIAG ? na : na * nev;
  bool active = false;
  int it = 0, pa = 0, pe = 0;
  int64_t gcur = 0;
  bool pulled = false;
  double lambda = 0.0;
  const double* A = mats;
  const double* L = LUs;
  const int32_t* P = Ps;
  unsigned long long my_iters = 0;
  for (;;) {
    while (!active) {
      // DIAG with pid (sorted copy): thread t keeps pair t -- the lanes of a
      // warp stay on one aligned group of 32 patches (coalesced patch loads)
      // that mostly share a centroid (broadcast factor loads); no refill
      int p;
      if (DIAG && pid) {
        p = pulled ? npairs : tid;
        pulled = true;
      } else {
        p = atomicAdd(&counter, 1);
      }
      // pruned assignment with long_prev: two passes over the block's pairs,
      // first those that ran past two power iterations in the previous Lloyd
      // iteration (likely long again), then the rest -- the long chains start
      // early instead of forming the block's tail
      const bool two = !DIAG && ru.long_prev != nullptr;
      if (p >= (two ? 2 * npairs : npairs)) break;
      const bool second = p >= npairs;
      if (second) p -= npairs;
      {
        pa = p % na;
        pe = p / na;
        if (two) {
          const int64_t q = (a0 + pa) * ne + e0 + pe;
          const bool lng = ru.long_prev[q] != 0;
          if (lng == second) continue;  // taken in the other pass
          ru.long_cur[q] = lng;         // carried when the pair is not run below
        }
        // DIAG with pid: position a0 + pa of a centroid-sorted copy of the
        // patches; g is the patch's own index for d / dprev / phi
        const int64_t g = (DIAG && pid) ? (int64_t)pid[a0 + pa] : a0 + pa;
        gcur = g;
        if (ru.chg != nullptr) {  // reuse across Lloyd iterations
          if (DIAG) {
            const int32_t f = diag_phi[g];
            if (!ru.chg[f]) {
              d[g] = ru.dprev[g * ru.mfull + f];
              continue;
            }
          } else if (ru.phi != nullptr && ru.phi[g] == e0 + pe) {
            d[g * ne + e0 + pe] = ub[g];  // the bound is this pair's distance, computed the same way
            continue;
          } else if (!ru.chg[e0 + pe]) {
            const int64_t q = g * ne + e0 + pe;
            if (isfinite(d[q])) continue;  // exact distance of the unchanged centroid
            if (isfinite(ub[g]) && ru.lbq[q] > fmax(ub[g] * ub[g] * (1.0 + 1e-4), 1e-8)) continue;  // still beaten
          }
        }
        active = true;
        if (DIAG) {
          const int64_t q = a0 + pa;
          A = mats + (q / kTileA) * LEN * kTileA + q % kTileA;
          L = lu + (int64_t)diag_phi[g] * LEN;
          P = piv + (int64_t)diag_phi[g] * PS;
        } else if (IL) {
          A = mats + tile * LEN * kTileA + pa;
          if (all_e) {  // factor pe of the interleaved groups of kTileE
            L = lu + (int64_t)(pe / kTileE) * LEN * kTileE + pe % kTileE;
            P = piv + (int64_t)(pe / kTileE) * PS * kTileE + pe % kTileE;
          } else {
            L = LUs + pe;
            P = Ps + pe;
          }
        } else {
          A = mats + (int64_t)(pid ? pid[g] : g) * LEN;
          L = LUs + pe * LEN;
          P = Ps + pe * PS;
        }
        it = 0;
        lambda = 0.0;
        // v0_i = 1 + 1e-6 i, normalised by division (dense.cpp:163-165)
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < PS; ++i) {
          const double vi = __dadd_rn(1.0, __dmul_rn(1e-6, (double)i));
          V[i * BD] = vi;
          s = __dadd_rn(s, __dmul_rn(vi, vi));
        }
        const double vn = __dsqrt_rn(s);
#pragma unroll
        for (int i = 0; i < PS; ++i) V[i * BD] = __ddiv_rn(V[i * BD], vn);
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
    if (!active) continue;
    // ---- t = B^{-1} v (lu_solve_into, dense.cpp:77-94)
    double T[PS];
#pragma unroll
    for (int i = 0; i < PS; ++i) T[i] = V[__ldg(P + i * SL) * BD];
    // column-oriented: once T[j] is final every later row takes its j-th
    // term -- each row still subtracts in ascending j, but the rows' chains
    // advance together (instruction-level parallelism PS - 1 - j)
#pragma unroll
    for (int j = 0; j < PS - 1; ++j) {
#pragma unroll
      for (int i = j + 1; i < PS; ++i) T[i] = __dsub_rn(T[i], __dmul_rn(__ldg(L + (i * PS + j) * SL), T[j]));
    }
#pragma unroll
    for (int i = PS - 1; i >= 0; --i) {
      double s = T[i];
#pragma unroll
      for (int j = i + 1; j < PS; ++j) s = __dsub_rn(s, __dmul_rn(__ldg(L + (i * PS + j) * SL), T[j]));
      T[i] = __ddiv_rn(s, __ldg(L + (i * PS + i) * SL));
    }
    // ---- w = v - A t (mat_vec) and s = A^T w (mat_tvec) in one pass over
    // A: row i gives w_i, then immediately its contribution to every s_j
    // (per-element order identical to mat_vec followed by mat_tvec).
    double S[PS];
#pragma unroll
    for (int j = 0; j < PS; ++j) S[j] = 0.0;
#pragma unroll 1
    for (int i = 0; i < PS; ++i) {
      const double* Ai = A + i * PS * SA;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < PS; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(Ai + j * SA), T[j]));
      const double wi = __dsub_rn(V[i * BD], acc);
      W[i * BD] = wi;
#pragma unroll
      for (int j = 0; j < PS; ++j) S[j] = __dadd_rn(S[j], __dmul_rn(__ldg(Ai + j * SA), wi));
    }
    // ---- t = B^{-T} s (lu_solve_transpose_into, dense.cpp:102-120)
#pragma unroll
    for (int j = 0; j < PS; ++j) {  // column-oriented, as the forward solve above
      S[j] = __ddiv_rn(S[j], __ldg(L + (j * PS + j) * SL));
#pragma unroll
      for (int i = j + 1; i < PS; ++i) S[i] = __dsub_rn(S[i], __dmul_rn(__ldg(L + (j * PS + i) * SL), S[j]));
    }
#pragma unroll
    for (int i = PS - 2; i >= 0; --i) {
      double s = S[i];
#pragma unroll
      for (int j = i + 1; j < PS; ++j) s = __dsub_rn(s, __dmul_rn(__ldg(L + (j * PS + i) * SL), S[j]));
      S[i] = s;
    }
#pragma unroll
    for (int i = 0; i < PS; ++i) Tv[__ldg(P + i * SL) * BD] = S[i];
    // ---- u = w - t, Rayleigh quotient, stopping rules (dense.cpp:170-188)
    double rq = 0.0;
#pragma unroll
    for (int i = 0; i < PS; ++i) {
      const double u = __dsub_rn(W[i * BD], Tv[i * BD]);
      Tv[i * BD] = u;
      rq = __dadd_rn(rq, __dmul_rn(V[i * BD], u));
    }
    rq = rq > 0.0 ? rq : 0.0;
    ++it;
    bool done = false;
    double result = 0.0;
    if (rq <= 1e-28) {
      done = true;
      result = __dsqrt_rn(rq);
    } else if (it > 1 && fabs(__dsub_rn(rq, lambda)) < __dmul_rn(1e-8, rq)) {
      done = true;
      result = __dsqrt_rn(rq);
    } else if ((ub != nullptr || ru.ubc > 0.0) && isfinite(ub ? ub[a0 + pa] : ru.ubc) &&
               rq > fmax((ub ? ub[a0 + pa] * ub[a0 + pa] : ru.ubc * ru.ubc) * (1.0 + 1e-4), 1e-8)) {
      // k-means pruning: the Rayleigh quotients of the power iteration rise
      // monotonically to the returned value, so this pair ends above the
      // patch's distance to its current centroid and cannot be the argmin.
      // The margin and the floor (distance 1e-4) keep the test clear of
      // rounding: near-identical pairs (quotients at noise level, not
      // monotone) always run to convergence.
      done = true;
      result = CUDART_INF;
      if (!DIAG && ru.lbq != nullptr) ru.lbq[(a0 + pa) * ne + e0 + pe] = rq;
    } else {
      lambda = rq;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < PS; ++i) s = __dadd_rn(s, __dmul_rn(Tv[i * BD], Tv[i * BD]));
      const double un2 = __dsqrt_rn(s);
      if (un2 == 0.0) {
        done = true;
        result = 0.0;
      } else {
#pragma unroll
        for (int i = 0; i < PS; ++i) V[i * BD] = __ddiv_rn(Tv[i * BD], un2);
        if (it == 200) {
          done = true;
          result = __dsqrt_rn(lambda);
        }
      }
    }
    if (done) {
      d[DIAG ? gcur : (a0 + pa) * ne + e0 + pe] = result;
      if (!DIAG && ru.long_cur) ru.long_cur[(a0 + pa) * ne + e0 + pe] = it > 2;
      if (DIAG && ru.it_out) ru.it_out[gcur] = it;
      my_iters += (unsigned long long)it;
      active = false;
    }
  }
  if (iters_total && my_iters) atomicAdd(iters_total, my_iters);
  if (!DIAG && ru.tile_iters && my_iters) atomicAdd(ru.tile_iters + tile, my_iters);
}

template <int PS, bool IL = false>
bool launch_spectral_tile(int64_t npat, const int32_t* pid, int64_t ne, const double* mats, const double* lu,
                          const int32_t* piv, double* d, unsigned long long* iters, cudaStream_t s,
                          KmeansReuse ru = KmeansReuse{}) {
  const size_t smem = (size_t)3 * PS * kTileThreads * sizeof(double);
  cudaFuncSetAttribute(spectral_tile_kernel<PS, IL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const bool all_e = IL && ru.ub != nullptr;  // must match the kernel's all_e
  dim3 grid(grid_for(npat, kTileA), all_e ? 1u : (unsigned)((ne + kTileE - 1) / kTileE));
  spectral_tile_kernel<PS, IL><<<grid, kTileThreads, smem, s>>>(npat, pid, ne, mats, lu, piv, d, iters, ru);
  return true;
}


// dst[((g * len) + q) * width + a] = src[(g * width + a) * len + q]; zero past `count` items
template <typename T>
__global__ void interleave_kernel(int64_t total, int64_t count, int width, int64_t len, const T* __restrict__ src,
                                  T* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int a = (int)(e % width);
  const int64_t q = (e / width) % len, g = e / (width * len);
  const int64_t item = g * width + a;
  dst[e] = item < count ? src[item * len + q] : T(0);
}

bool spectral_tiled(int64_t npat, const int32_t* pid, int64_t ne, int ps, const double* mats, const double* lu,
                    const int32_t* piv, double* d, unsigned long long* iters, cudaStream_t s, double bound) {
  const char* e = getenv("PDB_SPECTRAL_TILED");
  if (e && e[0] == '0') return false;
  KmeansReuse ru;
  ru.ubc = bound;
  switch (ps) {
    case 9: return launch_spectral_tile<9>(npat, pid, ne, mats, lu, piv, d, iters, s, ru);
    case 22: return launch_spectral_tile<22>(npat, pid, ne, mats, lu, piv, d, iters, s, ru);
    case 25: return launch_spectral_tile<25>(npat, pid, ne, mats, lu, piv, d, iters, s, ru);
    case 27: return launch_spectral_tile<27>(npat, pid, ne, mats, lu, piv, d, iters, s, ru);
    default: return false;
  }
}

// ------------------------------------------------------------ k-means ----
// Assignment (compress.cpp:150-166): strict <, so the lowest j wins ties;
// best starts at +inf with best_j = 0.
__global__ void argmin_kernel(int64_t n, int64_t ne, const double* __restrict__ d, const int32_t* __restrict__ phi,
                              int32_t* __restrict__ new_phi, double* __restrict__ min_dist, int32_t* changed) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double best = CUDART_INF;
  int32_t bj = 0;
  for (int64_t e = 0; e < ne; ++e) {
    const double v = d[t * ne + e];
    if (v < best) {
      best = v;
      bj = (int32_t)e;
    }
  }
  new_phi[t] = bj;
  min_dist[t] = best;
  if (bj != phi[t]) atomicOr(changed, 1);
}

__global__ void __launch_bounds__(kL1Threads) l1_argmin_kernel(int64_t n, int64_t ne, int len,
                                                               const double* __restrict__ mats,
                                                               const double* __restrict__ reps,
                                                               const int32_t* __restrict__ phi,
                                                               int32_t* __restrict__ new_phi,
                                                               double* __restrict__ min_dist, int32_t* changed) {
  __shared__ double R[kL1Ent][kL1Chunk];
  const int64_t t = (int64_t)blockIdx.x * kL1Threads + threadIdx.x;
  const bool live = t < n;
  const double* A = mats + (live ? t : 0) * len;
  double best = CUDART_INF;
  int32_t bj = 0;
  for (int64_t tile = 0; tile < ne; tile += kL1Ent) {
    double acc[kL1Ent];
#pragma unroll
    for (int c = 0; c < kL1Ent; ++c) acc[c] = 0.0;
    for (int q0 = 0; q0 < len; q0 += kL1Chunk) {
      const int qn = min(kL1Chunk, len - q0);
      __syncthreads();
      for (int c = 0; c < kL1Ent; ++c) {
        const int64_t e = tile + c;
        if (e >= ne) break;
        for (int q = threadIdx.x; q < qn; q += kL1Threads) R[c][q] = reps[e * len + q0 + q];
      }
      __syncthreads();
      if (live)
        for (int q = 0; q < qn; ++q) {
          const double a = A[q0 + q];
#pragma unroll
          for (int c = 0; c < kL1Ent; ++c) acc[c] = __dadd_rn(acc[c], fabs(__dsub_rn(a, R[c][q])));
        }
    }
    for (int c = 0; c < kL1Ent; ++c)
      if (tile + c < ne && acc[c] < best) {
        best = acc[c];
        bj = (int32_t)(tile + c);
      }
  }
  if (!live) return;
  new_phi[t] = bj;
  min_dist[t] = best;
  if (bj != phi[t]) atomicOr(changed, 1);
}

// entrywise_mean_indexed (dense.cpp:211-223): in-order sum from 0.0, then
// multiply by the reciprocal of the member count.  Thread per (cluster, entry).
__global__ void cluster_mean_kernel(int64_t m, int len, const int32_t* __restrict__ mem_ptr,
                                    const int32_t* __restrict__ mem, const double* __restrict__ mats,
                                    double* __restrict__ reps) {
  const int64_t j = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= len || j >= m) return;
  const int32_t lo = mem_ptr[j], hi = mem_ptr[j + 1];
  double s = 0.0;
  int32_t c = lo;
  // 8 member loads in flight, then the in-order additions
  for (; c + 8 <= hi; c += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = mats[(int64_t)__ldg(mem + c + u) * len + q];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
  }
  for (; c < hi; ++c) s = __dadd_rn(s, mats[(int64_t)mem[c] * len + q]);
  const double inv = __ddiv_rn(1.0, (double)(hi - lo));
  reps[j * len + q] = __dmul_rn(s, inv);
}

// Staged variant: block = one warp on 32 entries q of cluster j.  Each lane
// streams its own column through shared memory with 8-byte cp.async, kMeanD-1
// stages of kMeanS members ahead (160 loads in flight per lane without holding
// registers), and adds them in ascending member order -- the same sequential
// sum.  The register-pipelined kernel above exposes the full memory latency
// once per group of members, which dominates a large cluster's chain.
constexpr int kMeanS = 32, kMeanD = 6;

__global__ void __launch_bounds__(32) cluster_mean_staged_kernel(int64_t m, int len, const int32_t* __restrict__ mem_ptr,
                                                                 const int32_t* __restrict__ mem,
                                                                 const double* __restrict__ mats,
                                                                 double* __restrict__ reps) {
  __shared__ double buf[kMeanD][kMeanS][32];
  const int64_t j = blockIdx.y;
  const int t = threadIdx.x;
  const int q = blockIdx.x * 32 + t;
  const int32_t lo = mem_ptr[j], hi = mem_ptr[j + 1];
  const int cnt = hi - lo;
  const int nst = (cnt + kMeanS - 1) / kMeanS;
  const bool live = q < len;
  auto issue = [&](int st) {
    // lane t fetches member id t of the stage; the ids reach every lane by
    // shuffle (no dependent L1 load per copy)
    const int c0 = st * kMeanS;
    const int32_t my_id = c0 + t < cnt ? __ldg(mem + lo + c0 + t) : 0;
    const int un = cnt - c0 < kMeanS ? cnt - c0 : kMeanS;
    const unsigned base = (unsigned)__cvta_generic_to_shared(&buf[st % kMeanD][0][t]);
#pragma unroll 8
    for (int u = 0; u < kMeanS; ++u) {
      const int32_t id = __shfl_sync(0xffffffffu, my_id, u);
      if (u < un && live)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(base + u * 32 * 8),
                     "l"(mats + (int64_t)id * len + q)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int st = 0; st < kMeanD - 1; ++st) issue(st);  // (empty groups past the end keep the count uniform)
  double s = 0.0;
  for (int st = 0; st < nst; ++st) {
    issue(st + kMeanD - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(kMeanD - 1) : "memory");
    if (live) {
      const double* b = &buf[st % kMeanD][0][t];
      const int un = cnt - st * kMeanS < kMeanS ? cnt - st * kMeanS : kMeanS;
      for (int u = 0; u < un; ++u) s = __dadd_rn(s, b[u * 32]);
    }
  }
  if (!live) return;
  const double inv = __ddiv_rn(1.0, (double)cnt);
  reps[j * len + q] = __dmul_rn(s, inv);
}

}  // namespace

bool spectral_il_supported(int ps) { return ps == 9 || ps == 22 || ps == 25 || ps == 27; }

int64_t interleaved_len(int64_t count, int width, int64_t len) { return (count + width - 1) / width * width * len; }

void interleave_patches(int64_t count, int64_t len, const double* src, double* dst, cudaStream_t s) {
  const int64_t total = interleaved_len(count, kTileA, len);
  if (total > 0) interleave_kernel<double><<<grid_for(total, 256), 256, 0, s>>>(total, count, kTileA, len, src, dst);
}

void interleave_factors(int64_t count, int ps, const double* lu, const int32_t* piv, double* lu_il, int32_t* piv_il,
                        cudaStream_t s) {
  const int64_t len = (int64_t)ps * ps;
  const int64_t t1 = interleaved_len(count, kTileE, len), t2 = interleaved_len(count, kTileE, ps);
  if (t1 > 0) interleave_kernel<double><<<grid_for(t1, 256), 256, 0, s>>>(t1, count, kTileE, len, lu, lu_il);
  if (t2 > 0) interleave_kernel<int32_t><<<grid_for(t2, 256), 256, 0, s>>>(t2, count, kTileE, ps, piv, piv_il);
}

void spectral_tiled_il(int64_t npat, int64_t ne, int ps, const double* mats_il, const double* lu_il,
                       const int32_t* piv_il, double* d, unsigned long long* iters, cudaStream_t s, KmeansReuse ru) {
  switch (ps) {
    case 9: launch_spectral_tile<9, true>(npat, nullptr, ne, mats_il, lu_il, piv_il, d, iters, s, ru); break;
    case 22: launch_spectral_tile<22, true>(npat, nullptr, ne, mats_il, lu_il, piv_il, d, iters, s, ru); break;
    case 25: launch_spectral_tile<25, true>(npat, nullptr, ne, mats_il, lu_il, piv_il, d, iters, s, ru); break;
    case 27: launch_spectral_tile<27, true>(npat, nullptr, ne, mats_il, lu_il, piv_il, d, iters, s, ru); break;
    default: break;
  }
}


template <int PS>
void launch_spectral_diag(int64_t npat, const double* mats_il, const double* lu, const int32_t* piv, const int32_t* phi,
                          double* d, unsigned long long* iters, cudaStream_t s, KmeansReuse ru, const int32_t* perm) {
  const size_t smem = (size_t)3 * PS * kTileThreads * sizeof(double);
  cudaFuncSetAttribute(spectral_tile_kernel<PS, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ru.ub = nullptr;
  ru.lbq = nullptr;
  spectral_tile_kernel<PS, true, true>
      <<<grid_for(npat, perm ? kTileThreads : 2 * kTileThreads), kTileThreads, smem, s>>>(npat, perm, 1, mats_il, lu,
                                                                                         piv, d, iters, ru, phi);
}

void spectral_diag_il(int64_t npat, int ps, const double* mats_il, const double* lu, const int32_t* piv,
                      const int32_t* phi, double* d, unsigned long long* iters, cudaStream_t s, KmeansReuse ru,
                      const int32_t* perm) {
  if (npat <= 0) return;
  switch (ps) {
    case 9: launch_spectral_diag<9>(npat, mats_il, lu, piv, phi, d, iters, s, ru, perm); break;
    case 22: launch_spectral_diag<22>(npat, mats_il, lu, piv, phi, d, iters, s, ru, perm); break;
    case 25: launch_spectral_diag<25>(npat, mats_il, lu, piv, phi, d, iters, s, ru, perm); break;
    case 27: launch_spectral_diag<27>(npat, mats_il, lu, piv, phi, d, iters, s, ru, perm); break;
    default: break;
  }
}

// dst = the interleaved (width kTileA) copy of items perm[0..count) of src
__global__ void interleave_perm_kernel(int64_t total, int64_t count, int64_t len, const int32_t* __restrict__ perm,
                                       const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int a = (int)(e % kTileA);
  const int64_t q = (e / kTileA) % len, g = e / (kTileA * len);
  const int64_t item = g * kTileA + a;
  dst[e] = item < count ? src[(int64_t)__ldg(perm + item) * len + q] : 0.0;
}

void interleave_patches_perm(int64_t count, int64_t len, const int32_t* perm, const double* src, double* dst,
                             cudaStream_t s) {
  const int64_t total = interleaved_len(count, kTileA, len);
  if (total > 0) interleave_perm_kernel<<<grid_for(total, 256), 256, 0, s>>>(total, count, len, perm, src, dst);
}

void l1_pairs(int64_t npat, const int32_t* pid, int64_t ne, int len, const double* mats, const int32_t* rep_src,
              const double* reps, double* d, cudaStream_t s) {
  if (npat <= 0 || ne <= 0) return;
  if (l1_tiled_enabled()) {
    L1Args a{};
    a.npat = npat, a.pid = pid, a.len = len, a.mats = mats, a.e0 = 0, a.e1 = ne, a.rep_src = rep_src, a.reps = reps;
    a.d = d;
    l1_tile_launch<kL1Pairs>(a, s);
    return;
  }
  dim3 grid(grid_for(npat, kL1Threads), (unsigned)((ne + kL1Ent - 1) / kL1Ent));
  l1_pairs_kernel<<<grid, kL1Threads, 0, s>>>(npat, pid, ne, len, mats, rep_src, reps, d);
}

static int spectral_block(int ps) { return ps <= 40 ? 64 : ps <= 96 ? 32 : 16; }
static size_t spectral_vec_bytes(int ps, int bd) { return (size_t)4 * ps * bd * sizeof(double); }

void spectral_pairs(int64_t npat, const int32_t* pid, int64_t ne, int ps, const double* mats, const double* lu,
                    const int32_t* piv, double* d, unsigned long long* iters, cudaStream_t s, double bound) {
  if (npat <= 0 || ne <= 0) return;
  if (spectral_tiled(npat, pid, ne, ps, mats, lu, piv, d, iters, s, bound)) return;
  const int bd = spectral_block(ps);
  size_t smem = (size_t)ps * ps * sizeof(double) + (size_t)((ps + 1) / 2) * sizeof(double) +
                spectral_vec_bytes(ps, bd);
  const bool stage = smem <= 200 * 1024;
  if (!stage) smem = spectral_vec_bytes(ps, bd);
  cudaFuncSetAttribute(spectral_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(grid_for(npat, bd), (unsigned)ne);
  spectral_pairs_kernel<<<grid, bd, smem, s>>>(npat, pid, ne, ps, mats, lu, piv, d, iters, stage);
}

void spectral_list(int64_t npairs, const int32_t* pa, const int32_t* fb, int ps, const double* mats, const double* lu,
                   const int32_t* piv, double* d, unsigned long long* iters, cudaStream_t s) {
  if (npairs <= 0) return;
  const int bd = spectral_block(ps);
  const size_t smem = spectral_vec_bytes(ps, bd);
  cudaFuncSetAttribute(spectral_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  spectral_list_kernel<<<grid_for(npairs, bd), bd, smem, s>>>(npairs, pa, fb, ps, mats, lu, piv, d, iters);
}

void greedy_resolve(int B, const int32_t* S, const double* D, double eps, int best_match, int64_t abort_above,
                    const int32_t* lu_status, int32_t* phi, int32_t* creators, int32_t* entry_of, int64_t* state,
                    cudaStream_t s) {
  if (B <= 0) return;
  const char* e = getenv("PDB_RESOLVE_BITS");
  if (B <= kResolveMax && !(e && e[0] == '0')) {
    const size_t smem = (size_t)B * 32 * sizeof(uint32_t);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(greedy_resolve_bits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    uint32_t* cand = nullptr;
    PDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cand), smem, s));
    PDB_CUDA(cudaMemsetAsync(cand, 0, smem, s));
    greedy_cand_bits_kernel<<<4 * 148, 256, 0, s>>>(B, D, eps, cand);
    greedy_resolve_bits_kernel<<<1, 1024, smem, s>>>(B, S, D, eps, best_match, abort_above, lu_status, phi, creators,
                                                     entry_of, state, cand);
    PDB_CUDA(cudaFreeAsync(cand, s));
    return;
  }
  greedy_resolve_kernel<<<1, 32, 0, s>>>(B, S, D, eps, best_match, abort_above, lu_status, phi, creators, entry_of,
                                         state);
}

void l1_scan(int64_t nu, const int32_t* pid, int64_t e0, int64_t e1, int len, const double* mats,
             const int32_t* creators, double eps, int best_match, int32_t* phi, double* best_d, cudaStream_t s) {
  if (nu <= 0 || e1 <= e0) return;
  if (l1_tiled_enabled()) {
    L1Args a{};
    a.npat = nu, a.pid = pid, a.len = len, a.mats = mats, a.e0 = e0, a.e1 = e1, a.rep_src = creators;
    a.eps = eps, a.best_match = best_match, a.phi = phi, a.best_d = best_d;
    l1_tile_launch<kL1Scan>(a, s);
    return;
  }
  l1_scan_kernel<<<grid_for(nu, kL1Threads), kL1Threads, 0, s>>>(nu, pid, e0, e1, len, mats, creators, eps, best_match,
                                                                 phi, best_d);
}

void l1_scan_entries(int64_t nu, const int32_t* pid, int64_t id_offset, int64_t e0, int64_t e1, int len,
                     const double* mats, const double* entries, const int32_t* creators, double eps, int best_match,
                     int32_t* phi, double* best_d, cudaStream_t s) {
  if (nu <= 0 || e1 <= e0) return;
  L1Args a{};
  a.npat = nu, a.pid = pid, a.len = len, a.mats = mats, a.e0 = e0, a.e1 = e1, a.reps = entries;
  a.creator = creators, a.id_offset = id_offset;
  a.eps = eps, a.best_match = best_match, a.phi = phi, a.best_d = best_d;
  l1_tile_launch<kL1Scan>(a, s);
}

void apply_scan(int64_t nu, const int32_t* pid, int64_t e0, int64_t ne, const double* d, const int32_t* creators,
                double eps, int best_match, int32_t* phi, double* best_d, cudaStream_t s) {
  if (nu <= 0 || ne <= 0) return;
  apply_scan_kernel<<<grid_for(nu, 256), 256, 0, s>>>(nu, pid, e0, ne, d, creators, eps, best_match, phi, best_d);
}

void argmin_assign(int64_t n, int64_t ne, const double* d, const int32_t* phi, int32_t* new_phi, double* min_dist,
                   int32_t* changed, cudaStream_t s) {
  if (n > 0) argmin_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, ne, d, phi, new_phi, min_dist, changed);
}

void l1_argmin(int64_t n, int64_t ne, int len, const double* mats, const double* reps, const int32_t* phi,
               int32_t* new_phi, double* min_dist, int32_t* changed, cudaStream_t s) {
  if (n > 0 && l1_tiled_enabled()) {
    L1Args a{};
    a.npat = n, a.len = len, a.mats = mats, a.e0 = 0, a.e1 = ne, a.reps = reps;
    a.phi = const_cast<int32_t*>(phi), a.new_phi = new_phi, a.min_dist = min_dist, a.changed = changed;
    l1_tile_launch<kL1Argmin>(a, s);
    return;
  }
  if (n > 0)
    l1_argmin_kernel<<<grid_for(n, kL1Threads), kL1Threads, 0, s>>>(n, ne, len, mats, reps, phi, new_phi, min_dist,
                                                                    changed);
}

// In-order member sums continued from a previous rank's partial (the chain
// fold of entrywise_mean_indexed, dense.cpp:211-223, across ranks): out[j] =
// (init ? init[j] : 0) + members of j in ascending order; with counts (the
// last rank) multiplied by 1 / counts[j] as the reference's mean.
__global__ void cluster_sum_chain_kernel(int64_t m, int len, const int32_t* __restrict__ mem_ptr,
                                         const int32_t* __restrict__ mem, const double* __restrict__ mats,
                                         const double* __restrict__ init, const int64_t* __restrict__ counts,
                                         double* __restrict__ out) {
  const int64_t j = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= len || j >= m) return;
  double s = init ? init[j * len + q] : 0.0;
  const int32_t lo = mem_ptr[j], hi = mem_ptr[j + 1];
  int32_t c = lo;
  for (; c + 8 <= hi; c += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = mats[(int64_t)__ldg(mem + c + u) * len + q];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
  }
  for (; c < hi; ++c) s = __dadd_rn(s, mats[(int64_t)mem[c] * len + q]);
  if (counts) s = __dmul_rn(s, __ddiv_rn(1.0, (double)counts[j]));
  out[j * len + q] = s;
}

void cluster_sum_chain(int64_t m, int len, const int32_t* mem_ptr, const int32_t* mem, const double* mats,
                       const double* init, const int64_t* counts, double* out, cudaStream_t s) {
  if (m <= 0) return;
  cluster_sum_chain_kernel<<<dim3(grid_for(len, 128), (unsigned)m), 128, 0, s>>>(m, len, mem_ptr, mem, mats, init,
                                                                                counts, out);
}

void l1_argmin_ids(int64_t n, const int32_t* pid, int64_t ne, int len, const double* mats, const double* reps,
                   const int32_t* phi, int32_t* new_phi, double* min_dist, int32_t* changed, cudaStream_t s) {
  if (n <= 0) return;
  L1Args a{};
  a.npat = n, a.pid = pid, a.len = len, a.mats = mats, a.e0 = 0, a.e1 = ne, a.reps = reps;
  a.phi = const_cast<int32_t*>(phi), a.new_phi = new_phi, a.min_dist = min_dist, a.changed = changed;
  l1_tile_launch<kL1Argmin>(a, s);
}

void cluster_mean(int64_t m, int len, const int32_t* mem_ptr, const int32_t* mem, const double* mats, double* reps,
                  cudaStream_t s) {
  if (m <= 0) return;
  const char* e = getenv("PDB_MEAN_STAGED");
  if (!(e && e[0] == '0')) {
    cluster_mean_staged_kernel<<<dim3(grid_for(len, 32), (unsigned)m), 32, 0, s>>>(m, len, mem_ptr, mem, mats, reps);
    return;
  }
  dim3 grid(grid_for(len, 128), (unsigned)m);
  cluster_mean_kernel<<<grid, 128, 0, s>>>(m, len, mem_ptr, mem, mats, reps);
}

}  // namespace pdb::k
