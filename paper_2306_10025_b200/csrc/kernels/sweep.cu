// The relaxation sweep x <- x + omega W sum_k V_k^T B_phi(k)^{-1} V_k (b - A x)
// (reference: smooth precond.cpp:90-101, PatchPreconditioner::apply
// precond.cpp:58-88, spmv sparse.cpp:50-63).
//
// Patch stage and scatter (the residual is in spmv.cu):
//   patch_apply_dmma   compressed mode: tiles of <= 32 patches sharing a database
//                      entry, B^{-1} [r_k1 .. r_k32] on the FP64 tensor cores
//   patch_apply_inv    one patch per sub-block with its explicit inverse (exact
//                      mode, small databases); patch_solve: triangular solves
//                      on the LU factors (PDB_APPLY=lu)
//   scatter_update_csr x += omega W sum sols: owner-computes gather through the
//                      DoF -> (patch, slot) inverse map in ascending patch order,
//                      the reference's serial scatter order (precond.cpp:81-86),
//                      no atomics
// plus the setup kernels of these structures (inverses, inverse maps).
#include <algorithm>
#include <cstdlib>
#include <string>

#include <cuda.h>  // CUtensorMap (types only; the encoder is looked up through the runtime)
#include <cub/cub.cuh>

#include "../common.hpp"
#include "../kernels.hpp"
#include "pdl.cuh"

namespace pdb::k {

namespace {

constexpr int kBlock = 256;

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

// Solutions are written in patch order (sols[order[slot] * ps + i]).  Patch
// p's residuals are staged at rk[p * SP + k] with SP = 4 KS (+4 when KS is
// even), so the B-fragment loads of a half-warp (g = 0..3 or 4..7, tg = 0..3)
// fall in 16 distinct 8-byte banks (a stage of stride ps costs a 2-way
// conflict on every fragment load at ps = 25/27: config-3 apply 48.7 ->
// 45 us).  Rows k >= ps are zero in the stage itself, so a zero A entry never
// meets a neighbouring patch's (possibly non-finite) value.
template <int MT, int KS, bool SCALE>
__global__ void __launch_bounds__(MT * 32) patch_apply_dmma_kernel(int ps, const int32_t* __restrict__ tile_entry,
                                                                      const int32_t* __restrict__ tile_start,
                                                                      const int32_t* __restrict__ idx,
                                                                      const int32_t* __restrict__ order,
                                                                      const double* __restrict__ frag,
                                                                      const double* __restrict__ r,
                                                                      const double* __restrict__ in_scale,
                                                                      double* __restrict__ out) {
  constexpr int NTH = MT * 32;
  constexpr int SP = KS * 4 + ((KS & 1) ? 0 : 4);
  constexpr int TOT = kDmmaTile * SP;
  constexpr int ITER = (TOT + NTH - 1) / NTH;
  __shared__ double rk[TOT];
  __shared__ int32_t ko[kDmmaTile];
  const int t = blockIdx.x;
  const int f = __ldg(tile_entry + t);
  const int s0 = __ldg(tile_start + t), cnt = __ldg(tile_start + t + 1) - s0;
  if (threadIdx.x < cnt) ko[threadIdx.x] = __ldg(order + s0 + threadIdx.x);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a[KS];
  const double* fa = frag + ((int64_t)f * MT + w) * (KS * 32) + lane;
#pragma unroll
  for (int q = 0; q < KS; ++q) a[q] = __ldg(fa + q * 32);
  const int32_t* ti = idx + (int64_t)s0 * ps;
  int32_t gi[ITER];
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int e = threadIdx.x + it * NTH;
    const int p = e / SP, k = e - p * SP;
    gi[it] = (e < TOT && p < cnt && k < ps) ? __ldg(ti + p * ps + k) : -1;
  }
  grid_dep_wait();  // r is the residual kernel's output
  grid_dep_trigger();
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int e = threadIdx.x + it * NTH;
    double v = 0.0;
    if (gi[it] >= 0) {
      v = __ldg(r + gi[it]);
      if (SCALE) v *= __ldg(in_scale + gi[it]);
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
      const double* bp = rk + (nt * 8 + g) * SP + tg;
#pragma unroll
      for (int q = 0; q < KS; ++q) dmma_m8n8k4(c0, c1, a[q], bp[q * 4]);
      const int p0 = nt * 8 + 2 * tg;
      if (row < ps) {
        if (p0 < cnt) out[(int64_t)ko[p0] * ps + row] = c0;
        if (p0 + 1 < cnt) out[(int64_t)ko[p0 + 1] * ps + row] = c1;
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

// The same tile product with the entry's inverse staged by TMA.  The fragment
// array is a 2-D tensor: row (f * mt + w) holds warp w's ks * 32 fragment
// values of entry f, so the box {kTmaQ * 32 columns, mt rows} at column
// c * kTmaQ * 32 is k-step chunk c for every warp of the block -- one
// cp.async.bulk.tensor.2d per stage, landing as stage[w][q][lane] (each
// warp's fragment loads are 256 contiguous bytes: no bank conflicts).  The
// ring's first stages are issued before the tile's gathers and before
// griddepcontrol.wait (the inverses do not depend on the residual), so the
// 295 KB stream of a 192-DoF entry overlaps the gather latency instead of
// following it; a stage is refilled by warp 0 once every warp has released
// it (mbarrier full / empty pairs).  Columns past ks * 32 are zero-filled
// by the TMA unit (ks not a multiple of kTmaQ).
constexpr int kTmaQ = 8;         // k-steps per stage
constexpr int kTmaMaxIter = 10;  // gathers per thread: ceil(kstr / mt) <= 10 for 32 < ps <= 256
constexpr int kTmaMaxStages = 4;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

__global__ void __launch_bounds__(1024) patch_apply_dmma_tma_kernel(
    const __grid_constant__ CUtensorMap fmap, int ps, int mt, int ks, int kstr, int nst,
    const int32_t* __restrict__ tile_entry, const int32_t* __restrict__ tile_start,
    const int32_t* __restrict__ tile_idx, const int32_t* __restrict__ order, const double* __restrict__ r,
    const double* __restrict__ in_scale, double* __restrict__ sols) {
  extern __shared__ __align__(128) double dyn[];  // nst stages of mt * kTmaQ * 32, then the residual stage
  __shared__ __align__(8) uint64_t full[kTmaMaxStages], empty[kTmaMaxStages];
  __shared__ int32_t ko[kDmmaTile];
  const int stage_len = mt * kTmaQ * 32;
  double* rk = dyn + (size_t)nst * stage_len;  // kDmmaTile * kstr
  const int t = blockIdx.x;
  const int f = __ldg(tile_entry + t);
  const int s0 = __ldg(tile_start + t), cnt = __ldg(tile_start + t + 1) - s0;
  const int nth = blockDim.x;
  const int nchunks = (ks + kTmaQ - 1) / kTmaQ;
  const unsigned stage_bytes = (unsigned)stage_len * 8u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, (unsigned)mt);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int pre = nchunks < nst ? nchunks : nst;
    for (int c = 0; c < pre; ++c) {
      mbar_expect_tx(full + c, stage_bytes);
      tma_load_2d(dyn + (size_t)c * stage_len, &fmap, c * kTmaQ * 32, f * mt, full + c);
    }
  }
  if ((int)threadIdx.x < cnt) ko[threadIdx.x] = __ldg(order + s0 + threadIdx.x);
  const int32_t* ti = tile_idx + (int64_t)s0 * ps;
  const int tot = kDmmaTile * kstr;
  int32_t gi[kTmaMaxIter];
#pragma unroll
  for (int it = 0; it < kTmaMaxIter; ++it) {
    const int e = threadIdx.x + it * nth;
    const int p = e / kstr, k = e - p * kstr;
    gi[it] = (e < tot && p < cnt && k < ps) ? __ldg(ti + p * ps + k) : -1;
  }
  grid_dep_wait();  // r is the residual kernel's output
  grid_dep_trigger();
#pragma unroll
  for (int it = 0; it < kTmaMaxIter; ++it) {
    const int e = threadIdx.x + it * nth;
    double v = 0.0;
    if (gi[it] >= 0) {
      v = __ldg(r + gi[it]);
      if (in_scale) v *= __ldg(in_scale + gi[it]);
    }
    if (e < tot) rk[e] = v;
  }
  __syncthreads();  // residual stage complete; barrier inits visible to every warp
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tg = lane & 3;
  double c[kDmmaTile / 8][2];
#pragma unroll
  for (int nt = 0; nt < kDmmaTile / 8; ++nt) c[nt][0] = c[nt][1] = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch % nst;
    mbar_wait(full + st, (unsigned)((ch / nst) & 1));
    const double* sa = dyn + (size_t)st * stage_len + w * (kTmaQ * 32) + lane;
    double a[kTmaQ];
#pragma unroll
    for (int q = 0; q < kTmaQ; ++q) a[q] = sa[q * 32];
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);  // the fragments are in registers: the stage may be refilled
    const int kc = ch * kTmaQ;
#pragma unroll
    for (int nt = 0; nt < kDmmaTile / 8; ++nt) {
      if (nt * 8 < cnt) {
        const double* bp = rk + (nt * 8 + g) * kstr + kc * 4 + tg;
#pragma unroll
        for (int q = 0; q < kTmaQ; ++q)
          if (kc + q < ks) dmma_m8n8k4(c[nt][0], c[nt][1], a[q], bp[q * 4]);
      }
    }
    if (threadIdx.x == 0 && ch + nst < nchunks) {  // refill this stage with chunk ch + nst
      mbar_wait(empty + st, (unsigned)((ch / nst) & 1));
      mbar_expect_tx(full + st, stage_bytes);
      tma_load_2d(dyn + (size_t)st * stage_len, &fmap, (ch + nst) * kTmaQ * 32, f * mt, full + st);
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

// Persistent form of the TMA-staged apply: one block per SM walks tiles
// blockIdx.x, + gridDim.x, ...; the residual stage is double-buffered and the
// next tile's gathers are issued as 8-byte cp.async copies (index loads, then
// r -> shared memory, no register round trip) before the current tile's
// products, so the gather latency of tile j + 1 hides behind the tensor-core
// work of tile j; the TMA ring runs across tile boundaries (chunk gc belongs
// to tile gc / nchunks).  With in_scale (the PCG's W^1/2 gather scaling) the
// gathers go through registers instead (scaled before the store).
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

template <int MAXT>
__global__ void __launch_bounds__(MAXT) patch_apply_dmma_tma_persistent_kernel(
    const __grid_constant__ CUtensorMap fmap, int ps, int mt, int ks, int kstr, int nst, int ntiles,
    const int32_t* __restrict__ tile_entry, const int32_t* __restrict__ tile_start,
    const int32_t* __restrict__ tile_idx, const int32_t* __restrict__ order, const double* __restrict__ r,
    const double* __restrict__ in_scale, double* __restrict__ sols) {
  extern __shared__ __align__(128) double dyn[];  // nst stages of mt * kTmaQ * 32, then two residual stages
  __shared__ __align__(8) uint64_t full[kTmaMaxStages], empty[kTmaMaxStages];
  __shared__ int32_t ko[2][kDmmaTile];
  __shared__ int32_t kcnt[2];
  const int stage_len = mt * kTmaQ * 32;
  const int tot = kDmmaTile * kstr;
  double* rk0 = dyn + (size_t)nst * stage_len;
  const int nth = blockDim.x;
  const int nchunks = (ks + kTmaQ - 1) / kTmaQ;
  const unsigned stage_bytes = (unsigned)stage_len * 8u;
  const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int total_chunks = my_tiles * nchunks;
  auto issue = [&](int gc) {  // thread 0: chunk gc of this block's tile sequence into its ring stage
    const int j = gc / nchunks, c = gc - j * nchunks, st = gc % nst;
    const int f = __ldg(tile_entry + blockIdx.x + j * gridDim.x);
    mbar_expect_tx(full + st, stage_bytes);
    tma_load_2d(dyn + (size_t)st * stage_len, &fmap, c * kTmaQ * 32, f * mt, full + st);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, (unsigned)mt);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int pre = total_chunks < nst ? total_chunks : nst;
    for (int gc = 0; gc < pre; ++gc) issue(gc);
  }
  auto gather = [&](int j) {  // tile j's residuals -> stage j & 1 (asynchronously unless scaled)
    const int t = blockIdx.x + j * gridDim.x, buf = j & 1;
    const int s0 = __ldg(tile_start + t), cnt = __ldg(tile_start + t + 1) - s0;
    if (threadIdx.x < kDmmaTile) ko[buf][threadIdx.x] = (int)threadIdx.x < cnt ? __ldg(order + s0 + threadIdx.x) : 0;
    if (threadIdx.x == 0) kcnt[buf] = cnt;
    const int32_t* ti = tile_idx + (int64_t)s0 * ps;
    double* rk = rk0 + (size_t)buf * tot;
    int32_t gi[kTmaMaxIter];
#pragma unroll
    for (int it = 0; it < kTmaMaxIter; ++it) {
      const int e = threadIdx.x + it * nth;
      const int p = e / kstr, k = e - p * kstr;
      gi[it] = (e < tot && p < cnt && k < ps) ? __ldg(ti + p * ps + k) : -1;
    }
#pragma unroll
    for (int it = 0; it < kTmaMaxIter; ++it) {
      const int e = threadIdx.x + it * nth;
      if (e < tot) {
        if (gi[it] < 0)
          rk[e] = 0.0;
        else if (in_scale)
          rk[e] = __ldg(r + gi[it]) * __ldg(in_scale + gi[it]);
        else
          cp_async8(rk + e, r + gi[it]);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  grid_dep_wait();  // r is the residual kernel's output
  grid_dep_trigger();
  gather(0);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tg = lane & 3;
  const int row = w * 8 + g;
  int gc = 0;
  for (int j = 0; j < my_tiles; ++j) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // stage j & 1 complete; every warp is done with tile j - 1 (stage (j + 1) & 1 is free)
    if (j + 1 < my_tiles) gather(j + 1);
    const int buf = j & 1;
    const int cnt = kcnt[buf];
    const double* rk = rk0 + (size_t)buf * tot;
    double c[kDmmaTile / 8][2];
#pragma unroll
    for (int nt = 0; nt < kDmmaTile / 8; ++nt) c[nt][0] = c[nt][1] = 0.0;
    for (int ch = 0; ch < nchunks; ++ch, ++gc) {
      const int st = gc % nst;
      const unsigned par = (unsigned)((gc / nst) & 1);
      mbar_wait(full + st, par);
      const double* sa = dyn + (size_t)st * stage_len + w * (kTmaQ * 32) + lane;
      double a[kTmaQ];
#pragma unroll
      for (int q = 0; q < kTmaQ; ++q) a[q] = sa[q * 32];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);  // the fragments are in registers: the stage may be refilled
      const int kc = ch * kTmaQ;
#pragma unroll
      for (int nt = 0; nt < kDmmaTile / 8; ++nt) {
        if (nt * 8 < cnt) {
          const double* bp = rk + (nt * 8 + g) * kstr + kc * 4 + tg;
#pragma unroll
          for (int q = 0; q < kTmaQ; ++q)
            if (kc + q < ks) dmma_m8n8k4(c[nt][0], c[nt][1], a[q], bp[q * 4]);
        }
      }
      if (threadIdx.x == 0 && gc + nst < total_chunks) {
        mbar_wait(empty + st, par);
        issue(gc + nst);
      }
    }
    if (row < ps) {
#pragma unroll
      for (int nt = 0; nt < kDmmaTile / 8; ++nt) {
        const int p0 = nt * 8 + 2 * tg;
        if (p0 < cnt) sols[(int64_t)ko[buf][p0] * ps + row] = c[nt][0];
        if (p0 + 1 < cnt) sols[(int64_t)ko[buf][p0 + 1] * ps + row] = c[nt][1];
      }
    }
  }
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
  if (x) x[d] = __dadd_rn(__dmul_rn(z, omega_w[d]), x[d]);  // the serial scatter's rounding
}

__global__ void check_count_weights_kernel(int64_t n, double omega, const int32_t* __restrict__ inv_ptr,
                                         const double* __restrict__ omega_w, int32_t* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t cnt = inv_ptr[i + 1] - inv_ptr[i];
  const double w = cnt > 0 ? 1.0 / (double)cnt : 0.0;
  if (omega_w[i] != omega * w) atomicOr(bad, 1);
}

__global__ void scatter_ints_kernel(int64_t count, const int32_t* __restrict__ idx, const int32_t* __restrict__ src,
                                    int32_t* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) dst[idx[t]] = src[t];
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

// Scatter/update: DoF-parallel (owner computes) gather of a DoF's solution
// slots through the inverse map inv_ptr / inv (slots sorted by patch: the
// reference's serial scatter order, precond.cpp:81-86), no atomics.  The
// overlap weight is recomputed from the slot count exactly as
// compute_weights does (patch.cpp:12-20): scale = omega * (1.0 / count) (or
// omega * sqrt(1.0 / count) for the symmetric PCG weighting); setup checks
// that the patch set's weights are exactly that.  kScatterU DoFs per thread
// (blockDim apart, so every load stays coalesced), the slot loads of a DoF
// unrolled to MAXC and independent: all index, then all solution loads are
// in flight together (the kernel is latency-bound on the idx -> sols chain).
// (A padded slot-major map, 4 * MAXC bytes per DoF instead of 4 per slot,
// measured no faster: 37.3 vs 36.4 us at config 3.)

template <int MAXC, int kScatterU>
__global__ void scatter_update_csr_kernel(int64_t n, const int32_t* __restrict__ inv_ptr,
                                          const int32_t* __restrict__ inv, const double* __restrict__ sols,
                                          double omega, bool sym, const double* __restrict__ x_in,
                                          double* __restrict__ z_out, double* __restrict__ x_out) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x * kScatterU + threadIdx.x;
  int32_t lo[kScatterU], cn[kScatterU];
  double xi[kScatterU];
#pragma unroll
  for (int u = 0; u < kScatterU; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    lo[u] = i < n ? __ldcs(inv_ptr + i) : 0;
    cn[u] = i < n ? __ldcs(inv_ptr + i + 1) - lo[u] : 0;
    xi[u] = (x_out && i < n) ? __ldcs(x_in + i) : 0.0;
  }
  int32_t e[kScatterU][MAXC];
#pragma unroll
  for (int u = 0; u < kScatterU; ++u)
#pragma unroll
    for (int c = 0; c < MAXC; ++c) e[u][c] = c < cn[u] ? __ldcs(inv + lo[u] + c) : -1;
  grid_dep_wait();  // sols is the apply kernel's output
  grid_dep_trigger();
  double v[kScatterU][MAXC];
#pragma unroll
  for (int u = 0; u < kScatterU; ++u)
#pragma unroll
    for (int c = 0; c < MAXC; ++c) v[u][c] = e[u][c] >= 0 ? __ldg(sols + e[u][c]) : 0.0;
#pragma unroll
  for (int u = 0; u < kScatterU; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    if (i >= n) break;
    double z = 0.0;
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < cn[u]) z += v[u][c];
    double w = cn[u] > 0 ? 1.0 / (double)cn[u] : 0.0;
    if (sym) w = sqrt(w);
    z = __dmul_rn(z, omega * w);
    if (z_out) z_out[i] = z;
    if (x_out) x_out[i] = __dadd_rn(z, xi[u]);
  }
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

// Explicit inverse for larger patches (ps > 32): one CTA per (factor, block
// of 32 columns), the 32 right-hand sides P e_c held in shared memory
// [ps][33] (lane = column: conflict-free), L and U read as warp-uniform
// broadcasts.  Forward then backward substitution in row blocks of 8: each
// warp takes one row of the block and accumulates the contributions of all
// rows before the block (the dense part), warp 0 finishes the 8 rows in
// order.  Not bit-exact with the thread-per-column kernel (the sweep
// tolerance is 1e-9).
constexpr int kInvWarps = 8;
constexpr int kInvRows = 16;  // rows per block step: two per warp (each loaded X value feeds both)
constexpr int kInvLd = 33;

__global__ void __launch_bounds__(kInvWarps * 32)
    invert_block_kernel(int64_t nf, int ps, const double* __restrict__ lu, const int32_t* __restrict__ piv,
                        double* __restrict__ inv) {
  extern __shared__ double X[];  // [ps][kInvLd]
  double* part = X + (size_t)ps * kInvLd;  // [kInvRows][32]
  const int nb = (ps + 31) / 32;
  const int64_t f = blockIdx.x / nb;
  const int c0 = (int)(blockIdx.x % nb) * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* L = lu + f * (int64_t)ps * ps;
  const int32_t* P = piv + f * ps;
  for (int i = warp; i < ps; i += kInvWarps) X[i * kInvLd + lane] = P[i] == c0 + lane ? 1.0 : 0.0;
  __syncthreads();
  // forward: L y = P e_c (unit lower); rows b0 + w and b0 + 8 + w per warp
  for (int b0 = 0; b0 < ps; b0 += kInvRows) {
    const int i1 = b0 + warp, i2 = b0 + kInvWarps + warp;
    if (i1 < ps) {
      const double* L1 = L + (int64_t)i1 * ps;
      const double* L2 = L + (int64_t)(i2 < ps ? i2 : i1) * ps;
      double s1 = X[i1 * kInvLd + lane], s2 = i2 < ps ? X[i2 * kInvLd + lane] : 0.0, t1 = 0.0, t2 = 0.0;
      int j = 0;
      for (; j + 2 <= b0; j += 2) {
        const double x0 = X[j * kInvLd + lane], x1 = X[(j + 1) * kInvLd + lane];
        s1 -= L1[j] * x0;
        s2 -= L2[j] * x0;
        t1 -= L1[j + 1] * x1;
        t2 -= L2[j + 1] * x1;
      }
      for (; j < b0; ++j) {
        const double x0 = X[j * kInvLd + lane];
        s1 -= L1[j] * x0;
        s2 -= L2[j] * x0;
      }
      part[warp * 32 + lane] = s1 + t1;
      if (i2 < ps) part[(kInvWarps + warp) * 32 + lane] = s2 + t2;
    }
    __syncthreads();
    if (warp == 0)
      for (int r = 0; r < kInvRows && b0 + r < ps; ++r) {
        const int ii = b0 + r;
        const double* Li = L + (int64_t)ii * ps;
        double s = part[r * 32 + lane];
        for (int j = b0; j < ii; ++j) s -= Li[j] * X[j * kInvLd + lane];
        X[ii * kInvLd + lane] = s;
      }
    __syncthreads();
  }
  // backward: U x = y; rows e0 - 1 - w and e0 - 9 - w per warp
  for (int e0 = ps; e0 > 0; e0 -= kInvRows) {  // rows [max(e0 - 16, 0), e0)
    const int lo = e0 - kInvRows > 0 ? e0 - kInvRows : 0;
    const int i1 = e0 - 1 - warp, i2 = e0 - 1 - kInvWarps - warp;
    if (i1 >= lo) {
      const bool two = i2 >= lo;
      const double* U1 = L + (int64_t)i1 * ps;
      const double* U2 = L + (int64_t)(two ? i2 : i1) * ps;
      double s1 = X[i1 * kInvLd + lane], s2 = two ? X[i2 * kInvLd + lane] : 0.0, t1 = 0.0, t2 = 0.0;
      int j = e0;
      for (; j + 2 <= ps; j += 2) {
        const double x0 = X[j * kInvLd + lane], x1 = X[(j + 1) * kInvLd + lane];
        s1 -= U1[j] * x0;
        s2 -= U2[j] * x0;
        t1 -= U1[j + 1] * x1;
        t2 -= U2[j + 1] * x1;
      }
      for (; j < ps; ++j) {
        const double x0 = X[j * kInvLd + lane];
        s1 -= U1[j] * x0;
        s2 -= U2[j] * x0;
      }
      part[(e0 - 1 - i1) * 32 + lane] = s1 + t1;
      if (two) part[(e0 - 1 - i2) * 32 + lane] = s2 + t2;
    }
    __syncthreads();
    if (warp == 0)
      for (int ii = e0 - 1; ii >= lo; --ii) {
        const double* Ui = L + (int64_t)ii * ps;
        double s = part[(e0 - 1 - ii) * 32 + lane];
        for (int j = ii + 1; j < e0; ++j) s -= Ui[j] * X[j * kInvLd + lane];
        X[ii * kInvLd + lane] = s / Ui[ii];
      }
    __syncthreads();
  }
  // column-major output: column c0 + c, rows contiguous
  const int nc = ps - c0 < 32 ? ps - c0 : 32;
  double* out = inv + f * (int64_t)ps * ps + (int64_t)c0 * ps;
  for (int e = threadIdx.x; e < nc * ps; e += kInvWarps * 32) {
    const int c = e / ps, i = e % ps;
    out[(int64_t)c * ps + i] = X[i * kInvLd + c];
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
  z = __dmul_rn(z, omega_w[i]);
  if (z_out) z_out[i] = z;
  if (x_out) x_out[i] = __dadd_rn(z, x_in[i]);
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
    PDB_CUDA(cudaFuncSetAttribute(patch_apply_grouped_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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

// The fragment array as a 2-D FP64 tensor {ks * 32, nf * mt} with boxes {kTmaQ * 32, mt}.
void frag_tensor_map(int64_t nf, int ps, const double* frag, FragTensorMap* out) {
  static_assert(sizeof(CUtensorMap) <= sizeof(FragTensorMap::opaque), "CUtensorMap is 128 bytes");
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  PDB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess)
    fail(Errc::internal, "cuTensorMapEncodeTiled is not available from this driver");
  const int mt = (ps + 7) / 8, ks = (ps + 3) / 4;
  const cuuint64_t dims[2] = {(cuuint64_t)ks * 32, (cuuint64_t)nf * mt};
  const cuuint64_t strides[1] = {(cuuint64_t)ks * 32 * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)kTmaQ * 32, (cuuint32_t)mt};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = reinterpret_cast<Encode>(fn)(
      reinterpret_cast<CUtensorMap*>(out->opaque), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(frag), dims,
      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) fail(Errc::internal, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)rc));
}

void patch_apply_dmma(int ntiles, int ps, const int32_t* tile_entry, const int32_t* tile_start,
                      const int32_t* tile_idx, const int32_t* order, const double* frag,
                      const FragTensorMap* frag_map, const double* r, const double* in_scale, double* sols,
                      cudaStream_t s) {
  if (ntiles <= 0) return;
  const int mt = (ps + 7) / 8, ks = (ps + 3) / 4;
  static const bool no_tma = [] {
    const char* e = getenv("PDB_APPLY_TMA");  // PDB_APPLY_TMA=0: the register-streamed kernel (A/B)
    return e && e[0] == '0';
  }();
  if (ps > 32 && frag_map && !no_tma) {  // run-time shapes, inverse staged by TMA
    int kstr = ks * 4;
    if (kstr % 8 == 0) kstr += 4;
    const size_t stage = (size_t)mt * kTmaQ * 32 * sizeof(double);
    static const bool persistent = [] {
      const char* e = getenv("PDB_APPLY_TMA_PERSISTENT");  // 0: one tile per block (A/B)
      return !(e && e[0] == '0');
    }();
    const size_t rkb = (size_t)kDmmaTile * kstr * sizeof(double) * (persistent ? 2 : 1);
    const int nchunks = (ks + kTmaQ - 1) / kTmaQ;
    int nst = (int)((220 * 1024 - rkb) / stage);
    nst = std::min({nst, kTmaMaxStages, nchunks});
    static const int cap = [] {
      const char* e = getenv("PDB_APPLY_TMA_STAGES");  // ring depth cap (tuning)
      return e ? atoi(e) : 0;
    }();
    if (cap > 0) nst = std::min(nst, cap);
    if (nst < 1 || (kstr + mt - 1) / mt > kTmaMaxIter) fail(Errc::internal, "TMA apply: unsupported patch size");
    const size_t smem = nst * stage + rkb;
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    if (persistent) {
      // up to 24 warps (192 DoFs) the block is compiled for 768 threads (85 registers, no spills)
      auto kern = mt <= 24 ? patch_apply_dmma_tma_persistent_kernel<768> : patch_apply_dmma_tma_persistent_kernel<1024>;
      static size_t opted_p[64][2] = {};
      if (dev >= 64 || smem > opted_p[dev][mt <= 24]) {
        PDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (dev < 64) opted_p[dev][mt <= 24] = smem;
      }
      const int grid = std::min(ntiles, num_sms());
      launch_pdl(kern, dim3((unsigned)grid), dim3(mt * 32), smem, s,
                 *reinterpret_cast<const CUtensorMap*>(frag_map->opaque), ps, mt, ks, kstr, nst, ntiles, tile_entry,
                 tile_start, tile_idx, order, r, in_scale, sols);
      return;
    }
    static size_t opted[64] = {};  // the opt-in is per device: cache the largest size set on each
    if (dev >= 64 || smem > opted[dev]) {
      PDB_CUDA(cudaFuncSetAttribute(patch_apply_dmma_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      if (dev < 64) opted[dev] = smem;
    }
    launch_pdl(patch_apply_dmma_tma_kernel, dim3((unsigned)ntiles), dim3(mt * 32), smem, s,
               *reinterpret_cast<const CUtensorMap*>(frag_map->opaque), ps, mt, ks, kstr, nst, tile_entry, tile_start,
               tile_idx, order, r, in_scale, sols);
    return;
  }
  if (ps > 32) {  // run-time shapes, inverse streamed from L2 through registers
    int kstr = ks * 4;
    if (kstr % 8 == 0) kstr += 4;
    const size_t smem = (size_t)kDmmaTile * kstr * sizeof(double);
    // the opt-in is per device: cache the largest size set on each
    static size_t opted[64] = {};
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    if (smem > 48 * 1024 && (dev >= 64 || smem > opted[dev])) {
      PDB_CUDA(cudaFuncSetAttribute(patch_apply_dmma_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      if (dev < 64) opted[dev] = smem;
    }
    launch_pdl(patch_apply_dmma_large_kernel, dim3((unsigned)ntiles), dim3(mt * 32), smem, s, ps, mt, ks, kstr,
               tile_entry, tile_start, tile_idx, order, frag, r, in_scale, sols);
    return;
  }
#define PDB_DMMA_LAUNCH(KERN, GRID, BLOCK, ...)                                                               \
  launch_pdl(KERN, dim3((unsigned)(GRID)), dim3(BLOCK), 0, s, __VA_ARGS__, tile_entry, tile_start, tile_idx,   \
             order, frag, r, in_scale, sols)
#define PDB_DMMA_CASE(M, K)                                                                                   \
  if (mt == M && ks == K) {                                                                                   \
    if (in_scale)                                                                                             \
      PDB_DMMA_LAUNCH((patch_apply_dmma_kernel<M, K, true>), ntiles, M * 32, ps);                             \
    else                                                                                                      \
      PDB_DMMA_LAUNCH((patch_apply_dmma_kernel<M, K, false>), ntiles, M * 32, ps);                            \
    return;                                                                                                   \
  }
  PDB_DMMA_CASE(1, 1)
  PDB_DMMA_CASE(1, 2)
  PDB_DMMA_CASE(2, 3)
  PDB_DMMA_CASE(2, 4)
  PDB_DMMA_CASE(3, 5)
  PDB_DMMA_CASE(3, 6)
  PDB_DMMA_CASE(4, 7)
  PDB_DMMA_CASE(4, 8)
#undef PDB_DMMA_LAUNCH
#undef PDB_DMMA_CASE
}

void shard_scatter(int64_t count, const int32_t* list, const int32_t* inv_ptr, const int32_t* inv, const double* sols,
                   const double* init, const double* omega_w, double* z_out, double* x, cudaStream_t s) {
  if (count > 0)
    shard_scatter_kernel<<<grid_for(count, kBlock), kBlock, 0, s>>>(count, list, inv_ptr, inv, sols, init, omega_w,
                                                                    z_out, x);
}

void check_count_weights(int64_t n, double omega, const int32_t* inv_ptr, const double* omega_w, int32_t* bad,
                       cudaStream_t s) {
  if (n > 0) check_count_weights_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, omega, inv_ptr, omega_w, bad);
}

void scatter_ints(int64_t count, const int32_t* idx, const int32_t* src, int32_t* dst, cudaStream_t s) {
  if (count > 0) scatter_ints_kernel<<<grid_for(count, kBlock), kBlock, 0, s>>>(count, idx, src, dst);
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

void scatter_update_csr(int64_t n, int maxc, const int32_t* inv_ptr, const int32_t* inv, const double* sols,
                        double omega, bool sym, const double* x_in, double* z_out, double* x_out, cudaStream_t s) {
  if (n <= 0) return;
  // DoFs per thread: 1 with up to 8 slots per DoF (3D cell patches: config 3
  // scatter 33.0 vs 35.2 us at 2, 43.1 at 4), else 2 (config 2: 14.3 vs
  // 14.4 us); PDB_SCATTER_U = 1 / 2 / 4 overrides for A/B runs
  static const int u_env = [] {
    const char* e = getenv("PDB_SCATTER_U");
    return e ? atoi(e) : 0;
  }();
  const int u = u_env == 1 || u_env == 2 || u_env == 4 ? u_env : (maxc > 4 ? 1 : 2);
#define PDB_CSR_CASE(M, U)                                                                                   \
  launch_pdl(scatter_update_csr_kernel<M, U>, dim3(grid_for(n, kBlock * U)), dim3(kBlock), 0, s, n, inv_ptr, \
             inv, sols, omega, sym, x_in, z_out, x_out)
#define PDB_CSR_U(M)              \
  if (u == 1)                     \
    PDB_CSR_CASE(M, 1);           \
  else if (u == 4)                \
    PDB_CSR_CASE(M, 4);           \
  else                            \
    PDB_CSR_CASE(M, 2)
  switch (maxc) {
    case 1: PDB_CSR_U(1); break;
    case 2: PDB_CSR_U(2); break;
    case 3:
    case 4: PDB_CSR_U(4); break;
    default: PDB_CSR_U(8); break;
  }
#undef PDB_CSR_U
#undef PDB_CSR_CASE
}

void invert_factors(int64_t nf, int ps, const double* lu, const int32_t* piv, double* inv, cudaStream_t s) {
  if (nf <= 0) return;
  if (ps <= 32) {
    invert_factors_kernel<<<(unsigned)((nf + 3) / 4), 128, 0, s>>>(nf, ps, lu, piv, inv);
    return;
  }
  const size_t smem = ((size_t)ps * kInvLd + kInvRows * 32) * sizeof(double);  // rows x 33 + 16 x 32
  if (smem > 48 * 1024) {
    static int configured[64] = {};
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && !configured[dev]) {
      PDB_CUDA(cudaFuncSetAttribute(invert_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      configured[dev] = 1;
    }
  }
  const int64_t blocks = nf * ((ps + 31) / 32);
  invert_block_kernel<<<(unsigned)blocks, kInvWarps * 32, smem, s>>>(nf, ps, lu, piv, inv);
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
