// Host-callable launchers for the sm_100a kernels in kernels/*.cu.
// All launchers are asynchronous on the given stream.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "common.hpp"

namespace pdb::k {

// ---- spmv.cu : residual and SpMV ------------------------------------------
// r = b - A x (b may be null: y = A x when negate == false).  When sumsq !=
// null, per-block partial sums of r^2 are written to sumsq[blockIdx]
// (deterministic two-pass norm).
struct SpmvPlan {
  int version = 2;    // 9: SELL-C-sigma (default); 5: CSR warp items; 2: G lanes per row
  int blocks = 0;
  int group = 8;      // v2: lanes per row (power of two <= 32)
  int rows_per_block = 32;
  int entries = 8;    // v2: entries per lane per pass; v9: steps in flight per lane (4 or 8)
  const int32_t* blk_start = nullptr;  // v5: item row starts (nblk + 1 entries)
  const int64_t* blk_base = nullptr;   // v5: row_ptr at each item start
  int nblk = 0;                        // v5: warp items
  // v9: SELL-C-sigma slices (see DeviceCsr)
  const int64_t* sell_off = nullptr;
  const int32_t* sell_row = nullptr;
  const double* sell_val = nullptr;
  const int32_t* sell_col = nullptr;
  int64_t nslices = 0;
  // all rows in column-pattern classes (see DeviceCsr): no column stream
  const int32_t* sell_tab = nullptr;
  const int32_t* sell_tstart = nullptr;
  // half ("mirror") storage (sell_mirror.cpp): own slot t of slice s at
  // sell_off[s] + 32 t + lane; lower entry m of a class-c row at
  // mir_rbase[j] + mir_kslot[tstart[c] + m]
  const int32_t* mir_clo = nullptr;
  const int32_t* mir_rbase = nullptr;
  const int32_t* mir_kslot = nullptr;
  int mir_ntab = 0, mir_ncls = 0;
  int64_t mir_nval = 0;  // values stored
};
constexpr int kSellC = 32;          // rows per SELL slice (one warp)
constexpr int kSellSigma = 8192;    // sorting window (rows)
SpmvPlan spmv_plan(int64_t n, int64_t nnz);
// v5 plan over a warp-item partition (item_partition, built at upload).
SpmvPlan spmv_plan_items(int64_t n, int64_t nnz, const int32_t* item_start, const int64_t* item_base, int nitems);
// Host-side warp items: consecutive rows, <= 31 rows and <= 256 nonzeros (a longer row alone).
std::vector<int32_t> item_partition(int64_t n, const int64_t* row_ptr);
// SELL plans only: r = b - A x on slices [s0, s1) (whole sorting windows, i.e. rows
// [s0 * kSellC, min(s1 * kSellC, n))), plain launch (ordered after events by the caller).
void residual_slices(const SpmvPlan& plan, int64_t s0, int64_t s1, const double* x, const double* b, double* r,
                     cudaStream_t s);
void residual(const SpmvPlan& plan, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
              const double* x, const double* b, double* r, double* block_sumsq, cudaStream_t s);
void spmv(const SpmvPlan& plan, int64_t n, const int64_t* rp, const int32_t* col, const double* val, const double* x,
          double* y, cudaStream_t s);
// Deterministic sum of `count` partials -> out[0] = sqrt(sum) (sqrt_result) or sum.
void finish_sum(const double* partials, int count, double* out, bool sqrt_result, cudaStream_t s);
// y = A x with per-block partial sums of x_i y_i (plan.blocks partials; CG's (p, A p)).
void spmv_dot(const SpmvPlan& plan, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
              const double* x, double* y, double* partials, cudaStream_t s);
// CG building blocks (kernels/blas.cu): dot_partials() partials each.
void dot_partial(int64_t n, const double* a, const double* b, double* partials, cudaStream_t s);
void cg_update(int64_t n, const double* alpha, const double* p, const double* q, const double* x_in, double* x_out,
               double* r, double* partials, cudaStream_t s);  // x_out = x_in + a p, r -= a q, partials of r.r
// !beta: out = num / sum(partials);  beta: out = sum / num, then num = sum.
void finish_ratio(const double* partials, int count, double* num, double* out, bool beta, cudaStream_t s);

// ---- sweep.cu : patch stage and scatter -----------------------------------
// Per-patch gather + LU solve (column-major factors):
//   sols[k*ps + i] = (B_f^{-1} (r .* in_scale)[patch_k])_i,  f = phi ? phi[k] : k; in_scale may be null.
// Reproducible PCG (oracle orc_pcg order): reference-order patch solve on the
// column-major LU, chunk sums of the blocked inner product, unfused axpys
// (mode 0: y += a x, 1: y -= a x, 2: y = x + a y).
void patch_solve_ref(int64_t np, int ps, const int32_t* patches, const double* factors_cm, const int32_t* piv,
                     const int32_t* phi, const double* r, const double* in_scale, double* sols, cudaStream_t s);
void dot_chunks(int64_t n, int chunk, const double* a, const double* b, double* out, cudaStream_t s);
void axpy_ref(int64_t n, double alpha, const double* x, double* y, int mode, cudaStream_t s);
void patch_solve(int64_t np, int ps, const int32_t* patches, const double* factors_cm, const int32_t* piv,
                 const int32_t* phi, const double* r, const double* in_scale, double* sols, cudaStream_t s);
// Same product with explicit column-major inverses Binv (default sweep path).
void patch_apply_inv(int64_t np, int ps, const int32_t* patches, const double* Binv, const int32_t* phi,
                     const double* r, const double* in_scale, double* sols, cudaStream_t s);
// Scatter/update through the compact inverse map (maxc = the largest slot count, <= 8);
// the weight omega*(1/count) (sym: omega*sqrt(1/count)) is recomputed in-kernel.
void scatter_update_csr(int64_t n, int maxc, const int32_t* inv_ptr, const int32_t* inv, const double* sols,
                        double omega, bool sym, const double* x_in, double* z_out, double* x_out, cudaStream_t s);
int grouped_tile(int ps);  // patches per grouped-apply tile
// Cluster-grouped apply: tile t covers tile-order slots [tile_start[t], tile_start[t+1]) sharing entry
// tile_entry[t]; tile_idx holds the patch DoF lists in tile order.  Solutions are written in patch
// order (sols[order[slot] * ps + i]), so a DoF's contributions sit next to its neighbours' in memory.
void patch_apply_grouped(int ntiles, int ps, const int32_t* tile_entry, const int32_t* tile_start,
                         const int32_t* tile_idx, const int32_t* order, const double* Binv, const double* r,
                         const double* in_scale, double* sols, int max_tile, cudaStream_t s);
// Tensor-core grouped apply (FP64 mma.sync m8n8k4, ps <= 32, tiles <= 32 patches): sols_tile =
// B_f^{-1} [r_k1 .. r_k32] with each inverse pre-arranged in A-fragment order by build_frag_inverses.
bool dmma_apply_supported(int ps);
int apply_tile(int ps);  // patches per tile of the grouped apply (32 on the DMMA path)
int64_t frag_len(int ps);  // doubles per entry in fragment order
void build_frag_inverses(int64_t nf, int ps, const double* inv_cm, double* frag, cudaStream_t s);
// Patches above 32 DoFs (config 5: 192): an entry's fragment-ordered inverse (295 KB) does not fit in
// registers, so it is staged through shared memory by TMA (cp.async.bulk.tensor.2d over a tensor map of
// the fragment array: rows = (entry, 8-row block), columns = (k-step, lane)), a ring of 8-k-step stages
// filled ahead of the tile's gathers.  frag_tensor_map encodes the map once per preconditioner.
using ::pdb::FragTensorMap;
void frag_tensor_map(int64_t nf, int ps, const double* frag, FragTensorMap* out);
void patch_apply_dmma(int ntiles, int ps, const int32_t* tile_entry, const int32_t* tile_start,
                      const int32_t* tile_idx, const int32_t* order, const double* frag,
                      const FragTensorMap* frag_map, const double* r, const double* in_scale, double* sols,
                      cudaStream_t s);
void remap_inverse(int64_t count, int ps, const int32_t* slot_of, int32_t* inv, cudaStream_t s);
// Multi-GPU shard helpers: list-driven scatter (see shard.cu), pack / unpack.
void shard_scatter(int64_t count, const int32_t* list, const int32_t* inv_ptr, const int32_t* inv, const double* sols,
                   const double* init, const double* omega_w, double* z_out, double* x, cudaStream_t s);
void gather_vals(int64_t count, const int32_t* idx, const double* src, double* dst, cudaStream_t s);
void scatter_ints(int64_t count, const int32_t* idx, const int32_t* src, int32_t* dst, cudaStream_t s);
// bad = 1 when some omega_w[i] != omega * (1 / patches covering i) (the padded scatter's weight)
void check_count_weights(int64_t n, double omega, const int32_t* inv_ptr, const double* omega_w, int32_t* bad,
                       cudaStream_t s);
void scatter_vals(int64_t count, const int32_t* idx, const double* src, double* dst, cudaStream_t s);
// Binv (column-major) from row-major LU + pivots: column c = lu_solve(e_c).
void invert_factors(int64_t nf, int ps, const double* lu, const int32_t* piv, double* inv, cudaStream_t s);
// z[i] = (sum over (k,l) in inv(i), ascending k, of sols[k*ps+l]) * omega_w[i];
// x_out (may be null): x_out[i] = z[i] + x_in[i] (the smooth() update, precond.cpp:99).
void scatter_update(int64_t n, const int32_t* inv_ptr, const int32_t* inv, const double* sols, const double* omega_w,
                    const double* x_in, double* z_out, double* x_out, cudaStream_t s);

// Sweep-structure setup.
void build_inverse_count(int64_t np, int ps, const int32_t* patches, int32_t* counts, cudaStream_t s);
void build_inverse_fill(int64_t np, int ps, const int32_t* patches, const int32_t* inv_ptr, int32_t* cursor,
                        int32_t* inv, cudaStream_t s);
void sort_inverse_segments(int64_t n, const int32_t* inv_ptr, int32_t* inv, cudaStream_t s);
void transpose_factors(int64_t nf, int ps, const double* lu_rm, double* lu_cm, cudaStream_t s);
void scale_weights(int64_t n, double omega, const double* w, double* omega_w, cudaStream_t s);
void sqrt_weights(int64_t n, double omega, const double* w, double* sw, double* omega_sw, cudaStream_t s);

// ---- detect.cu : matrix-only cell-patch detection --------------------------
void detect_candidates(int64_t n, const int64_t* rp, int64_t ps, uint8_t* cand, int32_t* any, cudaStream_t s);
// For each candidate row listed in rows[0..nrows): consistent[t] (0/1) and hash[t] (FNV-1a of its columns).
void detect_consistency(int64_t nrows, const int32_t* rows, const int64_t* rp, const int32_t* col,
                        const uint8_t* cand, int ps, uint8_t* consistent, uint64_t* hash, cudaStream_t s);
// Positions sorted by (hash, position): keep_by_pos[p] = 0 when an earlier row of the same
// hash run has an identical column set (first occurrence wins), else 1.
void detect_dedupe(int64_t nrows, const uint64_t* hash_sorted, const int32_t* pos_sorted, const int32_t* rows,
                   const int64_t* rp, const int32_t* col, int ps, uint8_t* keep_by_pos, cudaStream_t s);
void iota(int64_t n, int32_t* out, cudaStream_t s);
void gather_patches(int64_t np, const int32_t* rows, const int32_t* order, const int64_t* rp, const int32_t* col,
                    int ps, int32_t* patches, cudaStream_t s);
void cover_weights(int64_t n, int64_t np, int ps, const int32_t* patches, int32_t* cover, double* w, cudaStream_t s);
void patch_fronts(int64_t np, int ps, const int32_t* patches, int32_t* fronts, cudaStream_t s);
// flags[0] |= 1: two sorted keys equal; flags[1] |= 1: order is not the identity
void front_order(int64_t np, const int32_t* key_sorted, const int32_t* order, int32_t* flags, cudaStream_t s);

// ---- extract.cu : batched A_k = V_k A V_k^T ---------------------------------
// ids == null: patches 0..count-1; else patches ids[0..count).
void extract(int64_t count, const int32_t* ids, int ps, const int32_t* patches, const int64_t* rp,
             const int32_t* col, const double* val, double* out, cudaStream_t s);

// ---- lu.cu : bit-exact batched partial-pivot LU (dense.cpp:31-75) ----------
// Factor mats[src[t]] (src == null: t) into lu[t], piv[t]; status[t] = 0 ok,
// else (column+1) of the failing pivot with fail_best[t] = |pivot|.
void lu_batched(int64_t count, int ps, const double* mats, const int32_t* src, double* lu, int32_t* piv,
                int32_t* status, double* fail_best, cudaStream_t s);

// ---- criterion.cu : bit-exact distance criteria ----------------------------
// L1: d[t*ne + e] = sum_q |mats[pid[t]] - reps_e| (sequential q), reps_e = mats[rep_src[e]] (rep_src != null) or reps[e].
void l1_pairs(int64_t npat, const int32_t* pid, int64_t ne, int len, const double* mats, const int32_t* rep_src,
              const double* reps, double* d, cudaStream_t s);
// Spectral: d[t*ne + e] = spectral_distance(mats[pid[t]], factor e) (dense.cpp:154-190).
// iters (may be null) accumulates power iterations (atomic, for work accounting).
// bound > 0 (greedy tolerance): pairs that provably end at d > bound stop early with d = +inf
// (patch sizes of the tiled kernel only; the others always run to convergence).
void spectral_pairs(int64_t npat, const int32_t* pid, int64_t ne, int ps, const double* mats, const double* lu,
                    const int32_t* piv, double* d, unsigned long long* iters, cudaStream_t s, double bound = 0.0);
// Interleaved spectral path (k-means assignment): patches interleaved in groups of 32
// (interleave_patches, once per patch set) and factors in groups of 8 (interleave_factors,
// per Lloyd iteration); then d[t*ne + e] as spectral_pairs with pid = null.
bool spectral_il_supported(int ps);
int64_t interleaved_len(int64_t count, int width, int64_t len);
void interleave_patches(int64_t count, int64_t len, const double* src, double* dst, cudaStream_t s);
void interleave_factors(int64_t count, int ps, const double* lu, const int32_t* piv, double* lu_il, int32_t* piv_il,
                        cudaStream_t s);
// k-means assignment reuse (all optional): ub = per-patch distance to its
// current centroid (pairs whose Rayleigh quotient exceeds
// max(ub^2 (1 + 1e-4), 1e-8) stop with d = +inf: they cannot be the argmin);
// chg = per-entry "centroid changed" flags -- pairs of unchanged centroids
// keep d from the previous launch (exact) or stay +inf when lbq (the quotient
// at which they were pruned) still exceeds the bound; dprev/mfull: the
// previous distance matrix for the DIAG (bound) launch.
struct KmeansReuse {
  const double* ub = nullptr;
  double ubc = 0.0;  // > 0: the same bound for every patch (greedy tolerance), when ub is null
  const int32_t* phi = nullptr;  // current assignment: the pair (i, phi[i]) is ub[i] itself
  const uint8_t* chg = nullptr;
  double* lbq = nullptr;
  const double* dprev = nullptr;
  int64_t mfull = 0;
  int32_t* it_out = nullptr;  // DIAG: power iterations each patch's pair took
  const int32_t* tile_order = nullptr;       // pruned pass: block b works on tile tile_order[b]
  unsigned long long* tile_iters = nullptr;  // ... and adds its power iterations to tile_iters[tile]
  const uint8_t* long_prev = nullptr;  // pruned pass: pair ran > 2 iterations last Lloyd iteration
  uint8_t* long_cur = nullptr;         // ... written for the next one
};
void spectral_tiled_il(int64_t npat, int64_t ne, int ps, const double* mats_il, const double* lu_il,
                       const int32_t* piv_il, double* d, unsigned long long* iters, cudaStream_t s,
                       KmeansReuse ru = KmeansReuse{});
// d[t] = dist(patch t, factor phi[t]) for interleaved patches and plain-layout factors;
// with perm, mats_il holds patches perm[0..npat) in that order, one pair per thread
// (d, phi, dprev, it_out stay indexed by patch).
void spectral_diag_il(int64_t npat, int ps, const double* mats_il, const double* lu, const int32_t* piv,
                      const int32_t* phi, double* d, unsigned long long* iters, cudaStream_t s,
                      KmeansReuse ru = KmeansReuse{}, const int32_t* perm = nullptr);
// Interleaved (width 32) copy of patches perm[0..count) of the plain layout src
// (the sorted copy for spectral_diag_il's perm).
void interleave_patches_perm(int64_t count, int64_t len, const int32_t* perm, const double* src, double* dst,
                             cudaStream_t s);
// Spectral distance of listed (patch, factor) pairs: d[t] = dist(mats[pa[t]], factor fb[t]).
void spectral_list(int64_t npairs, const int32_t* pa, const int32_t* fb, int ps, const double* mats, const double* lu,
                   const int32_t* piv, double* d, unsigned long long* iters, cudaStream_t s);

// Greedy (compress.cpp:40-95) round machinery.
// Sequential resolution of the batch S (size B, ascending patch ids) against
// the entries it creates itself; D is B x B (row a = patch S[a], col b = entry
// made from S[b]).  Outputs: phi for S, new entries appended to creators[] at
// *m, lu_status of S consulted for failures.  state[0] = m (in/out),
// state[1] = abort flag, state[2] = error batch index (-1 none).
void greedy_resolve(int B, const int32_t* S, const double* D, double eps, int best_match, int64_t abort_above,
                    const int32_t* lu_status, int32_t* phi, int32_t* creators, int32_t* entry_of_batch,
                    int64_t* state, cudaStream_t s);
// First-match / best-match scan of unresolved patches against entries [e0,e1)
// (L1 flavour, reps are patch matrices of creators).  For first-match,
// phi[pid] = first j with d < eps; best-match tracks (best_d, best_j) over
// entries with creator < patch.
// l1_scan with the entries' matrices in their own array (entries + e*len) and
// creator ids in the numbering pid[t] + id_offset (distributed greedy)
void l1_scan_entries(int64_t nu, const int32_t* pid, int64_t id_offset, int64_t e0, int64_t e1, int len,
                     const double* mats, const double* entries, const int32_t* creators, double eps, int best_match,
                     int32_t* phi, double* best_d, cudaStream_t s);
void l1_scan(int64_t nu, const int32_t* pid, int64_t e0, int64_t e1, int len, const double* mats,
             const int32_t* creators, double eps, int best_match, int32_t* phi, double* best_d, cudaStream_t s);
// Apply a precomputed distance block d[t*ne + e] (entries e0+e) to the match state.
void apply_scan(int64_t nu, const int32_t* pid, int64_t e0, int64_t ne, const double* d, const int32_t* creators,
                double eps, int best_match, int32_t* phi, double* best_d, cudaStream_t s);

// k-means (compress.cpp:138-262).
// argmin over e of d[t*ne+e] (strict <, lowest e wins): new_phi[t], min_dist[t]; changed flag set when != phi[t].
void argmin_assign(int64_t n, int64_t ne, const double* d, const int32_t* phi, int32_t* new_phi, double* min_dist,
                   int32_t* changed, cudaStream_t s);
// L1 argmin without materialising d (entries tiled through shared memory).
void l1_argmin(int64_t n, int64_t ne, int len, const double* mats, const double* reps, const int32_t* phi,
               int32_t* new_phi, double* min_dist, int32_t* changed, cudaStream_t s);
// In-order entrywise mean of each cluster (dense.cpp:211-223): members CSR (ascending).
void cluster_sum_chain(int64_t m, int len, const int32_t* mem_ptr, const int32_t* mem, const double* mats,
                       const double* init, const int64_t* counts, double* out, cudaStream_t s);
// l1 argmin (strict <) of the listed patch rows pid[t] against ne entries
void l1_argmin_ids(int64_t n, const int32_t* pid, int64_t ne, int len, const double* mats, const double* reps,
                   const int32_t* phi, int32_t* new_phi, double* min_dist, int32_t* changed, cudaStream_t s);
void cluster_mean(int64_t m, int len, const int32_t* mem_ptr, const int32_t* mem, const double* mats, double* reps,
                  cudaStream_t s);

// ---- cluster.cu : clustering data movement ---------------------------------
// masks[k*words + w] bit b: local row 64w+b of patch k holds exactly one value != 0.0.
void boundary_masks(int64_t np, int ps, const double* mats, int words, unsigned long long* masks, cudaStream_t s);
void gather_mats(int64_t count, const int32_t* ids, int64_t len, const double* src, double* dst, cudaStream_t s);
void gather_i32(int64_t count, const int32_t* ids, int64_t len, const int32_t* src, int32_t* dst, cudaStream_t s);

// ---- blas.cu : deterministic vector kernels for the Krylov drivers ---------
// out[0] = dot(a, b) via fixed two-level reduction (partials scratch >= dot_partials()).
int dot_partials();
void dot(int64_t n, const double* a, const double* b, double* partials, double* out, cudaStream_t s);
void axpy(int64_t n, const double* alpha, bool negate, const double* x, double* y, cudaStream_t s);  // y += (+-)alpha[0]*x
void xpay(int64_t n, const double* x, const double* beta, double* y, cudaStream_t s);                // y = x + beta[0]*y
void axpy_val(int64_t n, double a, const double* x, double* y, cudaStream_t s);                      // y += a*x
void div_scalar(int64_t n, const double* x, double sc, double* y, cudaStream_t s);                   // y = x / sc
void sub(int64_t n, const double* a, const double* b, double* y, cudaStream_t s);                    // y = a - b
void scalar_div(const double* a, const double* b, double* out, cudaStream_t s);                       // out = a/b (device scalars)
// Modified Gram-Schmidt step of the Arnoldi process in ONE cooperative launch:
// for i = 0..j: h[i] = (w, v_i), w -= h[i] v_i; then h[j+1] = (w, w).  The
// vector stays in registers across the j+2 grid-wide reductions.  Returns
// false (nothing launched) when n is too large for the register-resident form.
bool mgs_fused(int64_t n, int j, const double* V, int64_t ldv, double* w, double* h, cudaStream_t s);

}  // namespace pdb::k
