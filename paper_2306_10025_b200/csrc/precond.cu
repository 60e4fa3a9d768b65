// Patch preconditioner setup and application (reference
// PatchPreconditioner::{exact,compressed,apply} precond.cpp:11-88, smooth
// precond.cpp:90-101).
//
// Setup converts the database (reference row-major LU layout) into the sweep
// layout: column-major factors, int32 pivots, omega*W, and the DoF ->
// (patch, slot) inverse map sorted by patch so the gather-side scatter adds
// in the reference's ascending-k order.
#include <cstdlib>
#include <string>

#include <cub/cub.cuh>

#include "host.hpp"
#include "kernels.hpp"

namespace pdb {

bool use_dmma_apply(int ps);

// DoF -> solution-slot inverse map.  Entries are first k*ps + l sorted by k
// (the reference's scatter order, precond.cpp:81-86); remapped to
// slot_of[k]*ps + l only for callers that store solutions in tile order.
void build_inverse(pdb_precond_s& pc, cudaStream_t s, const int32_t* slot_of) {
  const int64_t n = pc.n;
  pc.inv_ptr.alloc(static_cast<size_t>(n + 1));
  pc.inv.alloc(static_cast<size_t>(std::max<int64_t>(pc.np * pc.ps, 1)));
  Scratch<int32_t> counts(static_cast<size_t>(n + 1), s);
  PDB_CUDA(cudaMemsetAsync(counts.get(), 0, (n + 1) * sizeof(int32_t), s));
  k::build_inverse_count(pc.np, static_cast<int>(pc.ps), pc.patches.get(), counts.get(), s);
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, counts.get(), pc.inv_ptr.get(), n + 1, s);
  Scratch<unsigned char> tmp(bytes, s);
  cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, counts.get(), pc.inv_ptr.get(), n + 1, s);
  PDB_CUDA(cudaMemsetAsync(counts.get(), 0, (n + 1) * sizeof(int32_t), s));
  k::build_inverse_fill(pc.np, static_cast<int>(pc.ps), pc.patches.get(), pc.inv_ptr.get(), counts.get(),
                        pc.inv.get(), s);
  k::sort_inverse_segments(n, pc.inv_ptr.get(), pc.inv.get(), s);
  if (slot_of) k::remap_inverse(pc.np * pc.ps, static_cast<int>(pc.ps), slot_of, pc.inv.get(), s);
  PDB_LAUNCH_CHECK();
  // largest slot count: the templated scatter handles up to 8 (cell patches)
  Scratch<int32_t> maxc(1, s);
  size_t mb = 0;
  cub::DeviceReduce::Max(nullptr, mb, counts.get(), maxc.get(), n, s);
  Scratch<unsigned char> mtmp(mb, s);
  // counts was consumed as the fill cursor: it now holds the final per-DoF counts
  cub::DeviceReduce::Max(mtmp.get(), mb, counts.get(), maxc.get(), n, s);
  int32_t mh = 0;
  PDB_CUDA(cudaMemcpyAsync(&mh, maxc.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync(s);
  pc.maxc = 0;
  if (mh <= 8) {
    pc.maxc = mh <= 1 ? 1 : mh <= 2 ? 2 : mh <= 4 ? 4 : 8;
    // the templated scatter recomputes omega * (1 / count); keep it only when
    // the patch set's weights are exactly that (detect_patches' compute_weights)
    if (pc.omega_w.get()) {
      Scratch<int32_t> bad(1, s);
      PDB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int32_t), s));
      k::check_count_weights(n, pc.omega, pc.inv_ptr.get(), pc.omega_w.get(), bad.get(), s);
      int32_t bh = 0;
      PDB_CUDA(cudaMemcpyAsync(&bh, bad.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      sync(s);
      if (bh) pc.maxc = 0;
    }
  }
}

namespace {

void scatter_stage(const pdb_precond_s& pc, const double* sols, bool symmetric, const double* x_in, double* z_out,
                   double* x_out, cudaStream_t s) {
  if (pc.maxc > 0)
    k::scatter_update_csr(pc.n, pc.maxc, pc.inv_ptr.get(), pc.inv.get(), sols, pc.omega, symmetric, x_in, z_out,
                          x_out, s);
  else
    k::scatter_update(pc.n, pc.inv_ptr.get(), pc.inv.get(), sols, symmetric ? pc.omega_sw.get() : pc.omega_w.get(),
                      x_in, z_out, x_out, s);
}

}  // namespace

void common_setup(const pdb_patchset_s& ps, double omega, pdb_precond_s& pc, cudaStream_t s) {
  require(ps.np * ps.ps < (int64_t{1} << 31), Errc::invalid_argument, "patch set too large for 32-bit slot ids");
  pc.n = ps.n;
  pc.np = ps.np;
  pc.ps = ps.ps;
  pc.omega = omega;
  pc.patches.alloc(static_cast<size_t>(ps.np * ps.ps));
  PDB_CUDA(cudaMemcpyAsync(pc.patches.get(), ps.patches.get(), ps.np * ps.ps * sizeof(int32_t),
                           cudaMemcpyDeviceToDevice, s));
  pc.omega_w.alloc(static_cast<size_t>(std::max<int64_t>(ps.n, 1)));
  k::scale_weights(ps.n, omega, ps.weights.get(), pc.omega_w.get(), s);
  pc.sqrt_w.alloc(static_cast<size_t>(std::max<int64_t>(ps.n, 1)));
  pc.omega_sw.alloc(static_cast<size_t>(std::max<int64_t>(ps.n, 1)));
  k::sqrt_weights(ps.n, omega, ps.weights.get(), pc.sqrt_w.get(), pc.omega_sw.get(), s);
}

namespace {

// Sweep factor layout: explicit column-major inverses (default) or the
// column-major LU for the triangular-solve kernel (PDB_APPLY=lu).
bool use_lu_apply() {
  const char* e = getenv("PDB_APPLY");
  return e && std::string(e) == "lu";
}

void set_factors(pdb_precond_s& pc, int64_t nf, int ps, const double* lu_rm, const int32_t* piv, cudaStream_t s) {
  pc.nf = nf;
  pc.lu_apply = use_lu_apply();
  pc.factors.alloc(static_cast<size_t>(nf * ps * ps));
  if (pc.lu_apply)
    k::transpose_factors(nf, ps, lu_rm, pc.factors.get(), s);
  else
    k::invert_factors(nf, ps, lu_rm, piv, pc.factors.get(), s);
  pc.piv.alloc(static_cast<size_t>(nf * ps));
  PDB_CUDA(cudaMemcpyAsync(pc.piv.get(), piv, nf * ps * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  PDB_LAUNCH_CHECK();
}

// Patches grouped by database entry (stable: ascending k inside a group) and
// cut into tiles of at most kTile patches; one block applies one tile.
void build_tiles(pdb_precond_s& pc, const std::vector<int32_t>& phi, cudaStream_t s) {
  const int kTile = use_dmma_apply(static_cast<int>(pc.ps)) ? k::apply_tile(static_cast<int>(pc.ps))
                                                            : k::grouped_tile(static_cast<int>(pc.ps));
  std::vector<int32_t> count(static_cast<size_t>(pc.nf), 0);
  for (int32_t j : phi) ++count[static_cast<size_t>(j)];
  std::vector<int32_t> start(static_cast<size_t>(pc.nf + 1), 0);
  for (int64_t j = 0; j < pc.nf; ++j) start[static_cast<size_t>(j + 1)] = start[static_cast<size_t>(j)] + count[static_cast<size_t>(j)];
  std::vector<int32_t> order(phi.size()), cursor(start.begin(), start.end() - 1);
  for (size_t k = 0; k < phi.size(); ++k) order[static_cast<size_t>(cursor[static_cast<size_t>(phi[k])]++)] = static_cast<int32_t>(k);
  std::vector<int32_t> te, ts;
  for (int64_t j = 0; j < pc.nf; ++j)
    for (int32_t a = start[static_cast<size_t>(j)]; a < start[static_cast<size_t>(j + 1)]; a += kTile) {
      te.push_back(static_cast<int32_t>(j));
      ts.push_back(a);
    }
  ts.push_back(static_cast<int32_t>(phi.size()));
  pc.ntiles = static_cast<int>(te.size());
  pc.max_tile = kTile;
  std::vector<int32_t> slot_of(order.size());
  for (size_t q = 0; q < order.size(); ++q) slot_of[static_cast<size_t>(order[q])] = static_cast<int32_t>(q);
  pc.order.alloc(order.size());
  pc.order.upload(order.data(), order.size(), s);
  pc.slot_of.alloc(slot_of.size());
  pc.slot_of.upload(slot_of.data(), slot_of.size(), s);
  pc.tile_entry.alloc(te.size());
  pc.tile_entry.upload(te.data(), te.size(), s);
  pc.tile_start.alloc(ts.size());
  pc.tile_start.upload(ts.data(), ts.size(), s);
  // patch DoF lists in tile order
  pc.tile_idx.alloc(static_cast<size_t>(pc.np * pc.ps));
  k::gather_i32(pc.np, pc.order.get(), pc.ps, pc.patches.get(), pc.tile_idx.get(), s);
  PDB_LAUNCH_CHECK();
  sync(s);
}

// Grouping pays when entries are shared: by default only with >= 4 patches
// per entry on average (an identity-phi database keeps the per-patch kernel,
// so Exact == Compressed holds bit for bit).  PDB_GROUPED=0/1 forces it.
bool use_grouped_apply(int64_t np, int64_t nf, int ps) {
  // the CUDA-core tile kernel stages B^{-1} and the tile's residuals in shared memory
  const bool fits = k::dmma_apply_supported(ps) ||
                    (static_cast<size_t>(ps) * ps + static_cast<size_t>(k::grouped_tile(ps)) * ps) * sizeof(double) <=
                        200 * 1024;
  if (!fits) return false;
  const char* e = getenv("PDB_GROUPED");
  if (e) return std::string(e) != "0";
  return np >= 4 * nf;
}

// Tensor-core (DMMA) tiles for ps <= 32 unless PDB_DMMA=0.
}  // namespace

bool use_dmma_apply(int ps) {
  const char* e = getenv("PDB_DMMA");
  return k::dmma_apply_supported(ps) && !(e && std::string(e) == "0");
}


// Solution scratch (patch order).
int64_t sols_len(const pdb_precond_s& pc) { return std::max<int64_t>(pc.np * pc.ps, 1); }

// sols_k = B_phi(k)^{-1} (r .* in_scale)|_k for every patch.
void patch_stage(const pdb_precond_s& pc, const double* r, const double* in_scale, double* sols, cudaStream_t s) {
  const int32_t* phi = pc.compressed ? pc.phi.get() : nullptr;
  if (!pc.lu_apply && pc.compressed && pc.ntiles > 0 && pc.frag.get() && use_dmma_apply(static_cast<int>(pc.ps)))
    k::patch_apply_dmma(pc.ntiles, static_cast<int>(pc.ps), pc.tile_entry.get(), pc.tile_start.get(),
                        pc.tile_idx.get(), pc.order.get(), pc.frag.get(), pc.has_frag_map ? &pc.frag_map : nullptr, r,
                        in_scale, sols, s);
  else if (!pc.lu_apply && pc.compressed && pc.ntiles > 0)
    k::patch_apply_grouped(pc.ntiles, static_cast<int>(pc.ps), pc.tile_entry.get(), pc.tile_start.get(),
                           pc.tile_idx.get(), pc.order.get(), pc.factors.get(), r, in_scale, sols, pc.max_tile, s);
  else if (pc.lu_apply)
    k::patch_solve(pc.np, static_cast<int>(pc.ps), pc.patches.get(), pc.factors.get(), pc.piv.get(), phi, r,
                   in_scale, sols, s);
  else
    k::patch_apply_inv(pc.np, static_cast<int>(pc.ps), pc.patches.get(), pc.factors.get(), phi, r, in_scale, sols,
                       s);
}

// Exact (all-patch) preconditioner, streamed in chunks of patches: extract,
// LU (bit-exact, dense.cpp:31-75) and invert each chunk straight into the
// factor array, so the transient memory is two chunks rather than three
// copies of every patch matrix (config 5: 295 KB per 192-DoF patch).  The
// first singular patch in ascending order fails the setup with the
// reference's "patch k: ..." message, as exact_database (compress.cpp:99-114).
void precond_exact(const DeviceCsr& a, const pdb_patchset_s& ps, double omega, pdb_precond_s& pc, cudaStream_t s) {
  require_device();
  require(ps.n == a.n, Errc::dimension_mismatch, "patch set weights do not match the matrix size");
  require(ps.np >= 1, Errc::invalid_argument, "exact_database needs at least one patch");
  const int p = static_cast<int>(ps.ps);
  const int64_t len = static_cast<int64_t>(p) * p;
  common_setup(ps, omega, pc, s);
  build_inverse(pc, s);
  pc.compressed = false;
  pc.nf = ps.np;
  pc.lu_apply = use_lu_apply();
  pc.factors.alloc(static_cast<size_t>(ps.np * len));
  pc.piv.alloc(static_cast<size_t>(ps.np * p));
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(ps.np, (int64_t{1} << 31) / (len * 8)));  // ~2 GB
  DevBuf<double> mats(static_cast<size_t>(chunk * len)), lu(static_cast<size_t>(chunk * len));
  DevBuf<int32_t> status(static_cast<size_t>(chunk));
  DevBuf<double> best(static_cast<size_t>(chunk));
  for (int64_t k0 = 0; k0 < ps.np; k0 += chunk) {
    const int64_t c = std::min(chunk, ps.np - k0);
    k::extract(c, nullptr, p, ps.patches.get() + k0 * p, a.row_ptr.get(), a.col.get(), a.val.get(), mats.get(), s);
    k::lu_batched(c, p, mats.get(), nullptr, lu.get(), pc.piv.get() + k0 * p, status.get(), best.get(), s);
    PDB_LAUNCH_CHECK();
    const std::vector<int32_t> st = status.to_host(s);
    for (int64_t t = 0; t < c; ++t)
      if (st[static_cast<size_t>(t)] != 0) {
        const std::vector<double> bh = best.to_host(s);
        fail(Errc::singular_matrix, "patch " + std::to_string(k0 + t) + ": " +
                                        singular_msg(st[static_cast<size_t>(t)], bh[static_cast<size_t>(t)]));
      }
    if (pc.lu_apply)
      k::transpose_factors(c, p, lu.get(), pc.factors.get() + k0 * len, s);
    else
      k::invert_factors(c, p, lu.get(), pc.piv.get() + k0 * p, pc.factors.get() + k0 * len, s);
    PDB_LAUNCH_CHECK();
  }
  sync(s);
}

static void precond_compressed_impl(const pdb_patchset_s& ps, const pdb_database_s& db, double omega,
                                    pdb_precond_s& pc, cudaStream_t s, bool check_onto);

void precond_compressed(const pdb_patchset_s& ps, const pdb_database_s& db, double omega, pdb_precond_s& pc,
                        cudaStream_t s) {
  precond_compressed_impl(ps, db, omega, pc, s, true);
}

// A shard's patches need not reference every database entry.
void precond_compressed_shard(const pdb_patchset_s& ps, const pdb_database_s& db, double omega, pdb_precond_s& pc,
                              cudaStream_t s) {
  precond_compressed_impl(ps, db, omega, pc, s, false);
}

static void precond_compressed_impl(const pdb_patchset_s& ps, const pdb_database_s& db, double omega,
                                    pdb_precond_s& pc, cudaStream_t s, bool check_onto) {
  require_device();
  require(db.np == ps.np, Errc::dimension_mismatch, "database does not cover the patch set");
  // phi onto the database (Database::phi_onto, compress.cpp:3-10)
  const std::vector<int32_t> phi = db.phi.to_host(s);
  if (!check_onto)  // shards: not onto, but out-of-range ids must never reach the apply kernels
    for (int32_t j : phi)
      require(j >= 0 && j < db.m, Errc::invalid_argument, "assignment map entry outside the database");
  if (check_onto) {
    std::vector<char> hit(static_cast<size_t>(db.m), 0);
    bool ok = true;
    for (int32_t j : phi) {
      if (j < 0 || j >= db.m) {
        ok = false;
        break;
      }
      hit[static_cast<size_t>(j)] = 1;
    }
    for (char h : hit) ok = ok && h;
    require(ok, Errc::invalid_argument, "assignment map must be onto the database");
  }
  require(db.ps == ps.ps, Errc::dimension_mismatch, "database entry dimension does not match the patch size");
  TraceScope tr_all("precond_compressed after phi check", s);
  common_setup(ps, omega, pc, s);
  pc.compressed = true;
  set_factors(pc, db.m, static_cast<int>(ps.ps), db.lu.get(), db.piv.get(), s);
  pc.phi.alloc(static_cast<size_t>(ps.np));
  PDB_CUDA(cudaMemcpyAsync(pc.phi.get(), db.phi.get(), ps.np * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if (!pc.lu_apply && use_grouped_apply(ps.np, db.m, static_cast<int>(ps.ps))) {
    {
      TraceScope tr("build_tiles", s);
      build_tiles(pc, phi, s);  // tiles in entry order; solutions stay in patch order
    }
    TraceScope tr("build_inverse", s);
    build_inverse(pc, s);
    if (use_dmma_apply(static_cast<int>(ps.ps))) {
      pc.frag.alloc(static_cast<size_t>(db.m * k::frag_len(static_cast<int>(ps.ps))));
      k::build_frag_inverses(db.m, static_cast<int>(ps.ps), pc.factors.get(), pc.frag.get(), s);
      if (ps.ps > 32) {
        k::frag_tensor_map(db.m, static_cast<int>(ps.ps), pc.frag.get(), &pc.frag_map);
        pc.has_frag_map = true;
      }
    }
  } else {
    build_inverse(pc, s);
  }
  PDB_LAUNCH_CHECK();
  sync(s);
}

void precond_apply_device(const pdb_precond_s& pc, const double* r, double* z, cudaStream_t s, bool symmetric,
                          bool reference_order) {
  Scratch<double> sols(static_cast<size_t>(sols_len(pc)), s);
  if (reference_order) {
    require(pc.lu_apply, Errc::invalid_argument,
            "reproducible mode needs the LU factors (preconditioner created with PDB_APPLY=lu)");
    k::patch_solve_ref(pc.np, static_cast<int>(pc.ps), pc.patches.get(), pc.factors.get(), pc.piv.get(),
                       pc.compressed ? pc.phi.get() : nullptr, r, symmetric ? pc.sqrt_w.get() : nullptr, sols.get(), s);
  } else {
    patch_stage(pc, r, symmetric ? pc.sqrt_w.get() : nullptr, sols.get(), s);
  }
  scatter_stage(pc, sols.get(), symmetric, nullptr, z, nullptr, s);
  if (pc.coarse) coarse_correct(*pc.coarse, r, z, s);  // combo: z += P0 Ac^{-1} R0 r
  PDB_LAUNCH_CHECK();
}

void relax_device(const DeviceCsr& a, const pdb_precond_s& pc, const double* b, double* x, int64_t sweeps,
                  double* history, cudaStream_t s) {
  require(pc.n == a.n, Errc::dimension_mismatch, "smooth length mismatch");
  const k::SpmvPlan plan = plan_of(a);
  Scratch<double> r(static_cast<size_t>(std::max<int64_t>(a.n, 1)), s);
  Scratch<double> sols(static_cast<size_t>(sols_len(pc)), s);
  double* const r_ptr = r.get();
  double* const sols_ptr = sols.get();
  Scratch<double> partials(static_cast<size_t>(std::max(plan.blocks, 1)), s);
  // combo: x + (patch term + coarse term), the reference's z += x order
  Scratch<double> z(pc.coarse ? static_cast<size_t>(std::max<int64_t>(a.n, 1)) : 1, s);
  for (int64_t sw = 0; sw <= sweeps; ++sw) {
    if (sw == sweeps && !history) break;
    k::residual(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, b, r_ptr, history ? partials.get() : nullptr,
                s);
    if (history) k::finish_sum(partials.get(), plan.blocks, history + sw, true, s);
    if (sw == sweeps) break;
    patch_stage(pc, r_ptr, nullptr, sols_ptr, s);
    if (pc.coarse) {
      scatter_stage(pc, sols_ptr, false, nullptr, z.get(), nullptr, s);
      coarse_correct(*pc.coarse, r_ptr, z.get(), s);
      k::axpy_val(a.n, 1.0, z.get(), x, s);
    } else {
      scatter_stage(pc, sols_ptr, false, x, nullptr, x, s);
    }
  }
  PDB_LAUNCH_CHECK();
}

// pdb_relax with host vectors.  With the SELL residual the first sweep is
// pipelined against the host link: x is copied first, b follows in chunks of
// whole sorting windows on a copy stream, and the residual of each chunk
// starts as soon as its rows of b have landed, so the b transfer hides the
// residual.  Remaining sweeps run as relax_device; x is copied back at the end.
void relax_host(const DeviceCsr& a, const pdb_precond_s& pc, const double* b_h, double* x_h, int64_t sweeps,
                double* history_h, cudaStream_t s) {
  require(pc.n == a.n, Errc::dimension_mismatch, "smooth length mismatch");
  const size_t n = static_cast<size_t>(a.n);
  Scratch<double> db(std::max<size_t>(n, 1), s), dx(std::max<size_t>(n, 1), s);
  const k::SpmvPlan plan = plan_of(a);
  const char* e = getenv("PDB_PIPELINE");
  const bool pipelined = plan.version == 9 && !a.win_slice.empty() && sweeps >= 1 && history_h == nullptr && n > 0 && !pc.coarse &&
                         !(e && std::string(e) == "0");
  if (!pipelined) {
    Scratch<double> dh(static_cast<size_t>(sweeps + 1), s);
    PDB_CUDA(cudaMemcpyAsync(db.get(), b_h, n * sizeof(double), cudaMemcpyHostToDevice, s));
    PDB_CUDA(cudaMemcpyAsync(dx.get(), x_h, n * sizeof(double), cudaMemcpyHostToDevice, s));
    relax_device(a, pc, db.get(), dx.get(), sweeps, history_h ? dh.get() : nullptr, s);
    PDB_CUDA(cudaMemcpyAsync(x_h, dx.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (history_h)
      PDB_CUDA(cudaMemcpyAsync(history_h, dh.get(), static_cast<size_t>(sweeps + 1) * sizeof(double),
                               cudaMemcpyDeviceToHost, s));
    sync(s);
    return;
  }
  static thread_local cudaStream_t cs_of[64] = {};  // per device (a stream belongs to one device)
  int dev = 0;
  PDB_CUDA(cudaGetDevice(&dev));
  require(dev < 64, Errc::internal, "device ordinal beyond the per-device caches");
  cudaStream_t& cs = cs_of[dev];
  if (!cs) PDB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  const int64_t nwin = (a.n + k::kSellSigma - 1) / k::kSellSigma;
  const int64_t chunks = std::min<int64_t>(8, nwin);
  std::vector<cudaEvent_t> ev(static_cast<size_t>(chunks + 2));
  for (auto& ee : ev) PDB_CUDA(cudaEventCreateWithFlags(&ee, cudaEventDisableTiming));
  PDB_CUDA(cudaEventRecord(ev[0], s));  // scratch allocations are ordered on s
  PDB_CUDA(cudaStreamWaitEvent(cs, ev[0], 0));
  PDB_CUDA(cudaMemcpyAsync(dx.get(), x_h, n * sizeof(double), cudaMemcpyHostToDevice, cs));
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t w0 = nwin * c / chunks, w1 = nwin * (c + 1) / chunks;
    const int64_t r0 = w0 * k::kSellSigma, r1 = std::min<int64_t>(a.n, w1 * k::kSellSigma);
    PDB_CUDA(cudaMemcpyAsync(db.get() + r0, b_h + r0, static_cast<size_t>(r1 - r0) * sizeof(double),
                             cudaMemcpyHostToDevice, cs));
    PDB_CUDA(cudaEventRecord(ev[static_cast<size_t>(c + 1)], cs));
  }
  Scratch<double> r(std::max<size_t>(n, 1), s);
  Scratch<double> sols(static_cast<size_t>(sols_len(pc)), s);
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t w0 = nwin * c / chunks, w1 = nwin * (c + 1) / chunks;
    PDB_CUDA(cudaStreamWaitEvent(s, ev[static_cast<size_t>(c + 1)], 0));
    k::residual_slices(plan, a.win_slice[static_cast<size_t>(w0)], a.win_slice[static_cast<size_t>(w1)], dx.get(), db.get(),
                       r.get(), s);
  }
  patch_stage(pc, r.get(), nullptr, sols.get(), s);
  scatter_stage(pc, sols.get(), false, dx.get(), nullptr, dx.get(), s);
  if (sweeps > 1) relax_device(a, pc, db.get(), dx.get(), sweeps - 1, nullptr, s);
  PDB_CUDA(cudaMemcpyAsync(x_h, dx.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
  PDB_LAUNCH_CHECK();
  sync(s);
  for (auto& ee : ev) cudaEventDestroy(ee);
}

void relax_profile(const DeviceCsr& a, const pdb_precond_s& pc, const double* b, double* x, int64_t sweeps,
                   double* ms_phase, cudaStream_t s) {
  require(pc.n == a.n, Errc::dimension_mismatch, "smooth length mismatch");
  const k::SpmvPlan plan = plan_of(a);
  Scratch<double> r(static_cast<size_t>(std::max<int64_t>(a.n, 1)), s);
  Scratch<double> sols(static_cast<size_t>(sols_len(pc)), s);
  if (const char* oe = getenv("PDB_PROFILE_OVERLAP"); oe && oe[0] == '1') {
    // Probe: residual on a low-priority stream concurrently with an
    // independent apply + scatter on a high-priority stream.  ms_phase =
    // {overlapped, residual alone, apply + scatter alone} per sweep.
    int lo = 0, hi = 0;
    PDB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    cudaStream_t sl = nullptr, sh = nullptr;
    PDB_CUDA(cudaStreamCreateWithPriority(&sl, cudaStreamNonBlocking, lo));
    PDB_CUDA(cudaStreamCreateWithPriority(&sh, cudaStreamNonBlocking, hi));
    Scratch<double> r2(static_cast<size_t>(std::max<int64_t>(a.n, 1)), s), x2(static_cast<size_t>(std::max<int64_t>(a.n, 1)), s);
    PDB_CUDA(cudaMemcpyAsync(x2.get(), x, a.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    k::residual(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, b, r2.get(), nullptr, s);
    cudaEvent_t t[6], j0, j1;
    for (auto& e : t) PDB_CUDA(cudaEventCreate(&e));
    PDB_CUDA(cudaEventCreateWithFlags(&j0, cudaEventDisableTiming));
    PDB_CUDA(cudaEventCreateWithFlags(&j1, cudaEventDisableTiming));
    PDB_CUDA(cudaEventRecord(j0, s));
    PDB_CUDA(cudaStreamWaitEvent(sl, j0, 0));
    PDB_CUDA(cudaEventRecord(t[0], sl));
    for (int64_t sw = 0; sw < sweeps; ++sw)
      k::residual(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, b, r.get(), nullptr, sl);
    PDB_CUDA(cudaEventRecord(t[1], sl));
    for (int64_t sw = 0; sw < sweeps; ++sw) {
      patch_stage(pc, r2.get(), nullptr, sols.get(), sl);
      scatter_stage(pc, sols.get(), false, x2.get(), nullptr, x2.get(), sl);
    }
    PDB_CUDA(cudaEventRecord(t[2], sl));
    for (int64_t sw = 0; sw < sweeps; ++sw) {
      PDB_CUDA(cudaEventRecord(j0, sl));
      PDB_CUDA(cudaStreamWaitEvent(sh, j0, 0));
      k::residual(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, b, r.get(), nullptr, sl);
      patch_stage(pc, r2.get(), nullptr, sols.get(), sh);
      scatter_stage(pc, sols.get(), false, x2.get(), nullptr, x2.get(), sh);
      PDB_CUDA(cudaEventRecord(j1, sh));
      PDB_CUDA(cudaStreamWaitEvent(sl, j1, 0));
    }
    PDB_CUDA(cudaEventRecord(t[3], sl));
    PDB_CUDA(cudaStreamSynchronize(sl));
    float m01 = 0.f, m12 = 0.f, m23 = 0.f;
    PDB_CUDA(cudaEventElapsedTime(&m01, t[0], t[1]));
    PDB_CUDA(cudaEventElapsedTime(&m12, t[1], t[2]));
    PDB_CUDA(cudaEventElapsedTime(&m23, t[2], t[3]));
    const double sw = static_cast<double>(std::max<int64_t>(sweeps, 1));
    ms_phase[0] = m23 / sw;
    ms_phase[1] = m01 / sw;
    ms_phase[2] = m12 / sw;
    for (auto& e : t) cudaEventDestroy(e);
    cudaEventDestroy(j0);
    cudaEventDestroy(j1);
    cudaStreamDestroy(sl);
    cudaStreamDestroy(sh);
    return;
  }
  std::vector<cudaEvent_t> ev(static_cast<size_t>(4 * std::max<int64_t>(sweeps, 1)));
  const char* he = getenv("PDB_PROFILE_HOT");
  const bool hot = he && he[0] == '1';
  for (auto& e : ev) PDB_CUDA(cudaEventCreate(&e));
  for (int64_t sw = 0; sw < sweeps; ++sw) {
    cudaEvent_t* e = ev.data() + 4 * sw;
    PDB_CUDA(cudaEventRecord(e[0], s));
    k::residual(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, b, r.get(), nullptr, s);
    if (hot) patch_stage(pc, r.get(), nullptr, sols.get(), s);  // PDB_PROFILE_HOT: time a second, L2-warm apply
    PDB_CUDA(cudaEventRecord(e[1], s));
    patch_stage(pc, r.get(), nullptr, sols.get(), s);
    PDB_CUDA(cudaEventRecord(e[2], s));
    scatter_stage(pc, sols.get(), false, x, nullptr, x, s);
    PDB_CUDA(cudaEventRecord(e[3], s));
  }
  PDB_LAUNCH_CHECK();
  sync(s);
  ms_phase[0] = ms_phase[1] = ms_phase[2] = 0.0;
  for (int64_t sw = 0; sw < sweeps; ++sw) {
    cudaEvent_t* e = ev.data() + 4 * sw;
    for (int p = 0; p < 3; ++p) {
      float ms = 0.f;
      PDB_CUDA(cudaEventElapsedTime(&ms, e[p], e[p + 1]));
      ms_phase[p] += ms / static_cast<double>(sweeps);
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

}  // namespace pdb
