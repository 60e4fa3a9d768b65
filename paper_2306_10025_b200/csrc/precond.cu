// Patch preconditioner setup and application (reference
// PatchPreconditioner::{exact,compressed,apply} precond.cpp:11-88, smooth
// precond.cpp:90-101).
//
// Setup converts the database (reference row-major LU layout) into the sweep
// layout: column-major factors, int32 pivots, omega*W, and the DoF ->
// (patch, slot) inverse map sorted by patch so the gather-side scatter adds
// in the reference's ascending-k order.
#include <cub/cub.cuh>

#include "host.hpp"
#include "kernels.hpp"

namespace pdb {

namespace {

void build_inverse(pdb_precond_s& pc, cudaStream_t s) {
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
  PDB_LAUNCH_CHECK();
}

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
  build_inverse(pc, s);
}

}  // namespace

void precond_exact(const DeviceCsr& a, const pdb_patchset_s& ps, double omega, pdb_precond_s& pc, cudaStream_t s) {
  require_device();
  require(ps.n == a.n, Errc::dimension_mismatch, "patch set weights do not match the matrix size");
  pdb_database_s db;
  BuildParams p;
  p.method = PDB_METHOD_EXACT;
  build_database(a, ps, p, db, s);  // extract + LU of every patch; "patch k: ..." on failure
  common_setup(ps, omega, pc, s);
  pc.compressed = false;
  pc.nf = db.m;
  pc.factors.alloc(static_cast<size_t>(db.m * ps.ps * ps.ps));
  k::transpose_factors(db.m, static_cast<int>(ps.ps), db.lu.get(), pc.factors.get(), s);
  pc.piv = std::move(db.piv);
  PDB_LAUNCH_CHECK();
  sync(s);
}

void precond_compressed(const pdb_patchset_s& ps, const pdb_database_s& db, double omega, pdb_precond_s& pc,
                        cudaStream_t s) {
  require_device();
  require(db.np == ps.np, Errc::dimension_mismatch, "database does not cover the patch set");
  // phi onto the database (Database::phi_onto, compress.cpp:3-10)
  {
    const std::vector<int32_t> phi = db.phi.to_host(s);
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
  common_setup(ps, omega, pc, s);
  pc.compressed = true;
  pc.nf = db.m;
  pc.factors.alloc(static_cast<size_t>(db.m * ps.ps * ps.ps));
  k::transpose_factors(db.m, static_cast<int>(ps.ps), db.lu.get(), pc.factors.get(), s);
  pc.piv.alloc(static_cast<size_t>(db.m * ps.ps));
  PDB_CUDA(cudaMemcpyAsync(pc.piv.get(), db.piv.get(), db.m * ps.ps * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  pc.phi.alloc(static_cast<size_t>(ps.np));
  PDB_CUDA(cudaMemcpyAsync(pc.phi.get(), db.phi.get(), ps.np * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  PDB_LAUNCH_CHECK();
  sync(s);
}

void precond_apply_device(const pdb_precond_s& pc, const double* r, double* z, cudaStream_t s, bool symmetric) {
  Scratch<double> sols(static_cast<size_t>(std::max<int64_t>(pc.np * pc.ps, 1)), s);
  k::patch_solve(pc.np, static_cast<int>(pc.ps), pc.patches.get(), pc.factors.get(), pc.piv.get(),
                 pc.compressed ? pc.phi.get() : nullptr, r, symmetric ? pc.sqrt_w.get() : nullptr, sols.get(), s);
  k::scatter_update(pc.n, pc.inv_ptr.get(), pc.inv.get(), sols.get(),
                    symmetric ? pc.omega_sw.get() : pc.omega_w.get(), nullptr, z, nullptr, s);
  PDB_LAUNCH_CHECK();
}

void relax_device(const DeviceCsr& a, const pdb_precond_s& pc, const double* b, double* x, int64_t sweeps,
                  double* history, cudaStream_t s) {
  require(pc.n == a.n, Errc::dimension_mismatch, "smooth length mismatch");
  const k::SpmvPlan plan = k::spmv_plan(a.n, a.nnz);
  Scratch<double> r(static_cast<size_t>(std::max<int64_t>(a.n, 1)), s);
  Scratch<double> sols(static_cast<size_t>(std::max<int64_t>(pc.np * pc.ps, 1)), s);
  Scratch<double> partials(static_cast<size_t>(std::max(plan.blocks, 1)), s);
  for (int64_t sw = 0; sw <= sweeps; ++sw) {
    if (sw == sweeps && !history) break;
    k::residual(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, b, r.get(), history ? partials.get() : nullptr,
                s);
    if (history) k::finish_sum(partials.get(), plan.blocks, history + sw, true, s);
    if (sw == sweeps) break;
    k::patch_solve(pc.np, static_cast<int>(pc.ps), pc.patches.get(), pc.factors.get(), pc.piv.get(),
                   pc.compressed ? pc.phi.get() : nullptr, r.get(), nullptr, sols.get(), s);
    k::scatter_update(pc.n, pc.inv_ptr.get(), pc.inv.get(), sols.get(), pc.omega_w.get(), x, nullptr, x, s);
  }
  PDB_LAUNCH_CHECK();
}

void relax_profile(const DeviceCsr& a, const pdb_precond_s& pc, const double* b, double* x, int64_t sweeps,
                   double* ms_phase, cudaStream_t s) {
  require(pc.n == a.n, Errc::dimension_mismatch, "smooth length mismatch");
  const k::SpmvPlan plan = k::spmv_plan(a.n, a.nnz);
  Scratch<double> r(static_cast<size_t>(std::max<int64_t>(a.n, 1)), s);
  Scratch<double> sols(static_cast<size_t>(std::max<int64_t>(pc.np * pc.ps, 1)), s);
  std::vector<cudaEvent_t> ev(static_cast<size_t>(4 * std::max<int64_t>(sweeps, 1)));
  for (auto& e : ev) PDB_CUDA(cudaEventCreate(&e));
  for (int64_t sw = 0; sw < sweeps; ++sw) {
    cudaEvent_t* e = ev.data() + 4 * sw;
    PDB_CUDA(cudaEventRecord(e[0], s));
    k::residual(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, b, r.get(), nullptr, s);
    PDB_CUDA(cudaEventRecord(e[1], s));
    k::patch_solve(pc.np, static_cast<int>(pc.ps), pc.patches.get(), pc.factors.get(), pc.piv.get(),
                   pc.compressed ? pc.phi.get() : nullptr, r.get(), nullptr, sols.get(), s);
    PDB_CUDA(cudaEventRecord(e[2], s));
    k::scatter_update(pc.n, pc.inv_ptr.get(), pc.inv.get(), sols.get(), pc.omega_w.get(), x, nullptr, x, s);
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
