// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// Thin extern "C" harness over the *unmodified* reference library
// (/root/reference/proj/src/core, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libpdbref.so).  The reference C-ABI can
// only ingest matrices from Matrix Market files or its own uniform-mesh
// assembler, so this harness builds patchdb::SparseMatrix directly from CSR
// arrays (its fields are public, sparse.hpp:20-25) and exposes the hot-path
// entry points the GPU implementation is checked against:
//   detect_patches (patch.cpp:37-90), extract_all (patch.cpp:92-99),
//   the pdb_database_build method switch (capi.cpp:249-284),
//   greedy_bisect_to_size (experiments.cpp:168-204),
//   PatchPreconditioner::{exact,compressed,apply} (precond.cpp:11-88),
//   smooth (precond.cpp:90-101), gmres (gmres.cpp:27-169),
//   lu_factor / spectral_distance / entrywise_l1_distance (dense.cpp).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load it.
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "core/compress.hpp"
#include "core/dense.hpp"
#include "core/errors.hpp"
#include "core/experiments.hpp"
#include "core/fem.hpp"
#include "core/gmres.hpp"
#include "core/matrix_market.hpp"
#include "core/patch.hpp"
#include "core/precond.hpp"
#include "core/sparse.hpp"

using namespace patchdb;

#define RH_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

// Same Errc -> status mapping as the reference C-ABI (capi.cpp:41-71).
int code_of(Errc c) {
  switch (c) {
    case Errc::invalid_argument: return 1;
    case Errc::dimension_mismatch: return 2;
    case Errc::singular_matrix: return 3;
    case Errc::index_out_of_range: return 4;
    case Errc::duplicate_index: return 5;
    case Errc::parse_error: return 6;
    case Errc::non_square_matrix: return 7;
    case Errc::no_patches_found: return 8;
    case Errc::empty_cluster: return 9;
    case Errc::budget_too_small: return 10;
    case Errc::invalid_degree: return 11;
    case Errc::non_positive_coefficient: return 12;
    case Errc::io_error: return 13;
  }
  return 14;
}

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const Exception& e) {
    g_err = e.what();
    return code_of(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 14;
  } catch (...) {
    g_err = "unknown error";
    return 14;
  }
}

DenseMatrix dense_from(int64_t n, const double* a) {
  DenseMatrix m(n, n);
  std::memcpy(m.a.data(), a, sizeof(double) * static_cast<size_t>(n * n));
  return m;
}

std::vector<DenseMatrix> mats_from(int64_t np, int64_t ps, const double* a) {
  std::vector<DenseMatrix> out(static_cast<size_t>(np));
  for (int64_t k = 0; k < np; ++k) out[static_cast<size_t>(k)] = dense_from(ps, a + k * ps * ps);
  return out;
}

struct RefPc {
  std::unique_ptr<Preconditioner> pc;
};

}  // namespace

RH_API const char* refh_last_error(void) { return g_err.c_str(); }

/* ---- matrices ---- */

// read_matrix_market(path) (matrix_market.cpp:87-91): status + matrix
RH_API int refh_read_mm(const char* path, void** out) {
  return guarded([&] { *out = new SparseMatrix(read_matrix_market(std::string(path))); });
}

// write_matrix_market(a, path) (matrix_market.cpp:105-110)
RH_API int refh_write_mm(void* m, const char* path) {
  return guarded([&] { write_matrix_market(*static_cast<SparseMatrix*>(m), std::string(path)); });
}

RH_API void* refh_matrix_new(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
  auto* m = new SparseMatrix();
  m->n = n;
  m->row_ptr.assign(rp, rp + n + 1);
  const int64_t nnz = rp[n];
  m->col_idx.assign(ci, ci + nnz);
  m->values.assign(v, v + nnz);
  return m;
}
RH_API void refh_matrix_free(void* m) { delete static_cast<SparseMatrix*>(m); }

RH_API int refh_spmv(void* m, const double* x, double* y, int threads) {
  auto* a = static_cast<SparseMatrix*>(m);
  return guarded([&] {
    const size_t n = static_cast<size_t>(a->n);
    spmv(*a, {x, n}, {y, n}, threads);
  });
}

/* ---- patch sets ---- */

RH_API int refh_detect(void* m, int64_t patch_size, void** out) {
  return guarded([&] { *out = new PatchSet(detect_patches(*static_cast<SparseMatrix*>(m), patch_size)); });
}
RH_API int64_t refh_ps_count(void* ps) { return static_cast<PatchSet*>(ps)->count(); }
RH_API int64_t refh_ps_size(void* ps) { return static_cast<PatchSet*>(ps)->patch_size; }
RH_API void refh_ps_patches(void* ps, int64_t* out) {
  auto* p = static_cast<PatchSet*>(ps);
  for (const auto& patch : p->patches) {
    std::memcpy(out, patch.data(), sizeof(int64_t) * patch.size());
    out += patch.size();
  }
}
RH_API void refh_ps_weights(void* ps, double* out) {
  auto* p = static_cast<PatchSet*>(ps);
  std::memcpy(out, p->weights.data(), sizeof(double) * p->weights.size());
}
RH_API void refh_ps_free(void* ps) { delete static_cast<PatchSet*>(ps); }

/* A patch set from explicit lists (weights recomputed as compute_weights). */
RH_API void* refh_ps_new(int64_t n, int64_t np, int64_t ps, const int64_t* patches) {
  auto* p = new PatchSet();
  p->patch_size = ps;
  p->patches.resize(static_cast<size_t>(np));
  for (int64_t k = 0; k < np; ++k) p->patches[static_cast<size_t>(k)].assign(patches + k * ps, patches + (k + 1) * ps);
  p->weights = compute_weights(n, p->patches);
  return p;
}

RH_API int refh_extract_all(void* m, void* ps, int threads, double* out) {
  return guarded([&] {
    const auto mats = extract_all(*static_cast<SparseMatrix*>(m), *static_cast<PatchSet*>(ps), threads);
    for (const auto& a : mats) {
      std::memcpy(out, a.a.data(), sizeof(double) * a.a.size());
      out += a.a.size();
    }
  });
}

/* ---- databases ---- */

// Mirrors the method switch of pdb_database_build (capi.cpp:249-284).
RH_API int refh_db_build(void* m, void* ps, int method, double eps, int64_t db_size, uint64_t seed, int max_iters,
                         int best_match, int threads, void** out) {
  return guarded([&] {
    const auto mats = extract_all(*static_cast<SparseMatrix*>(m), *static_cast<PatchSet*>(ps), threads);
    auto db = std::make_unique<Database>();
    switch (method) {
      case 0: *db = exact_database(mats, threads); break;
      case 1: *db = greedy_tolerance(mats, eps, Flavor::Spectral, best_match != 0, threads); break;
      case 2: *db = greedy_tolerance(mats, eps, Flavor::EntrywiseL1, best_match != 0, threads); break;
      case 3: *db = partitioned_build(mats, db_size, KmeansVariant::Entrywise, seed, max_iters, threads); break;
      case 4: *db = partitioned_build(mats, db_size, KmeansVariant::Spectral, seed, max_iters, threads); break;
      case 5: *db = partitioned_build(mats, db_size, KmeansVariant::VarianceMinimizing, seed, max_iters, threads); break;
      case 6: *db = bootstrapped(mats, eps, KmeansVariant::VarianceMinimizing, max_iters, threads); break;
      default: fail(Errc::invalid_argument, "unknown compression method");
    }
    *out = db.release();
  });
}

// evaluate_objective (compress.cpp:423-440) of a database on the set's patches.
RH_API int refh_evaluate_objective(void* m, void* ps, void* db, double beta, int threads, double* out) {
  return guarded([&] {
    const auto mats = extract_all(*static_cast<SparseMatrix*>(m), *static_cast<PatchSet*>(ps), threads);
    *out = evaluate_objective(*static_cast<Database*>(db), mats, beta, threads);
  });
}

// compressibility_curve (compress.cpp:442-456).
RH_API int refh_compressibility_curve(void* m, void* ps, int spectral, const double* grid, int64_t count, int threads,
                                      int64_t* sizes, double* ratios) {
  return guarded([&] {
    const auto mats = extract_all(*static_cast<SparseMatrix*>(m), *static_cast<PatchSet*>(ps), threads);
    const std::vector<double> g(grid, grid + count);
    const auto curve = compressibility_curve(mats, g, spectral ? Flavor::Spectral : Flavor::EntrywiseL1, threads);
    for (size_t k = 0; k < curve.size(); ++k) {
      sizes[k] = curve[k].db_size;
      ratios[k] = curve[k].ratio;
    }
  });
}

// greedy_tolerance_capped (compress.cpp:121-124); *out = NULL when aborted.
RH_API int refh_db_greedy_capped(void* m, void* ps, int spectral, double eps, int64_t abort_above, int best_match,
                                 int threads, void** out) {
  return guarded([&] {
    const auto mats = extract_all(*static_cast<SparseMatrix*>(m), *static_cast<PatchSet*>(ps), threads);
    auto db = greedy_tolerance_capped(mats, eps, spectral ? Flavor::Spectral : Flavor::EntrywiseL1, abort_above,
                                      best_match != 0, threads);
    *out = db.has_value() ? new Database(std::move(*db)) : nullptr;
  });
}

// greedy_bisect_to_size (experiments.cpp:168-204).
RH_API int refh_db_bisect(void* m, void* ps, int spectral, int64_t lo, int64_t hi, int best_match, int threads,
                          void** out, double* eps_out) {
  return guarded([&] {
    const auto mats = extract_all(*static_cast<SparseMatrix*>(m), *static_cast<PatchSet*>(ps), threads);
    GreedyBisectResult r =
        greedy_bisect_to_size(mats, spectral ? Flavor::Spectral : Flavor::EntrywiseL1, lo, hi, best_match != 0, threads);
    *eps_out = r.eps;
    *out = new Database(std::move(r.db));
  });
}

// A Database from explicit arrays (representatives, factors, pivots, phi):
// lets the CPU baseline time the reference sweep on a database built
// elsewhere (the sweep cost depends only on the sizes).
RH_API void* refh_db_from_arrays(int64_t m, int64_t ps, int64_t np, const double* reps, const double* lu,
                                 const int64_t* piv, const int64_t* phi) {
  auto* db = new Database();
  db->method = "external";
  db->entries.resize(static_cast<size_t>(m));
  const int64_t len = ps * ps;
  for (int64_t j = 0; j < m; ++j) {
    auto& e = db->entries[static_cast<size_t>(j)];
    e.representative = dense_from(ps, reps + j * len);
    e.factor.dim = ps;
    e.factor.lu = dense_from(ps, lu + j * len);
    e.factor.pivots.assign(piv + j * ps, piv + (j + 1) * ps);
  }
  db->phi.assign(phi, phi + np);
  return db;
}

RH_API int64_t refh_db_size(void* db) { return static_cast<Database*>(db)->size(); }
RH_API int64_t refh_db_n_patches(void* db) { return static_cast<Database*>(db)->n_patches(); }
RH_API double refh_db_eps(void* db) { return static_cast<Database*>(db)->eps; }
RH_API void refh_db_phi(void* db, int64_t* phi) {
  auto* d = static_cast<Database*>(db);
  std::memcpy(phi, d->phi.data(), sizeof(int64_t) * d->phi.size());
}
RH_API void refh_db_reps(void* db, double* out) {
  for (const auto& e : static_cast<Database*>(db)->entries) {
    std::memcpy(out, e.representative.a.data(), sizeof(double) * e.representative.a.size());
    out += e.representative.a.size();
  }
}
RH_API void refh_db_factors(void* db, double* lu, int64_t* piv) {
  for (const auto& e : static_cast<Database*>(db)->entries) {
    std::memcpy(lu, e.factor.lu.a.data(), sizeof(double) * e.factor.lu.a.size());
    lu += e.factor.lu.a.size();
    std::memcpy(piv, e.factor.pivots.data(), sizeof(int64_t) * e.factor.pivots.size());
    piv += e.factor.pivots.size();
  }
}
RH_API int64_t refh_db_n_patterns(void* db) {
  return static_cast<int64_t>(static_cast<Database*>(db)->entry_patterns.size());
}
RH_API void refh_db_patterns(void* db, uint8_t* out) {
  for (const auto& bp : static_cast<Database*>(db)->entry_patterns)
    for (bool b : bp.mask) *out++ = b ? 1 : 0;
}
RH_API void refh_db_method(void* db, char* out, int64_t cap) {
  const std::string& s = static_cast<Database*>(db)->method;
  std::strncpy(out, s.c_str(), static_cast<size_t>(cap));
}
RH_API void refh_db_free(void* db) { delete static_cast<Database*>(db); }

/* ---- preconditioners and the sweep ---- */

RH_API int refh_pc_new(void* m, void* ps, void* db, double omega, int threads, void** out) {
  return guarded([&] {
    auto h = std::make_unique<RefPc>();
    if (db == nullptr)
      h->pc = std::make_unique<PatchPreconditioner>(
          PatchPreconditioner::exact(*static_cast<SparseMatrix*>(m), *static_cast<PatchSet*>(ps), omega, threads));
    else
      h->pc = std::make_unique<PatchPreconditioner>(PatchPreconditioner::compressed(
          *static_cast<PatchSet*>(ps), *static_cast<Database*>(db), omega, threads));
    *out = h.release();
  });
}
RH_API int refh_pc_apply(void* pc, const double* r, double* z) {
  auto* h = static_cast<RefPc*>(pc);
  return guarded([&] {
    const size_t n = static_cast<size_t>(h->pc->size());
    h->pc->apply({r, n}, {z, n});
  });
}
RH_API void refh_pc_free(void* pc) { delete static_cast<RefPc*>(pc); }

// `sweeps` applications of smooth (precond.cpp:90-101); x is updated in place.
RH_API int refh_smooth(void* pc, void* m, double* x, const double* b, int64_t sweeps, int threads) {
  auto* h = static_cast<RefPc*>(pc);
  auto* a = static_cast<SparseMatrix*>(m);
  return guarded([&] {
    const size_t n = static_cast<size_t>(a->n);
    for (int64_t s = 0; s < sweeps; ++s) {
      std::vector<double> xn = smooth(*h->pc, *a, {x, n}, {b, n}, threads);
      std::memcpy(x, xn.data(), sizeof(double) * n);
    }
  });
}

RH_API int refh_gmres(void* m, const double* b, void* pc, int64_t restart, double tol, int64_t max_iters, int left,
                      int threads, double* x, int64_t* iters, int64_t* restarts, int* converged, double* relres,
                      double* hist, int64_t* hist_len) {
  auto* a = static_cast<SparseMatrix*>(m);
  return guarded([&] {
    GmresOptions go{restart, tol, max_iters, left != 0, threads};
    GmresResult r = gmres(*a, {b, static_cast<size_t>(a->n)},
                          pc == nullptr ? nullptr : static_cast<RefPc*>(pc)->pc.get(), go);
    std::memcpy(x, r.x.data(), sizeof(double) * r.x.size());
    *iters = r.report.iterations;
    *restarts = r.report.restarts;
    *converged = r.report.converged ? 1 : 0;
    *relres = r.report.final_relative_residual;
    const int64_t cap = *hist_len;
    const int64_t len = static_cast<int64_t>(r.report.residual_history.size());
    *hist_len = len;
    std::memcpy(hist, r.report.residual_history.data(), sizeof(double) * static_cast<size_t>(std::min(cap, len)));
  });
}

/* ---- dense kernels ---- */

RH_API int refh_lu_factor(int64_t n, const double* a, double* lu, int64_t* piv) {
  return guarded([&] {
    DenseFactor f = lu_factor(dense_from(n, a));
    std::memcpy(lu, f.lu.a.data(), sizeof(double) * static_cast<size_t>(n * n));
    std::memcpy(piv, f.pivots.data(), sizeof(int64_t) * static_cast<size_t>(n));
  });
}

RH_API int refh_lu_solve(int64_t n, const double* lu, const int64_t* piv, const double* rhs, double* out,
                         int transpose) {
  return guarded([&] {
    DenseFactor f;
    f.dim = n;
    f.lu = dense_from(n, lu);
    f.pivots.assign(piv, piv + n);
    const size_t un = static_cast<size_t>(n);
    if (transpose)
      lu_solve_transpose_into(f, {rhs, un}, {out, un});
    else
      lu_solve_into(f, {rhs, un}, {out, un});
  });
}

// spectral_distance(A, lu_factor(B)) (dense.cpp:154-190).
RH_API int refh_spectral_distance(int64_t n, const double* a, const double* b, double* out) {
  return guarded([&] { *out = spectral_distance(dense_from(n, a), lu_factor(dense_from(n, b))); });
}

RH_API double refh_l1_distance(int64_t n, const double* a, const double* b) {
  return entrywise_l1_distance(dense_from(n, a), dense_from(n, b));
}

RH_API int refh_split_budget(int64_t m_p, int64_t parts, const int64_t* sizes, int64_t* out) {
  return guarded([&] {
    std::vector<Index> s(sizes, sizes + parts);
    const auto alloc = split_budget(m_p, s);
    std::memcpy(out, alloc.data(), sizeof(int64_t) * alloc.size());
  });
}

// boundary_partition (patch.cpp:113-126) on explicit patch matrices:
// group_of[k] = group index; masks = ngroups x ps bytes.
RH_API int refh_boundary_partition(int64_t np, int64_t ps, const double* mats, int64_t* group_of, uint8_t* masks,
                                   int64_t* ngroups) {
  return guarded([&] {
    const auto m = mats_from(np, ps, mats);
    const auto groups = boundary_partition(m);
    *ngroups = static_cast<int64_t>(groups.size());
    for (size_t g = 0; g < groups.size(); ++g) {
      for (Index k : groups[g].second) group_of[k] = static_cast<int64_t>(g);
      for (int64_t i = 0; i < ps; ++i) masks[g * ps + i] = groups[g].first.mask[static_cast<size_t>(i)] ? 1 : 0;
    }
  });
}

/* ---- reference uniform-mesh assembler (fem.cpp:248-346) ---- */

RH_API int refh_assemble(int dim, int64_t cells, int degree, int coeff_kind, double coeff_value, int64_t bx,
                         int64_t by, const double* block_values, int64_t n_block_values, void** out_matrix,
                         double* rhs_out /* may be NULL */) {
  return guarded([&] {
    Coefficient c;
    if (coeff_kind == 0) c = Coefficient::constant(coeff_value);
    else if (coeff_kind == 1) c = Coefficient::smooth();
    else {
      c.kind = CoeffKind::PiecewiseConstant;
      c.blocks_x = bx;
      c.blocks_y = by;
      if (n_block_values > 0) c.block_values.assign(block_values, block_values + n_block_values);
      else c = Coefficient::checkerboard(bx, by, 1.0, 100.0);
    }
    StructuredMesh mesh{dim, cells, degree};
    DiscreteProblem p = assemble(mesh, c);
    if (rhs_out) std::memcpy(rhs_out, p.rhs.data(), sizeof(double) * p.rhs.size());
    *out_matrix = new SparseMatrix(std::move(p.matrix));
  });
}
RH_API int64_t refh_matrix_n(void* m) { return static_cast<SparseMatrix*>(m)->n; }
RH_API int64_t refh_matrix_nnz(void* m) { return static_cast<SparseMatrix*>(m)->nnz(); }
RH_API void refh_matrix_csr(void* m, int64_t* rp, int64_t* ci, double* v) {
  auto* a = static_cast<SparseMatrix*>(m);
  std::memcpy(rp, a->row_ptr.data(), sizeof(int64_t) * a->row_ptr.size());
  std::memcpy(ci, a->col_idx.data(), sizeof(int64_t) * a->col_idx.size());
  std::memcpy(v, a->values.data(), sizeof(double) * a->values.size());
}

/* ---- model problems and the combo preconditioner (capi.cpp:169-212, 320-333;
 *      fem.cpp:248-479; banded.cpp:11-84; precond.cpp:103-121) ---- */

// pdb_problem_assemble's exact recipe: parse_config + resolve_coefficient
// (constant fallback) + assemble.
RH_API int refh_problem_assemble(const char* json, void** out) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(json);
    const Coefficient coeff = resolve_coefficient(cfg, CoeffKind::Constant);
    StructuredMesh mesh{cfg.dim, cfg.cells, cfg.degree};
    *out = new DiscreteProblem(assemble(mesh, coeff));
  });
}
RH_API void refh_problem_free(void* p) { delete static_cast<DiscreteProblem*>(p); }
RH_API int64_t refh_problem_n(void* p) { return static_cast<DiscreteProblem*>(p)->matrix.n; }
RH_API int64_t refh_problem_nnz(void* p) { return static_cast<DiscreteProblem*>(p)->matrix.nnz(); }
RH_API void refh_problem_csr(void* p, int64_t* rp, int64_t* ci, double* v) {
  const SparseMatrix& a = static_cast<DiscreteProblem*>(p)->matrix;
  std::memcpy(rp, a.row_ptr.data(), sizeof(int64_t) * a.row_ptr.size());
  std::memcpy(ci, a.col_idx.data(), sizeof(int64_t) * a.col_idx.size());
  std::memcpy(v, a.values.data(), sizeof(double) * a.values.size());
}
RH_API void refh_problem_rhs(void* p, double* out) {
  const auto& r = static_cast<DiscreteProblem*>(p)->rhs;
  std::memcpy(out, r.data(), sizeof(double) * r.size());
}
RH_API void refh_problem_exact(void* p, double* out) {
  const std::vector<double> u = exact_solution(static_cast<DiscreteProblem*>(p)->mesh);
  std::memcpy(out, u.data(), sizeof(double) * u.size());
}
RH_API int refh_problem_l2_error(void* p, const double* u, double* out) {
  auto* pr = static_cast<DiscreteProblem*>(p);
  return guarded([&] { *out = l2_error(pr->mesh, {u, static_cast<size_t>(pr->matrix.n)}); });
}
// A copy of the problem's matrix as a harness matrix handle.
RH_API void* refh_problem_matrix(void* p) { return new SparseMatrix(static_cast<DiscreteProblem*>(p)->matrix); }

// Coarse space: sizes, then P0 and R0 A P0 as CSR, then the band factor.
RH_API int refh_coarse_sizes(void* p, int64_t* fine_n, int64_t* nc, int64_t* p0_nnz, int64_t* c_nnz) {
  auto* pr = static_cast<DiscreteProblem*>(p);
  return guarded([&] {
    const CoarseSpace cs = build_coarse_and_transfer(pr->mesh, pr->matrix);
    *fine_n = cs.p0.fine_n;
    *nc = cs.p0.coarse_n;
    *p0_nnz = static_cast<int64_t>(cs.p0.col.size());
    *c_nnz = cs.coarse_matrix.nnz();
  });
}
RH_API int refh_coarse_csr(void* p, int64_t* p0_rp, int64_t* p0_ci, double* p0_v, int64_t* c_rp, int64_t* c_ci,
                           double* c_v) {
  auto* pr = static_cast<DiscreteProblem*>(p);
  return guarded([&] {
    const CoarseSpace cs = build_coarse_and_transfer(pr->mesh, pr->matrix);
    std::memcpy(p0_rp, cs.p0.row_ptr.data(), sizeof(int64_t) * cs.p0.row_ptr.size());
    std::memcpy(p0_ci, cs.p0.col.data(), sizeof(int64_t) * cs.p0.col.size());
    std::memcpy(p0_v, cs.p0.val.data(), sizeof(double) * cs.p0.val.size());
    const SparseMatrix& c = cs.coarse_matrix;
    std::memcpy(c_rp, c.row_ptr.data(), sizeof(int64_t) * c.row_ptr.size());
    std::memcpy(c_ci, c.col_idx.data(), sizeof(int64_t) * c.col_idx.size());
    std::memcpy(c_v, c.values.data(), sizeof(double) * c.values.size());
  });
}
// band: (2kl+ku+1) x n row-major (BandedFactor::ab), ipiv absolute rows.
// Call with band == NULL first to get kl, ku.
RH_API int refh_coarse_factor(void* p, int64_t* kl, int64_t* ku, double* band, int64_t* ipiv) {
  auto* pr = static_cast<DiscreteProblem*>(p);
  return guarded([&] {
    const CoarseSpace cs = build_coarse_and_transfer(pr->mesh, pr->matrix);
    const BandedFactor f = band_factor(cs.coarse_matrix);
    *kl = f.kl;
    *ku = f.ku;
    if (band) std::memcpy(band, f.ab.data(), sizeof(double) * f.ab.size());
    if (ipiv) std::memcpy(ipiv, f.ipiv.data(), sizeof(int64_t) * f.ipiv.size());
  });
}
// Combo preconditioner exactly as pdb_precond_create_combo builds it.
RH_API int refh_combo_new(void* p, void* ps, void* db, double omega, int threads, void** out) {
  auto* pr = static_cast<DiscreteProblem*>(p);
  return guarded([&] {
    PatchPreconditioner patch_pc =
        db == nullptr ? PatchPreconditioner::exact(pr->matrix, *static_cast<PatchSet*>(ps), omega, threads)
                      : PatchPreconditioner::compressed(*static_cast<PatchSet*>(ps), *static_cast<Database*>(db),
                                                        omega, threads);
    const CoarseSpace cs = build_coarse_and_transfer(pr->mesh, pr->matrix);
    auto h = std::make_unique<RefPc>();
    h->pc = std::make_unique<ComboPreconditioner>(std::move(patch_pc), cs);
    *out = h.release();
  });
}

// pdb_export_matrix's recipe (capi.cpp:422-428, experiments.cpp:430-435).
RH_API int refh_export_matrix(const char* json, const char* path) {
  return guarded([&] { export_matrix(parse_config(json), path); });
}

// A reference DiscreteProblem around an external CSR on a uniform lattice
// (dim, cells, degree): lets the reference's combo run on generated configs.
RH_API void* refh_problem_from_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* rhs,
                                   int dim, int64_t cells, int degree) {
  auto* p = new DiscreteProblem();
  p->matrix.n = n;
  p->matrix.row_ptr.assign(rp, rp + n + 1);
  p->matrix.col_idx.assign(ci, ci + rp[n]);
  p->matrix.values.assign(v, v + rp[n]);
  p->rhs.assign(rhs, rhs + n);
  p->mesh = StructuredMesh{dim, cells, degree};
  return p;
}
