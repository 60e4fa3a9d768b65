// The C-ABI: every pdb_* symbol of include/patchdb/patchdb.h.
//
// Error handling mirrors the reference C-ABI (capi.cpp:37-135 of
// /root/reference/proj/src): null arguments -> PDB_ERR_INVALID_ARGUMENT
// "null argument"; library errors -> their code; anything else ->
// PDB_ERR_INTERNAL; the message is thread-local (pdb_last_error).  Getters
// return 0 on NULL handles; pdb_*_free(NULL) is a no-op.  All calls are
// synchronous and run on the calling thread's per-thread default stream,
// with per-call scratch, so concurrent applies on one handle are safe
// (reference precond.cpp:67-69 is const with per-call buffers).
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "host.hpp"

using namespace pdb;

namespace {

thread_local std::string g_last_error;

template <typename F>
pdb_status guarded(F&& fn) {
  try {
    fn();
    return PDB_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return static_cast<pdb_status>(static_cast<int>(e.code()));
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return PDB_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PDB_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return PDB_ERR_INTERNAL;
  }
}

pdb_status arg_error(const char* msg) {
  g_last_error = msg;
  return PDB_ERR_INVALID_ARGUMENT;
}

pdb_status unsupported(const char* what) {
  g_last_error = std::string(what) +
                 " is outside the B200 hot path of this build (reference experiment/FEM driver); see DESIGN.md";
  return PDB_ERR_INTERNAL;
}

cudaStream_t stream_of(void* s) { return s ? static_cast<cudaStream_t>(s) : default_stream(); }

template <typename T>
int64_t copy_out(const std::vector<T>& v, void* out) {
  if (out) {
    if (std::is_same<T, double>::value)
      std::memcpy(out, v.data(), v.size() * sizeof(double));
    else
      for (size_t i = 0; i < v.size(); ++i) static_cast<int64_t*>(out)[i] = static_cast<int64_t>(v[i]);
  }
  return static_cast<int64_t>(v.size());
}

// Plan arrays for pdb_shard_plan_get: integer arrays are widened to int64.
int64_t plan_array(const ShardPlan& p, int which, void* out) {
  switch (which) {
    case PDB_PLAN_DOFS: return copy_out(p.dofs, out);
    case PDB_PLAN_ROW_PTR: return copy_out(p.rp, out);
    case PDB_PLAN_COLS: return copy_out(p.ci, out);
    case PDB_PLAN_VALUES: return copy_out(p.val, out);
    case PDB_PLAN_PATCHES: return copy_out(p.patches, out);
    case PDB_PLAN_WEIGHTS: return copy_out(p.weights, out);
    case PDB_PLAN_OWNED: return copy_out(p.owned, out);
    case PDB_PLAN_UP: return copy_out(p.up, out);
    case PDB_PLAN_UP_PEER: return copy_out(p.up_peer, out);
    case PDB_PLAN_PIN: return copy_out(p.pin, out);
    case PDB_PLAN_PIN_PEER: return copy_out(p.pin_peer, out);
    case PDB_PLAN_XS: return copy_out(p.xs, out);
    case PDB_PLAN_XS_PEER: return copy_out(p.xs_peer, out);
    case PDB_PLAN_XR: return copy_out(p.xr, out);
    case PDB_PLAN_XR_PEER: return copy_out(p.xr_peer, out);
    case PDB_PLAN_PATCH_RANGE: {
      const std::vector<int64_t> r = {p.k0, p.k1};
      return copy_out(r, out);
    }
    default: return -1;
  }
}

}  // namespace

extern "C" {

PDB_API const char* pdb_status_string(pdb_status status) {
  switch (status) {
    case PDB_OK: return "ok";
    case PDB_ERR_INVALID_ARGUMENT: return "invalid argument";
    case PDB_ERR_DIMENSION_MISMATCH: return "dimension mismatch";
    case PDB_ERR_SINGULAR_MATRIX: return "singular matrix";
    case PDB_ERR_INDEX_OUT_OF_RANGE: return "index out of range";
    case PDB_ERR_DUPLICATE_INDEX: return "duplicate index";
    case PDB_ERR_PARSE: return "parse error";
    case PDB_ERR_NON_SQUARE_MATRIX: return "non-square matrix";
    case PDB_ERR_NO_PATCHES_FOUND: return "no patches found";
    case PDB_ERR_EMPTY_CLUSTER: return "empty cluster";
    case PDB_ERR_BUDGET_TOO_SMALL: return "budget too small";
    case PDB_ERR_INVALID_DEGREE: return "invalid degree";
    case PDB_ERR_NON_POSITIVE_COEFFICIENT: return "non-positive coefficient";
    case PDB_ERR_IO: return "io error";
    case PDB_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

PDB_API const char* pdb_last_error(void) { return g_last_error.c_str(); }

PDB_API const char* pdb_build_info(void) {
  return "patchdb-b200 0.1.0; device code sm_100a (B200); C-ABI of patchdb 0.1.0";
}

/* ---- matrices ---- */

PDB_API pdb_status pdb_matrix_read_matrix_market(const char* path, pdb_matrix* out) {
  if (path == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    HostCsr h = read_matrix_market_host(path);
    auto m = std::make_unique<pdb_matrix_s>();
    upload_csr(h, m->a, default_stream());
    *out = m.release();
  });
}

PDB_API pdb_status pdb_matrix_write_matrix_market(pdb_matrix m, const char* path) {
  if (m == nullptr || path == nullptr) return arg_error("null argument");
  return guarded([&] { write_matrix_market_host(download_csr(m->a, default_stream()), path); });
}

PDB_API int64_t pdb_matrix_rows(pdb_matrix m) { return m == nullptr ? 0 : m->a.n; }
PDB_API int64_t pdb_matrix_nnz(pdb_matrix m) { return m == nullptr ? 0 : m->a.nnz; }

PDB_API pdb_status pdb_matrix_spmv(pdb_matrix m, const double* x, double* y) {
  if (m == nullptr || x == nullptr || y == nullptr) return arg_error("null argument");
  return guarded([&] {
    require_device();
    cudaStream_t s = default_stream();
    const size_t n = static_cast<size_t>(m->a.n);
    Scratch<double> dx(std::max<size_t>(n, 1), s), dy(std::max<size_t>(n, 1), s);
    PDB_CUDA(cudaMemcpyAsync(dx.get(), x, n * sizeof(double), cudaMemcpyHostToDevice, s));
    spmv_device(m->a, dx.get(), dy.get(), s);
    PDB_CUDA(cudaMemcpyAsync(y, dy.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

PDB_API pdb_status pdb_matrix_spmv_device(pdb_matrix m, const double* d_x, double* d_y, void* stream) {
  if (m == nullptr || d_x == nullptr || d_y == nullptr) return arg_error("null argument");
  return guarded([&] {
    require_device();
    spmv_device(m->a, d_x, d_y, stream_of(stream));
  });
}

PDB_API void pdb_matrix_free(pdb_matrix m) { delete m; }

PDB_API pdb_status pdb_matrix_from_csr(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                       const double* values, pdb_matrix* out) {
  if (row_ptr == nullptr || out == nullptr || ((col_idx == nullptr || values == nullptr) && n > 0 && row_ptr[n] > 0))
    return arg_error("null argument");
  return guarded([&] {
    HostCsr h = validated_csr(n, row_ptr, col_idx, values);
    auto m = std::make_unique<pdb_matrix_s>();
    upload_csr(h, m->a, default_stream());
    *out = m.release();
  });
}

PDB_API pdb_status pdb_matrix_csr(pdb_matrix m, int64_t* row_ptr, int64_t* col_idx, double* values) {
  if (m == nullptr || row_ptr == nullptr || col_idx == nullptr || values == nullptr) return arg_error("null argument");
  return guarded([&] {
    HostCsr h = download_csr(m->a, default_stream());
    std::memcpy(row_ptr, h.row_ptr.data(), h.row_ptr.size() * sizeof(int64_t));
    for (size_t p = 0; p < h.col.size(); ++p) col_idx[p] = h.col[p];
    std::memcpy(values, h.val.data(), h.val.size() * sizeof(double));
  });
}

/* ---- problems ---- */

PDB_API pdb_status pdb_problem_assemble(const char* config_json, pdb_problem* out) {
  if (config_json == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    ModelConfig m = parse_model_config(config_json);
    resolve_model_coefficient(m);
    auto p = std::make_unique<pdb_problem_s>();
    assemble_model_problem(m, *p);
    *out = p.release();
  });
}

PDB_API int64_t pdb_problem_ndofs(pdb_problem p) { return p == nullptr ? 0 : p->a.n; }
PDB_API int64_t pdb_problem_nnz(pdb_problem p) { return p == nullptr ? 0 : p->a.nnz(); }

PDB_API pdb_status pdb_problem_matrix(pdb_problem p, pdb_matrix* out) {
  if (p == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(!p->is_slab(), Errc::invalid_argument,
            "slab problem holds a row block with global columns: use pdb_shard_create_local");
    auto m = std::make_unique<pdb_matrix_s>();
    upload_csr(p->a, m->a, default_stream());
    *out = m.release();
  });
}

PDB_API pdb_status pdb_problem_rhs(pdb_problem p, double* out) {
  if (p == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] { std::memcpy(out, p->rhs.data(), p->rhs.size() * sizeof(double)); });
}

PDB_API pdb_status pdb_problem_csr(pdb_problem p, int64_t* row_ptr, int64_t* col_idx, double* values) {
  if (p == nullptr || row_ptr == nullptr || col_idx == nullptr || values == nullptr) return arg_error("null argument");
  return guarded([&] {
    std::memcpy(row_ptr, p->a.row_ptr.data(), p->a.row_ptr.size() * sizeof(int64_t));
    for (size_t q = 0; q < p->a.col.size(); ++q) col_idx[q] = p->a.col[q];
    std::memcpy(values, p->a.val.data(), p->a.val.size() * sizeof(double));
  });
}

PDB_API pdb_status pdb_problem_exact_solution(pdb_problem p, double* out) {
  if (p == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(p->has_exact, Errc::invalid_argument, "problem has no manufactured solution (generated input)");
    std::memcpy(out, p->exact.data(), p->exact.size() * sizeof(double));
  });
}

PDB_API pdb_status pdb_problem_l2_error(pdb_problem p, const double* discrete_solution, double* out) {
  if (p == nullptr || discrete_solution == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] { *out = model_l2_error(*p, discrete_solution); });
}

PDB_API void pdb_problem_free(pdb_problem p) { delete p; }

PDB_API void pdb_gen_options_init(pdb_gen_options* o) { gen_options_defaults(o); }

// BASELINE.json configs, presets in generator.cpp.
PDB_API pdb_status pdb_gen_options_config(int config, int64_t cells, pdb_gen_options* o) {
  if (o == nullptr) return arg_error("null argument");
  if (!gen_options_preset(config, cells, o)) return arg_error("config must be 1..5");
  return PDB_OK;
}

PDB_API pdb_status pdb_problem_generate(const pdb_gen_options* o, pdb_problem* out) {
  if (o == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(o->physics >= 0 && o->physics <= 2, Errc::invalid_argument,
            "physics must be 0 (diffusion), 1 (Stokes) or 2 (elasticity)");
    require(o->bc_mode == 0, Errc::invalid_argument, "only Dirichlet row replacement (bc_mode 0) is supported");
    auto p = std::make_unique<pdb_problem_s>();
    if (o->physics == 0)
      generate_scalar(*o, *p);
    else
      generate_system(*o, *p);
    *out = p.release();
  });
}

PDB_API pdb_status pdb_problem_generate_slab(const pdb_gen_options* o, int rank, int nranks, pdb_problem* out) {
  if (o == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(o->physics >= 0 && o->physics <= 2, Errc::invalid_argument,
            "physics must be 0 (diffusion), 1 (Stokes) or 2 (elasticity)");
    require(o->bc_mode == 0, Errc::invalid_argument, "only Dirichlet row replacement (bc_mode 0) is supported");
    const RowWindow w = slab_window(*o, rank, nranks);
    auto p = std::make_unique<pdb_problem_s>();
    if (o->physics == 0)
      generate_scalar(*o, *p, &w);
    else
      generate_system(*o, *p, &w);
    p->slab_rank = rank;
    p->slab_ranks = nranks;
    *out = p.release();
  });
}

PDB_API pdb_status pdb_problem_generate_cells(const pdb_gen_options* o, int64_t c0, int64_t c1, int rank, int nranks,
                                              pdb_problem* out) {
  if (o == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(o->physics >= 0 && o->physics <= 2, Errc::invalid_argument,
            "physics must be 0 (diffusion), 1 (Stokes) or 2 (elasticity)");
    const RowWindow w = cells_window(*o, c0, c1);
    auto p = std::make_unique<pdb_problem_s>();
    if (o->physics == 0)
      generate_scalar(*o, *p, &w);
    else
      generate_system(*o, *p, &w);
    p->slab_rank = rank;
    p->slab_ranks = nranks;
    *out = p.release();
  });
}

PDB_API int64_t pdb_problem_rows_global(pdb_problem p) {
  return p == nullptr ? 0 : (p->is_slab() ? p->n_global : p->a.n);
}

PDB_API int64_t pdb_problem_row_range_count(pdb_problem p) {
  return p == nullptr ? 0 : (p->is_slab() ? static_cast<int64_t>(p->row_ranges.size()) : 1);
}

PDB_API pdb_status pdb_problem_row_ranges(pdb_problem p, int64_t* r) {
  if (p == nullptr || r == nullptr) return arg_error("null argument");
  return guarded([&] {
    if (!p->is_slab()) {
      r[0] = 0;
      r[1] = p->a.n;
      return;
    }
    for (size_t k = 0; k < p->row_ranges.size(); ++k) {
      r[2 * k] = p->row_ranges[k].first;
      r[2 * k + 1] = p->row_ranges[k].second;
    }
  });
}

/* ---- patch sets ---- */

PDB_API pdb_status pdb_patchset_detect(pdb_matrix m, int64_t patch_size, pdb_patchset* out) {
  if (m == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    auto ps = std::make_unique<pdb_patchset_s>();
    detect_patches(m->a, patch_size, *ps, default_stream());
    *out = ps.release();
  });
}

PDB_API int64_t pdb_patchset_count(pdb_patchset ps) { return ps == nullptr ? 0 : ps->np; }
PDB_API int64_t pdb_patchset_patch_size(pdb_patchset ps) { return ps == nullptr ? 0 : ps->ps; }
PDB_API int64_t pdb_patchset_rows(pdb_patchset ps) { return ps == nullptr ? 0 : ps->n; }

PDB_API pdb_status pdb_patchset_write_json(pdb_patchset ps, const char* path) {
  if (ps == nullptr || path == nullptr) return arg_error("null argument");
  return guarded([&] { write_patchset_json(*ps, path, default_stream()); });
}

PDB_API pdb_status pdb_patchset_patches(pdb_patchset ps, int64_t* patches) {
  if (ps == nullptr || patches == nullptr) return arg_error("null argument");
  return guarded([&] {
    const std::vector<int64_t> h = patches_host(*ps, default_stream());
    std::memcpy(patches, h.data(), h.size() * sizeof(int64_t));
  });
}

PDB_API pdb_status pdb_patchset_weights(pdb_patchset ps, double* weights) {
  if (ps == nullptr || weights == nullptr) return arg_error("null argument");
  return guarded([&] {
    ps->weights.download(weights, static_cast<size_t>(ps->n), default_stream());
    sync(default_stream());
  });
}

PDB_API pdb_status pdb_patchset_extract(pdb_matrix m, pdb_patchset ps, double* out) {
  if (m == nullptr || ps == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    DevBuf<double> mats;
    extract_patches(m->a, *ps, mats, default_stream());
    mats.download(out, mats.size(), default_stream());
    sync(default_stream());
  });
}

PDB_API void pdb_patchset_free(pdb_patchset ps) { delete ps; }

/* ---- databases ---- */

PDB_API void pdb_compress_options_init(pdb_compress_options* opts) {
  if (opts == nullptr) return;
  opts->method = PDB_METHOD_GREEDY_L1;
  opts->eps = 1e-7;
  opts->db_size = 0;
  opts->seed = 42;
  opts->max_iters = 50;
  opts->best_match = 0;
  opts->threads = 1;
}

static BuildParams params_of(const pdb_compress_options* o) {
  BuildParams p;
  p.method = o->method;
  p.eps = o->eps;
  p.db_size = o->db_size;
  p.seed = o->seed;
  p.max_iters = o->max_iters;
  p.best_match = o->best_match != 0;
  return p;
}

PDB_API pdb_status pdb_database_build(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                      pdb_database* out) {
  if (m == nullptr || ps == nullptr || opts == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    auto db = std::make_unique<pdb_database_s>();
    build_database(m->a, *ps, params_of(opts), *db, default_stream());
    *out = db.release();
  });
}

PDB_API pdb_status pdb_comm_create(const unsigned char* id128, int rank, int nranks, pdb_comm* out) {
  if (id128 == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] { *out = comm_create(id128, rank, nranks); });
}

PDB_API void pdb_comm_free(pdb_comm c) { comm_delete(c); }

PDB_API pdb_status pdb_database_build_sharded(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                              pdb_comm comm, pdb_database* out) {
  if (m == nullptr || ps == nullptr || opts == nullptr || comm == nullptr || out == nullptr)
    return arg_error("null argument");
  return guarded([&] {
    auto db = std::make_unique<pdb_database_s>();
    BuildParams p = params_of(opts);
    p.comm = &comm_of(comm);
    build_database(m->a, *ps, p, *db, default_stream());
    *out = db.release();
  });
}

PDB_API pdb_status pdb_database_build_to_size_sharded(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                                      int64_t target_lo, int64_t target_hi, pdb_comm comm,
                                                      pdb_database* out, double* eps_out) {
  if (m == nullptr || ps == nullptr || opts == nullptr || comm == nullptr || out == nullptr)
    return arg_error("null argument");
  return guarded([&] {
    auto db = std::make_unique<pdb_database_s>();
    BuildParams p = params_of(opts);
    p.comm = &comm_of(comm);
    const double eps = bisect_database(m->a, *ps, p, target_lo, target_hi, *db, default_stream());
    if (eps_out) *eps_out = eps;
    *out = db.release();
  });
}

PDB_API pdb_status pdb_database_build_to_size(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                              int64_t target_lo, int64_t target_hi, pdb_database* out,
                                              double* eps_out) {
  if (m == nullptr || ps == nullptr || opts == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    auto db = std::make_unique<pdb_database_s>();
    const double eps = bisect_database(m->a, *ps, params_of(opts), target_lo, target_hi, *db, default_stream());
    if (eps_out) *eps_out = eps;
    *out = db.release();
  });
}

PDB_API pdb_status pdb_database_objective(pdb_matrix m, pdb_patchset ps, pdb_database db, double beta,
                                          double* out) {
  if (m == nullptr || ps == nullptr || db == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] { *out = database_objective(m->a, *ps, *db, beta, default_stream()); });
}

PDB_API pdb_status pdb_compressibility_curve(pdb_matrix m, pdb_patchset ps, pdb_method method, const double* eps_grid,
                                             int64_t count, int64_t* db_sizes, double* ratios) {
  if (m == nullptr || ps == nullptr || db_sizes == nullptr || ratios == nullptr || (count > 0 && eps_grid == nullptr))
    return arg_error("null argument");
  return guarded([&] {
    require(method == PDB_METHOD_GREEDY_SPECTRAL || method == PDB_METHOD_GREEDY_L1, Errc::invalid_argument,
            "compressibility_curve needs a greedy method (spectral or l1)");
    compressibility_curve(m->a, *ps, method == PDB_METHOD_GREEDY_SPECTRAL, eps_grid, count, db_sizes, ratios,
                          default_stream());
  });
}

PDB_API int64_t pdb_database_size(pdb_database db) { return db == nullptr ? 0 : db->m; }
PDB_API int64_t pdb_database_n_patches(pdb_database db) { return db == nullptr ? 0 : db->np; }
PDB_API int64_t pdb_database_patch_size(pdb_database db) { return db == nullptr ? 0 : db->ps; }
PDB_API double pdb_database_eps(pdb_database db) { return db == nullptr ? 0.0 : db->eps; }

PDB_API pdb_status pdb_database_phi(pdb_database db, int64_t* phi) {
  if (db == nullptr || phi == nullptr) return arg_error("null argument");
  return guarded([&] {
    const std::vector<int32_t> h = db->phi.to_host(default_stream());
    for (int64_t k = 0; k < db->np; ++k) phi[k] = h[static_cast<size_t>(k)];
  });
}

PDB_API pdb_status pdb_database_representatives(pdb_database db, double* reps) {
  if (db == nullptr || reps == nullptr) return arg_error("null argument");
  return guarded([&] {
    db->reps.download(reps, static_cast<size_t>(db->m * db->ps * db->ps), default_stream());
    sync(default_stream());
  });
}

PDB_API pdb_status pdb_database_factors(pdb_database db, double* lu, int64_t* pivots) {
  if (db == nullptr || lu == nullptr || pivots == nullptr) return arg_error("null argument");
  return guarded([&] {
    db->lu.download(lu, static_cast<size_t>(db->m * db->ps * db->ps), default_stream());
    std::vector<int32_t> p(static_cast<size_t>(db->m * db->ps));
    db->piv.download(p.data(), p.size(), default_stream());
    sync(default_stream());
    for (size_t q = 0; q < p.size(); ++q) pivots[q] = p[q];
  });
}

PDB_API pdb_status pdb_database_work(pdb_database db, int64_t* pair_evals, int64_t* power_iters, int64_t* lu_count) {
  if (db == nullptr) return arg_error("null argument");
  if (pair_evals) *pair_evals = db->work.pair_evals;
  if (power_iters) *power_iters = db->work.power_iters;
  if (lu_count) *lu_count = db->work.lu_count;
  return PDB_OK;
}

PDB_API pdb_status pdb_database_import(const char* json_path, const char* bin_path, pdb_database* out) {
  if (json_path == nullptr || bin_path == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    auto db = std::make_unique<pdb_database_s>();
    import_database(json_path, bin_path, *db, default_stream());
    *out = db.release();
  });
}

PDB_API pdb_status pdb_database_export(pdb_database db, const char* json_path, const char* bin_path) {
  if (db == nullptr || json_path == nullptr || bin_path == nullptr) return arg_error("null argument");
  return guarded([&] { export_database(*db, json_path, bin_path, default_stream()); });
}

PDB_API void pdb_database_free(pdb_database db) { delete db; }

/* ---- preconditioners ---- */

PDB_API pdb_status pdb_precond_create(pdb_matrix m, pdb_patchset ps, pdb_database db, double omega, int threads,
                                      pdb_precond* out) {
  (void)threads;
  if (ps == nullptr || out == nullptr) return arg_error("null argument");
  if (db == nullptr && m == nullptr) return arg_error("exact preconditioner needs the matrix");
  return guarded([&] {
    auto pc = std::make_unique<pdb_precond_s>();
    if (db == nullptr)
      precond_exact(m->a, *ps, omega, *pc, default_stream());
    else
      precond_compressed(*ps, *db, omega, *pc, default_stream());
    *out = pc.release();
  });
}

PDB_API pdb_status pdb_precond_create_combo(pdb_problem p, pdb_patchset ps, pdb_database db, double omega,
                                            int threads, pdb_precond* out) {
  (void)threads;
  if (p == nullptr || ps == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    cudaStream_t s = default_stream();
    auto pc = std::make_unique<pdb_precond_s>();
    if (db == nullptr) {
      require_device();
      DeviceCsr a;
      upload_csr(p->a, a, s);
      precond_exact(a, *ps, omega, *pc, s);
    } else {
      precond_compressed(*ps, *db, omega, *pc, s);
    }
    const CoarseSpaceHost cs = build_coarse_space(*p);
    require(cs.p0.rows == pc->n, Errc::dimension_mismatch, "transfer operator does not match the patch term");
    pc->coarse = std::make_shared<CoarseDev>();
    coarse_setup(cs, *pc->coarse, s);
    *out = pc.release();
  });
}

PDB_API pdb_status pdb_precond_apply(pdb_precond pc, const double* r, double* z) {
  if (pc == nullptr || r == nullptr || z == nullptr) return arg_error("null argument");
  return guarded([&] {
    require_device();
    cudaStream_t s = default_stream();
    const size_t n = static_cast<size_t>(pc->n);
    Scratch<double> dr(std::max<size_t>(n, 1), s), dz(std::max<size_t>(n, 1), s);
    PDB_CUDA(cudaMemcpyAsync(dr.get(), r, n * sizeof(double), cudaMemcpyHostToDevice, s));
    precond_apply_device(*pc, dr.get(), dz.get(), s);
    PDB_CUDA(cudaMemcpyAsync(z, dz.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

PDB_API pdb_status pdb_precond_apply_device(pdb_precond pc, const double* d_r, double* d_z, void* stream) {
  if (pc == nullptr || d_r == nullptr || d_z == nullptr) return arg_error("null argument");
  return guarded([&] {
    require_device();
    precond_apply_device(*pc, d_r, d_z, stream_of(stream));
  });
}

PDB_API pdb_status pdb_relax(pdb_matrix m, pdb_precond pc, const double* b, double* x, int64_t sweeps,
                             double* history) {
  if (m == nullptr || pc == nullptr || b == nullptr || x == nullptr) return arg_error("null argument");
  return guarded([&] {
    require_device();
    require(sweeps >= 0, Errc::invalid_argument, "sweeps must be >= 0");
    relax_host(m->a, *pc, b, x, sweeps, history, default_stream());
  });
}

PDB_API pdb_status pdb_relax_device(pdb_matrix m, pdb_precond pc, const double* d_b, double* d_x, int64_t sweeps,
                                    double* d_history, void* stream) {
  if (m == nullptr || pc == nullptr || d_b == nullptr || d_x == nullptr) return arg_error("null argument");
  return guarded([&] {
    require_device();
    require(sweeps >= 0, Errc::invalid_argument, "sweeps must be >= 0");
    relax_device(m->a, *pc, d_b, d_x, sweeps, d_history, stream_of(stream));
  });
}

PDB_API pdb_status pdb_relax_profile(pdb_matrix m, pdb_precond pc, const double* d_b, double* d_x, int64_t sweeps,
                                     double* ms_phase, void* stream) {
  if (m == nullptr || pc == nullptr || d_b == nullptr || d_x == nullptr || ms_phase == nullptr)
    return arg_error("null argument");
  return guarded([&] {
    require_device();
    require(sweeps >= 1, Errc::invalid_argument, "sweeps must be >= 1");
    relax_profile(m->a, *pc, d_b, d_x, sweeps, ms_phase, stream_of(stream));
  });
}

PDB_API pdb_status pdb_matrix_sell_info(pdb_matrix m, int64_t* out4) {
  if (m == nullptr || out4 == nullptr) return arg_error("null argument");
  return guarded([&] {
    const DeviceCsr& a = m->a;
    const bool sell = a.nslices > 0;
    out4[0] = sell ? a.sell_classes : 0;
    out4[1] = sell && a.sell_classes == 0 ? static_cast<int64_t>(a.sell_col.size()) : 0;
    out4[2] = a.nslices;
    out4[3] = sell ? static_cast<int64_t>(a.sell_val.size()) : 0;
  });
}

PDB_API pdb_status pdb_matrix_mirror_info(pdb_matrix m, int64_t* out4, const char** why) {
  if (m == nullptr || out4 == nullptr) return arg_error("null argument");
  return guarded([&] {
    const DeviceCsr& a = m->a;
    out4[0] = a.mirror ? 1 : 0;
    out4[1] = a.mirror ? static_cast<int64_t>(a.sell_val.size()) : 0;
    out4[2] = a.mirror ? a.mir_virtual : 0;
    out4[3] = a.mirror ? static_cast<int64_t>(a.sell_tab.size()) : 0;
    if (why) *why = a.mir_why.c_str();
  });
}

PDB_API pdb_status pdb_debug_mirror_check(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                          const double* values, const double* x, double* y, int64_t* out6) {
  if (row_ptr == nullptr || out6 == nullptr || (n > 0 && (col_idx == nullptr || values == nullptr || x == nullptr ||
                                                          y == nullptr)))
    return arg_error("null argument");
  return guarded([&] {
    const HostCsr h = validated_csr(n, row_ptr, col_idx, values);
    std::vector<int32_t> cls, tab, tstart;
    MirrorHost M;
    const bool classed = sell_classes(h, cls, tab, tstart);
    const bool built = classed && build_mirror_host(h, cls, tab, tstart, k::kSellSigma, M);
    out6[0] = built ? 1 : 0;
    out6[1] = built ? M.nslices : 0;
    out6[2] = built ? static_cast<int64_t>(M.val.size()) : 0;
    out6[3] = built ? static_cast<int64_t>(tab.size()) : 0;
    out6[4] = built ? static_cast<int64_t>(tstart.size()) - 1 : 0;
    out6[5] = built ? M.virtual_rows : 0;
    if (built) mirror_spmv_host(M, tab, tstart, x, y);
    g_last_error = built ? "" : (classed ? M.why : std::string("rows do not share column patterns"));
  });
}

PDB_API int64_t pdb_precond_stored_factors(pdb_precond pc) { return pc == nullptr ? 0 : pc->nf; }
PDB_API int64_t pdb_precond_patch_count(pdb_precond pc) { return pc == nullptr ? 0 : pc->np; }
PDB_API int64_t pdb_precond_patch_size(pdb_precond pc) { return pc == nullptr ? 0 : pc->ps; }

PDB_API pdb_status pdb_precond_coarse_size(pdb_precond pc, int64_t* nc, int64_t* kl, int64_t* ku) {
  if (pc == nullptr || nc == nullptr || kl == nullptr || ku == nullptr) return arg_error("null argument");
  const CoarseDev* c = pc->coarse.get();
  *nc = c ? c->nc : 0;
  *kl = c ? c->kl : 0;
  *ku = c ? c->ku : 0;
  return PDB_OK;
}

PDB_API pdb_status pdb_precond_coarse_factor(pdb_precond pc, double* band, int64_t* ipiv) {
  if (pc == nullptr) return arg_error("null argument");
  return guarded([&] {
    const CoarseDev* c = pc->coarse.get();
    require(c != nullptr, Errc::invalid_argument, "not a combo preconditioner");
    cudaStream_t s = default_stream();
    const size_t n = static_cast<size_t>(c->nc), ld = static_cast<size_t>(c->ldab);
    if (band) {
      const std::vector<double> cm = c->band.to_host(s);  // column-major [n][ldab]
      for (size_t j = 0; j < n; ++j)
        for (size_t r = 0; r < ld; ++r) band[r * n + j] = cm[j * ld + r];
    }
    if (ipiv) {
      const std::vector<int32_t> p = c->ipiv.to_host(s);
      for (size_t j = 0; j < n; ++j) ipiv[j] = p[j];
    }
  });
}

PDB_API void pdb_precond_free(pdb_precond pc) { delete pc; }

/* ---- solvers ---- */

PDB_API void pdb_gmres_options_init(pdb_gmres_options* opts) {
  if (opts == nullptr) return;
  opts->restart = 20;
  opts->tol = 1e-8;
  opts->max_iters = 2000;
  opts->left_precond = 0;
  opts->threads = 1;
}

PDB_API pdb_status pdb_gmres_solve(pdb_matrix m, const double* b, pdb_precond pc, const pdb_gmres_options* opts,
                                   double* x, pdb_report* out_report) {
  if (m == nullptr || b == nullptr || opts == nullptr || x == nullptr) return arg_error("null argument");
  return guarded([&] {
    auto rep = std::make_unique<pdb_report_s>();
    gmres_device(m->a, b, pc, *opts, x, *rep, default_stream());
    if (out_report != nullptr) *out_report = rep.release();
  });
}

PDB_API pdb_status pdb_pcg_solve(pdb_matrix m, const double* b, pdb_precond pc, double tol, int64_t max_iters,
                                 double* x, pdb_report* out_report) {
  if (m == nullptr || b == nullptr || x == nullptr) return arg_error("null argument");
  return guarded([&] {
    auto rep = std::make_unique<pdb_report_s>();
    pcg_device(m->a, b, pc, tol, max_iters, x, *rep, default_stream());
    if (out_report != nullptr) *out_report = rep.release();
  });
}

PDB_API pdb_status pdb_pcg_solve_ex(pdb_matrix m, const double* b, pdb_precond pc, double tol, int64_t max_iters,
                                    int flags, double* x, pdb_report* out_report) {
  if (m == nullptr || b == nullptr || x == nullptr) return arg_error("null argument");
  return guarded([&] {
    auto rep = std::make_unique<pdb_report_s>();
    pcg_device(m->a, b, pc, tol, max_iters, x, *rep, default_stream(), (flags & PDB_PCG_REPRODUCIBLE) != 0);
    if (out_report != nullptr) *out_report = rep.release();
  });
}

PDB_API int64_t pdb_report_iterations(pdb_report rep) { return rep == nullptr ? 0 : rep->iterations; }
PDB_API int64_t pdb_report_restarts(pdb_report rep) { return rep == nullptr ? 0 : rep->restarts; }
PDB_API int pdb_report_converged(pdb_report rep) { return rep != nullptr && rep->converged ? 1 : 0; }
PDB_API double pdb_report_final_relative_residual(pdb_report rep) {
  return rep == nullptr ? 0.0 : rep->final_relative_residual;
}
PDB_API int64_t pdb_report_residual_history_size(pdb_report rep) {
  return rep == nullptr ? 0 : static_cast<int64_t>(rep->residual_history.size());
}
PDB_API pdb_status pdb_report_residual_history(pdb_report rep, double* out) {
  if (rep == nullptr || out == nullptr) return arg_error("null argument");
  std::memcpy(out, rep->residual_history.data(), rep->residual_history.size() * sizeof(double));
  return PDB_OK;
}
PDB_API void pdb_report_free(pdb_report rep) { delete rep; }

/* ---- multi-GPU shards ---- */

PDB_API pdb_status pdb_shard_plan_create(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                         const double* values, int64_t n_patches, int64_t patch_size,
                                         const int64_t* patches, const double* weights, int rank, int nranks,
                                         pdb_shard_plan* out) {
  if (row_ptr == nullptr || col_idx == nullptr || values == nullptr || patches == nullptr || weights == nullptr ||
      out == nullptr)
    return arg_error("null argument");
  return guarded([&] {
    HostCsr h = validated_csr(n, row_ptr, col_idx, values);
    std::vector<int32_t> p32(static_cast<size_t>(n_patches * patch_size));
    for (size_t q = 0; q < p32.size(); ++q) {
      require(patches[q] >= 0 && patches[q] < n, Errc::index_out_of_range, "patch index outside matrix");
      p32[q] = static_cast<int32_t>(patches[q]);
    }
    auto plan = std::make_unique<pdb_shard_plan_s>();
    plan->p = plan_shard(n, h.row_ptr.data(), h.col.data(), h.val.data(), n_patches, patch_size, p32.data(), weights,
                         rank, nranks);
    *out = plan.release();
  });
}

PDB_API int64_t pdb_shard_plan_size(pdb_shard_plan plan, int which) {
  return plan == nullptr ? 0 : plan_array(plan->p, which, nullptr);
}

PDB_API pdb_status pdb_shard_plan_get(pdb_shard_plan plan, int which, void* out) {
  if (plan == nullptr || out == nullptr) return arg_error("null argument");
  if (plan_array(plan->p, which, out) < 0) return arg_error("unknown plan array");
  return PDB_OK;
}

PDB_API void pdb_shard_plan_free(pdb_shard_plan plan) { delete plan; }

PDB_API pdb_status pdb_comm_unique_id(unsigned char* id128) {
  if (id128 == nullptr) return arg_error("null argument");
  return guarded([&] { comm_unique_id(id128); });
}

PDB_API pdb_status pdb_shard_create(pdb_matrix m, pdb_patchset ps, pdb_database db, double omega, int rank,
                                    int nranks, pdb_shard* out) {
  if (m == nullptr || ps == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    HostCsr h = download_csr(m->a, default_stream());
    pdb_shard sh = shard_new();
    try {
      shard_create(h, *ps, db, omega, rank, nranks, *sh, default_stream());
    } catch (...) {
      shard_delete(sh);
      throw;
    }
    *out = sh;
  });
}

PDB_API pdb_status pdb_shard_attach_comm(pdb_shard sh, const unsigned char* id128) {
  if (sh == nullptr || id128 == nullptr) return arg_error("null argument");
  return guarded([&] { shard_attach(*sh, id128); });
}

PDB_API int64_t pdb_shard_local_size(pdb_shard sh) { return sh == nullptr ? 0 : shard_local_size(*sh); }

PDB_API pdb_status pdb_shard_local_dofs(pdb_shard sh, int64_t* global_ids) {
  if (sh == nullptr || global_ids == nullptr) return arg_error("null argument");
  return guarded([&] { plan_array(shard_plan(*sh), PDB_PLAN_DOFS, global_ids); });
}

PDB_API int64_t pdb_shard_owned_count(pdb_shard sh) {
  return sh == nullptr ? 0 : static_cast<int64_t>(shard_plan(*sh).owned.size());
}

PDB_API pdb_status pdb_shard_owned(pdb_shard sh, int64_t* local_idx) {
  if (sh == nullptr || local_idx == nullptr) return arg_error("null argument");
  return guarded([&] { plan_array(shard_plan(*sh), PDB_PLAN_OWNED, local_idx); });
}

PDB_API pdb_status pdb_shard_relax_device(pdb_shard sh, const double* d_b, double* d_x, int64_t sweeps, void* stream) {
  if (sh == nullptr || d_b == nullptr || d_x == nullptr) return arg_error("null argument");
  return guarded([&] {
    require_device();
    require(sweeps >= 0, Errc::invalid_argument, "sweeps must be >= 0");
    shard_relax(*sh, d_b, d_x, sweeps, stream_of(stream));
  });
}

PDB_API void pdb_shard_free(pdb_shard sh) { shard_delete(sh); }

/* ---- rank-local multi-GPU shards (slab.cu) ---- */

PDB_API pdb_status pdb_slab_create(pdb_problem* slabs, int count, int rank, int nranks, int64_t patch_size,
                                   pdb_database db, double omega, const unsigned char* nccl_id, pdb_slab* out) {
  return pdb_slab_create_subset(slabs, count, nullptr, rank, nranks, patch_size, db, omega, nccl_id, out);
}

PDB_API pdb_status pdb_slab_create_subset(pdb_problem* slabs, int count, const int* ranks, int rank, int nranks,
                                          int64_t patch_size, pdb_database db, double omega,
                                          const unsigned char* nccl_id, pdb_slab* out) {
  if (slabs == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(count >= 1, Errc::invalid_argument, "need at least one slab");
    require(patch_size >= 1, Errc::invalid_argument, "patch_size must be >= 1");
    const bool emulated = nccl_id == nullptr && nranks > 1;
    std::vector<int> rl;
    if (emulated) {
      for (int i = 0; i < count; ++i) rl.push_back(ranks ? ranks[i] : i);
      for (int i = 0; i < count; ++i)
        require(rl[static_cast<size_t>(i)] >= 0 && rl[static_cast<size_t>(i)] < nranks &&
                    (i == 0 || rl[static_cast<size_t>(i)] > rl[static_cast<size_t>(i) - 1]),
                Errc::invalid_argument, "emulated ranks must be ascending in [0, nranks)");
      require(ranks != nullptr || count == nranks, Errc::invalid_argument,
              "an emulated group holds all nranks slabs (or name its subset of ranks)");
      require(ranks == nullptr || db == nullptr, Errc::invalid_argument,
              "a subset of ranks cannot place the database's phi: exact preconditioners only");
    } else {
      require(count == 1, Errc::invalid_argument, "one slab per process with a communicator");
    }
    std::vector<pdb_problem_s*> probs;
    for (int i = 0; i < count; ++i) {
      require(slabs[i] != nullptr, Errc::invalid_argument, "null argument");
      probs.push_back(slabs[i]);
    }
    std::unique_ptr<pdb_slab_s, void (*)(pdb_slab_s*)> g(slab_new(rank, nranks, emulated, rl), slab_delete);
    if (nccl_id != nullptr && nranks > 1) slab_attach(*g, nccl_id);
    slab_setup(*g, probs, patch_size, db, omega, default_stream());
    *out = g.release();
  });
}

PDB_API pdb_status pdb_slab_create_built(pdb_problem* slabs, int count, int rank, int nranks, int64_t patch_size,
                                         const pdb_compress_options* opts, double omega, const unsigned char* nccl_id,
                                         pdb_slab* out) {
  if (slabs == nullptr || opts == nullptr || out == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(count >= 1, Errc::invalid_argument, "need at least one slab");
    require(patch_size >= 1, Errc::invalid_argument, "patch_size must be >= 1");
    const bool emulated = nccl_id == nullptr && nranks > 1;
    require(emulated ? count == nranks : count == 1, Errc::invalid_argument,
            "one slab per process with a communicator, all nranks slabs for an emulated group");
    std::vector<pdb_problem_s*> probs;
    for (int i = 0; i < count; ++i) {
      require(slabs[i] != nullptr, Errc::invalid_argument, "null argument");
      probs.push_back(slabs[i]);
    }
    BuildParams p;
    p.method = opts->method;
    p.eps = opts->eps;
    p.best_match = opts->best_match != 0;
    p.db_size = opts->db_size;
    p.seed = opts->seed;
    p.max_iters = opts->max_iters;
    std::unique_ptr<pdb_slab_s, void (*)(pdb_slab_s*)> g(slab_new(rank, nranks, emulated), slab_delete);
    if (nccl_id != nullptr && nranks > 1) slab_attach(*g, nccl_id);
    slab_setup(*g, probs, patch_size, nullptr, omega, default_stream(), &p);
    *out = g.release();
  });
}

PDB_API int64_t pdb_slab_database_size(pdb_slab sh) { return sh == nullptr ? 0 : slab_database_size(*sh); }

PDB_API pdb_status pdb_slab_phi(pdb_slab sh, int i, int64_t* phi) {
  if (sh == nullptr || phi == nullptr) return arg_error("null argument");
  return guarded([&] { slab_phi(*sh, i, phi); });
}

PDB_API pdb_status pdb_slab_creators(pdb_slab sh, int64_t* creators) {
  if (sh == nullptr || creators == nullptr) return arg_error("null argument");
  return guarded([&] { slab_creators(*sh, creators); });
}

PDB_API int pdb_slab_local_ranks(pdb_slab sh) { return sh == nullptr ? 0 : slab_local_ranks(*sh); }

PDB_API double pdb_slab_upload_seconds(pdb_slab sh) { return sh == nullptr ? 0.0 : slab_upload_seconds(*sh); }

PDB_API pdb_status pdb_slab_info(pdb_slab sh, int i, int64_t* info) {
  if (sh == nullptr || info == nullptr) return arg_error("null argument");
  return guarded([&] {
    const SlabInfo f = slab_info(*sh, i);
    const int64_t v[12] = {f.rank, f.nranks, f.n_local, f.n_rows, f.n_patches, f.first_patch, f.split, f.n_owned,
                           f.n_up, f.n_pin, f.n_xs, f.n_xr};
    std::memcpy(info, v, sizeof(v));
  });
}

PDB_API pdb_status pdb_slab_local_dofs(pdb_slab sh, int i, int64_t* global_ids) {
  if (sh == nullptr || global_ids == nullptr) return arg_error("null argument");
  return guarded([&] { slab_local_dofs(*sh, i, global_ids); });
}

PDB_API pdb_status pdb_slab_owned(pdb_slab sh, int i, int64_t* local_idx) {
  if (sh == nullptr || local_idx == nullptr) return arg_error("null argument");
  return guarded([&] { slab_owned(*sh, i, local_idx); });
}

PDB_API pdb_status pdb_slab_relax_device(pdb_slab sh, const double* const* d_b, double* const* d_x, int64_t sweeps,
                                         void* stream) {
  if (sh == nullptr || d_b == nullptr || d_x == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(sweeps >= 0, Errc::invalid_argument, "sweeps must be >= 0");
    const int L = slab_local_ranks(*sh);
    std::vector<const double*> b(d_b, d_b + L);
    std::vector<double*> x(d_x, d_x + L);
    slab_relax(*sh, b, x, sweeps, stream_of(stream));
  });
}

PDB_API pdb_status pdb_slab_relax_rank_device(pdb_slab sh, int i, const double* d_b, double* d_x, int64_t sweeps,
                                              void* stream) {
  if (sh == nullptr || d_b == nullptr || d_x == nullptr) return arg_error("null argument");
  return guarded([&] {
    require(i >= 0 && i < slab_local_ranks(*sh), Errc::invalid_argument, "rank index out of range");
    slab_relax_one(*sh, i, d_b, d_x, sweeps, stream_of(stream));
  });
}

PDB_API void pdb_slab_free(pdb_slab sh) { slab_delete(sh); }

/* ---- experiment drivers (reference experiments.cpp; outside the hot path) ---- */

PDB_API pdb_status pdb_run_experiment(const char* config_json, const char* out_csv) {
  if (config_json == nullptr || out_csv == nullptr) return arg_error("null argument");
  return unsupported("pdb_run_experiment");
}

PDB_API pdb_status pdb_run_analyze(const char* config_json, const char* curve_csv, const char* histogram_csv) {
  if (config_json == nullptr || curve_csv == nullptr || histogram_csv == nullptr) return arg_error("null argument");
  return unsupported("pdb_run_analyze");
}

PDB_API pdb_status pdb_run_benchmark(const char* config_json, const char* out_csv) {
  if (config_json == nullptr || out_csv == nullptr) return arg_error("null argument");
  return unsupported("pdb_run_benchmark");
}

PDB_API pdb_status pdb_export_matrix(const char* config_json, const char* out_path) {
  if (config_json == nullptr || out_path == nullptr) return arg_error("null argument");
  return guarded([&] {  // experiments.cpp:430-435: smooth (experiment 1) or piecewise (2) fallback
    ModelConfig m = parse_model_config(config_json);
    resolve_model_coefficient(m, m.experiment == 2 ? "piecewise" : "smooth");
    pdb_problem_s p;
    assemble_model_problem(m, p);
    write_matrix_market_host(p.a, out_path);
  });
}

}  // extern "C"
