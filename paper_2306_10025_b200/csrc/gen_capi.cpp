// libpdbgen.so -- the seeded BASELINE input generator (generator.cpp) as a
// standalone host library with no CUDA and no patchdb symbols, so a process
// that runs only the reference (bench.py --impl reference, the golden-fixture
// scripts) can build the same inputs without loading libpatchdb.so.0.
// The same generator.cpp is linked into libpatchdb (pdb_problem_generate).
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "host.hpp"

#define GEN_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_error;
}

GEN_API const char* pdbgen_last_error() { return g_error.c_str(); }

// config 1..5, cells per axis (0 = the config's own size).  0 on success.
GEN_API int pdbgen_generate(int config, int64_t cells, void** out) {
  if (out == nullptr) return 1;
  try {
    pdb_gen_options o;
    if (!pdb::gen_options_preset(config, cells, &o)) {
      g_error = "config must be 1..5";
      return 1;
    }
    auto p = std::make_unique<pdb_problem_s>();
    if (o.physics == 0)
      pdb::generate_scalar(o, *p);
    else
      pdb::generate_system(o, *p);
    *out = p.release();
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 2;
  }
}

GEN_API int64_t pdbgen_n(void* p) { return p ? static_cast<pdb_problem_s*>(p)->a.n : 0; }
GEN_API int64_t pdbgen_nnz(void* p) { return p ? static_cast<pdb_problem_s*>(p)->a.nnz() : 0; }

GEN_API void pdbgen_csr(void* h, int64_t* row_ptr, int64_t* col_idx, double* values) {
  const auto& a = static_cast<pdb_problem_s*>(h)->a;
  std::memcpy(row_ptr, a.row_ptr.data(), a.row_ptr.size() * sizeof(int64_t));
  for (size_t q = 0; q < a.col.size(); ++q) col_idx[q] = a.col[q];
  std::memcpy(values, a.val.data(), a.val.size() * sizeof(double));
}

GEN_API void pdbgen_rhs(void* h, double* out) {
  const auto& r = static_cast<pdb_problem_s*>(h)->rhs;
  std::memcpy(out, r.data(), r.size() * sizeof(double));
}

GEN_API void pdbgen_free(void* h) { delete static_cast<pdb_problem_s*>(h); }
