/* Drop-in check driver (TEST INFRASTRUCTURE).  Plain C99 compiled against the
 * UNMODIFIED reference header (/root/reference/proj/include/patchdb/patchdb.h)
 * and linked by SONAME (libpatchdb.so.0), so the same binary runs against the
 * reference build (oracle/_ref/capi) or this repo's library, chosen with
 * LD_LIBRARY_PATH.  It walks the hot path the way an external host would:
 *
 *   read Matrix Market -> detect (patch size 9) -> write the patch set JSON
 *   -> for each of the 7 methods: build the database, phi, export JSON + bin,
 *      precondition (omega 0.8), one apply on a fixed vector, GMRES(20)
 *   -> error paths (null arguments, bad file, singular-free status strings)
 *
 * and writes everything under the output directory for tests/test_dropin.py. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "patchdb/patchdb.h"

static FILE* summary;

static void check(pdb_status st, const char* what) {
  fprintf(summary, "%s status=%d\n", what, (int)st);
  if (st != PDB_OK) fprintf(summary, "%s error=%s\n", what, pdb_last_error());
}

static void dump(const char* dir, const char* name, const void* data, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof(path), "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f) {
    fprintf(stderr, "cannot write %s\n", path);
    exit(2);
  }
  fwrite(data, 1, bytes, f);
  fclose(f);
}

int main(int argc, char** argv) {
  if (argc != 3) {
    fprintf(stderr, "usage: dropin <matrix.mtx> <out_dir>\n");
    return 2;
  }
  const char* dir = argv[2];
  char path[4096], path2[4096];
  snprintf(path, sizeof(path), "%s/summary.txt", dir);
  summary = fopen(path, "w");
  fprintf(summary, "sizeof_compress_options=%zu sizeof_gmres_options=%zu\n", sizeof(pdb_compress_options),
          sizeof(pdb_gmres_options));

  pdb_matrix m = NULL;
  check(pdb_matrix_read_matrix_market(argv[1], &m), "read");
  if (!m) return 1;
  const int64_t n = pdb_matrix_rows(m);
  fprintf(summary, "rows=%lld nnz=%lld\n", (long long)n, (long long)pdb_matrix_nnz(m));
  double* x = malloc(sizeof(double) * (size_t)n);
  double* y = malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) x[i] = (double)((i * 7919) % 2003) / 1001.0 - 1.0;
  check(pdb_matrix_spmv(m, x, y), "spmv");
  dump(dir, "spmv.bin", y, sizeof(double) * (size_t)n);

  pdb_patchset ps = NULL;
  check(pdb_patchset_detect(m, 9, &ps), "detect");
  fprintf(summary, "patches=%lld patch_size=%lld\n", (long long)pdb_patchset_count(ps),
          (long long)pdb_patchset_patch_size(ps));
  snprintf(path, sizeof(path), "%s/patchset.json", dir);
  check(pdb_patchset_write_json(ps, path), "write_json");

  const int64_t np = pdb_patchset_count(ps);
  int64_t* phi = malloc(sizeof(int64_t) * (size_t)np);
  for (int method = 0; method <= 6; ++method) {
    pdb_compress_options o;
    pdb_compress_options_init(&o);
    fprintf(summary, "m%d defaults method=%d eps=%.17g db_size=%lld seed=%llu max_iters=%d best_match=%d threads=%d\n",
            method, (int)o.method, o.eps, (long long)o.db_size, (unsigned long long)o.seed, o.max_iters, o.best_match,
            o.threads);
    o.method = (pdb_method)method;
    o.eps = method == 2 ? 2.0 : 0.5;
    o.db_size = 51;
    o.max_iters = 20;
    pdb_database db = NULL;
    char tag[64];
    snprintf(tag, sizeof(tag), "m%d build", method);
    check(pdb_database_build(m, ps, &o, &db), tag);
    if (!db) continue;
    fprintf(summary, "m%d size=%lld n_patches=%lld\n", method, (long long)pdb_database_size(db),
            (long long)pdb_database_n_patches(db));
    check(pdb_database_phi(db, phi), "phi");
    snprintf(tag, sizeof(tag), "phi_m%d.bin", method);
    dump(dir, tag, phi, sizeof(int64_t) * (size_t)np);
    snprintf(path, sizeof(path), "%s/db_m%d.json", dir, method);
    snprintf(path2, sizeof(path2), "%s/db_m%d.bin", dir, method);
    check(pdb_database_export(db, path, path2), "export");

    pdb_precond pc = NULL;
    check(pdb_precond_create(m, ps, method == 0 ? NULL : db, 0.8, 1, &pc), "precond");
    check(pdb_precond_apply(pc, x, y), "apply");
    snprintf(tag, sizeof(tag), "apply_m%d.bin", method);
    dump(dir, tag, y, sizeof(double) * (size_t)n);

    pdb_gmres_options go;
    pdb_gmres_options_init(&go);
    fprintf(summary, "gmres defaults restart=%lld tol=%.17g max_iters=%lld left=%d threads=%d\n",
            (long long)go.restart, go.tol, (long long)go.max_iters, go.left_precond, go.threads);
    pdb_report rep = NULL;
    check(pdb_gmres_solve(m, x, pc, &go, y, &rep), "gmres");
    if (rep) {
      const int64_t h = pdb_report_residual_history_size(rep);
      fprintf(summary, "m%d gmres iterations=%lld restarts=%lld converged=%d history=%lld\n", method,
              (long long)pdb_report_iterations(rep), (long long)pdb_report_restarts(rep), pdb_report_converged(rep),
              (long long)h);
      double* hist = malloc(sizeof(double) * (size_t)(h > 0 ? h : 1));
      check(pdb_report_residual_history(rep, hist), "history");
      snprintf(tag, sizeof(tag), "gmres_hist_m%d.bin", method);
      dump(dir, tag, hist, sizeof(double) * (size_t)h);
      snprintf(tag, sizeof(tag), "gmres_x_m%d.bin", method);
      dump(dir, tag, y, sizeof(double) * (size_t)n);
      free(hist);
      pdb_report_free(rep);
    }
    pdb_precond_free(pc);
    pdb_database_free(db);
  }

  /* error paths and conventions */
  pdb_database db = NULL;
  check(pdb_database_build(NULL, ps, NULL, &db), "err null build");
  pdb_matrix bad = NULL;
  snprintf(path, sizeof(path), "%s/missing.mtx", dir);
  check(pdb_matrix_read_matrix_market(path, &bad), "err missing file");
  fprintf(summary, "null getters %lld %lld %lld\n", (long long)pdb_matrix_rows(NULL), (long long)pdb_patchset_count(NULL),
          (long long)pdb_database_size(NULL));
  for (int st = 0; st <= 14; ++st) fprintf(summary, "status_string %d %s\n", st, pdb_status_string((pdb_status)st));
  pdb_matrix_free(NULL);
  pdb_patchset_free(NULL);
  pdb_database_free(NULL);
  pdb_precond_free(NULL);
  pdb_report_free(NULL);

  free(phi);
  free(x);
  free(y);
  pdb_patchset_free(ps);
  pdb_matrix_free(m);
  fclose(summary);
  return 0;
}
