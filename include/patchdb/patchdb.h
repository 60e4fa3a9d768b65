/*
 * patchdb-b200 -- B200-native drop-in for the reference `patchdb` C-ABI.
 *
 * Every declaration in the first part of this header has the signature,
 * struct layout and error semantics of the reference interface it replaces;
 * the citation after each one is /root/reference/proj/include/patchdb/patchdb.h
 * (abbreviated "ref.h:LINE").  Handles live on the GPU: matrices, patch
 * sets, databases and preconditioners keep their arrays in HBM and every
 * call is synchronous (device work is complete when the call returns).
 * Host arrays passed in or out are plain caller-owned pointers, exactly as
 * in the reference.  There is no CPU fallback: on a machine without a
 * usable sm_100 device the compute entry points fail with
 * PDB_ERR_INTERNAL and a "CUDA ..." message.
 *
 * The second part (below "extensions") adds new symbols only; nothing in
 * the reference interface changes meaning.
 */
#ifndef PATCHDB_B200_H
#define PATCHDB_B200_H

#include <stdint.h>

#if defined(_WIN32)
#define PDB_API __declspec(dllexport)
#else
#define PDB_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, values fixed by ref.h:25-41. */
typedef enum pdb_status {
  PDB_OK = 0,
  PDB_ERR_INVALID_ARGUMENT = 1,
  PDB_ERR_DIMENSION_MISMATCH = 2,
  PDB_ERR_SINGULAR_MATRIX = 3,
  PDB_ERR_INDEX_OUT_OF_RANGE = 4,
  PDB_ERR_DUPLICATE_INDEX = 5,
  PDB_ERR_PARSE = 6,
  PDB_ERR_NON_SQUARE_MATRIX = 7,
  PDB_ERR_NO_PATCHES_FOUND = 8,
  PDB_ERR_EMPTY_CLUSTER = 9,
  PDB_ERR_BUDGET_TOO_SMALL = 10,
  PDB_ERR_INVALID_DEGREE = 11,
  PDB_ERR_NON_POSITIVE_COEFFICIENT = 12,
  PDB_ERR_IO = 13,
  PDB_ERR_INTERNAL = 14
} pdb_status;

PDB_API const char* pdb_status_string(pdb_status status);       /* ref.h:43 */
PDB_API const char* pdb_last_error(void);                       /* ref.h:46, thread-local */

typedef struct pdb_matrix_s* pdb_matrix;     /* device CSR */
typedef struct pdb_problem_s* pdb_problem;   /* host-side assembled problem */
typedef struct pdb_patchset_s* pdb_patchset; /* device patch lists + weights */
typedef struct pdb_database_s* pdb_database; /* device representatives + factors + phi */
typedef struct pdb_precond_s* pdb_precond;   /* device sweep structures */
typedef struct pdb_report_s* pdb_report;

/* ---- sparse matrices (ref.h:57-63) ---- */
PDB_API pdb_status pdb_matrix_read_matrix_market(const char* path, pdb_matrix* out);
PDB_API pdb_status pdb_matrix_write_matrix_market(pdb_matrix m, const char* path);
PDB_API int64_t pdb_matrix_rows(pdb_matrix m);
PDB_API int64_t pdb_matrix_nnz(pdb_matrix m);
PDB_API pdb_status pdb_matrix_spmv(pdb_matrix m, const double* x, double* y);
PDB_API void pdb_matrix_free(pdb_matrix m);

/* ---- assembled model problems (ref.h:67-75) ---- */
PDB_API pdb_status pdb_problem_assemble(const char* config_json, pdb_problem* out);
PDB_API int64_t pdb_problem_ndofs(pdb_problem p);
PDB_API pdb_status pdb_problem_matrix(pdb_problem p, pdb_matrix* out);
PDB_API pdb_status pdb_problem_rhs(pdb_problem p, double* out);
PDB_API pdb_status pdb_problem_exact_solution(pdb_problem p, double* out);
PDB_API pdb_status pdb_problem_l2_error(pdb_problem p, const double* discrete_solution, double* out);
PDB_API void pdb_problem_free(pdb_problem p);

/* ---- patch detection (ref.h:80-84) ---- */
PDB_API pdb_status pdb_patchset_detect(pdb_matrix m, int64_t patch_size, pdb_patchset* out);
PDB_API int64_t pdb_patchset_count(pdb_patchset ps);
PDB_API int64_t pdb_patchset_patch_size(pdb_patchset ps);
PDB_API pdb_status pdb_patchset_write_json(pdb_patchset ps, const char* path);
PDB_API void pdb_patchset_free(pdb_patchset ps);

/* ---- factorization database (ref.h:88-117) ---- */
typedef enum pdb_method {
  PDB_METHOD_EXACT = 0,
  PDB_METHOD_GREEDY_SPECTRAL = 1,
  PDB_METHOD_GREEDY_L1 = 2,
  PDB_METHOD_KMEANS_ENTRYWISE = 3,
  PDB_METHOD_KMEANS_SPECTRAL = 4,
  PDB_METHOD_KMEANS_VARMIN = 5,
  PDB_METHOD_BOOTSTRAP = 6
} pdb_method;

/* 48 bytes, field offsets 0/8/16/24/32/36/40 as ref.h:98-106. */
typedef struct pdb_compress_options {
  pdb_method method;
  double eps;
  int64_t db_size;
  uint64_t seed;
  int max_iters;
  int best_match;
  int threads; /* accepted and ignored: the GPU sets its own parallelism */
} pdb_compress_options;

PDB_API void pdb_compress_options_init(pdb_compress_options* opts);
PDB_API pdb_status pdb_database_build(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                      pdb_database* out);
PDB_API int64_t pdb_database_size(pdb_database db);
PDB_API int64_t pdb_database_n_patches(pdb_database db);
PDB_API pdb_status pdb_database_phi(pdb_database db, int64_t* phi);
PDB_API pdb_status pdb_database_export(pdb_database db, const char* json_path, const char* bin_path);
PDB_API void pdb_database_free(pdb_database db);

/* ---- preconditioners (ref.h:121-130) ---- */
PDB_API pdb_status pdb_precond_create(pdb_matrix m, pdb_patchset ps, pdb_database db, double omega, int threads,
                                      pdb_precond* out);
PDB_API pdb_status pdb_precond_create_combo(pdb_problem p, pdb_patchset ps, pdb_database db, double omega,
                                            int threads, pdb_precond* out);
PDB_API pdb_status pdb_precond_apply(pdb_precond pc, const double* r, double* z);
PDB_API void pdb_precond_free(pdb_precond pc);

/* ---- solver (ref.h:134-158) ---- */
/* 32 bytes, offsets 0/8/16/24/28 as ref.h:134-140. */
typedef struct pdb_gmres_options {
  int64_t restart;
  double tol;
  int64_t max_iters;
  int left_precond;
  int threads;
} pdb_gmres_options;

PDB_API void pdb_gmres_options_init(pdb_gmres_options* opts);
PDB_API pdb_status pdb_gmres_solve(pdb_matrix m, const double* b, pdb_precond pc, const pdb_gmres_options* opts,
                                   double* x, pdb_report* out_report);
PDB_API int64_t pdb_report_iterations(pdb_report rep);
PDB_API int64_t pdb_report_restarts(pdb_report rep);
PDB_API int pdb_report_converged(pdb_report rep);
PDB_API double pdb_report_final_relative_residual(pdb_report rep);
PDB_API int64_t pdb_report_residual_history_size(pdb_report rep);
PDB_API pdb_status pdb_report_residual_history(pdb_report rep, double* out);
PDB_API void pdb_report_free(pdb_report rep);

/* ---- experiment drivers (ref.h:166-169) ----
 * Not part of this build (the paper's CSV study
 * drivers are outside the hot path).  The symbols exist so a host links;
 * every call returns PDB_ERR_INTERNAL with pdb_last_error() =
 * "<name> is outside the B200 hot path of this build (...)" -- distinguishable
 * from a real internal failure by that message.  pdb_export_matrix is built. */
PDB_API pdb_status pdb_run_experiment(const char* config_json, const char* out_csv);
PDB_API pdb_status pdb_run_analyze(const char* config_json, const char* curve_csv, const char* histogram_csv);
PDB_API pdb_status pdb_run_benchmark(const char* config_json, const char* out_csv);
PDB_API pdb_status pdb_export_matrix(const char* config_json, const char* out_path);

/* =====================================================================
 * extensions (new symbols only)
 * ===================================================================== */

/* Build a device matrix from host CSR arrays (the reference's SparseMatrix
 * fields, sparse.hpp:20-25): row_ptr[n+1], col_idx[nnz] strictly increasing
 * per row, values[nnz].  Validated like the reference's invariants. */
PDB_API pdb_status pdb_matrix_from_csr(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                       const double* values, pdb_matrix* out);
/* Copy the CSR arrays back to the host (sizes from rows / nnz). */
PDB_API pdb_status pdb_matrix_csr(pdb_matrix m, int64_t* row_ptr, int64_t* col_idx, double* values);
/* y = A x with device pointers on `stream` (cudaStream_t; NULL = per-thread default). */
PDB_API pdb_status pdb_matrix_spmv_device(pdb_matrix m, const double* d_x, double* d_y, void* stream);

/* Seeded synthetic problem generator for the BASELINE configurations
 * (DESIGN.md "Inputs").  Host-only: works without a GPU. */
typedef struct pdb_gen_options {
  int physics;         /* 0 = scalar diffusion -div(rho grad u); 1 = Stokes Q_p-Q_{p-1} (2D Taylor-Hood,
                          symmetric-gradient viscous term, no pressure-pressure block); 2 = linear elasticity */
  int dim;             /* 2 or 3 (Stokes: 2) */
  int degree;          /* Lagrange degree p >= 1 (velocity / displacement; Stokes pressure is p-1 >= 1) */
  int bc_mode;         /* 0 = Dirichlet row replacement, no column elimination (ref fem.cpp:323-342) */
  int64_t cells;       /* cells per axis */
  double jitter;       /* interior vertices moved by U(-jitter*h, +jitter*h) per coordinate */
  uint64_t seed;
  int coeff_kind;      /* 0 = constant coeff_value; 1 = random blocks of block_cells^dim cells from levels[];
                          2 = lognormal per cell, exp(coeff_value * N(0,1)) */
  int n_levels;        /* number of entries of levels[] used by coeff_kind 1 */
  double coeff_value;
  int64_t block_cells;
  double levels[8];
  int threads;         /* host threads for assembly (0 = all) */
  int reserved;
  double poisson_ratio; /* physics 2: nu (Lame lambda = E nu / ((1+nu)(1-2nu)), mu = E / (2(1+nu))) */
} pdb_gen_options;

PDB_API void pdb_gen_options_init(pdb_gen_options* opts);
/* Presets for BASELINE.json configs 1..5 at a given cells-per-axis (0 = the config's own size). */
PDB_API pdb_status pdb_gen_options_config(int config, int64_t cells, pdb_gen_options* opts);
PDB_API pdb_status pdb_problem_generate(const pdb_gen_options* opts, pdb_problem* out);
PDB_API int64_t pdb_problem_nnz(pdb_problem p);
/* Slab of rank `rank` of `nranks` along the slowest mesh axis (cells
 * [C rank / nranks, C (rank+1) / nranks), at least two cell layers each):
 * only the rows of the slab's DoFs are generated, bitwise equal to the same
 * rows of pdb_problem_generate, with GLOBAL column ids; pdb_problem_rows /
 * _nnz / _csr / _rhs describe those local rows.  Input of pdb_shard_create_local. */
PDB_API pdb_status pdb_problem_generate_slab(const pdb_gen_options* opts, int rank, int nranks, pdb_problem* out);
/* Global row count of the (slab) problem, and its global row ranges
 * [lo, hi) as 2 * count int64 values (count = pdb_problem_row_range_count). */
/* Rows of the DoFs of cell layers [c0, c1) along the slowest axis, labelled
 * rank `rank` of `nranks` (a slab, or a thin neighbour of one). */
PDB_API pdb_status pdb_problem_generate_cells(const pdb_gen_options* opts, int64_t c0, int64_t c1, int rank,
                                              int nranks, pdb_problem* out);
PDB_API int64_t pdb_problem_rows_global(pdb_problem p);
PDB_API int64_t pdb_problem_row_range_count(pdb_problem p);
PDB_API pdb_status pdb_problem_row_ranges(pdb_problem p, int64_t* ranges);
PDB_API pdb_status pdb_problem_csr(pdb_problem p, int64_t* row_ptr, int64_t* col_idx, double* values);

/* Patch-set contents (host copies): patches[count*patch_size] ascending per patch; weights[rows]. */
PDB_API pdb_status pdb_patchset_patches(pdb_patchset ps, int64_t* patches);
PDB_API pdb_status pdb_patchset_weights(pdb_patchset ps, double* weights);
PDB_API int64_t pdb_patchset_rows(pdb_patchset ps);
/* Dense patch matrices A_k = V_k A V_k^T, row-major, count*patch_size^2 doubles (host copy). */
PDB_API pdb_status pdb_patchset_extract(pdb_matrix m, pdb_patchset ps, double* out);

/* Database contents (host copies).  reps/lu: size*patch_size^2 row-major;
 * pivots: size*patch_size ("original row at position i", ref dense.hpp:35-39). */
PDB_API int64_t pdb_database_patch_size(pdb_database db);
PDB_API double pdb_database_eps(pdb_database db);
PDB_API pdb_status pdb_database_representatives(pdb_database db, double* reps);
PDB_API pdb_status pdb_database_factors(pdb_database db, double* lu, int64_t* pivots);
/* Tolerance bisection to a size band, ref experiments.cpp:168-204 (greedy methods only). */
/* Reference evaluate_objective (compress.hpp:74-75, compress.cpp:423-440):
 * *out = beta * |B| + sum_k ||I - A_k B_phi(k)^{-1}||_2^2, every distance the
 * reference's spectral_distance (bitwise), summed in ascending k.  beta > 0. */
PDB_API pdb_status pdb_database_objective(pdb_matrix m, pdb_patchset ps, pdb_database db, double beta,
                                          double* out);
/* Reference compressibility_curve (compress.hpp:77-85, compress.cpp:442-456):
 * greedy_tolerance (first match) over an ascending grid of count tolerances;
 * db_sizes[k] = |B|, ratios[k] = (n_p - |B|) / n_p.  method is
 * PDB_METHOD_GREEDY_SPECTRAL or PDB_METHOD_GREEDY_L1. */
PDB_API pdb_status pdb_compressibility_curve(pdb_matrix m, pdb_patchset ps, pdb_method method, const double* eps_grid,
                                             int64_t count, int64_t* db_sizes, double* ratios);
PDB_API pdb_status pdb_database_build_to_size(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                              int64_t target_lo, int64_t target_hi, pdb_database* out,
                                              double* eps_out);
/* Database import (setup reuse): the pair written by pdb_database_export
 * (ref.h:114); factors are recomputed on the device, so the result equals the
 * exported database bit for bit. */
PDB_API pdb_status pdb_database_import(const char* json_path, const char* bin_path, pdb_database* out);
/* Work counters of the last build on this thread: distance evaluations and
 * power iterations (spectral), for FP64 roofline accounting. */
PDB_API pdb_status pdb_database_work(pdb_database db, int64_t* pair_evals, int64_t* power_iters, int64_t* lu_count);

/* Device-pointer apply on a stream (NULL = per-thread default stream). */
PDB_API pdb_status pdb_precond_apply_device(pdb_precond pc, const double* d_r, double* d_z, void* stream);
/* `sweeps` damped patch-relaxation sweeps x <- x + M^{-1}(b - A x) (ref
 * smooth(), precond.cpp:90-101) with host b and x (x updated in place).
 * history (may be NULL) receives sweeps+1 values ||b - A x_s||_2. */
PDB_API pdb_status pdb_relax(pdb_matrix m, pdb_precond pc, const double* b, double* x, int64_t sweeps,
                             double* history);
/* Same on device pointers; d_history (may be NULL) is a device array. */
PDB_API pdb_status pdb_relax_device(pdb_matrix m, pdb_precond pc, const double* d_b, double* d_x, int64_t sweeps,
                                    double* d_history, void* stream);

/* pdb_relax_device with CUDA events around each sweep kernel: ms_phase[3]
 * (host) receives the average milliseconds of the residual SpMV, the patch
 * solve and the scatter/update kernels (roofline accounting in bench.py). */
PDB_API pdb_status pdb_relax_profile(pdb_matrix m, pdb_precond pc, const double* d_b, double* d_x, int64_t sweeps,
                                     double* ms_phase, void* stream);
/* Residual storage of a matrix (its SELL-C-sigma copy): out[0] = column-
 * pattern classes (0: explicit column indices), out[1] = column indices
 * stored, out[2] = slices, out[3] = values stored (padding included).  All
 * zero without a SELL copy.  (No reference counterpart: bench.py's roofline
 * accounting.) */
PDB_API pdb_status pdb_matrix_sell_info(pdb_matrix m, int64_t* out4);
/* Half-storage ("mirror") residual layout (opt-in with
 * PDB_SELL_MIRROR=1 at matrix creation): out[0] = 1 when in use, out[1] = values stored, out[2] = identity rows storing
 * mirrored values, out[3] = class offsets; *why (may be null) = why the
 * layout is not in use (empty when it is).  (No reference counterpart.) */
PDB_API pdb_status pdb_matrix_mirror_info(pdb_matrix m, int64_t* out4, const char** why);
/* Test hook, host only: builds the mirror layout of a CSR matrix and
 * evaluates y = A x through it in the GPU kernel's order (no device needed).
 * out[0] = built, out[1] = slices, out[2] = values stored, out[3] = class
 * offsets, out[4] = classes, out[5] = identity rows storing mirrored values;
 * y is untouched when not built (pdb_last_error says why). */
PDB_API pdb_status pdb_debug_mirror_check(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                          const double* values, const double* x, double* y, int64_t* out6);
/* Sweep-structure sizes: stored factors (n_p exact, m_p compressed), patches, patch size. */
PDB_API int64_t pdb_precond_stored_factors(pdb_precond pc);
PDB_API int64_t pdb_precond_patch_count(pdb_precond pc);
PDB_API int64_t pdb_precond_patch_size(pdb_precond pc);
/* Combo preconditioners (pdb_precond_create_combo): coarse-space size n_c and
 * the band widths kl, ku of R0 A P0 (0 and PDB_OK with *nc = 0 for a plain
 * patch preconditioner), and the device band LU copied out in the reference's
 * BandedFactor layout (banded.hpp:13-24): band[(2*kl+ku+1) * n_c] row-major by
 * band row, ipiv[n_c] absolute pivot rows.  Either output may be NULL. */
PDB_API pdb_status pdb_precond_coarse_size(pdb_precond pc, int64_t* nc, int64_t* kl, int64_t* ku);
PDB_API pdb_status pdb_precond_coarse_factor(pdb_precond pc, double* band, int64_t* ipiv);

/* Preconditioned conjugate gradients, x0 = 0, stop when ||r||/||b|| <= tol.
 * The patch preconditioner is applied with symmetric weighting
 * omega W^1/2 S W^1/2 (CG needs a symmetric preconditioner). */
PDB_API pdb_status pdb_pcg_solve(pdb_matrix m, const double* b, pdb_precond pc, double tol, int64_t max_iters,
                                 double* x, pdb_report* out_report);
/* pdb_pcg_solve with flags.  PDB_PCG_REPRODUCIBLE: the CPU restatement's
 * sequence bit for bit (reference-order patch solves -- the preconditioner
 * must be created with PDB_APPLY=lu -- the ordered scatter, unfused updates,
 * inner products in chunks of 256 summed in order): identical iteration
 * counts and residual histories; host-driven, for verification. */
#define PDB_PCG_REPRODUCIBLE 1
PDB_API pdb_status pdb_pcg_solve_ex(pdb_matrix m, const double* b, pdb_precond pc, double tol, int64_t max_iters,
                                    int flags, double* x, pdb_report* out_report);

/* ---- multi-GPU: slab-partitioned sweep ----------
 * Rank r of N owns the contiguous patch range [np*r/N, np*(r+1)/N); DoFs are
 * owned by the highest rank whose patches contain them.  Each sweep
 * exchanges interface partial sums (towards the owner, preserving the
 * reference's ascending-patch order) and the x halo over NCCL. */
typedef struct pdb_shard_plan_s* pdb_shard_plan;
typedef struct pdb_shard_s* pdb_shard;
typedef enum pdb_shard_plan_array {
  PDB_PLAN_DOFS = 0,      /* int64: local index -> global DoF */
  PDB_PLAN_ROW_PTR = 1,   /* int64: local CSR */
  PDB_PLAN_COLS = 2,      /* int64 (local indices) */
  PDB_PLAN_VALUES = 3,    /* double */
  PDB_PLAN_PATCHES = 4,   /* int64 (local indices) */
  PDB_PLAN_WEIGHTS = 5,   /* double (global overlap weights) */
  PDB_PLAN_OWNED = 6,     /* int64 local indices */
  PDB_PLAN_UP = 7, PDB_PLAN_UP_PEER = 8,    /* interface partials sent */
  PDB_PLAN_PIN = 9, PDB_PLAN_PIN_PEER = 10, /* interface partials received */
  PDB_PLAN_XS = 11, PDB_PLAN_XS_PEER = 12,  /* x halo sent */
  PDB_PLAN_XR = 13, PDB_PLAN_XR_PEER = 14,  /* x halo received */
  PDB_PLAN_PATCH_RANGE = 15                 /* int64[2]: first, last+1 global patch */
} pdb_shard_plan_array;

/* Host-only planning (no GPU needed): the exchange schedule of rank `rank`. */
PDB_API pdb_status pdb_shard_plan_create(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                         const double* values, int64_t n_patches, int64_t patch_size,
                                         const int64_t* patches, const double* weights, int rank, int nranks,
                                         pdb_shard_plan* out);
PDB_API int64_t pdb_shard_plan_size(pdb_shard_plan plan, int which);
PDB_API pdb_status pdb_shard_plan_get(pdb_shard_plan plan, int which, void* out);
PDB_API void pdb_shard_plan_free(pdb_shard_plan plan);

/* Device shard of (m, ps, db) for rank/nranks (db NULL = exact mode). */
PDB_API pdb_status pdb_comm_unique_id(unsigned char* id128);
PDB_API pdb_status pdb_shard_create(pdb_matrix m, pdb_patchset ps, pdb_database db, double omega, int rank,
                                    int nranks, pdb_shard* out);
PDB_API pdb_status pdb_shard_attach_comm(pdb_shard sh, const unsigned char* id128);
PDB_API int64_t pdb_shard_local_size(pdb_shard sh);
PDB_API pdb_status pdb_shard_local_dofs(pdb_shard sh, int64_t* global_ids);
PDB_API int64_t pdb_shard_owned_count(pdb_shard sh);
PDB_API pdb_status pdb_shard_owned(pdb_shard sh, int64_t* local_idx);
/* `sweeps` sweeps on shard-local device vectors (layout of pdb_shard_local_dofs). */
PDB_API pdb_status pdb_shard_relax_device(pdb_shard sh, const double* d_b, double* d_x, int64_t sweeps, void* stream);
PDB_API void pdb_shard_free(pdb_shard sh);

/* Multi-GPU sweep with rank-local data.
 * A rank passes only its slab problem (pdb_problem_generate_slab: its rows,
 * global column ids); patches, global weights, ownership and the exchange
 * lists are set up with the neighbours, factors of the rank's own patches
 * (db == NULL: exact) or the replicated database with the rank's phi slice.
 *   nccl_id != NULL: this process is rank `rank` of `nranks` (count == 1),
 *                    collective over the ranks; NCCL carries the exchanges;
 *   nccl_id == NULL, count == nranks: an emulated group of all ranks on this
 *                    GPU, exchanges as device copies (tests, single-GPU runs);
 *   nranks == 1: one rank, no exchanges. */
typedef struct pdb_slab_s* pdb_slab;
PDB_API pdb_status pdb_slab_create(pdb_problem* slabs, int count, int rank, int nranks, int64_t patch_size,
                                   pdb_database db, double omega, const unsigned char* nccl_id, pdb_slab* out);
/* Emulated group of a SUBSET of the ranks (ascending `ranks`, count of them;
 * exact preconditioners only): messages to or from absent ranks are dropped,
 * so a rank's slab plus thin neighbours (pdb_problem_generate_cells) runs one
 * rank's share of a job larger than one GPU (config 5 at 96^3). */
PDB_API pdb_status pdb_slab_create_subset(pdb_problem* slabs, int count, const int* ranks, int rank, int nranks,
                                          int64_t patch_size, pdb_database db, double omega,
                                          const unsigned char* nccl_id, pdb_slab* out);
/* The same, with the compressed database built from the ranks' OWN patches
 * (no rank sees the others' matrices).  opts->method:
 *   PDB_METHOD_GREEDY_L1 (eps, best_match): the round-batched greedy -- each
 *     round's batch matrices are broadcast by their owners, the resolution is
 *     replicated, every rank scans only its own patches;
 *   PDB_METHOD_KMEANS_ENTRYWISE (db_size, seed, max_iters): boundary-partitioned
 *     k-means -- local assignment, gathered reseed, the in-order member sums
 *     chain-folded along the ranks.
 * The database (entries replicated, phi per rank) is bitwise the single-GPU
 * pdb_database_build's. */
PDB_API pdb_status pdb_slab_create_built(pdb_problem* slabs, int count, int rank, int nranks, int64_t patch_size,
                                         const pdb_compress_options* opts, double omega, const unsigned char* nccl_id,
                                         pdb_slab* out);
PDB_API int64_t pdb_slab_database_size(pdb_slab sh);
/* phi of local rank i's patches (its slice of the global phi), and the global
 * creator patch of every entry (pdb_slab_database_size of them). */
PDB_API pdb_status pdb_slab_phi(pdb_slab sh, int i, int64_t* phi);
PDB_API pdb_status pdb_slab_creators(pdb_slab sh, int64_t* creators);
/* Local ranks held by the handle (1, or nranks for an emulated group). */
PDB_API int pdb_slab_local_ranks(pdb_slab sh);
/* Seconds of the handle's setup spent uploading the slab's matrix and building
 * the residual's storage (what pdb_matrix_from_csr does before a single-GPU
 * setup starts), summed over the local ranks. */
PDB_API double pdb_slab_upload_seconds(pdb_slab sh);
/* info[12]: rank, nranks, local DoFs, local rows, local patches, first global
 * patch, interface split, owned DoFs, partials sent / received, x halo sent / received. */
PDB_API pdb_status pdb_slab_info(pdb_slab sh, int i, int64_t* info);
PDB_API pdb_status pdb_slab_local_dofs(pdb_slab sh, int i, int64_t* global_ids);
/* Local indices of the DoFs rank i finishes (ascending). */
PDB_API pdb_status pdb_slab_owned(pdb_slab sh, int i, int64_t* local_idx);
/* Sweeps on device vectors of the local DoFs, one b / x per local rank. */
PDB_API pdb_status pdb_slab_relax_device(pdb_slab sh, const double* const* d_b, double* const* d_x, int64_t sweeps,
                                         void* stream);
/* Local rank i's sweep phases alone, exchanges skipped (per-rank timing of a
 * slice of a job larger than this GPU; the values are not a valid sweep). */
PDB_API pdb_status pdb_slab_relax_rank_device(pdb_slab sh, int i, const double* d_b, double* d_x, int64_t sweeps,
                                              void* stream);
PDB_API void pdb_slab_free(pdb_slab sh);

/* Sharded setup: a communicator over nranks processes (one GPU each; id from
 * pdb_comm_unique_id on one rank, shared out of band), and database builds
 * whose dominant step is split across the ranks -- the k-means assignment, the
 * greedy scan of the remaining patches against each round's new entries --
 * with every rank returning the same database, bitwise equal to
 * pdb_database_build.  EXACT and BOOTSTRAP build redundantly on every rank. */
typedef struct pdb_comm_s* pdb_comm;
PDB_API pdb_status pdb_comm_create(const unsigned char* id128, int rank, int nranks, pdb_comm* out);
PDB_API void pdb_comm_free(pdb_comm c);
PDB_API pdb_status pdb_database_build_sharded(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                              pdb_comm comm, pdb_database* out);
/* Sharded greedy tolerance bisection (each probe a sharded greedy pass). */
PDB_API pdb_status pdb_database_build_to_size_sharded(pdb_matrix m, pdb_patchset ps, const pdb_compress_options* opts,
                                                      int64_t target_lo, int64_t target_hi, pdb_comm comm,
                                                      pdb_database* out, double* eps_out);

/* Build information: "sm_100a" target, version. */
PDB_API const char* pdb_build_info(void);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* PATCHDB_B200_H */
