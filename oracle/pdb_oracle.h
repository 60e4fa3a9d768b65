/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 path.
 *
 * A plain-C restatement of the reference (patchdb, /root/reference/proj)
 * algorithms on the compressed patch-relaxation hot path.  Every function
 * cites the reference file:line it restates and keeps the reference's
 * floating-point operation order (no FMA: built with -ffp-contract=off), so
 * its outputs are bit-identical to the reference's.  It is pinned against the
 * reference itself (oracle/_ref/libpdbref.so, compiled from the unmodified
 * reference sources) and against the committed golden fixtures in
 * tests/golden/ (tests/test_oracle_pins.py).  The reference ships no tests or
 * golden vectors of its own (proj/tests/CMakeLists.txt:1), so those two are
 * the pins.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference legs) may load this library; the product never does.
 *
 * Status codes are the reference's pdb_status values (patchdb.h:25-41).
 * Indices are int64 like the reference's Index (types.hpp:7).
 */
#ifndef PDB_ORACLE_H
#define PDB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* ---- dense (dense.cpp) ---- */
int orc_lu_factor(int64_t n, const double* a, double* lu, int64_t* piv);
void orc_lu_solve(int64_t n, const double* lu, const int64_t* piv, const double* rhs, double* out);
void orc_lu_solve_t(int64_t n, const double* lu, const int64_t* piv, const double* rhs, double* out);
double orc_spectral_distance(int64_t n, const double* a, const double* lu, const int64_t* piv, int* iters);
double orc_l1_distance(int64_t len, const double* a, const double* b);
void orc_mean_indexed(int64_t len, const double* mats, const int64_t* members, int64_t count, double* out);

/* ---- sparse (sparse.cpp) ---- */
void orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x, double* y);
int orc_extract(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const int64_t* idx, int64_t m,
                double* out);

/* ---- patches (patch.cpp) ---- */
/* *patches_out is malloc'd (np * ps int64), caller frees with orc_free. */
int orc_detect(int64_t n, const int64_t* rp, const int64_t* ci, int64_t ps, int64_t* np_out, int64_t** patches_out,
               double* weights);
void orc_free(void* p);
int orc_extract_all(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t np, int64_t ps,
                    const int64_t* patches, double* out);
/* group_of[np]; masks[np*ps] (only the first *ngroups rows are written). */
int orc_boundary_partition(int64_t np, int64_t ps, const double* mats, int64_t* group_of, uint8_t* masks,
                           int64_t* ngroups);

/* ---- compression (compress.cpp) ---- */
/* Database output: reps[m*ps*ps], lu[m*ps*ps], piv[m*ps] sized for np entries
 * by the caller; phi[np]; *m_out = entries.  creators[m] (greedy only) = the
 * patch that created each entry.  Returns 0 and *aborted=1 when the capped
 * pass gives up (compress.cpp:90). */
int orc_greedy(int64_t np, int64_t ps, const double* mats, double eps, int spectral, int best_match,
               int64_t abort_above, int64_t* phi, int64_t* creators, double* reps, double* lu, int64_t* piv,
               int64_t* m_out, int* aborted);
int orc_split_budget(int64_t m_p, int64_t parts, const int64_t* sizes, int64_t* out);
/* variant: 0 entrywise, 1 spectral, 2 variance-minimizing. */
int orc_kmeans(int64_t np, int64_t ps, const double* mats, int64_t m_p, int variant, uint64_t seed, int max_iters,
               int64_t* phi, double* reps, double* lu, int64_t* piv, int64_t* m_out);
int orc_partitioned_build(int64_t np, int64_t ps, const double* mats, int64_t m_p, int variant, uint64_t seed,
                          int max_iters, int64_t* phi, double* reps, double* lu, int64_t* piv, int64_t* m_out);
int orc_bootstrapped(int64_t np, int64_t ps, const double* mats, double eps, int variant, int max_iters,
                     int64_t* phi, double* reps, double* lu, int64_t* piv, int64_t* m_out);
/* greedy_bisect_to_size (experiments.cpp:168-204). */
int orc_greedy_bisect(int64_t np, int64_t ps, const double* mats, int spectral, int64_t target_lo, int64_t target_hi,
                      int best_match, int64_t* phi, int64_t* creators, double* reps, double* lu, int64_t* piv,
                      int64_t* m_out, double* eps_out);
uint64_t orc_mt19937_64_first(uint64_t seed, int64_t k); /* k-th draw (0-based), for pinning */

/* ---- preconditioner and sweep (precond.cpp) ---- */
/* phi == NULL: exact mode, lu/piv hold one factor per patch. */
void orc_precond_apply(int64_t n, int64_t np, int64_t ps, const int64_t* patches, const double* weights,
                       double omega, const double* lu, const int64_t* piv, const int64_t* phi, const double* r,
                       double* z);
/* `sweeps` smooth() steps in place; hist[s] = ||b - A x_s||_2 for s = 0..sweeps (may be NULL). */
void orc_relax(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t np, int64_t ps,
               const int64_t* patches, const double* weights, double omega, const double* lu, const int64_t* piv,
               const int64_t* phi, const double* b, double* x, int64_t sweeps, double* hist);

/* ---- Krylov ---- */
int orc_gmres(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b, int64_t np,
              int64_t ps, const int64_t* patches, const double* weights, double omega, const double* lu,
              const int64_t* piv, const int64_t* phi, int have_pc, int64_t restart, double tol, int64_t max_iters,
              int left, double* x, int64_t* iters, int64_t* restarts, int* converged, double* relres, double* hist,
              int64_t* hist_len);
/* Preconditioned CG (not in the reference): x0 = 0, stop when
 * ||r||/||b|| <= tol; hist[k] = ||r_k||/||b||.  The preconditioner is the
 * symmetrically weighted patch relaxation omega W^1/2 S W^1/2 (CG needs a
 * symmetric M; the reference's omega W S is not). */
int orc_pcg(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b, int64_t np, int64_t ps,
            const int64_t* patches, const double* weights, double omega, const double* lu, const int64_t* piv,
            const int64_t* phi, int have_pc, double tol, int64_t max_iters, double* x, int64_t* iters,
            int* converged, double* hist, int64_t* hist_len);

#ifdef __cplusplus
}
#endif
#endif
