/* TEST INFRASTRUCTURE ONLY -- see pdb_oracle.h for the contract.
 *
 * Plain-C restatement of the reference patchdb hot path.  File:line
 * citations are relative to /root/reference/proj/src/core/.  Operation order
 * follows the reference exactly (sequential sums, division where the
 * reference divides, multiplication by a reciprocal where it multiplies),
 * and the file is compiled with -ffp-contract=off, so results are bitwise
 * equal to the reference binary (checked in tests/test_oracle_pins.py).
 */
#include "pdb_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum {
  ST_OK = 0,
  ST_INVALID = 1,
  ST_DIM = 2,
  ST_SINGULAR = 3,
  ST_RANGE = 4,
  ST_DUP = 5,
  ST_NO_PATCHES = 8,
  ST_EMPTY = 9,
  ST_BUDGET = 10,
  ST_INTERNAL = 14
};

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

void orc_free(void* p) { free(p); }

/* ======================================================================
 * dense.cpp
 * ==================================================================== */

/* lu_factor, dense.cpp:31-75.  Right-looking LU; pivot = first maximum |.|
 * (strict >, :49-58); singular when best == 0 or best < 1e-14*colmax (:59-61);
 * full row swap (:62-65); l_ik by division (:68); skip l_ik == 0 (:70). */
int orc_lu_factor(int64_t n, const double* a, double* lu, int64_t* piv) {
  if (n < 1) return set_err(ST_INVALID, "lu_factor requires dim >= 1");
  memcpy(lu, a, sizeof(double) * (size_t)(n * n));
  for (int64_t i = 0; i < n; ++i) piv[i] = i;
  double* colmax = (double*)calloc((size_t)n, sizeof(double));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const double v = fabs(a[i * n + j]);
      if (v > colmax[j]) colmax[j] = v; /* std::max(colmax, v) */
    }
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = fabs(lu[k * n + k]);
    for (int64_t i = k + 1; i < n; ++i) {
      const double v = fabs(lu[i * n + k]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    if (best == 0.0 || best < 1e-14 * colmax[k]) {
      free(colmax);
      /* std::to_string(double) is "%f" */
      return set_err(ST_SINGULAR, "singular matrix: pivot %f below threshold in column %lld", best, (long long)k);
    }
    if (p != k) {
      for (int64_t j = 0; j < n; ++j) {
        const double t = lu[k * n + j];
        lu[k * n + j] = lu[p * n + j];
        lu[p * n + j] = t;
      }
      const int64_t t = piv[k];
      piv[k] = piv[p];
      piv[p] = t;
    }
    const double pv = lu[k * n + k];
    for (int64_t i = k + 1; i < n; ++i) {
      const double lik = lu[i * n + k] / pv;
      lu[i * n + k] = lik;
      if (lik == 0.0) continue;
      for (int64_t j = k + 1; j < n; ++j) lu[i * n + j] -= lik * lu[k * n + j];
    }
  }
  free(colmax);
  return ST_OK;
}

/* lu_solve_into, dense.cpp:77-94. */
void orc_lu_solve(int64_t n, const double* lu, const int64_t* piv, const double* rhs, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = rhs[piv[i]];
  for (int64_t i = 1; i < n; ++i) {
    double s = out[i];
    for (int64_t j = 0; j < i; ++j) s -= lu[i * n + j] * out[j];
    out[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = out[i];
    for (int64_t j = i + 1; j < n; ++j) s -= lu[i * n + j] * out[j];
    out[i] = s / lu[i * n + i];
  }
}

/* lu_solve_transpose_into, dense.cpp:102-120 (w is a fresh copy of rhs). */
void orc_lu_solve_t(int64_t n, const double* lu, const int64_t* piv, const double* rhs, double* out) {
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(w, rhs, sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    double s = w[i];
    for (int64_t j = 0; j < i; ++j) s -= lu[j * n + i] * w[j];
    w[i] = s / lu[i * n + i];
  }
  for (int64_t i = n - 2; i >= 0; --i) {
    double s = w[i];
    for (int64_t j = i + 1; j < n; ++j) s -= lu[j * n + i] * w[j];
    w[i] = s;
  }
  for (int64_t i = 0; i < n; ++i) out[piv[i]] = w[i];
  free(w);
}

/* mat_vec dense.cpp:122-131, mat_tvec :133-142. */
static void mat_vec(int64_t n, const double* a, const double* x, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    const double* row = a + i * n;
    for (int64_t j = 0; j < n; ++j) s += row[j] * x[j];
    out[i] = s;
  }
}
static void mat_tvec(int64_t n, const double* a, const double* x, double* out) {
  for (int64_t j = 0; j < n; ++j) out[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double xi = x[i];
    const double* row = a + i * n;
    for (int64_t j = 0; j < n; ++j) out[j] += row[j] * xi;
  }
}

/* norm2, dense.cpp:146-150. */
static double norm2(int64_t n, const double* v) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

/* spectral_distance, dense.cpp:154-190: power iteration on C^T C with
 * C = I - A B^{-1}; v0_i = 1 + 1e-6 i normalised by division; stop on
 * rq <= 1e-28 or |rq - lambda| < 1e-8 rq (it > 0); <= 200 iterations.
 * *iters (optional) = iterations executed (for work accounting). */
double orc_spectral_distance(int64_t n, const double* a, const double* lu, const int64_t* piv, int* iters) {
  const size_t un = (size_t)n;
  double* buf = (double*)malloc(sizeof(double) * un * 5);
  double *v = buf, *t = buf + un, *w = buf + 2 * un, *s = buf + 3 * un, *u = buf + 4 * un;
  for (int64_t i = 0; i < n; ++i) v[i] = 1.0 + 1e-6 * (double)i;
  const double vn = norm2(n, v);
  for (int64_t i = 0; i < n; ++i) v[i] /= vn;
  double lambda = 0.0;
  double result = -1.0;
  int it;
  for (it = 0; it < 200; ++it) {
    orc_lu_solve(n, lu, piv, v, t);
    mat_vec(n, a, t, w);
    for (int64_t i = 0; i < n; ++i) w[i] = v[i] - w[i];
    mat_tvec(n, a, w, s);
    orc_lu_solve_t(n, lu, piv, s, t);
    for (int64_t i = 0; i < n; ++i) u[i] = w[i] - t[i];
    double rq = 0.0;
    for (int64_t i = 0; i < n; ++i) rq += v[i] * u[i];
    rq = rq > 0.0 ? rq : 0.0; /* std::max(rq, 0.0) */
    if (rq <= 1e-28) {
      result = sqrt(rq);
      break;
    }
    if (it > 0 && fabs(rq - lambda) < 1e-8 * rq) {
      result = sqrt(rq);
      break;
    }
    lambda = rq;
    const double un2 = norm2(n, u);
    if (un2 == 0.0) {
      result = 0.0;
      break;
    }
    for (int64_t i = 0; i < n; ++i) v[i] = u[i] / un2;
  }
  if (it == 200) result = sqrt(lambda);
  if (iters) *iters = it == 200 ? 200 : it + 1;
  free(buf);
  return result;
}

/* entrywise_l1_distance, dense.cpp:192-197. */
double orc_l1_distance(int64_t len, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t k = 0; k < len; ++k) s += fabs(a[k] - b[k]);
  return s;
}

/* entrywise_mean_indexed, dense.cpp:211-223: in-order sum from 0.0, then
 * multiply by the reciprocal of the count. */
void orc_mean_indexed(int64_t len, const double* mats, const int64_t* members, int64_t count, double* out) {
  for (int64_t q = 0; q < len; ++q) out[q] = 0.0;
  for (int64_t c = 0; c < count; ++c) {
    const double* m = mats + members[c] * len;
    for (int64_t q = 0; q < len; ++q) out[q] += m[q];
  }
  const double inv = 1.0 / (double)count;
  for (int64_t q = 0; q < len; ++q) out[q] *= inv;
}

/* ======================================================================
 * sparse.cpp
 * ==================================================================== */

/* spmv, sparse.cpp:50-63. */
void orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) s += v[p] * x[ci[p]];
    y[i] = s;
  }
}

typedef struct {
  int64_t g, l;
} pair_gl;

static int cmp_pair(const void* a, const void* b) {
  const pair_gl* x = (const pair_gl*)a;
  const pair_gl* y = (const pair_gl*)b;
  if (x->g != y->g) return x->g < y->g ? -1 : 1;
  return x->l < y->l ? -1 : (x->l > y->l);
}

/* extract_submatrix, sparse.cpp:71-103: merge of the sorted CSR row with the
 * sorted (global, local) list; absent entries stay 0. */
int orc_extract(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const int64_t* idx, int64_t m,
                double* out) {
  for (int64_t k = 0; k < m; ++k)
    if (idx[k] < 0 || idx[k] >= n) return set_err(ST_RANGE, "submatrix index outside matrix");
  pair_gl* loc = (pair_gl*)malloc(sizeof(pair_gl) * (size_t)(m > 0 ? m : 1));
  for (int64_t k = 0; k < m; ++k) {
    loc[k].g = idx[k];
    loc[k].l = k;
  }
  qsort(loc, (size_t)m, sizeof(pair_gl), cmp_pair);
  for (int64_t k = 1; k < m; ++k)
    if (loc[k].g == loc[k - 1].g) {
      free(loc);
      return set_err(ST_DUP, "duplicate submatrix index");
    }
  memset(out, 0, sizeof(double) * (size_t)(m * m));
  for (int64_t r = 0; r < m; ++r) {
    const int64_t gi = idx[r];
    int64_t p = rp[gi], q = 0;
    const int64_t pe = rp[gi + 1];
    while (p < pe && q < m) {
      if (ci[p] < loc[q].g)
        ++p;
      else if (ci[p] > loc[q].g)
        ++q;
      else {
        out[r * m + loc[q].l] = v[p];
        ++p;
        ++q;
      }
    }
  }
  free(loc);
  return ST_OK;
}

/* ======================================================================
 * patch.cpp
 * ==================================================================== */

/* compute_weights, patch.cpp:12-20. */
static void compute_weights(int64_t n, int64_t np, int64_t ps, const int64_t* patches, double* w) {
  int64_t* cover = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int64_t k = 0; k < np * ps; ++k) ++cover[patches[k]];
  for (int64_t i = 0; i < n; ++i) w[i] = cover[i] > 0 ? 1.0 / (double)cover[i] : 0.0;
  free(cover);
}

/* IndexVectorHash, patch.cpp:24-33 (FNV-1a over the 64-bit indices). */
static uint64_t fnv_vec(const int64_t* v, int64_t len) {
  uint64_t h = 1469598103934665603ull;
  for (int64_t k = 0; k < len; ++k) {
    h ^= (uint64_t)v[k];
    h *= 1099511628211ull;
  }
  return h;
}

typedef struct {
  int64_t front, seq;
} front_key;

/* Stable merge sort by front.  The reference uses std::sort, which is not
 * stable (patch.cpp:82-83); the two agree whenever fronts are unique, which
 * holds for cell patches (every cell patch contains its own lowest corner). */
static void sort_fronts(front_key* a, int64_t n) {
  front_key* tmp = (front_key*)malloc(sizeof(front_key) * (size_t)(n > 0 ? n : 1));
  for (int64_t width = 1; width < n; width *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * width) {
      int64_t mid = lo + width < n ? lo + width : n;
      int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      int64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) tmp[k++] = (a[j].front < a[i].front) ? a[j++] : a[i++];
      while (i < mid) tmp[k++] = a[i++];
      while (j < hi) tmp[k++] = a[j++];
    }
    memcpy(a, tmp, sizeof(front_key) * (size_t)n);
  }
  free(tmp);
}

/* detect_patches, patch.cpp:37-90. */
int orc_detect(int64_t n, const int64_t* rp, const int64_t* ci, int64_t ps, int64_t* np_out, int64_t** patches_out,
               double* weights) {
  *np_out = 0;
  *patches_out = NULL;
  if (ps < 2) return set_err(ST_INVALID, "patch size must be >= 2");
  char* cand = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  int any = 0;
  for (int64_t i = 0; i < n; ++i)
    if (rp[i + 1] - rp[i] == ps) {
      cand[i] = 1;
      any = 1;
    }
  if (!any) {
    free(cand);
    return set_err(ST_NO_PATCHES, "no row has exactly %lld stored entries", (long long)ps);
  }
  /* emitted set: open addressing over patch slots */
  int64_t cap = 1024;
  int64_t count = 0;
  int64_t* sets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap * ps));
  int64_t hcap = 2048;
  int64_t* table = (int64_t*)malloc(sizeof(int64_t) * (size_t)hcap);
  for (int64_t h = 0; h < hcap; ++h) table[h] = -1;
  int64_t* fi = (int64_t*)malloc(sizeof(int64_t) * (size_t)ps);
  int64_t* fj = (int64_t*)malloc(sizeof(int64_t) * (size_t)ps);
  for (int64_t i = 0; i < n; ++i) {
    if (!cand[i]) continue;
    const int64_t* set = ci + rp[i];
    const uint64_t h = fnv_vec(set, ps);
    int64_t slot = (int64_t)(h & (uint64_t)(hcap - 1));
    int dup = 0;
    while (table[slot] >= 0) {
      if (memcmp(sets + table[slot] * ps, set, sizeof(int64_t) * (size_t)ps) == 0) {
        dup = 1;
        break;
      }
      slot = (slot + 1) & (hcap - 1);
    }
    if (dup) continue; /* :64 */
    /* candidate footprints, :66-76 */
    int64_t nfi = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (cand[ci[p]]) fi[nfi++] = ci[p];
    int consistent = 1;
    for (int64_t q = 0; q < ps && consistent; ++q) {
      const int64_t j = set[q];
      if (!cand[j] || j == i) continue;
      /* j is a candidate, so its row has exactly ps entries and fj fits */
      int64_t nfj = 0;
      for (int64_t p = rp[j]; p < rp[j + 1]; ++p)
        if (cand[ci[p]]) fj[nfj++] = ci[p];
      if (nfj != nfi || memcmp(fi, fj, sizeof(int64_t) * (size_t)nfi) != 0) consistent = 0;
    }
    if (!consistent) continue;
    if (count == cap) {
      cap *= 2;
      sets = (int64_t*)realloc(sets, sizeof(int64_t) * (size_t)(cap * ps));
    }
    memcpy(sets + count * ps, set, sizeof(int64_t) * (size_t)ps);
    table[slot] = count;
    ++count;
    if (2 * count > hcap) { /* rehash */
      int64_t ncap = hcap * 4;
      int64_t* nt = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncap);
      for (int64_t hh = 0; hh < ncap; ++hh) nt[hh] = -1;
      for (int64_t e = 0; e < count; ++e) {
        int64_t s2 = (int64_t)(fnv_vec(sets + e * ps, ps) & (uint64_t)(ncap - 1));
        while (nt[s2] >= 0) s2 = (s2 + 1) & (ncap - 1);
        nt[s2] = e;
      }
      free(table);
      table = nt;
      hcap = ncap;
    }
  }
  free(fi);
  free(fj);
  free(table);
  free(cand);
  if (count == 0) {
    free(sets);
    return set_err(ST_NO_PATCHES, "no consistent patch candidates detected");
  }
  front_key* keys = (front_key*)malloc(sizeof(front_key) * (size_t)count);
  for (int64_t e = 0; e < count; ++e) {
    keys[e].front = sets[e * ps];
    keys[e].seq = e;
  }
  sort_fronts(keys, count);
  int64_t* out = (int64_t*)malloc(sizeof(int64_t) * (size_t)(count * ps));
  for (int64_t e = 0; e < count; ++e) memcpy(out + e * ps, sets + keys[e].seq * ps, sizeof(int64_t) * (size_t)ps);
  free(keys);
  free(sets);
  compute_weights(n, count, ps, out, weights);
  *np_out = count;
  *patches_out = out;
  return ST_OK;
}

/* extract_all, patch.cpp:92-99. */
int orc_extract_all(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t np, int64_t ps,
                    const int64_t* patches, double* out) {
  for (int64_t k = 0; k < np; ++k) {
    const int st = orc_extract(n, rp, ci, v, patches + k * ps, ps, out + k * ps * ps);
    if (st) return st;
  }
  return ST_OK;
}

/* boundary_pattern patch.cpp:101-111 (row has exactly one value != 0.0),
 * boundary_partition :113-126 (groups in first-occurrence order). */
int orc_boundary_partition(int64_t np, int64_t ps, const double* mats, int64_t* group_of, uint8_t* masks,
                           int64_t* ngroups) {
  if (np < 1) return set_err(ST_INVALID, "boundary_partition needs at least one patch");
  uint8_t* m = (uint8_t*)malloc((size_t)ps);
  int64_t g = 0;
  for (int64_t k = 0; k < np; ++k) {
    const double* a = mats + k * ps * ps;
    for (int64_t i = 0; i < ps; ++i) {
      int64_t nz = 0;
      for (int64_t j = 0; j < ps; ++j)
        if (a[i * ps + j] != 0.0) ++nz;
      m[i] = nz == 1;
    }
    int64_t found = -1;
    for (int64_t q = 0; q < g && found < 0; ++q)
      if (memcmp(masks + q * ps, m, (size_t)ps) == 0) found = q;
    if (found < 0) {
      memcpy(masks + g * ps, m, (size_t)ps);
      found = g++;
    }
    group_of[k] = found;
  }
  free(m);
  *ngroups = g;
  return ST_OK;
}

/* ======================================================================
 * compress.cpp
 * ==================================================================== */

/* A growable database: reps/lu/piv are caller arrays sized for the maximum
 * number of entries. */
typedef struct {
  int64_t ps, m;
  double* reps;
  double* lu;
  int64_t* piv;
  char* has_factor;
} db_t;

static double entry_distance_l1(const db_t* db, const double* a, int64_t j) {
  const int64_t len = db->ps * db->ps;
  return orc_l1_distance(len, a, db->reps + j * len);
}

static double entry_distance_spec(const db_t* db, const double* a, int64_t j) {
  const int64_t len = db->ps * db->ps;
  return orc_spectral_distance(db->ps, a, db->lu + j * len, db->piv + j * db->ps, NULL);
}

/* factor_patch, compress.cpp:25-33 -- prefixes "patch k: ". */
static int factor_patch(int64_t ps, const double* a, double* lu, int64_t* piv, int64_t k) {
  const int st = orc_lu_factor(ps, a, lu, piv);
  if (st == ST_SINGULAR) {
    char tmp[512];
    snprintf(tmp, sizeof tmp, "%s", g_err);
    return set_err(ST_SINGULAR, "patch %lld: %s", (long long)k, tmp);
  }
  return st;
}

/* greedy_impl, compress.cpp:40-95 (sequential resolution; the threaded
 * variant :55-73 resolves identically). */
int orc_greedy(int64_t np, int64_t ps, const double* mats, double eps, int spectral, int best_match,
               int64_t abort_above, int64_t* phi, int64_t* creators, double* reps, double* lu, int64_t* piv,
               int64_t* m_out, int* aborted) {
  *aborted = 0;
  *m_out = 0;
  if (np < 1) return set_err(ST_INVALID, "greedy_tolerance needs at least one patch");
  if (!(eps > 0.0)) return set_err(ST_INVALID, "tolerance must be positive");
  const int64_t len = ps * ps;
  db_t db = {ps, 0, reps, lu, piv, NULL};
  for (int64_t i = 0; i < np; ++i) phi[i] = -1;
  for (int64_t i = 0; i < np; ++i) {
    const double* a = mats + i * len;
    const int64_t m = db.m;
    int64_t match = -1;
    double best = eps;
    for (int64_t j = 0; j < m; ++j) {
      const double d = spectral ? entry_distance_spec(&db, a, j) : entry_distance_l1(&db, a, j);
      if (d < best) {
        match = j;
        if (!best_match) break;
        best = d;
      }
    }
    if (match >= 0) {
      phi[i] = match;
      continue;
    }
    if (abort_above > 0 && db.m + 1 > abort_above) {
      *aborted = 1;
      *m_out = db.m;
      return ST_OK;
    }
    memcpy(reps + db.m * len, a, sizeof(double) * (size_t)len);
    const int st = factor_patch(ps, a, lu + db.m * len, piv + db.m * ps, i);
    if (st) return st;
    if (creators) creators[db.m] = i;
    phi[i] = db.m;
    ++db.m;
  }
  *m_out = db.m;
  return ST_OK;
}

/* mt19937_64 (the standard 64-bit Mersenne twister, as std::mt19937_64). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64_t* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

uint64_t orc_mt19937_64_first(uint64_t seed, int64_t k) {
  mt64_t s;
  mt64_seed(&s, seed);
  uint64_t v = 0;
  for (int64_t i = 0; i <= k; ++i) v = mt64_next(&s);
  return v;
}

enum { V_ENTRYWISE = 0, V_SPECTRAL = 1, V_VARMIN = 2 };

static double variant_distance(const db_t* db, const double* a, int64_t j, int variant) {
  return variant == V_ENTRYWISE ? entry_distance_l1(db, a, j) : entry_distance_spec(db, a, j);
}

/* kmeans_loop, compress.cpp:138-262.  policy 0 = Reseed, 1 = Prune. */
static int kmeans_loop(int64_t n, int64_t ps, const double* mats, db_t* db, int64_t* phi, int variant, int max_iters,
                       int policy) {
  const int64_t len = ps * ps;
  for (int64_t i = 0; i < n; ++i) phi[i] = -1;
  double* min_dist = (double*)calloc((size_t)n, sizeof(double));
  int64_t* new_phi = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* mcount = (int64_t*)malloc(sizeof(int64_t) * (size_t)(db->m > 0 ? db->m : 1));
  int64_t* mstart = (int64_t*)malloc(sizeof(int64_t) * (size_t)(db->m + 1));
  int64_t* mlist = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + db->m + 1));
  int64_t* mcap = (int64_t*)malloc(sizeof(int64_t) * (size_t)(db->m > 0 ? db->m : 1));
  int st = ST_OK;
  for (int iter = 0; iter < max_iters; ++iter) {
    const int64_t m = db->m;
    int changed = 0;
    for (int64_t i = 0; i < n; ++i) { /* :150-166 */
      int64_t best_j = 0;
      double best = INFINITY;
      for (int64_t j = 0; j < m; ++j) {
        const double d = variant_distance(db, mats + i * len, j, variant);
        if (d < best) {
          best = d;
          best_j = j;
        }
      }
      new_phi[i] = best_j;
      min_dist[i] = best;
      if (best_j != phi[i]) changed = 1;
    }
    memcpy(phi, new_phi, sizeof(int64_t) * (size_t)n);
    if (!changed) break;
    /* members in ascending patch order (:176-177); each cluster gets room
     * for one extra member so a reseed can append. */
    for (int64_t j = 0; j < m; ++j) mcount[j] = 0;
    for (int64_t i = 0; i < n; ++i) ++mcount[phi[i]];
    mstart[0] = 0;
    for (int64_t j = 0; j < m; ++j) {
      mstart[j + 1] = mstart[j] + mcount[j] + 1;
      mcap[j] = mcount[j];
      mcount[j] = 0;
    }
    for (int64_t i = 0; i < n; ++i) {
      const int64_t j = phi[i];
      mlist[mstart[j] + mcount[j]++] = i;
    }
    (void)mcap;
    int64_t mc = m;
    if (policy == 1) { /* Prune, :179-194 */
      int64_t* remap = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
      int64_t kept = 0;
      for (int64_t j = 0; j < m; ++j) {
        remap[j] = -1;
        if (mcount[j] > 0) {
          remap[j] = kept;
          if (kept != j) {
            memmove(db->reps + kept * len, db->reps + j * len, sizeof(double) * (size_t)len);
            memmove(db->lu + kept * len, db->lu + j * len, sizeof(double) * (size_t)len);
            memmove(db->piv + kept * ps, db->piv + j * ps, sizeof(int64_t) * (size_t)ps);
            db->has_factor[kept] = db->has_factor[j];
            mstart[kept] = mstart[j];
            mcount[kept] = mcount[j];
          }
          ++kept;
        }
      }
      db->m = kept;
      mc = kept;
      for (int64_t i = 0; i < n; ++i) phi[i] = remap[phi[i]];
      free(remap);
    } else { /* Reseed, :195-217 */
      for (int64_t j = 0; j < m; ++j) {
        if (mcount[j] != 0) continue;
        int64_t far = -1;
        double far_d = -1.0;
        for (int64_t i = 0; i < n; ++i) {
          const int64_t owner = phi[i];
          if (mcount[owner] <= 1) continue;
          if (min_dist[i] > far_d) {
            far_d = min_dist[i];
            far = i;
          }
        }
        if (far < 0) continue;
        const int64_t owner = phi[far];
        int64_t* own = mlist + mstart[owner];
        int64_t pos = 0;
        while (own[pos] != far) ++pos;
        memmove(own + pos, own + pos + 1, sizeof(int64_t) * (size_t)(mcount[owner] - pos - 1));
        --mcount[owner];
        mlist[mstart[j] + mcount[j]++] = far;
        phi[far] = j;
        min_dist[far] = 0.0;
      }
    }
    /* representative update, :219-261 */
    char err_first[512] = {0};
    int64_t err_cluster = -1;
    for (int64_t j = 0; j < mc && err_cluster < 0; ++j) {
      const int64_t* mem = mlist + mstart[j];
      const int64_t cnt = mcount[j];
      if (variant == V_VARMIN) {
        int64_t best_c = -1;
        double best_var = INFINITY;
        double* flu = (double*)malloc(sizeof(double) * (size_t)len);
        int64_t* fpiv = (int64_t*)malloc(sizeof(int64_t) * (size_t)ps);
        double* best_lu = (double*)malloc(sizeof(double) * (size_t)len);
        int64_t* best_piv = (int64_t*)malloc(sizeof(int64_t) * (size_t)ps);
        int bad = 0;
        for (int64_t c = 0; c < cnt; ++c) {
          const int s2 = factor_patch(ps, mats + mem[c] * len, flu, fpiv, mem[c]);
          if (s2) {
            bad = s2;
            break;
          }
          double var = 0.0;
          for (int64_t k = 0; k < cnt; ++k) {
            const double d = orc_spectral_distance(ps, mats + mem[k] * len, flu, fpiv, NULL);
            var += d * d;
          }
          if (var < best_var) {
            best_var = var;
            best_c = mem[c];
            memcpy(best_lu, flu, sizeof(double) * (size_t)len);
            memcpy(best_piv, fpiv, sizeof(int64_t) * (size_t)ps);
          }
        }
        if (bad) {
          snprintf(err_first, sizeof err_first, "%s", g_err);
          err_cluster = j;
        } else if (cnt == 0) {
          /* entrywise_mean/empty member list: the reference indexes
           * patches[best_c = -1]; unreachable after reseed unless nothing
           * was movable. */
          snprintf(err_first, sizeof err_first, "empty cluster");
          err_cluster = j;
        } else {
          memcpy(db->reps + j * len, mats + best_c * len, sizeof(double) * (size_t)len);
          memcpy(db->lu + j * len, best_lu, sizeof(double) * (size_t)len);
          memcpy(db->piv + j * ps, best_piv, sizeof(int64_t) * (size_t)ps);
          db->has_factor[j] = 1;
        }
        free(flu);
        free(fpiv);
        free(best_lu);
        free(best_piv);
      } else {
        if (cnt == 0) {
          snprintf(err_first, sizeof err_first, "entrywise_mean of an empty cluster");
          st = ST_EMPTY;
          err_cluster = j;
          break;
        }
        orc_mean_indexed(len, mats, mem, cnt, db->reps + j * len);
        if (variant == V_SPECTRAL) {
          const int s2 = orc_lu_factor(ps, db->reps + j * len, db->lu + j * len, db->piv + j * ps);
          if (s2) {
            snprintf(err_first, sizeof err_first, "%s", g_err);
            err_cluster = j;
          } else
            db->has_factor[j] = 1;
        } else
          db->has_factor[j] = 0;
      }
    }
    if (err_cluster >= 0) {
      /* every per-cluster failure is re-raised as singular_matrix (:259-260) */
      st = set_err(ST_SINGULAR, "cluster %lld: %s", (long long)err_cluster, err_first);
      break;
    }
  }
  free(min_dist);
  free(new_phi);
  free(mcount);
  free(mstart);
  free(mlist);
  free(mcap);
  return st;
}

/* finalize_factors, compress.cpp:266-278. */
static int finalize_factors(db_t* db) {
  const int64_t len = db->ps * db->ps;
  for (int64_t j = 0; j < db->m; ++j) {
    if (db->has_factor[j]) continue;
    const int st = orc_lu_factor(db->ps, db->reps + j * len, db->lu + j * len, db->piv + j * db->ps);
    if (st == ST_SINGULAR) {
      char tmp[512];
      snprintf(tmp, sizeof tmp, "%s", g_err);
      return set_err(ST_SINGULAR, "cluster %lld: %s", (long long)j, tmp);
    }
    if (st) return st;
    db->has_factor[j] = 1;
  }
  return ST_OK;
}

/* kmeans, compress.cpp:294-324. */
int orc_kmeans(int64_t np, int64_t ps, const double* mats, int64_t m_p, int variant, uint64_t seed, int max_iters,
               int64_t* phi, double* reps, double* lu, int64_t* piv, int64_t* m_out) {
  *m_out = 0;
  if (np < 1) return set_err(ST_INVALID, "kmeans needs at least one patch");
  if (m_p < 1 || m_p > np) return set_err(ST_INVALID, "kmeans requires 1 <= m_p <= n_p");
  const int64_t len = ps * ps;
  mt64_t rng;
  mt64_seed(&rng, seed);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)np);
  for (int64_t i = 0; i < np; ++i) perm[i] = i;
  for (int64_t i = 0; i < m_p; ++i) {
    const int64_t j = i + (int64_t)(mt64_next(&rng) % (uint64_t)(np - i));
    const int64_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  db_t db = {ps, m_p, reps, lu, piv, (char*)calloc((size_t)m_p, 1)};
  int st = ST_OK;
  for (int64_t j = 0; j < m_p && !st; ++j) {
    const int64_t pick = perm[j];
    memcpy(reps + j * len, mats + pick * len, sizeof(double) * (size_t)len);
    if (variant != V_ENTRYWISE) {
      st = factor_patch(ps, reps + j * len, lu + j * len, piv + j * ps, pick);
      db.has_factor[j] = 1;
    }
  }
  free(perm);
  if (!st) st = kmeans_loop(np, ps, mats, &db, phi, variant, max_iters, 0);
  if (!st) st = finalize_factors(&db);
  *m_out = db.m;
  free(db.has_factor);
  return st;
}

/* bootstrapped, compress.cpp:326-334. */
int orc_bootstrapped(int64_t np, int64_t ps, const double* mats, double eps, int variant, int max_iters,
                     int64_t* phi, double* reps, double* lu, int64_t* piv, int64_t* m_out) {
  int aborted = 0;
  int st = orc_greedy(np, ps, mats, eps, 1, 0, -1, phi, NULL, reps, lu, piv, m_out, &aborted);
  if (st) return st;
  db_t db = {ps, *m_out, reps, lu, piv, (char*)malloc((size_t)(*m_out > 0 ? *m_out : 1))};
  memset(db.has_factor, 1, (size_t)(*m_out > 0 ? *m_out : 1));
  st = kmeans_loop(np, ps, mats, &db, phi, variant, max_iters, 1);
  if (!st) st = finalize_factors(&db);
  *m_out = db.m;
  free(db.has_factor);
  return st;
}

/* split_budget, compress.cpp:336-392. */
int orc_split_budget(int64_t m_p, int64_t parts, const int64_t* sizes, int64_t* alloc) {
  if (parts < 1) return set_err(ST_INVALID, "no partitions");
  int64_t total = 0;
  for (int64_t p = 0; p < parts; ++p) total += sizes[p];
  if (m_p < parts) return set_err(ST_BUDGET, "database budget smaller than the number of boundary partitions");
  if (m_p > total) return set_err(ST_INVALID, "database budget larger than the number of patches");
  double* rem = (double*)malloc(sizeof(double) * (size_t)parts);
  int64_t assigned = 0;
  for (int64_t p = 0; p < parts; ++p) {
    const double quota = (double)m_p * (double)sizes[p] / (double)total;
    alloc[p] = (int64_t)floor(quota);
    rem[p] = quota - floor(quota);
    assigned += alloc[p];
  }
  /* stable sort of partition ids by descending remainder */
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)parts);
  for (int64_t p = 0; p < parts; ++p) order[p] = p;
  for (int64_t a = 1; a < parts; ++a) { /* insertion sort is stable */
    const int64_t key = order[a];
    int64_t b = a - 1;
    while (b >= 0 && rem[key] > rem[order[b]]) {
      order[b + 1] = order[b];
      --b;
    }
    order[b + 1] = key;
  }
  for (int64_t k = 0; assigned < m_p; ++k) {
    ++alloc[order[k % parts]];
    ++assigned;
  }
  int st = ST_OK;
  for (int64_t p = 0; p < parts && !st; ++p)
    while (alloc[p] == 0) {
      int64_t donor = -1;
      for (int64_t q = 0; q < parts; ++q)
        if (alloc[q] >= 2 && (donor < 0 || alloc[q] > alloc[donor])) donor = q;
      if (donor < 0) {
        st = set_err(ST_BUDGET, "cannot satisfy one cluster per partition");
        break;
      }
      --alloc[donor];
      ++alloc[p];
    }
  for (int64_t p = 0; p < parts && !st; ++p)
    while (alloc[p] > sizes[p]) {
      --alloc[p];
      int64_t recv = -1;
      double best_rem = -1.0;
      for (int64_t q = 0; q < parts; ++q)
        if (alloc[q] < sizes[q] && rem[q] > best_rem) {
          best_rem = rem[q];
          recv = q;
        }
      if (recv < 0) {
        st = set_err(ST_INVALID, "budget exceeds total patch count");
        break;
      }
      ++alloc[recv];
    }
  free(rem);
  free(order);
  return st;
}

/* partitioned_build, compress.cpp:394-421. */
int orc_partitioned_build(int64_t np, int64_t ps, const double* mats, int64_t m_p, int variant, uint64_t seed,
                          int max_iters, int64_t* phi, double* reps, double* lu, int64_t* piv, int64_t* m_out) {
  *m_out = 0;
  const int64_t len = ps * ps;
  int64_t* group_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)(np > 0 ? np : 1));
  uint8_t* masks = (uint8_t*)malloc((size_t)((np > 0 ? np : 1) * ps));
  int64_t ng = 0;
  int st = orc_boundary_partition(np, ps, mats, group_of, masks, &ng);
  free(masks);
  if (st) {
    free(group_of);
    return st;
  }
  int64_t* sizes = (int64_t*)calloc((size_t)ng, sizeof(int64_t));
  for (int64_t k = 0; k < np; ++k) ++sizes[group_of[k]];
  int64_t* alloc = (int64_t*)malloc(sizeof(int64_t) * (size_t)ng);
  st = orc_split_budget(m_p, ng, sizes, alloc);
  int64_t offset = 0;
  for (int64_t g = 0; g < ng && !st; ++g) {
    const int64_t cnt = sizes[g];
    int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)cnt);
    int64_t c = 0;
    for (int64_t k = 0; k < np; ++k)
      if (group_of[k] == g) ids[c++] = k;
    double* sub = (double*)malloc(sizeof(double) * (size_t)(cnt * len));
    for (int64_t q = 0; q < cnt; ++q) memcpy(sub + q * len, mats + ids[q] * len, sizeof(double) * (size_t)len);
    int64_t* sphi = (int64_t*)malloc(sizeof(int64_t) * (size_t)cnt);
    int64_t sm = 0;
    st = orc_kmeans(cnt, ps, sub, alloc[g], variant, seed + (uint64_t)g, max_iters, sphi, reps + offset * len,
                    lu + offset * len, piv + offset * ps, &sm);
    if (!st)
      for (int64_t q = 0; q < cnt; ++q) phi[ids[q]] = offset + sphi[q];
    offset += sm;
    free(ids);
    free(sub);
    free(sphi);
  }
  free(group_of);
  free(sizes);
  free(alloc);
  *m_out = offset;
  return st;
}

/* greedy_bisect_to_size, experiments.cpp:168-204. */
int orc_greedy_bisect(int64_t np, int64_t ps, const double* mats, int spectral, int64_t target_lo, int64_t target_hi,
                      int best_match, int64_t* phi, int64_t* creators, double* reps, double* lu, int64_t* piv,
                      int64_t* m_out, double* eps_out) {
  const int64_t len = ps * ps;
  if (target_lo > np) target_lo = np;
  if (target_lo < 1) target_lo = 1;
  if (target_hi > np) target_hi = np;
  if (target_hi < target_lo) target_hi = target_lo;
  double lo = 1e-14, hi = 1e10;
  int64_t best_gap = INT64_MAX;
  int64_t* tphi = (int64_t*)malloc(sizeof(int64_t) * (size_t)np);
  int64_t* tcre = (int64_t*)malloc(sizeof(int64_t) * (size_t)np);
  double* treps = (double*)malloc(sizeof(double) * (size_t)(np * len));
  double* tlu = (double*)malloc(sizeof(double) * (size_t)(np * len));
  int64_t* tpiv = (int64_t*)malloc(sizeof(int64_t) * (size_t)(np * ps));
  int st = ST_OK;
  for (int it = 0; it < 60; ++it) {
    const double eps = sqrt(lo * hi);
    int64_t m = 0;
    int aborted = 0;
    st = orc_greedy(np, ps, mats, eps, spectral, best_match, target_hi, tphi, tcre, treps, tlu, tpiv, &m, &aborted);
    if (st) break;
    if (aborted) {
      lo = eps;
      continue;
    }
    const int64_t gap = m < target_lo ? target_lo - m : (m > target_hi ? m - target_hi : 0);
    if (gap < best_gap) {
      best_gap = gap;
      memcpy(phi, tphi, sizeof(int64_t) * (size_t)np);
      if (creators) memcpy(creators, tcre, sizeof(int64_t) * (size_t)m);
      memcpy(reps, treps, sizeof(double) * (size_t)(m * len));
      memcpy(lu, tlu, sizeof(double) * (size_t)(m * len));
      memcpy(piv, tpiv, sizeof(int64_t) * (size_t)(m * ps));
      *m_out = m;
      *eps_out = eps;
      if (gap == 0) break;
    }
    if (m < target_lo)
      hi = eps;
    else
      lo = eps;
  }
  if (!st && best_gap == INT64_MAX) st = set_err(ST_INVALID, "greedy bisection found no database");
  free(tphi);
  free(tcre);
  free(treps);
  free(tlu);
  free(tpiv);
  return st;
}

/* ======================================================================
 * precond.cpp
 * ==================================================================== */

/* PatchPreconditioner::apply, precond.cpp:58-88: per-patch gather + LU solve
 * into sols, serial scatter in ascending k, then z *= omega*w. */
void orc_precond_apply(int64_t n, int64_t np, int64_t ps, const int64_t* patches, const double* weights,
                       double omega, const double* lu, const int64_t* piv, const int64_t* phi, const double* r,
                       double* z) {
  const int64_t len = ps * ps;
  double* sols = (double*)malloc(sizeof(double) * (size_t)(np * ps));
  double* local = (double*)malloc(sizeof(double) * (size_t)ps);
  for (int64_t k = 0; k < np; ++k) {
    const int64_t* idx = patches + k * ps;
    for (int64_t i = 0; i < ps; ++i) local[i] = r[idx[i]];
    const int64_t f = phi ? phi[k] : k;
    orc_lu_solve(ps, lu + f * len, piv + f * ps, local, sols + k * ps);
  }
  for (int64_t i = 0; i < n; ++i) z[i] = 0.0;
  for (int64_t k = 0; k < np; ++k) {
    const int64_t* idx = patches + k * ps;
    const double* sol = sols + k * ps;
    for (int64_t i = 0; i < ps; ++i) z[idx[i]] += sol[i];
  }
  for (int64_t i = 0; i < n; ++i) z[i] *= omega * weights[i];
  free(sols);
  free(local);
}

/* smooth, precond.cpp:90-101, repeated; hist = ||b - A x|| before each sweep
 * and after the last. */
void orc_relax(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t np, int64_t ps,
               const int64_t* patches, const double* weights, double omega, const double* lu, const int64_t* piv,
               const int64_t* phi, const double* b, double* x, int64_t sweeps, double* hist) {
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t s = 0; s <= sweeps; ++s) {
    orc_spmv(n, rp, ci, v, x, r);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    if (hist) hist[s] = norm2(n, r);
    if (s == sweeps) break;
    orc_precond_apply(n, np, ps, patches, weights, omega, lu, piv, phi, r, z);
    for (int64_t i = 0; i < n; ++i) z[i] += x[i];
    memcpy(x, z, sizeof(double) * (size_t)n);
  }
  free(r);
  free(z);
}

/* ======================================================================
 * gmres.cpp
 * ==================================================================== */

static double dot(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

typedef struct {
  int64_t n, np, ps;
  const int64_t* patches;
  const double* weights;
  double omega;
  const double* lu;
  const int64_t* piv;
  const int64_t* phi;
} pc_t;

static void pc_apply(const pc_t* pc, const double* r, double* z) {
  orc_precond_apply(pc->n, pc->np, pc->ps, pc->patches, pc->weights, pc->omega, pc->lu, pc->piv, pc->phi, r, z);
}

/* gmres, gmres.cpp:27-169: restarted GMRES(m), MGS, Givens, right
 * preconditioning by default, true residual per cycle. */
int orc_gmres(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b, int64_t np,
              int64_t ps, const int64_t* patches, const double* weights, double omega, const double* lu,
              const int64_t* piv, const int64_t* phi, int have_pc, int64_t restart, double tol, int64_t max_iters,
              int left, double* x, int64_t* iters_out, int64_t* restarts_out, int* converged_out, double* relres_out,
              double* hist, int64_t* hist_len) {
  if (restart < 1) return set_err(ST_INVALID, "restart length must be >= 1");
  pc_t pc = {n, np, ps, patches, weights, omega, lu, piv, phi};
  const int64_t hcap = *hist_len;
  int64_t hl = 0;
#define PUSH_HIST(val)               \
  do {                               \
    if (hl < hcap) hist[hl] = (val); \
    ++hl;                            \
  } while (0)
  int64_t iterations = 0, restarts = 0;
  int converged = 0;
  double final_relres = 0.0;
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  const double bnorm = norm2(n, b);
  if (bnorm == 0.0) {
    *iters_out = 0;
    *restarts_out = 0;
    *converged_out = 1;
    *relres_out = 0.0;
    *hist_len = 0;
    return ST_OK;
  }
  const size_t m = (size_t)restart;
  double* V = (double*)malloc(sizeof(double) * (size_t)n * (m + 1));
  double* H = (double*)calloc((m + 1) * m, sizeof(double));
  double* cs = (double*)calloc(m, sizeof(double));
  double* sn = (double*)calloc(m, sizeof(double));
  double* g = (double*)calloc(m + 1, sizeof(double));
  double* y = (double*)calloc(m, sizeof(double));
  double* r0 = (double*)malloc(sizeof(double) * (size_t)n);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
  double* corr = (double*)malloc(sizeof(double) * (size_t)n);
#define Hm(i, j) H[(i) * m + (j)]
  double refnorm = 0.0;
  int first_cycle = 1;
  for (;;) {
    if (first_cycle) {
      memcpy(r0, b, sizeof(double) * (size_t)n);
    } else {
      orc_spmv(n, rp, ci, v, x, r0);
      for (int64_t i = 0; i < n; ++i) r0[i] = b[i] - r0[i];
    }
    if (have_pc && left) {
      pc_apply(&pc, r0, tmp);
      double* t = r0;
      r0 = tmp;
      tmp = t;
    }
    const double beta = norm2(n, r0);
    if (first_cycle) {
      PUSH_HIST(beta);
      refnorm = beta;
    }
    if (beta == 0.0) {
      converged = 1;
      break;
    }
    for (int64_t i = 0; i < n; ++i) V[i] = r0[i] / beta;
    for (size_t i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    size_t steps = 0;
    int breakdown = 0;
    for (size_t j = 0; j < m; ++j) {
      double* vj = V + j * (size_t)n;
      double* vj1 = V + (j + 1) * (size_t)n;
      if (!have_pc) {
        orc_spmv(n, rp, ci, v, vj, vj1);
      } else if (left) {
        orc_spmv(n, rp, ci, v, vj, tmp);
        pc_apply(&pc, tmp, vj1);
      } else {
        pc_apply(&pc, vj, tmp);
        orc_spmv(n, rp, ci, v, tmp, vj1);
      }
      for (size_t i = 0; i <= j; ++i) {
        const double hij = dot(n, vj1, V + i * (size_t)n);
        Hm(i, j) = hij;
        const double* vi = V + i * (size_t)n;
        for (int64_t k = 0; k < n; ++k) vj1[k] -= hij * vi[k];
      }
      const double hj1 = norm2(n, vj1);
      Hm(j + 1, j) = hj1;
      if (hj1 > 0.0)
        for (int64_t k = 0; k < n; ++k) vj1[k] /= hj1;
      for (size_t i = 0; i < j; ++i) {
        const double t1 = cs[i] * Hm(i, j) + sn[i] * Hm(i + 1, j);
        const double t2 = -sn[i] * Hm(i, j) + cs[i] * Hm(i + 1, j);
        Hm(i, j) = t1;
        Hm(i + 1, j) = t2;
      }
      const double denom = hypot(Hm(j, j), Hm(j + 1, j));
      cs[j] = Hm(j, j) / denom;
      sn[j] = Hm(j + 1, j) / denom;
      Hm(j, j) = denom;
      Hm(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++steps;
      ++iterations;
      const double est = fabs(g[j + 1]);
      PUSH_HIST(est > 2.2250738585072014e-308 ? est : 2.2250738585072014e-308);
      if (hj1 == 0.0) {
        breakdown = 1;
        break;
      }
      if (est <= tol * refnorm || iterations >= max_iters) break;
    }
    for (size_t i = steps; i-- > 0;) {
      double s = g[i];
      for (size_t k = i + 1; k < steps; ++k) s -= Hm(i, k) * y[k];
      y[i] = s / Hm(i, i);
    }
    for (int64_t k = 0; k < n; ++k) tmp[k] = 0.0;
    for (size_t i = 0; i < steps; ++i) {
      const double* vi = V + i * (size_t)n;
      for (int64_t k = 0; k < n; ++k) tmp[k] += y[i] * vi[k];
    }
    if (have_pc && !left) {
      pc_apply(&pc, tmp, corr);
      for (int64_t k = 0; k < n; ++k) x[k] += corr[k];
    } else {
      for (int64_t k = 0; k < n; ++k) x[k] += tmp[k];
    }
    orc_spmv(n, rp, ci, v, x, corr);
    for (int64_t i = 0; i < n; ++i) corr[i] = b[i] - corr[i];
    final_relres = norm2(n, corr) / bnorm;
    if (final_relres <= tol || breakdown) {
      converged = final_relres <= tol || breakdown;
      break;
    }
    if (iterations >= max_iters) break;
    ++restarts;
    first_cycle = 0;
  }
  orc_spmv(n, rp, ci, v, x, corr);
  for (int64_t i = 0; i < n; ++i) corr[i] = b[i] - corr[i];
  final_relres = norm2(n, corr) / bnorm;
#undef Hm
#undef PUSH_HIST
  *iters_out = iterations;
  *restarts_out = restarts;
  *converged_out = converged;
  *relres_out = final_relres;
  *hist_len = hl;
  free(V);
  free(H);
  free(cs);
  free(sn);
  free(g);
  free(y);
  free(r0);
  free(tmp);
  free(corr);
  return ST_OK;
}

/* Symmetrically weighted patch preconditioner used by PCG:
 *   z = omega W^{1/2} sum_k V_k^T B_phi(k)^{-1} V_k W^{1/2} r.
 * CG needs a symmetric preconditioner; the reference's left scaling
 * omega W S (precond.cpp:87) is not symmetric and makes CG stagnate, so the
 * weight is split evenly between gather and scatter.
 * Same patch solves and scatter order as orc_precond_apply. */
static void pc_apply_sym(const pc_t* pc, const double* r, double* z) {
  const int64_t ps = pc->ps, len = ps * ps;
  double* sols = (double*)malloc(sizeof(double) * (size_t)(pc->np * ps));
  double* local = (double*)malloc(sizeof(double) * (size_t)ps);
  for (int64_t k = 0; k < pc->np; ++k) {
    const int64_t* idx = pc->patches + k * ps;
    for (int64_t i = 0; i < ps; ++i) local[i] = r[idx[i]] * sqrt(pc->weights[idx[i]]);
    const int64_t f = pc->phi ? pc->phi[k] : k;
    orc_lu_solve(ps, pc->lu + f * len, pc->piv + f * ps, local, sols + k * ps);
  }
  for (int64_t i = 0; i < pc->n; ++i) z[i] = 0.0;
  for (int64_t k = 0; k < pc->np; ++k) {
    const int64_t* idx = pc->patches + k * ps;
    for (int64_t i = 0; i < ps; ++i) z[idx[i]] += sols[k * ps + i];
  }
  for (int64_t i = 0; i < pc->n; ++i) z[i] *= pc->omega * sqrt(pc->weights[i]);
  free(sols);
  free(local);
}

/* Inner products of the PCG restatement in a fixed blocked order, so that a
 * parallel implementation can reproduce them bit for bit: chunks of
 * PCG_CHUNK consecutive elements summed from 0.0 in order (a[i] * b[i] rounded,
 * then added), the chunk sums summed in groups of PCG_CHUNK in order, the
 * group sums in order.  (The reference has no CG; this order is part of the
 * restatement's definition.) */
#define PCG_CHUNK 256
static double dot_blocked(int64_t n, const double* a, const double* b) {
  const int64_t nch = (n + PCG_CHUNK - 1) / PCG_CHUNK;
  const int64_t ngr = (nch + PCG_CHUNK - 1) / PCG_CHUNK;
  double total = 0.0;
  for (int64_t g = 0; g < ngr; ++g) {
    double gs = 0.0;
    for (int64_t c = g * PCG_CHUNK; c < nch && c < (g + 1) * PCG_CHUNK; ++c) {
      double cs = 0.0;
      for (int64_t i = c * PCG_CHUNK; i < n && i < (c + 1) * PCG_CHUNK; ++i) cs += a[i] * b[i];
      gs += cs;
    }
    total += gs;
  }
  return total;
}

/* Preconditioned CG (not in the reference; SPEC.md:509 lists CG as absent).
 * Textbook Hestenes-Stiefel form with z = M_sym^{-1} r (pc_apply_sym) and the
 * blocked inner products above; the GPU's reproducible mode
 * (pdb_pcg_solve_ex with PDB_PCG_REPRODUCIBLE) computes the same sequence. */
int orc_pcg(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b, int64_t np, int64_t ps,
            const int64_t* patches, const double* weights, double omega, const double* lu, const int64_t* piv,
            const int64_t* phi, int have_pc, double tol, int64_t max_iters, double* x, int64_t* iters_out,
            int* converged_out, double* hist, int64_t* hist_len) {
  pc_t pc = {n, np, ps, patches, weights, omega, lu, piv, phi};
  const int64_t hcap = *hist_len;
  int64_t hl = 0;
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  double* q = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    x[i] = 0.0;
    r[i] = b[i];
  }
  const double bnorm = sqrt(dot_blocked(n, b, b));
  int converged = 0;
  int64_t it = 0;
  if (bnorm == 0.0) {
    converged = 1;
  } else {
    if (hl < hcap) hist[hl] = 1.0;
    ++hl;
    if (have_pc) pc_apply_sym(&pc, r, z);
    else memcpy(z, r, sizeof(double) * (size_t)n);
    memcpy(p, z, sizeof(double) * (size_t)n);
    double rz = dot_blocked(n, r, z);
    while (it < max_iters) {
      orc_spmv(n, rp, ci, v, p, q);
      const double alpha = rz / dot_blocked(n, p, q);
      for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
      for (int64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
      ++it;
      const double rel = sqrt(dot_blocked(n, r, r)) / bnorm;
      if (hl < hcap) hist[hl] = rel;
      ++hl;
      if (rel <= tol) {
        converged = 1;
        break;
      }
      if (have_pc) pc_apply_sym(&pc, r, z);
      else memcpy(z, r, sizeof(double) * (size_t)n);
      const double rz_new = dot_blocked(n, r, z);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
  }
  *iters_out = it;
  *converged_out = converged;
  *hist_len = hl;
  free(r);
  free(z);
  free(p);
  free(q);
  return ST_OK;
}
