// Half-storage ("mirror") residual layout.
//
// The residual r = b - A x streams every stored value once per sweep, so the
// sweep's floor is the matrix bytes over the HBM rate.  The FEM matrices of
// the BASELINE configurations 1-3 are symmetric bit for bit between their
// non-Dirichlet rows (one element kernel, one assembly order for a_ij and
// a_ji); only the Dirichlet rows (identity rows, columns kept: generator.cpp
// apply_dirichlet) break symmetry.  This layout stores, per row, only its
// upper entries (column >= row, diagonal first) and reads each lower entry
// a_ij from row j's storage, where a_ji == a_ij sits -- the second read of a
// value that another warp streamed from HBM shortly before, an L2 hit.  HBM
// traffic per residual drops from 8 B to ~4 B per nonzero.  The summation
// order of every row is the CSR order (lower entries first, columns are
// ascending), so the residual stays bitwise the reference spmv's
// (sparse.cpp:50-63).
//
// Layout.  Rows carry the column-pattern class of build_sell (offsets
// col - row per class).  A "group" is a storage shape: the upper-offset list
// of a class.  Rows are cut into windows of kSellSigma rows (L2 locality of
// the mirrored reads); inside a window they are ordered by (group, row), and
// each run of one group (a section) is cut into slices of 32 rows stored as
// the plain SELL copy stores them: slot t of the slice's lane l at
// soff + 32 t + l, one contiguous block per slice (a warp streams it behind
// one bulk L2 prefetch, HBM pages read whole).  Identity rows that are
// mirror targets ("virtual" rows: a non-Dirichlet neighbour reads a_ij from
// them) take the group their readers expect and store those a_ij in the
// matching slots next to their own diagonal.
//
// A lower entry (i, j = i + d) of a row of class c, ordinal m, reads value
// index rbase[j] + 32 * slot(c, m): rbase (int32 per row, the index of the
// row's slot 0) is gathered at the same index as x[j], and slot(c, m) -- the
// position of -d in the upper list of j's storage shape -- is one per
// (class, ordinal) (kslot, next to the class offsets).  No per-slice
// addressing data.  Any precondition that fails (explicit columns,
// non-symmetric values, targets of one (class, ordinal) needing different
// slots, storage beyond int32 indices) leaves the regular classed SELL copy
// in use.
#include <algorithm>
#include <cstring>
#include <thread>

#include "host.hpp"

namespace pdb {

namespace {

inline uint64_t bits(double v) {
  uint64_t u;
  std::memcpy(&u, &v, sizeof u);
  return u;
}

template <class F>
void parallel_for(int64_t count, F&& body) {
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  if (count < 4096 || T == 1) {
    body(0, count, 0);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) pool.emplace_back([&, t] { body(count * t / T, count * (t + 1) / T, t); });
  for (auto& th : pool) th.join();
}

int num_threads() { return static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency()))); }

}  // namespace

bool build_mirror_host(const HostCsr& h, const std::vector<int32_t>& cls, const std::vector<int32_t>& tab,
                       const std::vector<int32_t>& tstart, int64_t sigma, MirrorHost& M) {
  const int64_t n = h.n;
  const int ncls = static_cast<int>(tstart.size()) - 1;
  auto fail_with = [&](const char* why) {
    M = MirrorHost();
    M.why = why;
    return false;
  };
  if (n == 0 || ncls <= 0 || static_cast<int64_t>(cls.size()) != n) return fail_with("no column-pattern classes");
  // ---- per class: lower count, own width, virtual (diagonal-only / empty)
  std::vector<int32_t> clo(static_cast<size_t>(ncls)), wid(static_cast<size_t>(ncls));
  std::vector<char> virt(static_cast<size_t>(ncls)), used(static_cast<size_t>(ncls), 0);
  for (int c = 0; c < ncls; ++c) {
    const int32_t* t = tab.data() + tstart[static_cast<size_t>(c)];
    const int len = tstart[static_cast<size_t>(c) + 1] - tstart[static_cast<size_t>(c)];
    int lo = 0;
    while (lo < len && t[lo] < 0) ++lo;
    for (int k = 1; k < len; ++k)
      if (t[k] <= t[k - 1]) return fail_with("class offsets not ascending");
    clo[static_cast<size_t>(c)] = lo;
    wid[static_cast<size_t>(c)] = len - lo;
    virt[static_cast<size_t>(c)] = len == 0 || (len == 1 && t[0] == 0);
  }
  for (int64_t i = 0; i < n; ++i) used[static_cast<size_t>(cls[static_cast<size_t>(i)])] = 1;
  // slot of upper offset o in class g's own list (-1: absent)
  auto slot_of = [&](int g, int32_t o) -> int32_t {
    const int32_t* b = tab.data() + tstart[static_cast<size_t>(g)] + clo[static_cast<size_t>(g)];
    const int32_t* e = tab.data() + tstart[static_cast<size_t>(g) + 1];
    const int32_t* p = std::lower_bound(b, e, o);
    return p != e && *p == o ? static_cast<int32_t>(p - b) : -1;
  };

  // ---- scan every lower entry: the class of its target row (one per (class,
  // ordinal)), the slot it reads there, bitwise symmetry; virtual demands
  const size_t nkey = tab.size();
  const int T = num_threads();
  std::vector<std::vector<int32_t>> ecl_t(static_cast<size_t>(T)), esl_t(static_cast<size_t>(T));
  struct Demand {
    int32_t j, key, i;
  };
  std::vector<std::vector<Demand>> dem_t(static_cast<size_t>(T));
  std::vector<const char*> bad_t(static_cast<size_t>(T), nullptr);
  parallel_for(n, [&](int64_t r0, int64_t r1, int t) {
    auto& ecl = ecl_t[static_cast<size_t>(t)];
    auto& esl = esl_t[static_cast<size_t>(t)];
    ecl.assign(nkey, -1);
    esl.assign(nkey, -1);
    auto& dem = dem_t[static_cast<size_t>(t)];
    for (int64_t i = r0; i < r1; ++i) {
      const int c = cls[static_cast<size_t>(i)];
      const int32_t ts = tstart[static_cast<size_t>(c)];
      const int64_t p0 = h.row_ptr[static_cast<size_t>(i)];
      for (int m = 0; m < clo[static_cast<size_t>(c)]; ++m) {
        const int32_t key = ts + m;
        const int64_t j = i + tab[static_cast<size_t>(key)];
        const int cj = cls[static_cast<size_t>(j)];
        if (virt[static_cast<size_t>(cj)]) {
          dem.push_back({static_cast<int32_t>(j), key, static_cast<int32_t>(i)});
          continue;
        }
        // the targets of one (class, ordinal) may fall in different classes
        // (clipped stencils), but must hold the value in the same slot
        int32_t& ec = ecl[static_cast<size_t>(key)];
        int32_t& es = esl[static_cast<size_t>(key)];
        if (ec != cj) {
          const int32_t sj = slot_of(cj, -tab[static_cast<size_t>(key)]);
          if (sj < 0) {
            bad_t[static_cast<size_t>(t)] = "pattern not symmetric";
            return;
          }
          if (es != -1 && es != sj) {
            bad_t[static_cast<size_t>(t)] = "mirror slot differs between target classes";
            return;
          }
          ec = cj;
          es = sj;
        }
        const double vj = h.val[static_cast<size_t>(h.row_ptr[static_cast<size_t>(j)] + clo[static_cast<size_t>(cj)] + es)];
        if (bits(vj) != bits(h.val[static_cast<size_t>(p0 + m)])) {
          bad_t[static_cast<size_t>(t)] = "values not bitwise symmetric";
          return;
        }
      }
    }
  });
  for (const char* b : bad_t)
    if (b) return fail_with(b);
  std::vector<int32_t> ecl(nkey, -1), esl(nkey, -1);  // a target class and the slot, per (class, ordinal)
  for (size_t t = 0; t < ecl_t.size(); ++t)
    for (size_t q = 0; q < ecl_t[t].size(); ++q) {
      if (ecl_t[t][q] == -1) continue;
      if (esl[q] != -1 && esl[q] != esl_t[t][q]) return fail_with("mirror slot differs between target classes");
      ecl[q] = ecl_t[t][q];
      esl[q] = esl_t[t][q];
    }
  for (int c = 0; c < ncls; ++c)
    if (used[static_cast<size_t>(c)])
      for (int m = 0; m < clo[static_cast<size_t>(c)]; ++m)
        if (ecl[static_cast<size_t>(tstart[static_cast<size_t>(c)] + m)] < 0) {
          // only identity-row targets: any storage shape holding the offset
          const size_t key = static_cast<size_t>(tstart[static_cast<size_t>(c)] + m);
          for (int g = 0; g < ncls && ecl[key] < 0; ++g)
            if (used[static_cast<size_t>(g)] && !virt[static_cast<size_t>(g)] && slot_of(g, -tab[key]) >= 0) {
              ecl[key] = g;
              esl[key] = slot_of(g, -tab[key]);
            }
          if (ecl[key] < 0) return fail_with("no storage shape holds a mirrored offset");
        }
  // ---- groups: own class, or for a demanded virtual row the class its readers expect
  std::vector<int32_t> group(cls.begin(), cls.end());
  std::vector<char> is_virt(static_cast<size_t>(n), 0);
  int64_t nvirt = 0;
  for (const auto& dv : dem_t)
    for (const Demand& d : dv) {
      if (is_virt[static_cast<size_t>(d.j)]) {
        if (slot_of(group[static_cast<size_t>(d.j)], -tab[static_cast<size_t>(d.key)]) != esl[static_cast<size_t>(d.key)])
          return fail_with("virtual row demanded by two storage shapes");
        continue;
      }
      const int32_t g = ecl[static_cast<size_t>(d.key)];
      const int cj = cls[static_cast<size_t>(d.j)];
      if (wid[static_cast<size_t>(cj)] == 1 && slot_of(g, 0) != 0) return fail_with("storage shape without a leading diagonal");
      is_virt[static_cast<size_t>(d.j)] = 1;
      group[static_cast<size_t>(d.j)] = g;
      ++nvirt;
    }

  // the kernel holds the class tables in shared memory (8 B per offset)
  if (tab.size() > 16384) return fail_with("class tables too large for shared memory");
  // ---- order: windows of sigma rows, (group, row) inside; sections
  const int64_t nwin = (n + sigma - 1) / sigma;
  struct Section {
    int64_t first;   // first perm position
    int64_t rows;    // rows in the section
    int32_t g;
    int64_t base;    // value index of (slot 0, row 0)
    int64_t slice0;  // first slice
  };
  std::vector<int32_t> perm(static_cast<size_t>(n));
  std::vector<std::vector<Section>> secs(static_cast<size_t>(nwin));
  parallel_for(nwin, [&](int64_t w0, int64_t w1, int) {
    for (int64_t w = w0; w < w1; ++w) {
      const int64_t r0 = w * sigma, r1 = std::min(n, r0 + sigma);
      for (int64_t i = r0; i < r1; ++i) perm[static_cast<size_t>(i)] = static_cast<int32_t>(i);
      std::stable_sort(perm.begin() + r0, perm.begin() + r1, [&](int32_t a, int32_t b) {
        return group[static_cast<size_t>(a)] < group[static_cast<size_t>(b)];
      });
      auto& sv = secs[static_cast<size_t>(w)];
      for (int64_t p = r0; p < r1;) {
        const int32_t g = group[static_cast<size_t>(perm[static_cast<size_t>(p)])];
        int64_t q = p;
        while (q < r1 && group[static_cast<size_t>(perm[static_cast<size_t>(q)])] == g) ++q;
        sv.push_back({p, q - p, g, 0, 0});
        p = q;
      }
    }
  });
  int64_t vbase = 0, nslices = 0;
  M.win_slice.assign(static_cast<size_t>(nwin) + 1, 0);
  for (int64_t w = 0; w < nwin; ++w) {
    M.win_slice[static_cast<size_t>(w)] = nslices;
    for (Section& s : secs[static_cast<size_t>(w)]) {
      const int64_t hgt = (s.rows + 31) / 32 * 32;
      s.base = vbase;
      s.slice0 = nslices;
      vbase += hgt * wid[static_cast<size_t>(s.g)];
      nslices += hgt / 32;
    }
  }
  M.win_slice[static_cast<size_t>(nwin)] = nslices;
  if (vbase >= INT32_MAX) return fail_with("storage beyond int32 value indices");
  // per row: value index of its slot 0 (slot t at + 32 t)
  std::vector<int64_t> rbase(static_cast<size_t>(n));
  M.nslices = nslices;
  M.soff.assign(static_cast<size_t>(nslices), 0);
  M.rows.assign(static_cast<size_t>(2 * nslices * 32), 0);
  parallel_for(nwin, [&](int64_t w0, int64_t w1, int) {
    for (int64_t w = w0; w < w1; ++w)
      for (const Section& s : secs[static_cast<size_t>(w)]) {
        const int64_t hgt = (s.rows + 31) / 32 * 32;  // <= sigma
        const int64_t W = wid[static_cast<size_t>(s.g)];
        // (slot t, row q) at base + (q / 32) * 32 W + 32 t + q % 32
        auto at0 = [&](int64_t q) { return s.base + (q / 32) * 32 * W + q % 32; };
        for (int64_t q = 0; q < hgt; ++q) {
          const int64_t sl = s.slice0 + q / 32;
          const size_t ri = static_cast<size_t>(2 * (sl * 32 + q % 32));
          if (q % 32 == 0) {
            M.soff[static_cast<size_t>(sl)] = at0(q);
          }
          if (q >= s.rows) {
            M.rows[ri] = -1;
            M.rows[ri + 1] = 0;
            continue;
          }
          const int32_t row = perm[static_cast<size_t>(s.first + q)];
          const int c = cls[static_cast<size_t>(row)];
          const int32_t len = tstart[static_cast<size_t>(c) + 1] - tstart[static_cast<size_t>(c)];
          M.rows[ri] = row;
          M.rows[ri + 1] = len | ((c + 1) << 16);
          rbase[static_cast<size_t>(row)] = at0(q);
        }
      }
  });
  // ---- values: own upper entries, then the virtual rows' demanded slots
  M.val.assign(static_cast<size_t>(vbase), 0.0);
  parallel_for(n, [&](int64_t r0, int64_t r1, int) {
    for (int64_t i = r0; i < r1; ++i) {
      const int c = cls[static_cast<size_t>(i)];
      const int64_t p = h.row_ptr[static_cast<size_t>(i)] + clo[static_cast<size_t>(c)];
      for (int t = 0; t < wid[static_cast<size_t>(c)]; ++t)
        M.val[static_cast<size_t>(rbase[static_cast<size_t>(i)] + 32 * int64_t{t})] =
            h.val[static_cast<size_t>(p + t)];
    }
  });
  for (const auto& dv : dem_t)
    for (const Demand& d : dv) {
      const int32_t t = esl[static_cast<size_t>(d.key)];
      const int c = cls[static_cast<size_t>(d.i)];
      const int m = d.key - tstart[static_cast<size_t>(c)];
      M.val[static_cast<size_t>(rbase[static_cast<size_t>(d.j)] + 32 * int64_t{t})] =
          h.val[static_cast<size_t>(h.row_ptr[static_cast<size_t>(d.i)] + m)];
    }
  // ---- per row its slot-0 index, per (class, lower ordinal) 32 * slot
  M.rbase.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    M.rbase[static_cast<size_t>(i)] = static_cast<int32_t>(rbase[static_cast<size_t>(i)]);
  }
  M.kslot.assign(tab.size(), 0);
  for (size_t q = 0; q < tab.size(); ++q)
    if (esl[q] >= 0) M.kslot[q] = 32 * esl[q];
  M.clo = clo;
  M.virtual_rows = nvirt;
  return true;
}

// Host emulation of residual_mirror_kernel's arithmetic (y = A x in the
// kernel's order): the layout self-check of pdb_debug_mirror_check.
void mirror_spmv_host(const MirrorHost& M, const std::vector<int32_t>& tab, const std::vector<int32_t>& tstart,
                      const double* x, double* y) {
  for (int64_t sl = 0; sl < M.nslices; ++sl) {
    const int64_t so = M.soff[static_cast<size_t>(sl)];
    for (int l = 0; l < 32; ++l) {
      const int32_t row = M.rows[static_cast<size_t>(2 * (sl * 32 + l))];
      if (row < 0) continue;
      const int32_t rl = M.rows[static_cast<size_t>(2 * (sl * 32 + l)) + 1];
      const int len = rl & 0xFFFF, c = (rl >> 16) - 1;
      const int lo = M.clo[static_cast<size_t>(c)];
      const int32_t ts = tstart[static_cast<size_t>(c)];
      double acc = 0.0;
      for (int m = 0; m < lo; ++m) {
        const int64_t j = row + tab[static_cast<size_t>(ts + m)];
        acc += M.val[static_cast<size_t>(M.rbase[static_cast<size_t>(j)] + M.kslot[static_cast<size_t>(ts + m)])] * x[j];
      }
      for (int t = 0; t < len - lo; ++t) acc += M.val[static_cast<size_t>(so + 32 * t + l)] * x[row + tab[static_cast<size_t>(ts + lo + t)]];
      y[row] = acc;
    }
  }
}

}  // namespace pdb
