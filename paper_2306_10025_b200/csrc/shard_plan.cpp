// Slab partition of the relaxation sweep across ranks.
//
// Patches are ordered by their smallest DoF (detect_patches sorts by front,
// patch.cpp:82-83), so contiguous patch ranges are slabs of cells.  Rank r
// owns patches [np*r/N, np*(r+1)/N).  A DoF is owned by the highest rank
// whose patches contain it: that rank finishes the reference's
// ascending-patch scatter sum (precond.cpp:81-86) -- the lower neighbour
// sends its partial sum (0 + s_k1 + s_k2 ...), the owner continues adding its
// own contributions, so interface sums are bitwise the serial ones.  Every
// DoF may be touched by at most two adjacent ranks (slabs at least one patch
// layer thick).  Each sweep exchanges (a) those interface partials upward and
// (b) the updated x of owned DoFs that other ranks' residual rows read.
//
// This file is host-only planning (no CUDA), so the exchange schedule is
// testable on the CPU (tests/test_shard.py runs it with world_size 2 over
// gloo against the serial oracle).
#include <algorithm>
#include <cstring>

#include "host.hpp"

namespace pdb {

namespace {

// Pairwise exchange lists, grouped by peer rank, each group sorted by global DoF.
void group_lists(std::vector<std::pair<int32_t, int64_t>>& entries, std::vector<int32_t>& peer_of,
                 std::vector<int64_t>& global_of) {
  std::sort(entries.begin(), entries.end());
  peer_of.clear();
  global_of.clear();
  for (const auto& e : entries) {
    peer_of.push_back(e.first);
    global_of.push_back(e.second);
  }
}

}  // namespace

ShardPlan plan_shard(Index n, const int64_t* rp, const int32_t* ci, const double* val, Index np, Index ps,
                     const int32_t* patches, const double* weights, int rank, int nranks) {
  require(nranks >= 1 && rank >= 0 && rank < nranks, Errc::invalid_argument, "rank out of range");
  require(np >= nranks, Errc::invalid_argument, "fewer patches than ranks");
  ShardPlan P;
  P.rank = rank;
  P.nranks = nranks;
  auto k_lo = [&](int r) { return np * r / nranks; };
  P.k0 = k_lo(rank);
  P.k1 = k_lo(rank + 1);

  // contributor ranks of every DoF
  std::vector<int32_t> lo_rank(static_cast<size_t>(n), -1), hi_rank(static_cast<size_t>(n), -1);
  for (int r = 0; r < nranks; ++r)
    for (Index k = k_lo(r); k < k_lo(r + 1); ++k)
      for (Index q = 0; q < ps; ++q) {
        const int32_t d = patches[k * ps + q];
        if (lo_rank[static_cast<size_t>(d)] < 0) lo_rank[static_cast<size_t>(d)] = r;
        hi_rank[static_cast<size_t>(d)] = r;
      }
  std::vector<int32_t> owner(static_cast<size_t>(n));
  for (Index d = 0; d < n; ++d) {
    const int32_t lo = lo_rank[static_cast<size_t>(d)], hi = hi_rank[static_cast<size_t>(d)];
    if (lo >= 0)
      require(hi - lo <= 1, Errc::invalid_argument,
              "slab partition too thin: a DoF is shared by non-adjacent ranks (use fewer ranks)");
    owner[static_cast<size_t>(d)] = lo >= 0 ? hi : 0;  // uncovered DoFs (z = 0) belong to rank 0
  }

  // local DoF set of a rank: its patch DoFs, its owned DoFs, and the columns of its patch-DoF rows
  auto local_set = [&](int r, std::vector<int64_t>& dofs, std::vector<char>& is_row) {
    std::vector<char> mark(static_cast<size_t>(n), 0);
    for (Index k = k_lo(r); k < k_lo(r + 1); ++k)
      for (Index q = 0; q < ps; ++q) mark[static_cast<size_t>(patches[k * ps + q])] = 2;  // residual row
    for (Index d = 0; d < n; ++d)
      if (owner[static_cast<size_t>(d)] == r && !mark[static_cast<size_t>(d)]) mark[static_cast<size_t>(d)] = 1;
    for (Index d = 0; d < n; ++d)
      if (mark[static_cast<size_t>(d)] == 2)
        for (int64_t p = rp[d]; p < rp[d + 1]; ++p)
          if (!mark[static_cast<size_t>(ci[p])]) mark[static_cast<size_t>(ci[p])] = 1;
    dofs.clear();
    is_row.clear();
    for (Index d = 0; d < n; ++d)
      if (mark[static_cast<size_t>(d)]) {
        dofs.push_back(d);
        is_row.push_back(mark[static_cast<size_t>(d)] == 2);
      }
  };

  std::vector<char> is_row;
  local_set(rank, P.dofs, is_row);
  const Index nl = static_cast<Index>(P.dofs.size());
  std::vector<int32_t> g2l(static_cast<size_t>(n), -1);
  for (Index l = 0; l < nl; ++l) g2l[static_cast<size_t>(P.dofs[static_cast<size_t>(l)])] = static_cast<int32_t>(l);

  // local CSR: patch-DoF rows carry their entries, every other local row is empty
  P.rp.assign(static_cast<size_t>(nl + 1), 0);
  for (Index l = 0; l < nl; ++l) {
    const Index d = P.dofs[static_cast<size_t>(l)];
    P.rp[static_cast<size_t>(l + 1)] = P.rp[static_cast<size_t>(l)] + (is_row[static_cast<size_t>(l)] ? rp[d + 1] - rp[d] : 0);
  }
  P.ci.resize(static_cast<size_t>(P.rp.back()));
  P.val.resize(static_cast<size_t>(P.rp.back()));
  for (Index l = 0; l < nl; ++l) {
    if (!is_row[static_cast<size_t>(l)]) continue;
    const Index d = P.dofs[static_cast<size_t>(l)];
    int64_t o = P.rp[static_cast<size_t>(l)];
    for (int64_t p = rp[d]; p < rp[d + 1]; ++p, ++o) {
      P.ci[static_cast<size_t>(o)] = g2l[static_cast<size_t>(ci[p])];
      P.val[static_cast<size_t>(o)] = val[p];
    }
  }
  // local patches and weights (global cover counts)
  const Index npl = P.k1 - P.k0;
  P.patches.resize(static_cast<size_t>(npl * ps));
  for (Index k = 0; k < npl; ++k)
    for (Index q = 0; q < ps; ++q)
      P.patches[static_cast<size_t>(k * ps + q)] = g2l[static_cast<size_t>(patches[(P.k0 + k) * ps + q])];
  P.weights.resize(static_cast<size_t>(nl));
  for (Index l = 0; l < nl; ++l) P.weights[static_cast<size_t>(l)] = weights[P.dofs[static_cast<size_t>(l)]];

  // owned DoFs; interface partials out (to the owner) and in (from the lower contributor)
  std::vector<std::pair<int32_t, int64_t>> up, pin;
  for (Index l = 0; l < nl; ++l) {
    const Index d = P.dofs[static_cast<size_t>(l)];
    const int32_t own = owner[static_cast<size_t>(d)];
    if (own == rank) {
      P.owned.push_back(static_cast<int32_t>(l));
      if (lo_rank[static_cast<size_t>(d)] >= 0 && lo_rank[static_cast<size_t>(d)] < rank)
        pin.emplace_back(lo_rank[static_cast<size_t>(d)], d);
    } else if (is_row[static_cast<size_t>(l)]) {
      up.emplace_back(own, d);  // this rank contributes to a DoF finished by `own`
    }
  }
  std::vector<int64_t> g;
  group_lists(up, P.up_peer, g);
  P.up.clear();
  for (int64_t d : g) P.up.push_back(g2l[static_cast<size_t>(d)]);
  group_lists(pin, P.pin_peer, g);
  P.pin.clear();
  for (int64_t d : g) P.pin.push_back(g2l[static_cast<size_t>(d)]);

  // x halo: receive every non-owned local DoF from its owner; send owned DoFs
  // to every other rank whose local set contains them.
  std::vector<std::pair<int32_t, int64_t>> xr, xs;
  for (Index l = 0; l < nl; ++l) {
    const Index d = P.dofs[static_cast<size_t>(l)];
    if (owner[static_cast<size_t>(d)] != rank) xr.emplace_back(owner[static_cast<size_t>(d)], d);
  }
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) continue;
    std::vector<int64_t> other;
    std::vector<char> other_rows;
    local_set(r, other, other_rows);
    for (int64_t d : other)
      if (owner[static_cast<size_t>(d)] == rank) xs.emplace_back(r, d);
  }
  group_lists(xr, P.xr_peer, g);
  P.xr.clear();
  for (int64_t d : g) P.xr.push_back(g2l[static_cast<size_t>(d)]);
  group_lists(xs, P.xs_peer, g);
  P.xs.clear();
  for (int64_t d : g) P.xs.push_back(g2l[static_cast<size_t>(d)]);
  return P;
}

}  // namespace pdb
