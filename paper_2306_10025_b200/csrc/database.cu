// Factorization database construction (reference compress.cpp, method
// switch of pdb_database_build capi.cpp:249-284).
//
// All matrix arithmetic (extraction, distances, means, LU) runs in the
// bit-exact kernels of kernels/{extract,criterion,lu}.cu; the host keeps the
// integer bookkeeping the reference does serially (greedy round control,
// k-means membership lists, reseed/prune, budget split).  Decisions are
// therefore identical to the reference's: phi is bit-exact.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <limits>
#include <map>
#include <numeric>
#include <random>

#include <cub/cub.cuh>

#include <nccl.h>

#include "host.hpp"

#define PDB_NCCL_DB(call)                                                                                 \
  do {                                                                                                    \
    ncclResult_t r_ = (call);                                                                             \
    if (r_ != ncclSuccess)                                                                                \
      ::pdb::fail(::pdb::Errc::internal, std::string("NCCL error in " #call ": ") + ncclGetErrorString(r_)); \
  } while (0)

#include "kernels.hpp"

namespace pdb {

namespace {

std::string fmt_f(double v) {  // std::to_string(double)
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", v);
  return buf;
}

}  // namespace

std::string singular_msg(int32_t status, double best) {
  return "singular matrix: pivot " + fmt_f(best) + " below threshold in column " + std::to_string(status - 1);
}

namespace {

template <typename T>
std::vector<T> d2h(const T* d, size_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) PDB_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  sync(s);
  return h;
}

template <typename T>
void h2d(T* d, const std::vector<T>& h, cudaStream_t s) {
  if (!h.empty()) PDB_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

// LU of mats[src[t]] for t < count.  Returns index of the first failing t (or -1) and its message.
int64_t lu_many(int64_t count, int ps, const double* mats, const int32_t* src, double* lu, int32_t* piv,
                std::string& msg, BuildWork& work, cudaStream_t s, std::vector<int32_t>* status_out = nullptr,
                std::vector<double>* best_out = nullptr) {
  if (count <= 0) return -1;
  Scratch<int32_t> status(static_cast<size_t>(count), s);
  Scratch<double> best(static_cast<size_t>(count), s);
  k::lu_batched(count, ps, mats, src, lu, piv, status.get(), best.get(), s);
  PDB_LAUNCH_CHECK();
  work.lu_count += count;
  std::vector<int32_t> st = d2h(status.get(), static_cast<size_t>(count), s);
  std::vector<double> bh = d2h(best.get(), static_cast<size_t>(count), s);
  int64_t first = -1;
  for (int64_t t = 0; t < count; ++t)
    if (st[static_cast<size_t>(t)] != 0) {
      first = t;
      msg = singular_msg(st[static_cast<size_t>(t)], bh[static_cast<size_t>(t)]);
      break;
    }
  if (status_out) *status_out = std::move(st);
  if (best_out) *best_out = std::move(bh);
  return first;
}

// Device entry storage with geometric growth.
struct EntryStore {
  int ps = 0;
  int64_t len = 0, m = 0, cap = 0;
  DevBuf<double> lu;
  DevBuf<int32_t> piv;
  void init(int ps_, int64_t cap0) {
    ps = ps_;
    len = static_cast<int64_t>(ps_) * ps_;
    cap = std::max<int64_t>(cap0, 1);
    lu.alloc(static_cast<size_t>(cap * len));
    piv.alloc(static_cast<size_t>(cap * ps));
  }
  void reserve(int64_t need, cudaStream_t s) {
    if (need <= cap) return;
    int64_t nc = std::max(need, cap * 2);
    DevBuf<double> l2(static_cast<size_t>(nc * len));
    DevBuf<int32_t> p2(static_cast<size_t>(nc * ps));
    if (m) {
      PDB_CUDA(cudaMemcpyAsync(l2.get(), lu.get(), m * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
      PDB_CUDA(cudaMemcpyAsync(p2.get(), piv.get(), m * ps * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
    sync(s);
    lu = std::move(l2);
    piv = std::move(p2);
    cap = nc;
  }
};

// ------------------------------------------------ device compaction --
struct Unmatched {
  const int32_t* phi;
  __device__ bool operator()(int32_t v) const { return phi[v] < 0; }
};

// out = the ids in[0..n) with phi[id] < 0, in order; returns their count.
int64_t select_unmatched(const int32_t* in, int64_t n, const int32_t* phi, int32_t* out, int64_t* num,
                         cudaStream_t s) {
  size_t bytes = 0;
  cub::DeviceSelect::If(nullptr, bytes, in, out, num, n, Unmatched{phi}, s);
  Scratch<unsigned char> tmp(bytes, s);
  cub::DeviceSelect::If(tmp.get(), bytes, in, out, num, n, Unmatched{phi}, s);
  int64_t c = 0;
  PDB_CUDA(cudaMemcpyAsync(&c, num, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  sync(s);
  return c;
}

// ---------------------------------------------------------------- greedy --
// greedy_impl (compress.cpp:40-95), exact round-batched form:
//   U = patches unmatched so far (ascending).  Each round takes the first B
//   of U as the batch S.  Every member of S was unmatched against all
//   existing entries, so the sequential pass would now process S in order
//   against entries created inside S only: greedy_resolve does exactly that.
//   The rest of U (first-match) -- or every later patch (best-match) -- is
//   then compared with the new entries only, in creation order.
// Sharding (comm, or PDB_SHARD_EMULATE=W on one GPU): every rank runs the
// same rounds -- batch distances, the sequential resolution and the list
// bookkeeping are replicated -- and only the dominant step, comparing the
// remaining patches R with the round's new entries, is split: rank r scans
// the r-th contiguous chunk of R.  Each patch is scanned by exactly one rank
// and entry ids only grow, so an all-reduce MAX of phi (and MIN of the best
// distance) merges the ranks' updates exactly; the database is bitwise the
// single-GPU one.
bool greedy_build(const DevBuf<double>& mats, int64_t np, int ps, double eps, bool spectral, bool best_match,
                  int64_t abort_above, pdb_database_s& out, cudaStream_t s, const ShardComm* comm = nullptr) {
  int W = comm ? comm->nranks : 1;
  if (!comm)
    if (const char* e = getenv("PDB_SHARD_EMULATE")) W = std::max(1, atoi(e));
  require(np >= 1, Errc::invalid_argument, "greedy_tolerance needs at least one patch");
  require(eps > 0.0, Errc::invalid_argument, "tolerance must be positive");
  const int64_t len = static_cast<int64_t>(ps) * ps;
  BuildWork& work = out.work;
  DevBuf<int32_t> phi(static_cast<size_t>(np));
  PDB_CUDA(cudaMemsetAsync(phi.get(), 0xff, np * sizeof(int32_t), s));  // -1
  // temporaries are stream-ordered (Scratch): no device-wide synchronisation per buffer
  Scratch<double> best_d(best_match ? static_cast<size_t>(np) : 0, s);
  if (best_match) {
    std::vector<double> init(static_cast<size_t>(np), eps);
    h2d(best_d.get(), init, s);
  }
  Scratch<int32_t> creators(static_cast<size_t>(np), s);
  Scratch<int32_t> U(static_cast<size_t>(np), s), U2(static_cast<size_t>(np), s);
  k::iota(np, U.get(), s);
  int64_t nu = np;
  EntryStore store;
  if (spectral) store.init(ps, std::min<int64_t>(np, 1024));
  const int64_t Bmax = spectral ? 128 : 1024;
  Scratch<double> D(static_cast<size_t>(Bmax * Bmax), s);
  Scratch<int32_t> luS_status(static_cast<size_t>(Bmax), s);
  Scratch<double> luS(spectral ? static_cast<size_t>(Bmax * len) : 0, s);
  Scratch<int32_t> pivS(spectral ? static_cast<size_t>(Bmax * ps) : 0, s);
  Scratch<int32_t> entry_of(static_cast<size_t>(Bmax), s);
  Scratch<int64_t> state(3, s);
  Scratch<uint8_t> flags(static_cast<size_t>(np), s);
  Scratch<int32_t> all_ids(static_cast<size_t>(np), s);
  k::iota(np, all_ids.get(), s);
  Scratch<unsigned long long> iters(1, s);
  PDB_CUDA(cudaMemsetAsync(iters.get(), 0, sizeof(unsigned long long), s));
  Scratch<int64_t> num_sel(1, s);
  size_t sel_bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, sel_bytes, U.get(), flags.get(), U2.get(), num_sel.get(), np, s);
  Scratch<unsigned char> sel_tmp(sel_bytes, s);
  auto select = [&](const int32_t* in, const uint8_t* fl, int32_t* o, int64_t n) -> int64_t {
    if (n <= 0) return 0;
    size_t b = sel_bytes;
    cub::DeviceSelect::Flagged(sel_tmp.get(), b, in, fl, o, num_sel.get(), n, s);
    int64_t c = 0;
    PDB_CUDA(cudaMemcpyAsync(&c, num_sel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    sync(s);
    return c;
  };
  int64_t m = 0;
  bool aborted = false;
  std::vector<int64_t> state_h(3);
  // Only distances below eps matter (first match: d < eps; best match: the
  // smallest d < eps), so spectral pairs that provably end above eps stop
  // early (Rayleigh-quotient bound, as the k-means pruning); PDB_GREEDY_PRUNE=0
  // runs every pair to convergence.
  const char* gp = getenv("PDB_GREEDY_PRUNE");
  const double bound = (gp && gp[0] == '0') ? 0.0 : eps;
  while (nu > 0) {
    const int64_t B = std::min(nu, Bmax);
    const int32_t* S = U.get();
    // distances among the batch
    TraceScope tr_round("greedy round (batch pairs + resolve)", s);
    if (spectral) {
      std::string msg;
      std::vector<int32_t> st;
      lu_many(B, ps, mats.get(), S, luS.get(), pivS.get(), msg, work, s, &st);
      h2d(luS_status.get(), st, s);
      k::spectral_pairs(B, S, B, ps, mats.get(), luS.get(), pivS.get(), D.get(), iters.get(), s, bound);
    } else {
      k::l1_pairs(B, S, B, static_cast<int>(len), mats.get(), S, nullptr, D.get(), s);
    }
    PDB_LAUNCH_CHECK();
    work.pair_evals += B * (B - 1) / 2;
    PDB_CUDA(cudaMemsetAsync(entry_of.get(), 0xff, B * sizeof(int32_t), s));
    state_h = {m, 0, -1};
    PDB_CUDA(cudaMemcpyAsync(state.get(), state_h.data(), 3 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    k::greedy_resolve(static_cast<int>(B), S, D.get(), eps, best_match ? 1 : 0, abort_above,
                      spectral ? luS_status.get() : nullptr, phi.get(), creators.get(), entry_of.get(), state.get(),
                      s);
    PDB_LAUNCH_CHECK();
    PDB_CUDA(cudaMemcpyAsync(state_h.data(), state.get(), 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    sync(s);
    const int64_t m_new = state_h[0];
    if (spectral) {
      // factors of the new entries (recomputed: bitwise identical to luS)
      store.reserve(m_new, s);
      std::string msg;
      const int64_t bad = lu_many(m_new - m, ps, mats.get(), creators.get() + m, store.lu.get() + m * len,
                                  store.piv.get() + m * ps, msg, work, s);
      if (bad >= 0) fail(Errc::internal, "greedy: factor of a new entry failed after a successful batch factor");
      store.m = m_new;
      if (state_h[2] >= 0) {
        const int64_t a = state_h[2];
        std::vector<int32_t> sh = d2h(S + a, 1, s);
        std::string msg2;
        std::vector<int32_t> st;
        std::vector<double> bst;
        Scratch<double> tl(static_cast<size_t>(len), s);
        Scratch<int32_t> tp(static_cast<size_t>(ps), s);
        lu_many(1, ps, mats.get(), S + a, tl.get(), tp.get(), msg2, work, s, &st, &bst);
        fail(Errc::singular_matrix, "patch " + std::to_string(sh[0]) + ": " + msg2);
      }
    }
    if (state_h[1]) {
      aborted = true;
      m = m_new;
      break;
    }
    // compare the remaining patches with the new entries [m, m_new)
    TraceScope tr_scan("greedy scan", s);
    if (m_new > m) {
      int64_t nr = 0;
      int32_t* R = U2.get();
      if (best_match) {
        // every patch above S[0] except the batch itself
        std::vector<int32_t> s0 = d2h(S, 1, s);
        std::vector<uint8_t> fl(static_cast<size_t>(np), 0);
        for (int64_t i = s0[0] + 1; i < np; ++i) fl[static_cast<size_t>(i)] = 1;
        std::vector<int32_t> Sh = d2h(S, static_cast<size_t>(B), s);
        for (int32_t v : Sh) fl[static_cast<size_t>(v)] = 0;
        h2d(flags.get(), fl, s);
        nr = select(all_ids.get(), flags.get(), R, np);
      } else {
        nr = nu - B;
        if (nr > 0)
          PDB_CUDA(cudaMemcpyAsync(R, U.get() + B, nr * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      }
      const int64_t rchunk = (nr + W - 1) / W;
      for (int rk = 0; rk < W && nr > 0; ++rk) {
        if (comm && rk != comm->rank) continue;
        const int64_t r0 = std::min<int64_t>(nr, rk * rchunk), r1 = std::min<int64_t>(nr, (rk + 1) * rchunk);
        int32_t* Rr = R + r0;
        const int64_t nrr = r1 - r0;
        if (nrr <= 0) continue;
        if (!spectral) {
          k::l1_scan(nrr, Rr, m, m_new, static_cast<int>(len), mats.get(), creators.get(), eps, best_match ? 1 : 0,
                     phi.get(), best_d.get(), s);
          PDB_LAUNCH_CHECK();
        } else {
          // chunks of new entries; first-match drops matched patches between chunks
          const int64_t CH = 16;
          Scratch<double> dch(static_cast<size_t>(nrr * CH), s);
          int64_t live = nrr;
          for (int64_t c0 = m; c0 < m_new && live > 0; c0 += CH) {
            const int64_t ne = std::min(CH, m_new - c0);
            k::spectral_pairs(live, Rr, ne, ps, mats.get(), store.lu.get() + c0 * len, store.piv.get() + c0 * ps,
                              dch.get(), iters.get(), s, bound);
            k::apply_scan(live, Rr, c0, ne, dch.get(), creators.get(), eps, best_match ? 1 : 0, phi.get(),
                          best_d.get(), s);
            PDB_LAUNCH_CHECK();
            if (!best_match && c0 + CH < m_new) {
              // keep unmatched
              std::vector<int32_t> ph = d2h(phi.get(), static_cast<size_t>(np), s);
              std::vector<int32_t> Rh = d2h(Rr, static_cast<size_t>(live), s);
              std::vector<int32_t> keep;
              keep.reserve(Rh.size());
              for (int32_t v : Rh)
                if (ph[static_cast<size_t>(v)] < 0) keep.push_back(v);
              live = static_cast<int64_t>(keep.size());
              h2d(Rr, keep, s);
            }
          }
        }
      }
      if (nr > 0) work.pair_evals += nr * (m_new - m);  // upper bound (early exits not counted)
      if (comm && nr > 0) {  // merge: phi only grows (entry ids), best distances only shrink
        PDB_NCCL_DB(ncclGroupStart());
        PDB_NCCL_DB(ncclAllReduce(phi.get(), phi.get(), static_cast<size_t>(np), ncclInt32, ncclMax, comm->comm, s));
        if (best_match)
          PDB_NCCL_DB(ncclAllReduce(best_d.get(), best_d.get(), static_cast<size_t>(np), ncclDouble, ncclMin,
                                    comm->comm, s));
        PDB_NCCL_DB(ncclGroupEnd());
      }
    }
    m = m_new;
    // U <- unmatched patches among U[B..nu)
    TraceScope tr_compact("greedy compact", s);
    const int64_t rest = nu - B;
    if (rest > 0) {
      // stream compaction on the device (order kept): U2 is free here
      nu = select_unmatched(U.get() + B, rest, phi.get(), U2.get(), num_sel.get(), s);
      PDB_CUDA(cudaMemcpyAsync(U.get(), U2.get(), nu * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    } else {
      nu = 0;
    }
  }
  if (comm) PDB_NCCL_DB(ncclAllReduce(iters.get(), iters.get(), 1, ncclUint64, ncclSum, comm->comm, s));
  unsigned long long it_h = 0;
  PDB_CUDA(cudaMemcpyAsync(&it_h, iters.get(), sizeof(it_h), cudaMemcpyDeviceToHost, s));
  sync(s);
  work.power_iters += static_cast<int64_t>(it_h);

  out.m = m;
  out.np = np;
  out.ps = ps;
  out.eps = eps;
  out.method = spectral ? "greedy" : "greedy-l1";
  out.reps.alloc(static_cast<size_t>(std::max<int64_t>(m, 1) * len));
  k::gather_mats(m, creators.get(), len, mats.get(), out.reps.get(), s);
  out.lu.alloc(static_cast<size_t>(std::max<int64_t>(m, 1) * len));
  out.piv.alloc(static_cast<size_t>(std::max<int64_t>(m, 1) * ps));
  if (spectral) {
    if (m) {
      PDB_CUDA(cudaMemcpyAsync(out.lu.get(), store.lu.get(), m * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
      PDB_CUDA(cudaMemcpyAsync(out.piv.get(), store.piv.get(), m * ps * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
  } else {
    // factor_patch at entry creation (compress.cpp:91): first failure in creation order wins,
    // and it precedes an abort that happens later in the sequence.
    std::string msg;
    const int64_t bad = lu_many(m, ps, mats.get(), creators.get(), out.lu.get(), out.piv.get(), msg, work, s);
    if (bad >= 0) {
      std::vector<int32_t> cr = d2h(creators.get() + bad, 1, s);
      fail(Errc::singular_matrix, "patch " + std::to_string(cr[0]) + ": " + msg);
    }
  }
  out.phi = std::move(phi);
  sync(s);
  return !aborted;
}

// ---------------------------------------------------------------- exact ---
void exact_build(const DevBuf<double>& mats, int64_t np, int ps, pdb_database_s& out, cudaStream_t s) {
  require(np >= 1, Errc::invalid_argument, "exact_database needs at least one patch");
  const int64_t len = static_cast<int64_t>(ps) * ps;
  out.m = np;
  out.np = np;
  out.ps = ps;
  out.method = "exact";
  out.reps.alloc(static_cast<size_t>(np * len));
  PDB_CUDA(cudaMemcpyAsync(out.reps.get(), mats.get(), np * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
  out.lu.alloc(static_cast<size_t>(np * len));
  out.piv.alloc(static_cast<size_t>(np * ps));
  std::string msg;
  const int64_t bad = lu_many(np, ps, mats.get(), nullptr, out.lu.get(), out.piv.get(), msg, out.work, s);
  if (bad >= 0) fail(Errc::singular_matrix, "patch " + std::to_string(bad) + ": " + msg);
  out.phi.alloc(static_cast<size_t>(np));
  k::iota(np, out.phi.get(), s);
  sync(s);
}

// --------------------------------------------------------------- k-means --
enum class Variant { Entrywise, Spectral, VarMin };
enum class Empty { Reseed, Prune };

std::string variant_name(Variant v) {
  switch (v) {
    case Variant::Entrywise: return "kmeans-entrywise";
    case Variant::Spectral: return "kmeans-spectral";
    case Variant::VarMin: return "kmeans-varmin";
  }
  return "kmeans";
}

struct KDb {
  int ps = 0;
  int64_t len = 0, m = 0;
  DevBuf<double> reps, lu;
  DevBuf<int32_t> piv;
  std::vector<char> has_factor;
};

// Factors of every patch of the group, computed once (VarMin candidates).
struct PatchFactors {
  bool ready = false;
  DevBuf<double> lu;
  DevBuf<int32_t> piv;
  std::vector<int32_t> status;
  std::vector<double> best;
};

void ensure_patch_factors(const double* sub, int64_t n, int ps, PatchFactors& pf, BuildWork& work, cudaStream_t s) {
  if (pf.ready) return;
  const int64_t len = static_cast<int64_t>(ps) * ps;
  pf.lu.alloc(static_cast<size_t>(n * len));
  pf.piv.alloc(static_cast<size_t>(n * ps));
  std::string msg;
  lu_many(n, ps, sub, nullptr, pf.lu.get(), pf.piv.get(), msg, work, s, &pf.status, &pf.best);
  pf.ready = true;
}

// kmeans_loop (compress.cpp:138-262).  phi_h receives the final assignment.
// Sharded assignment (SURVEY §8e "Setup"): the n patches are cut into W
// chunks of ceil(n/W); rank r evaluates the distances and the argmin of
// chunk r only, and an in-place ncclAllGather of the new assignment and the
// minimum distances gives every rank the full arrays, so the rest of the
// Lloyd iteration (reseed / prune, means in ascending member order, LU) runs
// redundantly and identically on all ranks -- the result is bitwise the
// single-GPU build.  PDB_SHARD_EMULATE=W runs all W chunks on one GPU (no
// NCCL), which tests the decomposition without W devices.

// Entrywise assignment: below this many patches per slot (or for patches of
// >= 4096 entries), one thread per (patch, entry tile) instead of one per
// patch (l1_pairs + argmin).
constexpr int64_t kL1PairsBelow = 16384;

struct AssignSlot {
  int64_t lo = 0, hi = 0;
  DevBuf<double> sub_il;
  DevBuf<double> dist, lbq;  // pruned spectral assignment: distances / quotient bounds kept across iterations
  int64_t m = 0;             // columns of dist / lbq
  DevBuf<double> sub_sorted;  // bound pass: the slot's patches interleaved in work order
  DevBuf<int32_t> perm, itc;  // work order; power iterations of each patch's last bound pair
  DevBuf<int32_t> tile_order;  // pruned pass: tiles of 32 patches, most power iterations first
  DevBuf<unsigned long long> tile_iters;
  DevBuf<uint8_t> lng[2];  // pruned pass: "ran long" per pair, by Lloyd iteration parity
};

// Work order of the bound pass (one pair per thread, aligned groups of 32 =
// one warp): patches whose centroid changed, sorted by centroid (the lanes of
// a warp share the factor: broadcast loads) and by the power iterations their
// previous bound pair took, descending (lanes of a warp finish together); the
// groups of 32 then run longest first (a short tail), and the patches whose
// centroid did not change (their distance is reused) come last.  The sorted
// interleaved copy makes every patch load of a warp one 256-byte span.
void diag_order(int64_t cnt, int64_t m, const std::vector<int32_t>& cur, const std::vector<uint8_t>& chg, int64_t len,
                const double* sub, AssignSlot& sl, cudaStream_t s) {
  if (sl.perm.size() < static_cast<size_t>(cnt)) {
    sl.perm.alloc(static_cast<size_t>(cnt));
    sl.itc.alloc(static_cast<size_t>(cnt));
    sl.itc.zero(s);
    sl.sub_sorted.alloc(static_cast<size_t>(k::interleaved_len(cnt, 32, len)));
  }
  const std::vector<int32_t> prev = d2h(sl.itc.get(), static_cast<size_t>(cnt), s);
  std::vector<int32_t> live, idle;
  for (int64_t i = 0; i < cnt; ++i) {
    const int32_t f = cur[static_cast<size_t>(i)];
    const bool c = f < 0 || f >= m || static_cast<size_t>(f) >= chg.size() || chg[static_cast<size_t>(f)];
    (c ? live : idle).push_back(static_cast<int32_t>(i));
  }
  // two stable counting sorts (O(n) per Lloyd iteration): iterations descending, then centroid
  auto counting = [](std::vector<int32_t>& v, int64_t nkeys, auto key) {
    std::vector<int32_t> start(static_cast<size_t>(nkeys + 1), 0), out(v.size());
    for (int32_t i : v) ++start[static_cast<size_t>(key(i) + 1)];
    for (int64_t k = 0; k < nkeys; ++k) start[static_cast<size_t>(k + 1)] += start[static_cast<size_t>(k)];
    for (int32_t i : v) out[static_cast<size_t>(start[static_cast<size_t>(key(i))]++)] = i;
    v.swap(out);
  };
  constexpr int32_t kMaxIt = 200;  // the power iteration's cap (dense.cpp:169)
  counting(live, kMaxIt + 1, [&](int32_t i) {
    return kMaxIt - std::min(std::max(prev[static_cast<size_t>(i)], 0), kMaxIt);
  });
  counting(live, m, [&](int32_t i) {
    const int32_t f = cur[static_cast<size_t>(i)];
    return (f >= 0 && f < m) ? f : 0;
  });
  const size_t full = live.size() / 32;  // whole groups; the partial one stays last (alignment)
  std::vector<std::pair<int32_t, size_t>> grp(full);
  for (size_t g = 0; g < full; ++g) {
    int32_t mx = 0;
    for (size_t a = 0; a < 32; ++a) mx = std::max(mx, prev[static_cast<size_t>(live[g * 32 + a])]);
    grp[g] = {mx, g};
  }
  std::stable_sort(grp.begin(), grp.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  std::vector<int32_t> perm;
  perm.reserve(static_cast<size_t>(cnt));
  for (const auto& gg : grp) perm.insert(perm.end(), live.begin() + static_cast<long>(gg.second * 32),
                                         live.begin() + static_cast<long>(gg.second * 32 + 32));
  perm.insert(perm.end(), live.begin() + static_cast<long>(full * 32), live.end());
  perm.insert(perm.end(), idle.begin(), idle.end());
  h2d(sl.perm.get(), perm, s);
  k::interleave_patches_perm(cnt, len, sl.perm.get(), sub, sl.sub_sorted.get(), s);
}

void kmeans_loop(const double* sub, int64_t n, KDb& db, Variant variant, int max_iters, Empty policy,
                 std::vector<int32_t>& phi_h, PatchFactors& pf, BuildWork& work, cudaStream_t s,
                 const ShardComm* comm = nullptr) {
  const int ps = db.ps;
  const int64_t len = db.len;
  const bool sharded = comm != nullptr;  // (a 1-rank communicator still runs the NCCL path)
  int W = sharded ? comm->nranks : 1;
  if (!sharded)
    if (const char* e = getenv("PDB_SHARD_EMULATE")) W = std::max(1, atoi(e));
  const int64_t chunk = (n + W - 1) / W;
  const size_t cap = static_cast<size_t>(std::max<int64_t>(chunk * W, n));
  phi_h.assign(static_cast<size_t>(n), -1);
  std::vector<double> min_dist(static_cast<size_t>(n), 0.0);
  DevBuf<int32_t> d_phi(cap), d_new(cap);
  DevBuf<double> d_min(cap);
  h2d(d_phi.get(), phi_h, s);
  Scratch<int32_t> changed(1, s);
  Scratch<unsigned long long> iters(1, s);
  PDB_CUDA(cudaMemsetAsync(iters.get(), 0, sizeof(unsigned long long), s));
  DevBuf<double> dist;
  // interleaved copies for the spectral assignment (PDB_SPECTRAL_IL=0 keeps the plain layout)
  const char* il_env = getenv("PDB_SPECTRAL_IL");
  const bool il = variant != Variant::Entrywise && k::spectral_il_supported(ps) && !(il_env && il_env[0] == '0');
  std::vector<AssignSlot> slots;
  for (int r = 0; r < W; ++r) {
    if (sharded && r != comm->rank) continue;
    AssignSlot sl;
    sl.lo = std::min<int64_t>(n, r * chunk);
    sl.hi = std::min<int64_t>(n, (r + 1) * chunk);
    if (il && sl.hi > sl.lo) {
      sl.sub_il.alloc(static_cast<size_t>(k::interleaved_len(sl.hi - sl.lo, 32, len)));
      k::interleave_patches(sl.hi - sl.lo, len, sub + sl.lo * len, sl.sub_il.get(), s);
    }
    slots.push_back(std::move(sl));
  }
  DevBuf<double> lu_il;
  DevBuf<int32_t> piv_il;
  // Assignment pruning (spectral variants, Lloyd iterations >= 1): each
  // patch's distance to its current centroid is evaluated first; every
  // other pair stops as soon as its Rayleigh quotient proves it larger
  // (spectral_tiled_il ub).  The argmin, its distance and so the whole
  // k-means run are unchanged; only the losing pairs' power iterations are
  // cut short.  PDB_KMEANS_PRUNE=0 evaluates every pair to convergence.
  const char* pr_env = getenv("PDB_KMEANS_PRUNE");
  const bool prune = il && !(pr_env && pr_env[0] == '0');
  const char* ds_env = getenv("PDB_DIAG_SORT");  // 0: bound pass in patch order with in-block refill
  const bool diag_sort = !(ds_env && ds_env[0] == '0');
  std::vector<uint8_t> chg_h;  // host copy of d_chg
  const char* lpt_env = getenv("PDB_TILE_LPT");  // 0: pruned-pass tiles in patch order
  const bool tile_lpt = !(lpt_env && lpt_env[0] == '0');
  const char* lf_env = getenv("PDB_LONG_FIRST");  // 0: pairs of a tile in plain order
  const bool long_first = !(lf_env && lf_env[0] == '0');
  DevBuf<double> ub;
  DevBuf<int32_t> guess;  // iteration 0: l1-nearest entry, for the first bound
  DevBuf<double> gmin;
  Scratch<int32_t> gchanged(1, s);
  DevBuf<uint8_t> d_chg;  // per entry: centroid changed since the previous assignment
  std::vector<std::vector<int32_t>> prev_members;
  if (prune) ub.alloc(cap);
  // PDB_KMEANS_TRACE=1: wall time per phase on stderr (assignment incl. its
  // device time / host update / means + LU)
  const char* tr_env = getenv("PDB_KMEANS_TRACE");
  const bool trace = tr_env && tr_env[0] == '1';
  double tr[3] = {0, 0, 0};
  auto tnow = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double tmark = tnow();
  for (int iter = 0; iter < max_iters; ++iter) {
    const int64_t m = db.m;
    if (trace) {
      sync(s);
      const double t = tnow();
      tr[2] += t - tmark;
      tmark = t;
    }
    PDB_CUDA(cudaMemsetAsync(changed.get(), 0, sizeof(int32_t), s));
    // one centroid: the argmin over a single entry is entry 0 whatever the
    // distances (strict <, best_j starts at 0: compress.cpp:154-160), and with
    // every patch in it no cluster is empty, so the distances are never read
    // (the reseed needs an empty cluster): skip them.  phi, the means and the
    // factors are those of the full computation; only the work counters differ.
    const bool single = m == 1;
    if (single) {
      PDB_CUDA(cudaMemsetAsync(d_new.get(), 0, cap * sizeof(int32_t), s));
      PDB_CUDA(cudaMemsetAsync(d_min.get(), 0, cap * sizeof(double), s));
    }
    if (!single && variant != Variant::Entrywise && il) {
      lu_il.alloc(static_cast<size_t>(k::interleaved_len(m, 8, len)));
      piv_il.alloc(static_cast<size_t>(k::interleaved_len(m, 8, ps)));
      k::interleave_factors(m, ps, db.lu.get(), db.piv.get(), lu_il.get(), piv_il.get(), s);
    }
    for (AssignSlot& sl : slots) {
      if (single) break;
      const int64_t cnt = sl.hi - sl.lo;
      if (cnt <= 0) continue;
      if (variant == Variant::Entrywise) {
        if ((cnt < kL1PairsBelow || len >= 4096) && m > 1) {
          // few patches (large ps): a thread per patch leaves the GPU idle, so
          // every (patch, entry tile) pair gets its own thread, then the
          // argmin -- the same sequential sums and strict-< scan, bitwise
          if (dist.size() < static_cast<size_t>(cnt * m)) dist.alloc(static_cast<size_t>(cnt * m));
          k::l1_pairs(cnt, nullptr, m, static_cast<int>(len), sub + sl.lo * len, nullptr, db.reps.get(), dist.get(),
                      s);
          k::argmin_assign(cnt, m, dist.get(), d_phi.get() + sl.lo, d_new.get() + sl.lo, d_min.get() + sl.lo,
                           changed.get(), s);
        } else {
          k::l1_argmin(cnt, m, static_cast<int>(len), sub + sl.lo * len, db.reps.get(), d_phi.get() + sl.lo,
                       d_new.get() + sl.lo, d_min.get() + sl.lo, changed.get(), s);
        }
      } else {
        double* dd = nullptr;
        if (prune) {  // per-slot distance matrix, kept for the next iteration
          if (sl.m != m) {
            sl.dist.alloc(static_cast<size_t>(cnt * m));
            sl.lbq.alloc(static_cast<size_t>(cnt * m));
            sl.lbq.zero(s);
            for (auto& lb : sl.lng) {
              lb.alloc(static_cast<size_t>(cnt * m));
              lb.zero(s);
            }
            sl.m = m;
          }
          dd = sl.dist.get();
        } else {
          if (dist.size() < static_cast<size_t>(cnt * m)) dist.alloc(static_cast<size_t>(cnt * m));
          dd = dist.get();
        }
        const bool pr = prune;
        k::KmeansReuse ru;
        const int32_t* cur_phi = d_phi.get() + sl.lo;
        if (pr && iter == 0) {
          // no assignment yet: bound each patch by its distance to the entry
          // nearest in the entrywise l1 sense (any entry's distance bounds the min)
          if (guess.size() < static_cast<size_t>(cap)) {
            guess.alloc(cap);
            gmin.alloc(cap);
          }
          k::l1_argmin(cnt, m, static_cast<int>(len), sub + sl.lo * len, db.reps.get(), d_phi.get() + sl.lo,
                       guess.get() + sl.lo, gmin.get() + sl.lo, gchanged.get(), s);
          cur_phi = guess.get() + sl.lo;
          std::vector<uint8_t> ones(static_cast<size_t>(m), 1);
          d_chg.alloc(static_cast<size_t>(m));
          h2d(d_chg.get(), ones, s);
          chg_h = ones;
        }
        if (pr) {
          ru.chg = d_chg.get();
          ru.dprev = dd;
          ru.mfull = m;
          const double* diag_mats = sl.sub_il.get();
          const int32_t* dperm = nullptr;
          if (diag_sort) {
            diag_order(cnt, m, iter == 0 ? d2h(cur_phi, static_cast<size_t>(cnt), s)
                                         : std::vector<int32_t>(phi_h.begin() + sl.lo, phi_h.begin() + sl.hi),
                       chg_h, len, sub + sl.lo * len, sl, s);
            diag_mats = sl.sub_sorted.get();
            dperm = sl.perm.get();
            ru.it_out = sl.itc.get();
          }
          k::spectral_diag_il(cnt, ps, diag_mats, db.lu.get(), db.piv.get(), cur_phi, ub.get() + sl.lo,
                              iters.get(), s, ru, dperm);
          ru.it_out = nullptr;
          work.pair_evals += cnt;
          ru.ub = ub.get() + sl.lo;
          ru.phi = cur_phi;
          ru.lbq = sl.lbq.get();
          ru.dprev = nullptr;
          if (tile_lpt) {
            // tiles in descending order of the power iterations they took in
            // the previous Lloyd iteration (stable: ties keep tile order)
            const int64_t nt = (cnt + 31) / 32;
            std::vector<int32_t> order(static_cast<size_t>(nt));
            std::iota(order.begin(), order.end(), 0);
            if (sl.tile_iters.size() == static_cast<size_t>(nt)) {
              const std::vector<unsigned long long> ti = d2h(sl.tile_iters.get(), static_cast<size_t>(nt), s);
              std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
                return ti[static_cast<size_t>(a)] > ti[static_cast<size_t>(b)];
              });
            } else {
              sl.tile_iters.alloc(static_cast<size_t>(nt));
              sl.tile_order.alloc(static_cast<size_t>(nt));
            }
            h2d(sl.tile_order.get(), order, s);
            sl.tile_iters.zero(s);
            ru.tile_order = sl.tile_order.get();
            ru.tile_iters = sl.tile_iters.get();
          }
          if (long_first) {
            ru.long_prev = sl.lng[iter & 1].get();
            ru.long_cur = sl.lng[(iter + 1) & 1].get();
          }
        }
        if (il)
          k::spectral_tiled_il(cnt, m, ps, sl.sub_il.get(), lu_il.get(), piv_il.get(), dd, iters.get(), s, ru);
        else
          k::spectral_pairs(cnt, nullptr, m, ps, sub + sl.lo * len, db.lu.get(), db.piv.get(), dd, iters.get(), s);
        k::argmin_assign(cnt, m, dd, d_phi.get() + sl.lo, d_new.get() + sl.lo, d_min.get() + sl.lo, changed.get(),
                         s);
      }
    }
    PDB_LAUNCH_CHECK();
    if (sharded) {
      PDB_NCCL_DB(ncclGroupStart());
      PDB_NCCL_DB(ncclAllGather(d_new.get() + comm->rank * chunk, d_new.get(), static_cast<size_t>(chunk), ncclInt32,
                                comm->comm, s));
      PDB_NCCL_DB(ncclAllGather(d_min.get() + comm->rank * chunk, d_min.get(), static_cast<size_t>(chunk),
                                ncclDouble, comm->comm, s));
      PDB_NCCL_DB(ncclGroupEnd());
    }
    if (!single) work.pair_evals += n * m;
    const std::vector<int32_t> prev = phi_h;
    phi_h = d2h(d_new.get(), static_cast<size_t>(n), s);
    if (trace) {
      const double t = tnow();
      tr[0] += t - tmark;
      tmark = t;
    }
    const bool ch = prev != phi_h;  // every rank sees the gathered assignment
    if (!ch) break;
    min_dist = d2h(d_min.get(), static_cast<size_t>(n), s);

    std::vector<std::vector<int32_t>> members(static_cast<size_t>(m));
    for (int64_t i = 0; i < n; ++i) members[static_cast<size_t>(phi_h[static_cast<size_t>(i)])].push_back(static_cast<int32_t>(i));
    const int64_t m_before = m;

    if (policy == Empty::Prune) {  // compress.cpp:179-194
      std::vector<int32_t> remap(static_cast<size_t>(m), -1), kept_ids;
      int64_t kept = 0;
      for (int64_t j = 0; j < m; ++j)
        if (!members[static_cast<size_t>(j)].empty()) {
          remap[static_cast<size_t>(j)] = static_cast<int32_t>(kept);
          kept_ids.push_back(static_cast<int32_t>(j));
          if (kept != j) {
            members[static_cast<size_t>(kept)] = std::move(members[static_cast<size_t>(j)]);
            db.has_factor[static_cast<size_t>(kept)] = db.has_factor[static_cast<size_t>(j)];
          }
          ++kept;
        }
      if (kept != m) {
        Scratch<int32_t> ids(static_cast<size_t>(kept), s);
        h2d(ids.get(), kept_ids, s);
        DevBuf<double> r2(static_cast<size_t>(kept * len)), l2(static_cast<size_t>(kept * len));
        DevBuf<int32_t> p2(static_cast<size_t>(kept * ps));
        k::gather_mats(kept, ids.get(), len, db.reps.get(), r2.get(), s);
        k::gather_mats(kept, ids.get(), len, db.lu.get(), l2.get(), s);
        k::gather_i32(kept, ids.get(), ps, db.piv.get(), p2.get(), s);
        sync(s);
        db.reps = std::move(r2);
        db.lu = std::move(l2);
        db.piv = std::move(p2);
      }
      members.resize(static_cast<size_t>(kept));
      db.has_factor.resize(static_cast<size_t>(kept));
      db.m = kept;
      for (int64_t i = 0; i < n; ++i)
        phi_h[static_cast<size_t>(i)] = remap[static_cast<size_t>(phi_h[static_cast<size_t>(i)])];
    } else {  // reseed, compress.cpp:195-217
      for (int64_t j = 0; j < m; ++j) {
        if (!members[static_cast<size_t>(j)].empty()) continue;
        int64_t far = -1;
        double far_d = -1.0;
        for (int64_t i = 0; i < n; ++i) {
          const int32_t owner = phi_h[static_cast<size_t>(i)];
          if (members[static_cast<size_t>(owner)].size() <= 1) continue;
          if (min_dist[static_cast<size_t>(i)] > far_d) {
            far_d = min_dist[static_cast<size_t>(i)];
            far = i;
          }
        }
        if (far < 0) continue;
        const int32_t owner = phi_h[static_cast<size_t>(far)];
        auto& own = members[static_cast<size_t>(owner)];
        own.erase(std::find(own.begin(), own.end(), static_cast<int32_t>(far)));
        members[static_cast<size_t>(j)].push_back(static_cast<int32_t>(far));
        phi_h[static_cast<size_t>(far)] = static_cast<int32_t>(j);
        min_dist[static_cast<size_t>(far)] = 0.0;
      }
    }
    h2d(d_phi.get(), phi_h, s);
    if (prune) {
      // the update below is a deterministic function of each cluster's
      // (ascending) member list: unchanged members -> bitwise unchanged centroid
      const int64_t mc = db.m;
      std::vector<uint8_t> chg(static_cast<size_t>(mc), 1);
      if (iter > 0 && mc == m_before && static_cast<int64_t>(prev_members.size()) == mc)
        for (int64_t j = 0; j < mc; ++j)
          chg[static_cast<size_t>(j)] = members[static_cast<size_t>(j)] != prev_members[static_cast<size_t>(j)];
      d_chg.alloc(static_cast<size_t>(std::max<int64_t>(mc, 1)));
      h2d(d_chg.get(), chg, s);
      chg_h = chg;
      prev_members = members;
    }

    if (trace) {
      const double t = tnow();
      tr[1] += t - tmark;
      tmark = t;
    }
    // representative update (compress.cpp:219-261); failures re-raised as
    // singular_matrix "cluster j: ..." for the lowest failing j.
    const int64_t mc = db.m;
    if (variant == Variant::VarMin) {
      ensure_patch_factors(sub, n, ps, pf, work, s);
      std::vector<int32_t> best_c(static_cast<size_t>(mc), -1);
      for (int64_t j = 0; j < mc; ++j) {
        const auto& mem = members[static_cast<size_t>(j)];
        for (int32_t c : mem)
          if (pf.status[static_cast<size_t>(c)] != 0)
            fail(Errc::singular_matrix, "cluster " + std::to_string(j) + ": patch " + std::to_string(c) + ": " +
                                            singular_msg(pf.status[static_cast<size_t>(c)], pf.best[static_cast<size_t>(c)]));
        if (mem.empty()) fail(Errc::singular_matrix, "cluster " + std::to_string(j) + ": empty cluster");
      }
      // all (k, c) pairs per cluster, in chunks
      const int64_t chunk_pairs = int64_t{1} << 22;
      std::vector<int32_t> pa, fb;
      for (int64_t j = 0; j < mc; ++j) {
        const auto& mem = members[static_cast<size_t>(j)];
        const int64_t cs = static_cast<int64_t>(mem.size());
        double best_var = std::numeric_limits<double>::infinity();
        int32_t bc = -1;
        // candidates processed in groups so each launch has <= chunk_pairs pairs
        const int64_t cand_per = std::max<int64_t>(1, chunk_pairs / std::max<int64_t>(cs, 1));
        for (int64_t c0 = 0; c0 < cs; c0 += cand_per) {
          const int64_t cn = std::min(cand_per, cs - c0);
          pa.resize(static_cast<size_t>(cn * cs));
          fb.resize(static_cast<size_t>(cn * cs));
          for (int64_t ci = 0; ci < cn; ++ci)
            for (int64_t kk = 0; kk < cs; ++kk) {
              pa[static_cast<size_t>(ci * cs + kk)] = mem[static_cast<size_t>(kk)];
              fb[static_cast<size_t>(ci * cs + kk)] = mem[static_cast<size_t>(c0 + ci)];
            }
          Scratch<int32_t> dpa(pa.size(), s), dfb(fb.size(), s);
          Scratch<double> dd(pa.size(), s);
          h2d(dpa.get(), pa, s);
          h2d(dfb.get(), fb, s);
          k::spectral_list(static_cast<int64_t>(pa.size()), dpa.get(), dfb.get(), ps, sub, pf.lu.get(), pf.piv.get(),
                           dd.get(), iters.get(), s);
          PDB_LAUNCH_CHECK();
          work.pair_evals += static_cast<int64_t>(pa.size());
          std::vector<double> dh = d2h(dd.get(), pa.size(), s);
          for (int64_t ci = 0; ci < cn; ++ci) {
            double var = 0.0;
            for (int64_t kk = 0; kk < cs; ++kk) {
              const double dv = dh[static_cast<size_t>(ci * cs + kk)];
              var += dv * dv;
            }
            if (var < best_var) {
              best_var = var;
              bc = mem[static_cast<size_t>(c0 + ci)];
            }
          }
        }
        best_c[static_cast<size_t>(j)] = bc;
      }
      Scratch<int32_t> ids(static_cast<size_t>(mc), s);
      h2d(ids.get(), best_c, s);
      k::gather_mats(mc, ids.get(), len, sub, db.reps.get(), s);
      k::gather_mats(mc, ids.get(), len, pf.lu.get(), db.lu.get(), s);
      k::gather_i32(mc, ids.get(), ps, pf.piv.get(), db.piv.get(), s);
      for (int64_t j = 0; j < mc; ++j) db.has_factor[static_cast<size_t>(j)] = 1;
    } else {
      for (int64_t j = 0; j < mc; ++j)
        if (members[static_cast<size_t>(j)].empty())
          fail(Errc::singular_matrix, "cluster " + std::to_string(j) + ": entrywise_mean of an empty cluster");
      std::vector<int32_t> mem_ptr(static_cast<size_t>(mc + 1), 0), mem;
      mem.reserve(static_cast<size_t>(n));
      for (int64_t j = 0; j < mc; ++j) {
        mem.insert(mem.end(), members[static_cast<size_t>(j)].begin(), members[static_cast<size_t>(j)].end());
        mem_ptr[static_cast<size_t>(j + 1)] = static_cast<int32_t>(mem.size());
      }
      Scratch<int32_t> dptr(mem_ptr.size(), s), dmem(std::max<size_t>(mem.size(), 1), s);
      h2d(dptr.get(), mem_ptr, s);
      h2d(dmem.get(), mem, s);
      k::cluster_mean(mc, static_cast<int>(len), dptr.get(), dmem.get(), sub, db.reps.get(), s);
      PDB_LAUNCH_CHECK();
      if (variant == Variant::Spectral) {
        std::string msg;
        const int64_t bad = lu_many(mc, ps, db.reps.get(), nullptr, db.lu.get(), db.piv.get(), msg, work, s);
        if (bad >= 0) fail(Errc::singular_matrix, "cluster " + std::to_string(bad) + ": " + msg);
        for (int64_t j = 0; j < mc; ++j) db.has_factor[static_cast<size_t>(j)] = 1;
      } else {
        for (int64_t j = 0; j < mc; ++j) db.has_factor[static_cast<size_t>(j)] = 0;
      }
      sync(s);
    }
  }
  if (trace)
    fprintf(stderr, "[kmeans] n=%lld m=%lld assign %.1f ms, host update %.1f ms, means+LU %.1f ms\n",
            static_cast<long long>(n), static_cast<long long>(db.m), tr[0] * 1e3, tr[1] * 1e3,
            (tr[2] + tnow() - tmark) * 1e3);
  if (sharded)  // every rank reports the whole job's power iterations
    PDB_NCCL_DB(ncclAllReduce(iters.get(), iters.get(), 1, ncclUint64, ncclSum, comm->comm, s));
  unsigned long long it_h = 0;
  PDB_CUDA(cudaMemcpyAsync(&it_h, iters.get(), sizeof(it_h), cudaMemcpyDeviceToHost, s));
  sync(s);
  work.power_iters += static_cast<int64_t>(it_h);
}

// finalize_factors (compress.cpp:266-278).
void finalize_factors(KDb& db, BuildWork& work, cudaStream_t s) {
  std::vector<int32_t> need;
  for (int64_t j = 0; j < db.m; ++j)
    if (!db.has_factor[static_cast<size_t>(j)]) need.push_back(static_cast<int32_t>(j));
  if (need.empty()) return;
  const int64_t cnt = static_cast<int64_t>(need.size());
  Scratch<int32_t> ids(need.size(), s);
  h2d(ids.get(), need, s);
  Scratch<double> lu(static_cast<size_t>(cnt * db.len), s);
  Scratch<int32_t> piv(static_cast<size_t>(cnt * db.ps), s);
  std::string msg;
  const int64_t bad = lu_many(cnt, db.ps, db.reps.get(), ids.get(), lu.get(), piv.get(), msg, work, s);
  if (bad >= 0) fail(Errc::singular_matrix, "cluster " + std::to_string(need[static_cast<size_t>(bad)]) + ": " + msg);
  // scatter back (need is ascending; contiguous in the common all-entries case)
  for (int64_t t = 0; t < cnt; ++t) {
    const int64_t j = need[static_cast<size_t>(t)];
    PDB_CUDA(cudaMemcpyAsync(db.lu.get() + j * db.len, lu.get() + t * db.len, db.len * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
    PDB_CUDA(cudaMemcpyAsync(db.piv.get() + j * db.ps, piv.get() + t * db.ps, db.ps * sizeof(int32_t),
                             cudaMemcpyDeviceToDevice, s));
    db.has_factor[static_cast<size_t>(j)] = 1;
  }
  sync(s);
}

// kmeans (compress.cpp:294-324) on a contiguous group of n patch matrices.
void kmeans_group(const double* sub, int64_t n, int ps, int64_t m_p, Variant variant, uint64_t seed, int max_iters,
                  KDb& db, std::vector<int32_t>& phi_h, BuildWork& work, cudaStream_t s,
                  const ShardComm* comm = nullptr) {
  require(n >= 1, Errc::invalid_argument, "kmeans needs at least one patch");
  require(m_p >= 1 && m_p <= n, Errc::invalid_argument, "kmeans requires 1 <= m_p <= n_p");
  const int64_t len = static_cast<int64_t>(ps) * ps;
  std::mt19937_64 rng(seed);
  std::vector<int32_t> perm(static_cast<size_t>(n));
  std::iota(perm.begin(), perm.end(), 0);
  for (int64_t i = 0; i < m_p; ++i) {
    const int64_t j = i + static_cast<int64_t>(rng() % static_cast<uint64_t>(n - i));
    std::swap(perm[static_cast<size_t>(i)], perm[static_cast<size_t>(j)]);
  }
  db.ps = ps;
  db.len = len;
  db.m = m_p;
  db.reps.alloc(static_cast<size_t>(m_p * len));
  db.lu.alloc(static_cast<size_t>(m_p * len));
  db.piv.alloc(static_cast<size_t>(m_p * ps));
  db.has_factor.assign(static_cast<size_t>(m_p), 0);
  std::vector<int32_t> picks(perm.begin(), perm.begin() + m_p);
  Scratch<int32_t> ids(picks.size(), s);
  h2d(ids.get(), picks, s);
  k::gather_mats(m_p, ids.get(), len, sub, db.reps.get(), s);
  if (variant != Variant::Entrywise) {
    std::string msg;
    const int64_t bad = lu_many(m_p, ps, db.reps.get(), nullptr, db.lu.get(), db.piv.get(), msg, work, s);
    if (bad >= 0) fail(Errc::singular_matrix, "patch " + std::to_string(picks[static_cast<size_t>(bad)]) + ": " + msg);
    std::fill(db.has_factor.begin(), db.has_factor.end(), 1);
  }
  PatchFactors pf;
  {
    TraceScope tk("kmeans_loop", s);
    kmeans_loop(sub, n, db, variant, max_iters, Empty::Reseed, phi_h, pf, work, s,
                variant == Variant::VarMin ? nullptr : comm);
  }
  TraceScope tf("finalize_factors", s);
  finalize_factors(db, work, s);
}

}  // namespace

// split_budget (compress.cpp:336-392).
std::vector<int64_t> split_budget(int64_t m_p, const std::vector<int64_t>& sizes) {
  const int64_t parts = static_cast<int64_t>(sizes.size());
  require(parts >= 1, Errc::invalid_argument, "no partitions");
  int64_t total = 0;
  for (int64_t v : sizes) total += v;
  require(m_p >= parts, Errc::budget_too_small, "database budget smaller than the number of boundary partitions");
  require(m_p <= total, Errc::invalid_argument, "database budget larger than the number of patches");
  std::vector<int64_t> alloc(static_cast<size_t>(parts), 0);
  std::vector<double> rem(static_cast<size_t>(parts), 0.0);
  int64_t assigned = 0;
  for (int64_t p = 0; p < parts; ++p) {
    const double quota = static_cast<double>(m_p) * static_cast<double>(sizes[static_cast<size_t>(p)]) / static_cast<double>(total);
    alloc[static_cast<size_t>(p)] = static_cast<int64_t>(std::floor(quota));
    rem[static_cast<size_t>(p)] = quota - std::floor(quota);
    assigned += alloc[static_cast<size_t>(p)];
  }
  std::vector<int64_t> order(static_cast<size_t>(parts));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t x, int64_t y) { return rem[static_cast<size_t>(x)] > rem[static_cast<size_t>(y)]; });
  for (int64_t k = 0; assigned < m_p; ++k) {
    ++alloc[static_cast<size_t>(order[static_cast<size_t>(k % parts)])];
    ++assigned;
  }
  auto take_from_largest = [&](int64_t needy) {
    int64_t donor = -1;
    for (int64_t p = 0; p < parts; ++p)
      if (alloc[static_cast<size_t>(p)] >= 2 && (donor < 0 || alloc[static_cast<size_t>(p)] > alloc[static_cast<size_t>(donor)]))
        donor = p;
    require(donor >= 0, Errc::budget_too_small, "cannot satisfy one cluster per partition");
    --alloc[static_cast<size_t>(donor)];
    ++alloc[static_cast<size_t>(needy)];
  };
  for (int64_t p = 0; p < parts; ++p)
    while (alloc[static_cast<size_t>(p)] == 0) take_from_largest(p);
  for (int64_t p = 0; p < parts; ++p)
    while (alloc[static_cast<size_t>(p)] > sizes[static_cast<size_t>(p)]) {
      --alloc[static_cast<size_t>(p)];
      int64_t recv = -1;
      double best_rem = -1.0;
      for (int64_t q = 0; q < parts; ++q)
        if (alloc[static_cast<size_t>(q)] < sizes[static_cast<size_t>(q)] && rem[static_cast<size_t>(q)] > best_rem) {
          best_rem = rem[static_cast<size_t>(q)];
          recv = q;
        }
      require(recv >= 0, Errc::invalid_argument, "budget exceeds total patch count");
      ++alloc[static_cast<size_t>(recv)];
    }
  return alloc;
}

namespace {

// boundary_partition (patch.cpp:113-126): groups in first-occurrence order.
void boundary_partition(const DevBuf<double>& mats, int64_t np, int ps, std::vector<std::vector<int32_t>>& groups,
                        std::vector<std::vector<uint8_t>>& patterns, cudaStream_t s) {
  require(np >= 1, Errc::invalid_argument, "boundary_partition needs at least one patch");
  const int words = (ps + 63) / 64;
  Scratch<unsigned long long> masks(static_cast<size_t>(np * words), s);
  k::boundary_masks(np, ps, mats.get(), words, masks.get(), s);
  PDB_LAUNCH_CHECK();
  std::vector<unsigned long long> mh = d2h(masks.get(), static_cast<size_t>(np * words), s);
  std::map<std::vector<unsigned long long>, size_t> index;
  std::vector<unsigned long long> key(static_cast<size_t>(words));
  for (int64_t k = 0; k < np; ++k) {
    std::copy(mh.begin() + k * words, mh.begin() + (k + 1) * words, key.begin());
    auto it = index.find(key);
    if (it == index.end()) {
      it = index.emplace(key, groups.size()).first;
      groups.emplace_back();
      std::vector<uint8_t> pat(static_cast<size_t>(ps));
      for (int i = 0; i < ps; ++i) pat[static_cast<size_t>(i)] = (key[static_cast<size_t>(i / 64)] >> (i % 64)) & 1ull;
      patterns.push_back(std::move(pat));
    }
    groups[it->second].push_back(static_cast<int32_t>(k));
  }
}

// partitioned_build (compress.cpp:394-421).
void partitioned_build(const DevBuf<double>& mats, int64_t np, int ps, int64_t m_p, Variant variant, uint64_t seed,
                       int max_iters, pdb_database_s& out, cudaStream_t s, const ShardComm* comm = nullptr) {
  const int64_t len = static_cast<int64_t>(ps) * ps;
  std::vector<std::vector<int32_t>> groups;
  std::vector<std::vector<uint8_t>> patterns;
  {
    TraceScope tb("boundary_partition", s);
    boundary_partition(mats, np, ps, groups, patterns, s);
  }
  std::vector<int64_t> sizes;
  for (const auto& g : groups) sizes.push_back(static_cast<int64_t>(g.size()));
  const std::vector<int64_t> alloc = split_budget(m_p, sizes);
  std::vector<KDb> parts(groups.size());
  std::vector<int32_t> phi(static_cast<size_t>(np), -1);
  int64_t total = 0;
  DevBuf<double> sub;
  for (size_t g = 0; g < groups.size(); ++g) {
    const int64_t cnt = static_cast<int64_t>(groups[g].size());
    TraceScope tg("partition (gather + kmeans_group)", s);
    sub.alloc(static_cast<size_t>(cnt * len));
    Scratch<int32_t> ids(static_cast<size_t>(cnt), s);
    h2d(ids.get(), groups[g], s);
    k::gather_mats(cnt, ids.get(), len, mats.get(), sub.get(), s);
    std::vector<int32_t> lphi;
    kmeans_group(sub.get(), cnt, ps, alloc[g], variant, seed + static_cast<uint64_t>(g), max_iters, parts[g], lphi,
                 out.work, s, comm);
    for (int64_t q = 0; q < cnt; ++q)
      phi[static_cast<size_t>(groups[g][static_cast<size_t>(q)])] = static_cast<int32_t>(total + lphi[static_cast<size_t>(q)]);
    total += parts[g].m;
  }
  out.m = total;
  out.np = np;
  out.ps = ps;
  out.method = variant_name(variant) + "-partitioned";
  out.reps.alloc(static_cast<size_t>(total * len));
  out.lu.alloc(static_cast<size_t>(total * len));
  out.piv.alloc(static_cast<size_t>(total * ps));
  int64_t off = 0;
  out.entry_patterns.clear();
  for (size_t g = 0; g < groups.size(); ++g) {
    const int64_t m = parts[g].m;
    PDB_CUDA(cudaMemcpyAsync(out.reps.get() + off * len, parts[g].reps.get(), m * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
    PDB_CUDA(cudaMemcpyAsync(out.lu.get() + off * len, parts[g].lu.get(), m * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
    PDB_CUDA(cudaMemcpyAsync(out.piv.get() + off * ps, parts[g].piv.get(), m * ps * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    for (int64_t j = 0; j < m; ++j) out.entry_patterns.push_back(patterns[g]);
    off += m;
  }
  out.phi.alloc(static_cast<size_t>(np));
  h2d(out.phi.get(), phi, s);
  sync(s);
}

// bootstrapped (compress.cpp:326-334): greedy (spectral, first match), then
// Lloyd iterations with pruning, then factors for any entry without one.
void bootstrap_build(const DevBuf<double>& mats, int64_t np, int ps, double eps, int max_iters, pdb_database_s& out,
                     cudaStream_t s) {
  pdb_database_s g;
  greedy_build(mats, np, ps, eps, true, false, -1, g, s);
  out.work = g.work;
  KDb db;
  db.ps = ps;
  db.len = static_cast<int64_t>(ps) * ps;
  db.m = g.m;
  db.reps = std::move(g.reps);
  db.lu = std::move(g.lu);
  db.piv = std::move(g.piv);
  db.has_factor.assign(static_cast<size_t>(db.m), 1);
  std::vector<int32_t> phi_h;
  PatchFactors pf;
  kmeans_loop(mats.get(), np, db, Variant::VarMin, max_iters, Empty::Prune, phi_h, pf, out.work, s);
  finalize_factors(db, out.work, s);
  out.m = db.m;
  out.np = np;
  out.ps = ps;
  out.eps = eps;
  out.method = "bootstrap-kmeans-varmin";
  out.reps = std::move(db.reps);
  out.lu = std::move(db.lu);
  out.piv = std::move(db.piv);
  out.phi.alloc(static_cast<size_t>(np));
  h2d(out.phi.get(), phi_h, s);
  sync(s);
}

}  // namespace

bool build_database_from_mats(const DevBuf<double>& mats, int64_t np, int64_t ps, const BuildParams& p,
                              pdb_database_s& out, cudaStream_t s) {
  const int ips = static_cast<int>(ps);
  switch (p.method) {
    case PDB_METHOD_EXACT: exact_build(mats, np, ips, out, s); return true;
    case PDB_METHOD_GREEDY_SPECTRAL:
      return greedy_build(mats, np, ips, p.eps, true, p.best_match, p.abort_above, out, s, p.comm);
    case PDB_METHOD_GREEDY_L1:
      return greedy_build(mats, np, ips, p.eps, false, p.best_match, p.abort_above, out, s, p.comm);
    case PDB_METHOD_KMEANS_ENTRYWISE:
      partitioned_build(mats, np, ips, p.db_size, Variant::Entrywise, p.seed, p.max_iters, out, s, p.comm);
      return true;
    case PDB_METHOD_KMEANS_SPECTRAL:
      partitioned_build(mats, np, ips, p.db_size, Variant::Spectral, p.seed, p.max_iters, out, s, p.comm);
      return true;
    case PDB_METHOD_KMEANS_VARMIN:
      partitioned_build(mats, np, ips, p.db_size, Variant::VarMin, p.seed, p.max_iters, out, s);
      return true;
    case PDB_METHOD_BOOTSTRAP: bootstrap_build(mats, np, ips, p.eps, p.max_iters, out, s); return true;
    default: fail(Errc::invalid_argument, "unknown compression method");
  }
}

// evaluate_objective (compress.cpp:423-440): beta |B| + sum_k d(A_k, B_phi(k))^2
// with the bit-exact spectral distance of every (patch, its entry) pair on the
// device and the terms summed in ascending k on the host, as the reference.
double database_objective(const DeviceCsr& a, const pdb_patchset_s& ps, const pdb_database_s& db, double beta,
                          cudaStream_t s) {
  require_device();
  require(beta > 0.0, Errc::invalid_argument, "beta must be positive");
  require(db.np == ps.np, Errc::dimension_mismatch, "database does not match the patch list");
  require(db.ps == ps.ps, Errc::dimension_mismatch, "spectral_distance dimension mismatch");
  const int64_t n = ps.np;
  DevBuf<double> mats;
  extract_patches(a, ps, mats, s);
  std::vector<int32_t> pa(static_cast<size_t>(n));
  std::iota(pa.begin(), pa.end(), 0);
  Scratch<int32_t> dpa(static_cast<size_t>(std::max<int64_t>(n, 1)), s);
  Scratch<double> d(static_cast<size_t>(std::max<int64_t>(n, 1)), s);
  Scratch<unsigned long long> iters(1, s);
  h2d(dpa.get(), pa, s);
  k::spectral_list(n, dpa.get(), db.phi.get(), static_cast<int>(ps.ps), mats.get(), db.lu.get(), db.piv.get(), d.get(),
                   iters.get(), s);
  PDB_LAUNCH_CHECK();
  const std::vector<double> dh = d2h(d.get(), static_cast<size_t>(n), s);
  double sum = 0.0;
  for (double v : dh) sum += v * v;
  return beta * static_cast<double>(db.m) + sum;
}

// compressibility_curve (compress.cpp:442-456): greedy_tolerance (first match)
// at every tolerance of an ascending grid; the patches are extracted once.
void compressibility_curve(const DeviceCsr& a, const pdb_patchset_s& ps, bool spectral, const double* grid,
                           int64_t count, int64_t* sizes, double* ratios, cudaStream_t s) {
  require_device();
  require(count > 0, Errc::invalid_argument, "empty tolerance grid");
  for (int64_t k = 0; k < count; ++k) {
    require(grid[k] > 0.0, Errc::invalid_argument, "tolerances must be positive");
    if (k > 0) require(grid[k] > grid[k - 1], Errc::invalid_argument, "tolerance grid must be ascending");
  }
  DevBuf<double> mats;
  extract_patches(a, ps, mats, s);
  const double n_p = static_cast<double>(ps.np);
  for (int64_t k = 0; k < count; ++k) {
    pdb_database_s db;
    greedy_build(mats, ps.np, static_cast<int>(ps.ps), grid[k], spectral, false, -1, db, s);
    sizes[k] = db.m;
    ratios[k] = (n_p - static_cast<double>(db.m)) / n_p;
  }
}

bool build_database(const DeviceCsr& a, const pdb_patchset_s& ps, const BuildParams& p, pdb_database_s& out,
                    cudaStream_t s) {
  require_device();
  TraceScope tr("build_database", s);
  DevBuf<double> mats;
  {
    TraceScope te("extract_patches", s);
    extract_patches(a, ps, mats, s);
  }
  return build_database_from_mats(mats, ps.np, ps.ps, p, out, s);
}

// greedy_bisect_to_size (experiments.cpp:168-204).
double bisect_database(const DeviceCsr& a, const pdb_patchset_s& ps, const BuildParams& p, int64_t target_lo,
                       int64_t target_hi, pdb_database_s& out, cudaStream_t s) {
  require(p.method == PDB_METHOD_GREEDY_L1 || p.method == PDB_METHOD_GREEDY_SPECTRAL, Errc::invalid_argument,
          "size bisection needs a greedy method");
  require_device();
  DevBuf<double> mats;
  extract_patches(a, ps, mats, s);
  const int64_t n_p = ps.np;
  target_lo = std::max<int64_t>(1, std::min(target_lo, n_p));
  target_hi = std::max(target_lo, std::min(target_hi, n_p));
  double lo = 1e-14, hi = 1e10;
  int64_t best_gap = std::numeric_limits<int64_t>::max();
  double best_eps = 0.0;
  BuildWork total;
  for (int it = 0; it < 60; ++it) {
    const double eps = std::sqrt(lo * hi);
    pdb_database_s db;
    const bool ok = greedy_build(mats, n_p, static_cast<int>(ps.ps), eps, p.method == PDB_METHOD_GREEDY_SPECTRAL,
                                 p.best_match, target_hi, db, s, p.comm);
    total.pair_evals += db.work.pair_evals;
    total.power_iters += db.work.power_iters;
    total.lu_count += db.work.lu_count;
    if (!ok) {
      lo = eps;
      continue;
    }
    const int64_t size = db.m;
    const int64_t gap = size < target_lo ? target_lo - size : (size > target_hi ? size - target_hi : 0);
    if (gap < best_gap) {
      best_gap = gap;
      out = std::move(db);
      best_eps = eps;
      if (gap == 0) break;
    }
    if (size < target_lo) hi = eps;
    else lo = eps;
  }
  require(best_gap != std::numeric_limits<int64_t>::max(), Errc::invalid_argument, "greedy bisection found no database");
  out.work = total;
  return best_eps;
}

// export_database (compress.cpp:458-485): raw representatives + JSON index.
void export_database(const pdb_database_s& db, const std::string& json_path, const std::string& bin_path,
                     cudaStream_t s) {
  const std::vector<double> reps = db.reps.to_host(s);
  std::ofstream bin(bin_path, std::ios::binary);
  if (!bin) fail(Errc::io_error, "cannot open '" + bin_path + "' for writing");
  bin.write(reinterpret_cast<const char*>(reps.data()),
            static_cast<std::streamsize>(static_cast<size_t>(db.m * db.ps * db.ps) * sizeof(double)));
  if (!bin) fail(Errc::io_error, "error while writing '" + bin_path + "'");
  const std::vector<int32_t> phi = db.phi.to_host(s);
  std::ofstream out(json_path);
  if (!out) fail(Errc::io_error, "cannot open '" + json_path + "' for writing");
  out << "{\n  \"method\": \"" << db.method << "\",\n  \"eps\": " << db.eps << ",\n  \"m_p\": " << db.m
      << ",\n  \"n_p\": " << db.np << ",\n  \"entries\": [";
  for (int64_t j = 0; j < db.m; ++j) {
    out << (j == 0 ? "\n    " : ",\n    ");
    out << "{\"rows\": " << db.ps << ", \"cols\": " << db.ps;
    if (!db.entry_patterns.empty()) {
      out << ", \"partition\": \"";
      for (uint8_t b : db.entry_patterns[static_cast<size_t>(j)]) out << (b ? '1' : '0');
      out << "\"";
    }
    out << "}";
  }
  out << "\n  ],\n  \"phi\": [";
  for (int64_t k = 0; k < db.np; ++k) out << (k == 0 ? "" : ", ") << phi[static_cast<size_t>(k)];
  out << "]\n}\n";
  if (!out) fail(Errc::io_error, "error while writing '" + json_path + "'");
}


// Import of an export_database pair (setup reuse across solves):
// the JSON's phi, method, eps and entry partitions plus the binary
// representatives; the factors are recomputed on the device by the same
// bit-exact LU, so the imported database equals the exported one bit for
// bit.  The files are parsed before any device work (errors: PDB_ERR_IO /
// PDB_ERR_PARSE).
namespace {

struct JsonCursor {
  const std::string& t;
  const std::string& name;
  size_t i = 0;
  [[noreturn]] void bad(const std::string& what) const {
    fail(Errc::parse_error, name + ": " + what + " at byte " + std::to_string(i));
  }
  void skip() {
    while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
  }
  bool key(const std::string& k) {  // moves to the value of "k"
    const size_t at = t.find("\"" + k + "\"", i);
    if (at == std::string::npos) return false;
    i = at + k.size() + 2;
    skip();
    if (i >= t.size() || t[i] != ':') bad("expected ':' after \"" + k + "\"");
    ++i;
    skip();
    return true;
  }
  std::string str() {
    if (i >= t.size() || t[i] != '"') bad("expected a string");
    const size_t e = t.find('"', i + 1);
    if (e == std::string::npos) bad("unterminated string");
    std::string v = t.substr(i + 1, e - i - 1);
    i = e + 1;
    return v;
  }
  double num() {
    const char* b = t.c_str() + i;
    char* e = nullptr;
    const double v = std::strtod(b, &e);
    if (e == b) bad("expected a number");
    i += static_cast<size_t>(e - b);
    return v;
  }
};

}  // namespace

void import_database(const std::string& json_path, const std::string& bin_path, pdb_database_s& db, cudaStream_t s) {
  std::ifstream jf(json_path);
  if (!jf) fail(Errc::io_error, "cannot open '" + json_path + "' for reading");
  const std::string text((std::istreambuf_iterator<char>(jf)), std::istreambuf_iterator<char>());
  JsonCursor c{text, json_path};
  if (!c.key("method")) c.bad("missing \"method\"");
  const std::string method = c.str();
  c.i = 0;
  if (!c.key("eps")) c.bad("missing \"eps\"");
  const double eps = c.num();
  c.i = 0;
  if (!c.key("m_p")) c.bad("missing \"m_p\"");
  const double mp = c.num();
  c.i = 0;
  if (!c.key("n_p")) c.bad("missing \"n_p\"");
  const double np = c.num();
  if (!(mp >= 1 && np >= mp && mp == std::floor(mp) && np == std::floor(np))) c.bad("invalid m_p / n_p");
  const int64_t m = static_cast<int64_t>(mp), n = static_cast<int64_t>(np);
  c.i = 0;
  if (!c.key("entries")) c.bad("missing \"entries\"");
  int64_t ps = -1;
  std::vector<std::vector<uint8_t>> patterns;
  for (int64_t j = 0; j < m; ++j) {
    const size_t open = text.find('{', c.i);
    const size_t close = text.find('}', open == std::string::npos ? c.i : open);
    if (open == std::string::npos || close == std::string::npos) c.bad("entry list shorter than m_p");
    c.i = open;
    if (!c.key("rows") || c.i > close) c.bad("entry without \"rows\"");
    const double rows = c.num();
    if (!(rows >= 1 && rows == std::floor(rows))) c.bad("invalid entry size");
    if (ps < 0) ps = static_cast<int64_t>(rows);
    if (static_cast<int64_t>(rows) != ps) c.bad("entries of different sizes");
    const size_t part = text.find("\"partition\"", open);
    if (part != std::string::npos && part < close) {
      c.i = part;
      c.key("partition");
      const std::string bits = c.str();
      if (static_cast<int64_t>(bits.size()) != ps) c.bad("partition pattern length differs from the entry size");
      std::vector<uint8_t> pat(bits.size());
      for (size_t q = 0; q < bits.size(); ++q) pat[q] = bits[q] == '1';
      patterns.push_back(std::move(pat));
    }
    c.i = close + 1;
  }
  if (!patterns.empty() && static_cast<int64_t>(patterns.size()) != m) c.bad("partition patterns on some entries only");
  if (!c.key("phi")) c.bad("missing \"phi\"");
  if (c.i >= text.size() || text[c.i] != '[') c.bad("expected '['");
  ++c.i;
  std::vector<int32_t> phi(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) {
    c.skip();
    if (k > 0) {
      if (c.i >= text.size() || text[c.i] != ',') c.bad("expected ','");
      ++c.i;
      c.skip();
    }
    const double v = c.num();
    if (!(v >= 0 && v < static_cast<double>(m) && v == std::floor(v))) c.bad("phi entry outside [0, m_p)");
    phi[static_cast<size_t>(k)] = static_cast<int32_t>(v);
  }
  const int64_t len = ps * ps;
  std::vector<double> reps(static_cast<size_t>(m * len));
  std::ifstream bf(bin_path, std::ios::binary);
  if (!bf) fail(Errc::io_error, "cannot open '" + bin_path + "' for reading");
  bf.read(reinterpret_cast<char*>(reps.data()), static_cast<std::streamsize>(reps.size() * sizeof(double)));
  if (bf.gcount() != static_cast<std::streamsize>(reps.size() * sizeof(double)))
    fail(Errc::parse_error, bin_path + ": expected " + std::to_string(m * len) + " doubles");
  require_device();
  db.m = m;
  db.np = n;
  db.ps = ps;
  db.eps = eps;
  db.method = method;
  db.entry_patterns = std::move(patterns);
  db.reps.alloc(reps.size());
  db.reps.upload(reps.data(), reps.size(), s);
  db.lu.alloc(reps.size());
  db.piv.alloc(static_cast<size_t>(m * ps));
  std::string msg;
  const int64_t bad = lu_many(m, static_cast<int>(ps), db.reps.get(), nullptr, db.lu.get(), db.piv.get(), msg,
                              db.work, s);
  if (bad >= 0) fail(Errc::singular_matrix, "entry " + std::to_string(bad) + ": " + msg);
  db.phi.alloc(phi.size());
  db.phi.upload(phi.data(), phi.size(), s);
  sync(s);
}

}  // namespace pdb
