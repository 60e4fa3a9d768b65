// Multi-GPU relaxation sweep with rank-local data.
//
// Every rank holds only its own rows: the rows of the DoFs of its patches
// (a slab of cells from pdb_problem_generate_slab, or any row block), with
// global column ids.  Nothing global is ever materialised:
//
// setup (per rank, exchanges with the ranks whose DoF ranges overlap)
//   local index space L = rows + their columns (sorted global ids), local CSR
//   patches detected on the local rows (detect_patches, patch.cpp:37-90): a
//     slab's candidate rows and their footprints are all local
//   global patch offset k0 = patches of lower ranks (patches are ordered by
//     front, so the slabs' patch ranges are consecutive)
//   cover counts of shared DoFs summed with the neighbours -> the global
//     weights 1 / count (compute_weights, patch.cpp:12-20)
//   ownership: a DoF is finished by the HIGHEST rank whose patches touch it;
//     the reference's scatter adds contributions in ascending patch order
//     (precond.cpp:81-86), so a lower rank's partial sum is a prefix of the
//     owner's sum: the lower rank sends it, the owner continues from it
//   x halo: every local DoF the rank does not own is requested from the
//     ranks whose ranges contain it; exactly one must own it
//   factors: exact -> extract + LU of the local patches only; compressed ->
//     the small replicated database and the rank's phi slice
//
// sweep (per rank), the interface first so the exchange hides behind the
// interior work:
//   r = b - A x on the local rows                               [main]
//   patches touching DoFs finished by the upper neighbour (the top cell
//   layer: a suffix of the local patches) -> their partial sums  [main]
//   -> ncclSend up / ncclRecv from below                         [comm stream]
//   the other patches; owned DoFs without a lower contribution   [main]
//   owned DoFs with a lower contribution, from the received sum  [main]
//   x of owned DoFs the neighbours read -> x halo exchange       [comm stream]
// On one GPU an emulated group runs W ranks' phases in order and moves the
// exchanged values with device copies: the same code, bitwise the single-GPU
// pdb_relax (tests/test_slab.py).
#include <nccl.h>

#include <atomic>
#include <optional>

#include <algorithm>
#include <mutex>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <random>
#include <thread>

#include "host.hpp"
#include "kernels.hpp"

#define PDB_NCCL_S(call)                                                                            \
  do {                                                                                              \
    ncclResult_t r_ = (call);                                                                       \
    if (r_ != ncclSuccess) ::pdb::fail(::pdb::Errc::internal, std::string("NCCL error in " #call ": ") + \
                                                             ncclGetErrorString(r_));               \
  } while (0)

namespace pdb {

namespace {

struct Seg {
  int peer;
  int64_t off, cnt;
};

int64_t seg_total(const std::vector<Seg>& v) { return v.empty() ? 0 : v.back().off + v.back().cnt; }

template <typename T>
void put(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  d.alloc(std::max<size_t>(h.size(), 1));
  if (!h.empty()) d.upload(h.data(), h.size(), s);
}

// contiguous patch range [k0, k1) of a local patch set as its own patch set
void sub_patchset(const pdb_patchset_s& ps, int64_t k0, int64_t k1, pdb_patchset_s& out, cudaStream_t s) {
  out.n = ps.n;
  out.np = k1 - k0;
  out.ps = ps.ps;
  out.patches.alloc(static_cast<size_t>(std::max<int64_t>(out.np * out.ps, 1)));
  if (out.np > 0)
    PDB_CUDA(cudaMemcpyAsync(out.patches.get(), ps.patches.get() + k0 * ps.ps, out.np * ps.ps * sizeof(int32_t),
                             cudaMemcpyDeviceToDevice, s));
  out.weights.alloc(static_cast<size_t>(std::max<int64_t>(ps.n, 1)));
  PDB_CUDA(cudaMemcpyAsync(out.weights.get(), ps.weights.get(), ps.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

}  // namespace

// One rank's state.
struct SlabRank {
  int rank = 0, nranks = 1;
  std::vector<int32_t> pt_host;  // setup only: the local patch lists on the host (released after phase 2)
  double upload_s = 0.0;  // matrix upload + residual structures (what pdb_matrix_from_csr does on one GPU)
  std::vector<int64_t> gid;  // local -> global DoF (ascending)
  int64_t nl = 0;
  std::vector<int32_t> rows;  // local ids of the rank's rows (its patch DoFs)
  DeviceCsr a;
  pdb_patchset_s ps;  // local patches, global weights
  int64_t np = 0, k0 = 0, kb = 0;  // local patches; global offset; start of the top-interface suffix
  pdb_precond_s pc_lo, pc_hi;      // patches [0, kb) and [kb, np)
  pdb_precond_s map;               // DoF -> (patch, slot) over all local patches
  DevBuf<double> omega_w;
  DevBuf<int32_t> own_plain, own_pin, up, pin, xs, xr;
  std::vector<Seg> up_seg, pin_seg, xs_seg, xr_seg;
  DevBuf<double> zup, zin, init, xsend, xrecv, r, sols;
  int64_t n_own = 0;
  std::vector<int32_t> phi;  // compressed: the rank's slice of phi
  // NCCL mode
  ncclComm_t comm = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev[4] = {};
  ~SlabRank() {
    if (comm) ncclCommDestroy(comm);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
  }
};

}  // namespace pdb

struct pdb_slab_s {
  std::vector<std::unique_ptr<pdb::SlabRank>> ranks;  // 1 (NCCL rank), or the emulated ranks (ascending)
  bool emulated = false;
  int64_t n_global = 0;
  std::vector<int64_t> k0_of, np_of;  // every rank's first global patch and patch count
  int64_t m = 0;                       // database entries (compressed)
  std::vector<int64_t> creators;       // global patch id of each entry (distributed greedy)
  std::vector<int> slot;  // emulated: rank -> index in `ranks`, -1 when absent
  int slot_of(int rank) const { return slot.empty() ? rank : slot[static_cast<size_t>(rank)]; }
};

namespace pdb {

namespace {

// ---- setup message passing: out[r][q] -> in[q][r] for the local ranks ----
using Mail = std::vector<std::vector<int64_t>>;  // [peer] -> payload

void deliver(pdb_slab_s& g, std::vector<Mail>& out, std::vector<Mail>& in, cudaStream_t s) {
  const int W = g.ranks[0]->nranks;
  in.assign(out.size(), Mail(static_cast<size_t>(W)));
  if (g.emulated) {  // messages to absent ranks are dropped, absent ranks send nothing
    for (size_t i = 0; i < g.ranks.size(); ++i)
      for (int q = 0; q < W; ++q) {
        const int j = g.slot_of(q);
        if (j >= 0) in[static_cast<size_t>(j)][static_cast<size_t>(g.ranks[i]->rank)] = out[i][static_cast<size_t>(q)];
      }
    return;
  }
  SlabRank& R = *g.ranks[0];
  if (W == 1) {
    in[0][0] = out[0][0];
    return;
  }
  const Mail& o = out[0];
  // sizes, then payloads (grouped point-to-point on device buffers)
  DevBuf<int64_t> ssz(static_cast<size_t>(W)), rsz(static_cast<size_t>(W));
  std::vector<int64_t> sz(static_cast<size_t>(W));
  for (int q = 0; q < W; ++q) sz[static_cast<size_t>(q)] = static_cast<int64_t>(o[static_cast<size_t>(q)].size());
  ssz.upload(sz.data(), sz.size(), s);
  PDB_NCCL_S(ncclGroupStart());
  for (int q = 0; q < W; ++q) {
    if (q == R.rank) continue;
    PDB_NCCL_S(ncclSend(ssz.get() + q, 1, ncclInt64, q, R.comm, s));
    PDB_NCCL_S(ncclRecv(rsz.get() + q, 1, ncclInt64, q, R.comm, s));
  }
  PDB_NCCL_S(ncclGroupEnd());
  std::vector<int64_t> rs = rsz.to_host(s);
  std::vector<int64_t> so(static_cast<size_t>(W + 1), 0), ro(static_cast<size_t>(W + 1), 0);
  for (int q = 0; q < W; ++q) {
    so[static_cast<size_t>(q) + 1] = so[static_cast<size_t>(q)] + (q == R.rank ? 0 : sz[static_cast<size_t>(q)]);
    ro[static_cast<size_t>(q) + 1] = ro[static_cast<size_t>(q)] + (q == R.rank ? 0 : rs[static_cast<size_t>(q)]);
  }
  std::vector<int64_t> flat(static_cast<size_t>(so[static_cast<size_t>(W)]));
  for (int q = 0; q < W; ++q)
    if (q != R.rank) std::copy(o[static_cast<size_t>(q)].begin(), o[static_cast<size_t>(q)].end(), flat.begin() + so[static_cast<size_t>(q)]);
  DevBuf<int64_t> sb(std::max<size_t>(flat.size(), 1)), rb(static_cast<size_t>(std::max<int64_t>(ro[static_cast<size_t>(W)], 1)));
  if (!flat.empty()) sb.upload(flat.data(), flat.size(), s);
  PDB_NCCL_S(ncclGroupStart());
  for (int q = 0; q < W; ++q) {
    if (q == R.rank) continue;
    if (sz[static_cast<size_t>(q)] > 0)
      PDB_NCCL_S(ncclSend(sb.get() + so[static_cast<size_t>(q)], static_cast<size_t>(sz[static_cast<size_t>(q)]), ncclInt64, q, R.comm, s));
    if (rs[static_cast<size_t>(q)] > 0)
      PDB_NCCL_S(ncclRecv(rb.get() + ro[static_cast<size_t>(q)], static_cast<size_t>(rs[static_cast<size_t>(q)]), ncclInt64, q, R.comm, s));
  }
  PDB_NCCL_S(ncclGroupEnd());
  std::vector<int64_t> all = rb.to_host(s);
  for (int q = 0; q < W; ++q)
    if (q != R.rank)
      in[0][static_cast<size_t>(q)].assign(all.begin() + ro[static_cast<size_t>(q)], all.begin() + ro[static_cast<size_t>(q) + 1]);
  in[0][static_cast<size_t>(R.rank)] = o[static_cast<size_t>(R.rank)];
}

std::vector<Seg> segments_of(const std::vector<int32_t>& peer) {
  std::vector<Seg> out;
  for (size_t i = 0; i < peer.size(); ++i) {
    if (out.empty() || out.back().peer != peer[i]) out.push_back({peer[i], static_cast<int64_t>(i), 0});
    ++out.back().cnt;
  }
  return out;
}

template <typename F>
void parallel_rows(int64_t n, F&& fn) {
  const int T = static_cast<int>(std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
  if (n < (1 << 16) || T == 1) {
    fn(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) pool.emplace_back([&, t] { fn(n * t / T, n * (t + 1) / T); });
  for (auto& th : pool) th.join();
}

// col[q] <- g2l[col[q] - gmin]: global column ids to the rank's local ids
__global__ void remap_cols_kernel(int64_t nnz, int64_t gmin, const int32_t* __restrict__ g2l, int32_t* col) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nnz) col[q] = g2l[col[q] - gmin];
}

// Phase A: local index space, local CSR, patches, touched set.
void local_structure(SlabRank& R, pdb_problem_s& prob, int64_t patch_size, cudaStream_t s,
                     std::vector<int64_t>& touched, std::vector<int64_t>& tcount) {
  HostCsr& h = prob.a;
  TraceScope tr_ls("slab local_structure: index space", s);
  std::vector<int64_t> rows_g;
  rows_g.reserve(static_cast<size_t>(h.n));
  for (const auto& g : prob.row_ranges)
    for (int64_t i = g.first; i < g.second; ++i) rows_g.push_back(i);
  require(static_cast<int64_t>(rows_g.size()) == h.n, Errc::invalid_argument, "slab rows do not match the row ranges");
  int64_t gmin = rows_g.empty() ? 0 : rows_g.front(), gmax = rows_g.empty() ? -1 : rows_g.back();
  // column range: rows hold ascending columns (the CSR contract, validated at creation and kept by the
  // generator), so a row's first and last entry bound it -- one pass over the rows, not the entries
  // (config 5 at 96^3: 3.5G entries per rank); the marking pass below checks every column against it
  {
    std::mutex mu;
    parallel_rows(h.n, [&](int64_t r0, int64_t r1) {
      int64_t lo = gmin, hi = gmax;
      for (int64_t i = r0; i < r1; ++i) {
        const int64_t a = h.row_ptr[static_cast<size_t>(i)], b = h.row_ptr[static_cast<size_t>(i) + 1];
        if (b > a) {
          lo = std::min<int64_t>(lo, h.col[static_cast<size_t>(a)]);
          hi = std::max<int64_t>(hi, h.col[static_cast<size_t>(b - 1)]);
        }
      }
      std::lock_guard<std::mutex> g(mu);
      gmin = std::min(gmin, lo);
      gmax = std::max(gmax, hi);
    });
  }
  const int64_t span = gmax - gmin + 1;
  std::vector<int32_t> g2l(static_cast<size_t>(std::max<int64_t>(span, 1)), -1);
  for (int64_t gi : rows_g) g2l[static_cast<size_t>(gi - gmin)] = 0;
  // mark every referenced column (threads may store the same 0: relaxed atomic stores)
  std::atomic<bool> in_range{true};
  parallel_rows(static_cast<int64_t>(h.col.size()), [&](int64_t b, int64_t e) {
    bool ok = true;
    for (int64_t q = b; q < e; ++q) {
      const int64_t c = h.col[static_cast<size_t>(q)];
      if (c < gmin || c > gmax) {
        ok = false;
        continue;
      }
      __atomic_store_n(&g2l[static_cast<size_t>(c - gmin)], 0, __ATOMIC_RELAXED);
    }
    if (!ok) in_range.store(false, std::memory_order_relaxed);
  });
  require(in_range.load(), Errc::invalid_argument, "slab rows must hold ascending column indices");
  R.gid.clear();
  for (int64_t q = 0; q < span; ++q)
    if (g2l[static_cast<size_t>(q)] == 0) {
      g2l[static_cast<size_t>(q)] = static_cast<int32_t>(R.gid.size());
      R.gid.push_back(gmin + q);
    }
  R.nl = static_cast<int64_t>(R.gid.size());
  // local CSR: the rank's rows keep their entries, the halo rows are empty
  HostCsr loc;
  loc.n = R.nl;
  loc.row_ptr.assign(static_cast<size_t>(R.nl + 1), 0);
  R.rows.resize(rows_g.size());
  for (size_t i = 0; i < rows_g.size(); ++i) {
    const int32_t l = g2l[static_cast<size_t>(rows_g[i] - gmin)];
    R.rows[i] = l;
    loc.row_ptr[static_cast<size_t>(l) + 1] = h.row_ptr[i + 1] - h.row_ptr[i];
  }
  for (int64_t l = 0; l < R.nl; ++l) loc.row_ptr[static_cast<size_t>(l) + 1] += loc.row_ptr[static_cast<size_t>(l)];
  // rows keep their order and the halo rows are empty, so the local entry
  // arrays are the slab's in the same order: the global columns and the
  // values are uploaded as they are and the columns remapped on the device
  // (config 5: 3.5G entries per rank -- no host copy of them is made); the
  // opt-in host-built half storage needs the local CSR on the host
  const char* me = getenv("PDB_SELL_MIRROR");
  std::optional<TraceScope> tr_up;
  tr_up.emplace("slab local_structure: upload + SELL", s, &R.upload_s);
  if (!(me && me[0] == '1')) {
    const int64_t nnz = static_cast<int64_t>(h.col.size());
    alloc_csr(R.nl, nnz, R.a, s);
    h2d_staged(R.a.row_ptr.get(), loc.row_ptr.data(), loc.row_ptr.size() * sizeof(int64_t), s);
    h2d_staged(R.a.col.get(), h.col.data(), h.col.size() * sizeof(int32_t), s);
    h2d_staged(R.a.val.get(), h.val.data(), h.val.size() * sizeof(double), s);
    {
      Scratch<int32_t> dg2l(g2l.size(), s);
      dg2l.upload(g2l.data(), g2l.size());
      if (nnz > 0)
        remap_cols_kernel<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(nnz, gmin, dg2l.get(), R.a.col.get());
      PDB_LAUNCH_CHECK();
      sync(s);
    }
    HostCsr none;
    finish_csr(none, loc.row_ptr, R.a, s);
  } else {
    loc.col.resize(h.col.size());
    parallel_rows(static_cast<int64_t>(h.col.size()), [&](int64_t b, int64_t e) {
      for (int64_t q = b; q < e; ++q)
        loc.col[static_cast<size_t>(q)] = g2l[static_cast<size_t>(h.col[static_cast<size_t>(q)] - gmin)];
    });
    loc.val.swap(h.val);  // lent for the upload (config 5 holds 46 GB of them)
    try {
      upload_csr(loc, R.a, s);
    } catch (...) {
      loc.val.swap(h.val);
      throw;
    }
    loc.val.swap(h.val);
  }
  tr_up.reset();
  {
    TraceScope tr_d("slab local_structure: detect", s);
    detect_patches(R.a, patch_size, R.ps, s);
  }
  TraceScope tr_t("slab local_structure: touched lists", s);
  R.np = R.ps.np;
  // touched DoFs (global ids, ascending) and the local cover counts
  R.pt_host = R.ps.patches.to_host(s);
  const std::vector<int32_t>& pt = R.pt_host;
  std::vector<int32_t> cnt(static_cast<size_t>(R.nl), 0);
  for (int32_t l : pt) ++cnt[static_cast<size_t>(l)];
  touched.clear();
  tcount.clear();
  touched.reserve(static_cast<size_t>(R.nl));
  tcount.reserve(static_cast<size_t>(R.nl));
  for (int64_t l = 0; l < R.nl; ++l)
    if (cnt[static_cast<size_t>(l)]) {
      touched.push_back(R.gid[static_cast<size_t>(l)]);
      tcount.push_back(cnt[static_cast<size_t>(l)]);
    }
}

int64_t local_of(const SlabRank& R, int64_t g) {
  auto it = std::lower_bound(R.gid.begin(), R.gid.end(), g);
  return it != R.gid.end() && *it == g ? static_cast<int64_t>(it - R.gid.begin()) : -1;
}

}  // namespace

// Collective setup of the ranks in g (each with its slab problem).
// Distributed greedy-l1 over the ranks' own patches (greedy_impl,
// compress.cpp:40-95, in the round-batched exact form of database.cu
// section "Greedy on the GPU").  Global patch order is rank-major, so each
// round's batch -- the first B unresolved patches -- is the unresolved prefix
// of rank 0, then of rank 1, ...: the owners contribute those matrices
// (broadcast), every rank computes the same batch distances and the same
// sequential resolution, keeps the new entries' matrices (the small
// replicated set), and scans only its OWN remaining patches against them.
// The decisions are those of the single-GPU build, hence the reference's.
void slab_greedy(pdb_slab_s& g, int64_t patch_size, const BuildParams& bp, pdb_database_s& out, cudaStream_t s) {
  require(bp.method == PDB_METHOD_GREEDY_L1, Errc::invalid_argument,
          "rank-local database build: greedy-l1 only (other methods need the whole patch set)");
  require(bp.eps > 0.0, Errc::invalid_argument, "tolerance must be positive");
  const int L = static_cast<int>(g.ranks.size());
  const int W = g.ranks[0]->nranks;
  const int ps = static_cast<int>(patch_size);
  const int64_t len = static_cast<int64_t>(ps) * ps;
  const int64_t Bmax = 1024;
  const bool best = bp.best_match;
  // per local rank: patch matrices, unresolved list, phi / best distances
  std::vector<DevBuf<double>> mats(static_cast<size_t>(L));
  std::vector<std::vector<int32_t>> U(static_cast<size_t>(L));
  std::vector<DevBuf<int32_t>> phi(static_cast<size_t>(L));
  std::vector<DevBuf<double>> bd(static_cast<size_t>(L));
  for (int i = 0; i < L; ++i) {
    SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    extract_patches(R.a, R.ps, mats[static_cast<size_t>(i)], s);
    U[static_cast<size_t>(i)].resize(static_cast<size_t>(R.np));
    for (int64_t k = 0; k < R.np; ++k) U[static_cast<size_t>(i)][static_cast<size_t>(k)] = static_cast<int32_t>(k);
    phi[static_cast<size_t>(i)].alloc(static_cast<size_t>(std::max<int64_t>(R.np, 1)));
    PDB_CUDA(cudaMemsetAsync(phi[static_cast<size_t>(i)].get(), 0xff, R.np * sizeof(int32_t), s));
    if (best) {
      std::vector<double> init(static_cast<size_t>(std::max<int64_t>(R.np, 1)), bp.eps);
      put(bd[static_cast<size_t>(i)], init, s);
    }
  }
  DevBuf<double> batch(static_cast<size_t>(Bmax * len)), D(static_cast<size_t>(Bmax * Bmax));
  DevBuf<int32_t> S(static_cast<size_t>(Bmax)), phib(static_cast<size_t>(Bmax)), entry_of(static_cast<size_t>(Bmax));
  DevBuf<int64_t> state(3);
  k::iota(Bmax, S.get(), s);
  int64_t cap = 1024, m = 0;
  DevBuf<double> entries(static_cast<size_t>(cap * len));
  DevBuf<int32_t> cre_b(static_cast<size_t>(cap)), cre_g(static_cast<size_t>(cap));
  g.creators.clear();
  auto grow = [&](int64_t need) {
    if (need <= cap) return;
    int64_t nc = cap;
    while (nc < need) nc *= 2;
    DevBuf<double> e2(static_cast<size_t>(nc * len));
    DevBuf<int32_t> b2(static_cast<size_t>(nc)), g2(static_cast<size_t>(nc));
    if (m > 0) {
      PDB_CUDA(cudaMemcpyAsync(e2.get(), entries.get(), m * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
      PDB_CUDA(cudaMemcpyAsync(g2.get(), cre_g.get(), m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
    entries = std::move(e2);
    cre_b = std::move(b2);
    cre_g = std::move(g2);
    cap = nc;
  };
  std::vector<Mail> outm(static_cast<size_t>(L), Mail(static_cast<size_t>(W))), inm;
  for (;;) {
    // unresolved counts of every rank
    std::vector<int64_t> cnt(static_cast<size_t>(W), 0);
    for (int i = 0; i < L; ++i)
      for (int q = 0; q < W; ++q) outm[static_cast<size_t>(i)][static_cast<size_t>(q)] = {static_cast<int64_t>(U[static_cast<size_t>(i)].size())};
    deliver(g, outm, inm, s);
    for (int q = 0; q < W; ++q)
      if (!inm[0][static_cast<size_t>(q)].empty()) cnt[static_cast<size_t>(q)] = inm[0][static_cast<size_t>(q)][0];
    int64_t total = 0;
    for (int64_t c : cnt) total += c;
    if (total == 0) break;
    const int64_t B = std::min(total, Bmax);
    std::vector<int64_t> take(static_cast<size_t>(W)), off(static_cast<size_t>(W) + 1, 0);
    for (int q = 0; q < W; ++q) {
      take[static_cast<size_t>(q)] = std::min(cnt[static_cast<size_t>(q)], B - off[static_cast<size_t>(q)]);
      off[static_cast<size_t>(q) + 1] = off[static_cast<size_t>(q)] + take[static_cast<size_t>(q)];
    }
    // the owners' batch matrices and the batch's global ids
    std::vector<int32_t> Sg(static_cast<size_t>(B));
    for (int i = 0; i < L; ++i) {
      const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
      const int64_t t = take[static_cast<size_t>(R.rank)];
      if (t == 0) continue;
      std::vector<int32_t> ids(U[static_cast<size_t>(i)].begin(), U[static_cast<size_t>(i)].begin() + t);
      DevBuf<int32_t> d_ids;
      put(d_ids, ids, s);
      k::gather_mats(t, d_ids.get(), len, mats[static_cast<size_t>(i)].get(), batch.get() + off[static_cast<size_t>(R.rank)] * len, s);
      sync(s);
    }
    if (!g.emulated && W > 1) {
      SlabRank& R = *g.ranks[0];
      PDB_NCCL_S(ncclGroupStart());
      for (int q = 0; q < W; ++q)
        if (take[static_cast<size_t>(q)] > 0)
          PDB_NCCL_S(ncclBroadcast(batch.get() + off[static_cast<size_t>(q)] * len, batch.get() + off[static_cast<size_t>(q)] * len,
                                   static_cast<size_t>(take[static_cast<size_t>(q)] * len), ncclDouble, q, R.comm, s));
      PDB_NCCL_S(ncclGroupEnd());
    }
    // global ids: every rank's unresolved prefix (ids exchanged with the counts' partners)
    for (int i = 0; i < L; ++i) {
      const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
      std::vector<int64_t> mine;
      for (int64_t j = 0; j < take[static_cast<size_t>(R.rank)]; ++j)
        mine.push_back(g.k0_of[static_cast<size_t>(R.rank)] + U[static_cast<size_t>(i)][static_cast<size_t>(j)]);
      for (int q = 0; q < W; ++q) outm[static_cast<size_t>(i)][static_cast<size_t>(q)] = mine;
    }
    deliver(g, outm, inm, s);
    for (int q = 0; q < W; ++q)
      for (int64_t j = 0; j < take[static_cast<size_t>(q)]; ++j)
        Sg[static_cast<size_t>(off[static_cast<size_t>(q)] + j)] = static_cast<int32_t>(inm[0][static_cast<size_t>(q)][static_cast<size_t>(j)]);
    // batch distances and the sequential resolution (replicated)
    k::l1_pairs(B, nullptr, B, static_cast<int>(len), batch.get(), nullptr, batch.get(), D.get(), s);
    PDB_CUDA(cudaMemsetAsync(entry_of.get(), 0xff, B * sizeof(int32_t), s));
    PDB_CUDA(cudaMemsetAsync(phib.get(), 0xff, B * sizeof(int32_t), s));
    grow(m + B);
    std::vector<int64_t> st = {m, 0, -1};
    PDB_CUDA(cudaMemcpyAsync(state.get(), st.data(), 3 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    k::greedy_resolve(static_cast<int>(B), S.get(), D.get(), bp.eps, best ? 1 : 0, -1, nullptr, phib.get(),
                      cre_b.get(), entry_of.get(), state.get(), s);
    PDB_LAUNCH_CHECK();
    PDB_CUDA(cudaMemcpyAsync(st.data(), state.get(), 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    sync(s);
    const int64_t m_new = st[0];
    // new entries: matrices and global creator ids
    if (m_new > m) {
      k::gather_mats(m_new - m, cre_b.get() + m, len, batch.get(), entries.get() + m * len, s);
      const std::vector<int32_t> cb = cre_b.to_host(s);
      std::vector<int32_t> cg(static_cast<size_t>(m_new - m));
      for (int64_t e = m; e < m_new; ++e) {
        cg[static_cast<size_t>(e - m)] = Sg[static_cast<size_t>(cb[static_cast<size_t>(e)])];
        g.creators.push_back(cg[static_cast<size_t>(e - m)]);
      }
      PDB_CUDA(cudaMemcpyAsync(cre_g.get() + m, cg.data(), cg.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    const std::vector<int32_t> pb = phib.to_host(s);
    // owners record their batch members' phi; scan their other patches against the new entries
    for (int i = 0; i < L; ++i) {
      SlabRank& R = *g.ranks[static_cast<size_t>(i)];
      auto& Ui = U[static_cast<size_t>(i)];
      const int64_t t = take[static_cast<size_t>(R.rank)], o = off[static_cast<size_t>(R.rank)];
      if (t > 0) {
        std::vector<int32_t> vals(pb.begin() + o, pb.begin() + o + t);
        std::vector<int32_t> ids(Ui.begin(), Ui.begin() + t);
        DevBuf<int32_t> d_ids, d_vals;
        put(d_ids, ids, s);
        put(d_vals, vals, s);
        k::scatter_ints(t, d_ids.get(), d_vals.get(), phi[static_cast<size_t>(i)].get(), s);
      }
      if (m_new > m) {
        std::vector<int32_t> rest;
        if (best) {  // every patch after the batch start except the batch itself (database.cu best match)
          const int64_t first = Sg[0];
          std::vector<char> inb(static_cast<size_t>(std::max<int64_t>(R.np, 1)), 0);
          for (int64_t j = 0; j < t; ++j) inb[static_cast<size_t>(Ui[static_cast<size_t>(j)])] = 1;
          for (int64_t k = 0; k < R.np; ++k)
            if (g.k0_of[static_cast<size_t>(R.rank)] + k > first && !inb[static_cast<size_t>(k)]) rest.push_back(static_cast<int32_t>(k));
        } else {
          rest.assign(Ui.begin() + t, Ui.end());
        }
        if (!rest.empty()) {
          DevBuf<int32_t> d_rest;
          put(d_rest, rest, s);
          k::l1_scan_entries(static_cast<int64_t>(rest.size()), d_rest.get(), g.k0_of[static_cast<size_t>(R.rank)], m,
                             m_new, static_cast<int>(len), mats[static_cast<size_t>(i)].get(), entries.get(),
                             cre_g.get(), bp.eps, best ? 1 : 0, phi[static_cast<size_t>(i)].get(),
                             best ? bd[static_cast<size_t>(i)].get() : nullptr, s);
          PDB_LAUNCH_CHECK();
        }
      }
      // unresolved: the unmatched among the rank's remaining patches
      const std::vector<int32_t> ph = phi[static_cast<size_t>(i)].to_host(s);
      std::vector<int32_t> keep;
      for (size_t j = static_cast<size_t>(t); j < Ui.size(); ++j)
        if (ph[static_cast<size_t>(Ui[j])] < 0) keep.push_back(Ui[j]);
      Ui.swap(keep);
    }
    m = m_new;
  }
  // factors of the entries (replicated; the reference factors each new entry, compress.cpp:91)
  out.m = m;
  out.ps = ps;
  out.np = 0;
  for (int64_t c : g.np_of) out.np += c;
  out.method = "greedy-l1";
  out.eps = bp.eps;
  out.lu.alloc(static_cast<size_t>(std::max<int64_t>(m, 1) * len));
  out.piv.alloc(static_cast<size_t>(std::max<int64_t>(m, 1) * ps));
  DevBuf<int32_t> status(static_cast<size_t>(std::max<int64_t>(m, 1)));
  DevBuf<double> bst(static_cast<size_t>(std::max<int64_t>(m, 1)));
  k::lu_batched(m, ps, entries.get(), nullptr, out.lu.get(), out.piv.get(), status.get(), bst.get(), s);
  PDB_LAUNCH_CHECK();
  const std::vector<int32_t> sth = status.to_host(s);
  for (int64_t e = 0; e < m; ++e)
    if (sth[static_cast<size_t>(e)] != 0) {
      const std::vector<double> bh = bst.to_host(s);
      fail(Errc::singular_matrix, "patch " + std::to_string(g.creators[static_cast<size_t>(e)]) + ": " +
                                      singular_msg(sth[static_cast<size_t>(e)], bh[static_cast<size_t>(e)]));
    }
  out.reps = std::move(entries);
  g.m = m;
  for (int i = 0; i < L; ++i) g.ranks[static_cast<size_t>(i)]->phi = phi[static_cast<size_t>(i)].to_host(s);
  sync(s);
}



// Distributed entrywise k-means, boundary-partitioned (partitioned_build,
// compress.cpp:394-421; kmeans / kmeans_loop, compress.cpp:138-324) over the
// ranks' own patches.  Partitions in global first-occurrence order (every
// rank's pattern list in rank order), budgets by split_budget, per partition:
// the seeded partial Fisher-Yates picks (their owners broadcast the initial
// representatives), then Lloyd iterations whose assignment is local (l1
// argmin, strict <) and whose assignment vector and distances are gathered so
// every rank applies the same reseed rule; the new means are the in-order
// member sums folded along the ranks (rank r continues rank r-1's partial
// sums, the last rank scales by 1/size, exactly entrywise_mean_indexed) and
// broadcast.  The database is bitwise the single-GPU partitioned_build's.
void slab_kmeans(pdb_slab_s& g, int64_t patch_size, const BuildParams& bp, pdb_database_s& out, cudaStream_t s) {
  require(bp.method == PDB_METHOD_KMEANS_ENTRYWISE, Errc::invalid_argument,
          "rank-local k-means: the entrywise variant only");
  const int L = static_cast<int>(g.ranks.size());
  const int W = g.ranks[0]->nranks;
  const int ps = static_cast<int>(patch_size);
  const int64_t len = static_cast<int64_t>(ps) * ps;
  const int words = (ps + 63) / 64;
  const bool nccl = !g.emulated && W > 1;
  std::vector<DevBuf<double>> mats(static_cast<size_t>(L));
  std::vector<std::vector<std::vector<unsigned long long>>> keys(static_cast<size_t>(L));  // per local patch
  for (int i = 0; i < L; ++i) {
    SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    extract_patches(R.a, R.ps, mats[static_cast<size_t>(i)], s);
    DevBuf<unsigned long long> mk(static_cast<size_t>(std::max<int64_t>(R.np * words, 1)));
    if (R.np > 0) k::boundary_masks(R.np, ps, mats[static_cast<size_t>(i)].get(), words, mk.get(), s);
    const std::vector<unsigned long long> mh = mk.to_host(s);
    keys[static_cast<size_t>(i)].resize(static_cast<size_t>(R.np));
    for (int64_t kk = 0; kk < R.np; ++kk)
      keys[static_cast<size_t>(i)][static_cast<size_t>(kk)].assign(mh.begin() + kk * words, mh.begin() + (kk + 1) * words);
  }
  // every rank's distinct patterns in local first-occurrence order, with counts
  std::vector<Mail> outm(static_cast<size_t>(L), Mail(static_cast<size_t>(W))), inm;
  std::vector<std::vector<std::vector<unsigned long long>>> lpat(static_cast<size_t>(L));
  std::vector<std::vector<int64_t>> lcnt(static_cast<size_t>(L));
  std::vector<std::vector<int32_t>> lpid(static_cast<size_t>(L));  // local pattern index per patch
  for (int i = 0; i < L; ++i) {
    std::map<std::vector<unsigned long long>, int32_t> idx;
    for (const auto& kv : keys[static_cast<size_t>(i)]) {
      auto it = idx.find(kv);
      if (it == idx.end()) {
        it = idx.emplace(kv, static_cast<int32_t>(lpat[static_cast<size_t>(i)].size())).first;
        lpat[static_cast<size_t>(i)].push_back(kv);
        lcnt[static_cast<size_t>(i)].push_back(0);
      }
      ++lcnt[static_cast<size_t>(i)][static_cast<size_t>(it->second)];
      lpid[static_cast<size_t>(i)].push_back(it->second);
    }
    std::vector<int64_t> msg;
    for (size_t p = 0; p < lpat[static_cast<size_t>(i)].size(); ++p) {
      msg.push_back(lcnt[static_cast<size_t>(i)][p]);
      for (unsigned long long w : lpat[static_cast<size_t>(i)][p]) msg.push_back(static_cast<int64_t>(w));
    }
    for (int q = 0; q < W; ++q) outm[static_cast<size_t>(i)][static_cast<size_t>(q)] = msg;
  }
  deliver(g, outm, inm, s);
  // global partitions: first occurrence over the ranks in order; per-rank counts
  std::map<std::vector<unsigned long long>, int32_t> gidx;
  std::vector<std::vector<unsigned long long>> gpat;
  std::vector<std::vector<int64_t>> gcnt;  // [partition][rank]
  for (int q = 0; q < W; ++q) {
    const auto& m = inm[0][static_cast<size_t>(q)];
    for (size_t o = 0; o + 1 + static_cast<size_t>(words) <= m.size(); o += 1 + static_cast<size_t>(words)) {
      std::vector<unsigned long long> kv(static_cast<size_t>(words));
      for (int w = 0; w < words; ++w) kv[static_cast<size_t>(w)] = static_cast<unsigned long long>(m[o + 1 + static_cast<size_t>(w)]);
      auto it = gidx.find(kv);
      if (it == gidx.end()) {
        it = gidx.emplace(kv, static_cast<int32_t>(gpat.size())).first;
        gpat.push_back(kv);
        gcnt.emplace_back(static_cast<size_t>(W), 0);
      }
      gcnt[static_cast<size_t>(it->second)][static_cast<size_t>(q)] += m[o];
    }
  }
  const size_t G = gpat.size();
  std::vector<int64_t> sizes(G);
  for (size_t p = 0; p < G; ++p)
    for (int q = 0; q < W; ++q) sizes[p] += gcnt[p][static_cast<size_t>(q)];
  const std::vector<int64_t> alloc = split_budget(bp.db_size, sizes);
  // per local rank: its patches of each partition (ascending local ids)
  std::vector<std::vector<std::vector<int32_t>>> mine(static_cast<size_t>(L), std::vector<std::vector<int32_t>>(G));
  for (int i = 0; i < L; ++i)
    for (size_t kk = 0; kk < lpid[static_cast<size_t>(i)].size(); ++kk) {
      const int32_t gp = gidx[lpat[static_cast<size_t>(i)][static_cast<size_t>(lpid[static_cast<size_t>(i)][kk])]];
      mine[static_cast<size_t>(i)][static_cast<size_t>(gp)].push_back(static_cast<int32_t>(kk));
    }
  int64_t total = 0;
  for (int64_t c : alloc) total += c;
  DevBuf<double> reps_all(static_cast<size_t>(std::max<int64_t>(total, 1) * len));
  for (int i = 0; i < L; ++i) g.ranks[static_cast<size_t>(i)]->phi.assign(static_cast<size_t>(g.ranks[static_cast<size_t>(i)]->np), -1);
  int64_t eoff = 0;
  DevBuf<int32_t> changed(1);
  for (size_t p = 0; p < G; ++p) {
    const int64_t n = sizes[p], m = alloc[p];
    std::vector<int64_t> off(static_cast<size_t>(W) + 1, 0);
    for (int q = 0; q < W; ++q) off[static_cast<size_t>(q) + 1] = off[static_cast<size_t>(q)] + gcnt[p][static_cast<size_t>(q)];
    auto owner_of = [&](int64_t o) {
      int q = 0;
      while (off[static_cast<size_t>(q) + 1] <= o) ++q;
      return q;
    };
    require(n >= 1 && m >= 1 && m <= n, Errc::invalid_argument, "kmeans requires 1 <= m_p <= n_p");
    // seeded picks (compress.cpp:302-308) and the initial representatives from their owners
    std::mt19937_64 rng(bp.seed + p);
    std::vector<int64_t> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), int64_t{0});
    for (int64_t i2 = 0; i2 < m; ++i2) {
      const int64_t j = i2 + static_cast<int64_t>(rng() % static_cast<uint64_t>(n - i2));
      std::swap(perm[static_cast<size_t>(i2)], perm[static_cast<size_t>(j)]);
    }
    double* reps = reps_all.get() + eoff * len;
    std::vector<int> pick_owner(static_cast<size_t>(m));
    for (int i = 0; i < L; ++i) {
      const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
      std::vector<int32_t> src, dst;
      for (int64_t c = 0; c < m; ++c) {
        const int64_t o = perm[static_cast<size_t>(c)];
        const int q = owner_of(o);
        pick_owner[static_cast<size_t>(c)] = q;
        if (q != R.rank) continue;
        src.push_back(mine[static_cast<size_t>(i)][p][static_cast<size_t>(o - off[static_cast<size_t>(q)])]);
        dst.push_back(static_cast<int32_t>(c));
      }
      for (size_t t = 0; t < src.size(); ++t)
        PDB_CUDA(cudaMemcpyAsync(reps + dst[t] * len, mats[static_cast<size_t>(i)].get() + static_cast<int64_t>(src[t]) * len,
                                 len * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    if (nccl) {
      SlabRank& R = *g.ranks[0];
      PDB_NCCL_S(ncclGroupStart());
      for (int64_t c = 0; c < m; ++c)
        PDB_NCCL_S(ncclBroadcast(reps + c * len, reps + c * len, static_cast<size_t>(len), ncclDouble,
                                 pick_owner[static_cast<size_t>(c)], R.comm, s));
      PDB_NCCL_S(ncclGroupEnd());
    }
    // Lloyd iterations (kmeans_loop, Reseed policy)
    std::vector<int32_t> phi_h(static_cast<size_t>(n), -1);
    std::vector<DevBuf<int32_t>> dpid(static_cast<size_t>(L)), dphi(static_cast<size_t>(L)), dnew(static_cast<size_t>(L));
    std::vector<DevBuf<double>> dmin(static_cast<size_t>(L));
    for (int i = 0; i < L; ++i) {
      const auto& li = mine[static_cast<size_t>(i)][p];
      put(dpid[static_cast<size_t>(i)], li, s);
      dphi[static_cast<size_t>(i)].alloc(std::max<size_t>(li.size(), 1));
      PDB_CUDA(cudaMemsetAsync(dphi[static_cast<size_t>(i)].get(), 0xff, li.size() * sizeof(int32_t), s));
      dnew[static_cast<size_t>(i)].alloc(std::max<size_t>(li.size(), 1));
      dmin[static_cast<size_t>(i)].alloc(std::max<size_t>(li.size(), 1));
    }
    DevBuf<double> partial(static_cast<size_t>(m * len)), next(static_cast<size_t>(m * len));
    for (int iter = 0; iter < bp.max_iters; ++iter) {
      for (int i = 0; i < L; ++i) {
        const auto& li = mine[static_cast<size_t>(i)][p];
        k::l1_argmin_ids(static_cast<int64_t>(li.size()), dpid[static_cast<size_t>(i)].get(), m, static_cast<int>(len),
                         mats[static_cast<size_t>(i)].get(), reps, dphi[static_cast<size_t>(i)].get(),
                         dnew[static_cast<size_t>(i)].get(), dmin[static_cast<size_t>(i)].get(), changed.get(), s);
        PDB_LAUNCH_CHECK();
        const std::vector<int32_t> nh = dnew[static_cast<size_t>(i)].to_host(s);
        const std::vector<double> mh = dmin[static_cast<size_t>(i)].to_host(s);
        std::vector<int64_t> msg(2 * li.size());
        for (size_t t = 0; t < li.size(); ++t) {
          msg[2 * t] = nh[t];
          std::memcpy(&msg[2 * t + 1], &mh[t], sizeof(double));
        }
        for (int q = 0; q < W; ++q) outm[static_cast<size_t>(i)][static_cast<size_t>(q)] = msg;
      }
      deliver(g, outm, inm, s);
      const std::vector<int32_t> prev = phi_h;
      std::vector<double> min_dist(static_cast<size_t>(n));
      for (int q = 0; q < W; ++q) {
        const auto& mm = inm[0][static_cast<size_t>(q)];
        for (int64_t t = 0; t < gcnt[p][static_cast<size_t>(q)]; ++t) {
          phi_h[static_cast<size_t>(off[static_cast<size_t>(q)] + t)] = static_cast<int32_t>(mm[static_cast<size_t>(2 * t)]);
          std::memcpy(&min_dist[static_cast<size_t>(off[static_cast<size_t>(q)] + t)], &mm[static_cast<size_t>(2 * t + 1)], sizeof(double));
        }
      }
      if (prev == phi_h) break;
      std::vector<std::vector<int32_t>> members(static_cast<size_t>(m));
      for (int64_t o = 0; o < n; ++o) members[static_cast<size_t>(phi_h[static_cast<size_t>(o)])].push_back(static_cast<int32_t>(o));
      for (int64_t j = 0; j < m; ++j) {  // reseed empty clusters (compress.cpp:195-217)
        if (!members[static_cast<size_t>(j)].empty()) continue;
        int64_t far = -1;
        double far_d = -1.0;
        for (int64_t o = 0; o < n; ++o) {
          const int32_t own = phi_h[static_cast<size_t>(o)];
          if (members[static_cast<size_t>(own)].size() <= 1) continue;
          if (min_dist[static_cast<size_t>(o)] > far_d) {
            far_d = min_dist[static_cast<size_t>(o)];
            far = o;
          }
        }
        if (far < 0) continue;
        auto& ow = members[static_cast<size_t>(phi_h[static_cast<size_t>(far)])];
        ow.erase(std::find(ow.begin(), ow.end(), static_cast<int32_t>(far)));
        members[static_cast<size_t>(j)].push_back(static_cast<int32_t>(far));
        phi_h[static_cast<size_t>(far)] = static_cast<int32_t>(j);
        min_dist[static_cast<size_t>(far)] = 0.0;
      }
      for (int64_t j = 0; j < m; ++j)
        if (members[static_cast<size_t>(j)].empty())
          fail(Errc::singular_matrix, "cluster " + std::to_string(j) + ": entrywise_mean of an empty cluster");
      std::vector<int64_t> counts(static_cast<size_t>(m));
      for (int64_t j = 0; j < m; ++j) counts[static_cast<size_t>(j)] = static_cast<int64_t>(members[static_cast<size_t>(j)].size());
      DevBuf<int64_t> dcounts;
      put(dcounts, counts, s);
      // each rank's members (local ids), cluster-major, ascending
      auto local_members = [&](int q, int i) {
        std::vector<int32_t> ptr(static_cast<size_t>(m) + 1, 0), mem;
        for (int64_t j = 0; j < m; ++j) {
          for (int32_t o : members[static_cast<size_t>(j)])
            if (o >= off[static_cast<size_t>(q)] && o < off[static_cast<size_t>(q) + 1])
              mem.push_back(mine[static_cast<size_t>(i)][p][static_cast<size_t>(o - off[static_cast<size_t>(q)])]);
          ptr[static_cast<size_t>(j) + 1] = static_cast<int32_t>(mem.size());
        }
        return std::make_pair(ptr, mem);
      };
      // the chain fold: ranks in order continue the partial sums, the last scales
      const int last = W - 1;
      if (g.emulated || W == 1) {
        for (int i = 0; i < L; ++i) {
          const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
          auto pm = local_members(R.rank, i);
          DevBuf<int32_t> dp, dm;
          put(dp, pm.first, s);
          put(dm, pm.second, s);
          k::cluster_sum_chain(m, static_cast<int>(len), dp.get(), dm.get(), mats[static_cast<size_t>(i)].get(),
                               i == 0 ? nullptr : partial.get(), R.rank == last ? dcounts.get() : nullptr,
                               R.rank == last ? reps : next.get(), s);
          sync(s);
          std::swap(partial, next);
        }
      } else {
        SlabRank& R = *g.ranks[0];
        auto pm = local_members(R.rank, 0);
        DevBuf<int32_t> dp, dm;
        put(dp, pm.first, s);
        put(dm, pm.second, s);
        if (R.rank > 0) PDB_NCCL_S(ncclRecv(partial.get(), static_cast<size_t>(m * len), ncclDouble, R.rank - 1, R.comm, s));
        k::cluster_sum_chain(m, static_cast<int>(len), dp.get(), dm.get(), mats[0].get(), R.rank > 0 ? partial.get() : nullptr,
                             R.rank == last ? dcounts.get() : nullptr, R.rank == last ? reps : next.get(), s);
        if (R.rank < last) PDB_NCCL_S(ncclSend(next.get(), static_cast<size_t>(m * len), ncclDouble, R.rank + 1, R.comm, s));
        PDB_NCCL_S(ncclBroadcast(reps, reps, static_cast<size_t>(m * len), ncclDouble, last, R.comm, s));
        sync(s);
      }
      // the next assignment compares against this one
      for (int i = 0; i < L; ++i) {
        const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
        const std::vector<int32_t> mp(phi_h.begin() + off[static_cast<size_t>(R.rank)],
                                      phi_h.begin() + off[static_cast<size_t>(R.rank) + 1]);
        if (!mp.empty()) dphi[static_cast<size_t>(i)].upload(mp.data(), mp.size(), s);
      }
    }
    // phi of this partition -> the ranks' patches
    for (int i = 0; i < L; ++i) {
      SlabRank& R = *g.ranks[static_cast<size_t>(i)];
      const auto& li = mine[static_cast<size_t>(i)][p];
      for (size_t t = 0; t < li.size(); ++t)
        R.phi[static_cast<size_t>(li[t])] = static_cast<int32_t>(eoff + phi_h[static_cast<size_t>(off[static_cast<size_t>(R.rank)] + static_cast<int64_t>(t))]);
    }
    eoff += m;
  }
  // factors of the representatives (finalize_factors; replicated)
  out.m = total;
  out.ps = ps;
  out.np = 0;
  for (int64_t c : g.np_of) out.np += c;
  out.method = "kmeans-entrywise-partitioned";
  out.lu.alloc(static_cast<size_t>(std::max<int64_t>(total, 1) * len));
  out.piv.alloc(static_cast<size_t>(std::max<int64_t>(total, 1) * ps));
  DevBuf<int32_t> status(static_cast<size_t>(std::max<int64_t>(total, 1)));
  DevBuf<double> bst(static_cast<size_t>(std::max<int64_t>(total, 1)));
  k::lu_batched(total, ps, reps_all.get(), nullptr, out.lu.get(), out.piv.get(), status.get(), bst.get(), s);
  PDB_LAUNCH_CHECK();
  const std::vector<int32_t> sth = status.to_host(s);
  for (int64_t e = 0; e < total; ++e)
    if (sth[static_cast<size_t>(e)] != 0) {
      const std::vector<double> bh = bst.to_host(s);
      fail(Errc::singular_matrix, "cluster " + std::to_string(e) + ": " +
                                      singular_msg(sth[static_cast<size_t>(e)], bh[static_cast<size_t>(e)]));
    }
  out.reps = std::move(reps_all);
  g.m = total;
  g.creators.clear();
  sync(s);
}

void slab_setup(pdb_slab_s& g, std::vector<pdb_problem_s*>& probs, int64_t patch_size, const pdb_database_s* db,
                double omega, cudaStream_t s, const BuildParams* build) {
  require_device();
  const int L = static_cast<int>(g.ranks.size());
  const int W = g.ranks[0]->nranks;
  std::vector<std::vector<int64_t>> T(static_cast<size_t>(L)), Tc(static_cast<size_t>(L));
  for (int i = 0; i < L; ++i) {
    require(probs[static_cast<size_t>(i)]->is_slab() || W == 1, Errc::invalid_argument,
            "shard needs a slab problem (pdb_problem_generate_slab)");
    if (!probs[static_cast<size_t>(i)]->is_slab()) probs[static_cast<size_t>(i)]->row_ranges = {{0, probs[static_cast<size_t>(i)]->a.n}};
    local_structure(*g.ranks[static_cast<size_t>(i)], *probs[static_cast<size_t>(i)], patch_size, s, T[static_cast<size_t>(i)], Tc[static_cast<size_t>(i)]);
  }
  g.n_global = probs[0]->n_global > 0 ? probs[0]->n_global : probs[0]->a.n;
  std::optional<TraceScope> tph;
  tph.emplace("slab setup: phase 1 (counts, ranges)", s);
  // (1) all ranks: patch count and touched range
  std::vector<Mail> out(static_cast<size_t>(L), Mail(static_cast<size_t>(W))), in;
  for (int i = 0; i < L; ++i) {
    const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    const auto& t = T[static_cast<size_t>(i)];
    for (int q = 0; q < W; ++q)
      out[static_cast<size_t>(i)][static_cast<size_t>(q)] = {R.np, t.empty() ? INT64_MAX : t.front(), t.empty() ? -1 : t.back()};
  }
  deliver(g, out, in, s);
  std::vector<std::vector<int64_t>> info(static_cast<size_t>(L));  // [i] -> np, tmin, tmax per rank
  for (int i = 0; i < L; ++i) {
    SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    R.k0 = 0;
    for (int q = 0; q < W; ++q) {
      auto m = in[static_cast<size_t>(i)][static_cast<size_t>(q)];
      if (m.empty()) m = {0, INT64_MAX, -1};  // absent rank (emulated subset)
      info[static_cast<size_t>(i)].insert(info[static_cast<size_t>(i)].end(), m.begin(), m.end());
      if (q < R.rank) R.k0 += m[0];
    }
  }
  int64_t np_total = 0;
  for (int q = 0; q < W; ++q) np_total += info[0][static_cast<size_t>(3 * q)];
  g.k0_of.assign(static_cast<size_t>(W), 0);
  g.np_of.assign(static_cast<size_t>(W), 0);
  for (int q = 0; q < W; ++q) {
    g.np_of[static_cast<size_t>(q)] = info[0][static_cast<size_t>(3 * q)];
    if (q > 0) g.k0_of[static_cast<size_t>(q)] = g.k0_of[static_cast<size_t>(q) - 1] + g.np_of[static_cast<size_t>(q) - 1];
  }
  tph.emplace("slab setup: phase 2 (touched DoFs, weights, ownership)", s);
  // (2) touched DoFs (with counts) to every rank whose touched range overlaps
  for (int i = 0; i < L; ++i) {
    const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    const auto& t = T[static_cast<size_t>(i)];
    const auto& c = Tc[static_cast<size_t>(i)];
    for (int q = 0; q < W; ++q) {
      auto& m = out[static_cast<size_t>(i)][static_cast<size_t>(q)];
      m.clear();
      if (q == R.rank) continue;
      const int64_t lo = info[static_cast<size_t>(i)][static_cast<size_t>(3 * q + 1)], hi = info[static_cast<size_t>(i)][static_cast<size_t>(3 * q + 2)];
      for (size_t k = std::lower_bound(t.begin(), t.end(), lo) - t.begin(); k < t.size() && t[k] <= hi; ++k) {
        m.push_back(t[k]);
        m.push_back(c[k]);
      }
    }
  }
  deliver(g, out, in, s);
  std::vector<std::vector<int64_t>> need(static_cast<size_t>(L));       // local ids whose x comes from elsewhere
  std::vector<std::vector<int32_t>> owner_of(static_cast<size_t>(L));  // per touched DoF
  for (int i = 0; i < L; ++i) {
    SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    const auto& t = T[static_cast<size_t>(i)];
    std::vector<int64_t> total(Tc[static_cast<size_t>(i)]);
    std::vector<int32_t> lo_rank(t.size(), R.rank), hi_rank(t.size(), R.rank);
    for (int q = 0; q < W; ++q) {
      const auto& m = in[static_cast<size_t>(i)][static_cast<size_t>(q)];
      for (size_t k = 0; k + 1 < m.size(); k += 2) {
        const auto it = std::lower_bound(t.begin(), t.end(), m[k]);
        if (it == t.end() || *it != m[k]) continue;  // in my range but not touched by me
        const size_t j = static_cast<size_t>(it - t.begin());
        total[j] += m[k + 1];
        lo_rank[j] = std::min(lo_rank[j], q);
        hi_rank[j] = std::max(hi_rank[j], q);
      }
    }
    std::vector<double> w(static_cast<size_t>(R.nl), 0.0);
    std::vector<int32_t> up_l, up_p, pin_l, pin_p, plain;
    std::vector<char> owned(static_cast<size_t>(R.nl), 0);
    plain.reserve(t.size());
    int64_t l = 0;  // t and R.gid are both ascending and t is a subset: one merge walk
    for (size_t j = 0; j < t.size(); ++j) {
      while (R.gid[static_cast<size_t>(l)] != t[j]) ++l;
      w[static_cast<size_t>(l)] = 1.0 / static_cast<double>(total[j]);  // compute_weights (patch.cpp:12-20)
      require(hi_rank[j] - lo_rank[j] <= 1, Errc::invalid_argument,
              "slab partition too thin: a DoF is shared by non-adjacent ranks (use fewer ranks)");
      if (hi_rank[j] > R.rank) {
        up_l.push_back(static_cast<int32_t>(l));
        up_p.push_back(hi_rank[j]);
      } else {
        owned[static_cast<size_t>(l)] = 1;
        if (lo_rank[j] < R.rank) {
          pin_l.push_back(static_cast<int32_t>(l));
          pin_p.push_back(lo_rank[j]);
        } else {
          plain.push_back(static_cast<int32_t>(l));
        }
      }
    }
    // lists are in ascending global order already; group by peer (stable)
    auto group = [](std::vector<int32_t>& l, std::vector<int32_t>& p) {
      std::vector<size_t> o(l.size());
      for (size_t k = 0; k < o.size(); ++k) o[k] = k;
      std::stable_sort(o.begin(), o.end(), [&](size_t a, size_t b) { return p[a] < p[b]; });
      std::vector<int32_t> l2, p2;
      for (size_t k : o) l2.push_back(l[k]), p2.push_back(p[k]);
      l.swap(l2);
      p.swap(p2);
    };
    group(up_l, up_p);
    group(pin_l, pin_p);
    R.up_seg = segments_of(up_p);
    R.pin_seg = segments_of(pin_p);
    put(R.up, up_l, s);
    put(R.pin, pin_l, s);
    put(R.own_plain, plain, s);
    put(R.own_pin, pin_l, s);
    R.n_own = static_cast<int64_t>(plain.size() + pin_l.size());
    R.zup.alloc(std::max<size_t>(up_l.size(), 1));
    R.zin.alloc(std::max<size_t>(pin_l.size(), 1));
    // global weights for the local patch set
    R.ps.weights.alloc(static_cast<size_t>(std::max<int64_t>(R.nl, 1)));
    R.ps.weights.upload(w.data(), w.size(), s);
    std::vector<double> ow(w.size());
    for (size_t k = 0; k < w.size(); ++k) ow[k] = omega * w[k];
    put(R.omega_w, ow, s);
    for (int64_t l = 0; l < R.nl; ++l)
      if (!owned[static_cast<size_t>(l)]) need[static_cast<size_t>(i)].push_back(l);
    // split point: the patches touching a DoF finished above must be a suffix
    std::vector<char> is_up(static_cast<size_t>(R.nl), 0);
    for (int32_t l : up_l) is_up[static_cast<size_t>(l)] = 1;
    const std::vector<int32_t>& pt = R.pt_host;
    int64_t first = R.np;
    bool suffix = true;
    for (int64_t k = 0; k < R.np; ++k) {
      bool touches = false;
      for (int64_t q = 0; q < patch_size; ++q) touches = touches || is_up[static_cast<size_t>(pt[static_cast<size_t>(k * patch_size + q)])];
      if (touches && first == R.np) first = k;
      if (!touches && first < R.np) suffix = false;
    }
    R.kb = suffix ? first : R.np;
    std::vector<int32_t>().swap(R.pt_host);
  }
  tph.emplace("slab setup: phase 3 (halo requests)", s);
  // (3) x halo requests to every rank whose touched range holds the DoF
  for (int i = 0; i < L; ++i) {
    const SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    for (int q = 0; q < W; ++q) out[static_cast<size_t>(i)][static_cast<size_t>(q)].clear();
    for (int64_t l : need[static_cast<size_t>(i)]) {
      const int64_t gd = R.gid[static_cast<size_t>(l)];
      for (int q = 0; q < W; ++q)
        if (q != R.rank && gd >= info[static_cast<size_t>(i)][static_cast<size_t>(3 * q + 1)] && gd <= info[static_cast<size_t>(i)][static_cast<size_t>(3 * q + 2)])
          out[static_cast<size_t>(i)][static_cast<size_t>(q)].push_back(gd);
    }
  }
  deliver(g, out, in, s);
  std::vector<Mail> req = in;
  tph.emplace("slab setup: phase 4 (replies, lists)", s);
  // (4) replies: 1 where the requested DoF is owned here; those become xs
  for (int i = 0; i < L; ++i) {
    SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    std::vector<char> own(static_cast<size_t>(R.nl), 0);
    if (R.n_own > 0) {
      const std::vector<int32_t> plain = R.own_plain.to_host(s), pinv = R.own_pin.to_host(s);
      const int64_t npin = seg_total(R.pin_seg);
      for (int64_t k = 0; k < R.n_own - npin; ++k) own[static_cast<size_t>(plain[static_cast<size_t>(k)])] = 1;
      for (int64_t k = 0; k < npin; ++k) own[static_cast<size_t>(pinv[static_cast<size_t>(k)])] = 1;
    }
    std::vector<int32_t> xs_l, xs_p;
    for (int q = 0; q < W; ++q) {
      auto& m = out[static_cast<size_t>(i)][static_cast<size_t>(q)];
      m.clear();
      for (int64_t gd : req[static_cast<size_t>(i)][static_cast<size_t>(q)]) {
        const int64_t l = local_of(R, gd);
        const bool mine = l >= 0 && own[static_cast<size_t>(l)];
        m.push_back(mine ? 1 : 0);
        if (mine) xs_l.push_back(static_cast<int32_t>(l)), xs_p.push_back(q);
      }
    }
    R.xs_seg = segments_of(xs_p);
    put(R.xs, xs_l, s);
    R.xsend.alloc(std::max<size_t>(xs_l.size(), 1));
  }
  deliver(g, out, in, s);
  for (int i = 0; i < L; ++i) {
    SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    std::vector<int32_t> xr_l, xr_p;
    std::vector<int> got(static_cast<size_t>(R.nl), 0);
    // re-derive what this rank asked each peer (same order as step 3)
    std::vector<std::vector<int64_t>> asked(static_cast<size_t>(W));
    for (int64_t l : need[static_cast<size_t>(i)]) {
      const int64_t gd = R.gid[static_cast<size_t>(l)];
      for (int q = 0; q < W; ++q)
        if (q != R.rank && gd >= info[static_cast<size_t>(i)][static_cast<size_t>(3 * q + 1)] && gd <= info[static_cast<size_t>(i)][static_cast<size_t>(3 * q + 2)])
          asked[static_cast<size_t>(q)].push_back(gd);
    }
    for (int q = 0; q < W; ++q) {
      const auto& rep = in[static_cast<size_t>(i)][static_cast<size_t>(q)];
      if (g.emulated && g.slot_of(q) < 0) continue;  // absent rank: no reply
      require(rep.size() == asked[static_cast<size_t>(q)].size(), Errc::internal, "slab setup: reply size mismatch");
      for (size_t k = 0; k < rep.size(); ++k)
        if (rep[k]) {
          const int64_t l = local_of(R, asked[static_cast<size_t>(q)][k]);
          ++got[static_cast<size_t>(l)];
          xr_l.push_back(static_cast<int32_t>(l));
          xr_p.push_back(q);
        }
    }
    for (int64_t l : need[static_cast<size_t>(i)])
      require(got[static_cast<size_t>(l)] <= 1, Errc::internal, "slab setup: a DoF has two owners");
    // DoFs no rank touches keep their initial x (the serial sweep leaves them unchanged)
    R.xr_seg = segments_of(xr_p);
    put(R.xr, xr_l, s);
    R.xrecv.alloc(std::max<size_t>(xr_l.size(), 1));
  }
  tph.reset();
  // (5) factors and the DoF -> slot map
  TraceScope tr_f("slab setup: database + factors + maps", s);
  pdb_database_s built;  // distributed greedy: replicated entries, per-rank phi in R.phi
  if (!db && build) {
    if (build->method == PDB_METHOD_KMEANS_ENTRYWISE)
      slab_kmeans(g, patch_size, *build, built, s);
    else
      slab_greedy(g, patch_size, *build, built, s);
    db = &built;
  }
  for (int i = 0; i < L; ++i) {
    SlabRank& R = *g.ranks[static_cast<size_t>(i)];
    pdb_patchset_s lo, hi;
    sub_patchset(R.ps, 0, R.kb, lo, s);
    sub_patchset(R.ps, R.kb, R.np, hi, s);
    if (db == &built) {
      auto part = [&](pdb_patchset_s& sp, int64_t off, pdb_precond_s& pc) {
        if (sp.np == 0) return;
        pdb_database_s ldb;
        ldb.m = built.m;
        ldb.np = sp.np;
        ldb.ps = built.ps;
        const size_t len = static_cast<size_t>(built.ps * built.ps);
        ldb.lu.alloc(built.m * len);
        PDB_CUDA(cudaMemcpyAsync(ldb.lu.get(), built.lu.get(), built.m * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
        ldb.piv.alloc(static_cast<size_t>(built.m * built.ps));
        PDB_CUDA(cudaMemcpyAsync(ldb.piv.get(), built.piv.get(), built.m * built.ps * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        std::vector<int32_t> ph(R.phi.begin() + off, R.phi.begin() + off + sp.np);
        put(ldb.phi, ph, s);
        precond_compressed_shard(sp, ldb, omega, pc, s);
      };
      part(lo, 0, R.pc_lo);
      part(hi, R.kb, R.pc_hi);
    } else if (db) {
      require(db->np == np_total, Errc::dimension_mismatch, "database does not cover the global patch set");
      require(db->ps == patch_size, Errc::dimension_mismatch, "database entry dimension does not match the patch size");
      auto part = [&](pdb_patchset_s& sp, int64_t off, pdb_precond_s& pc) {
        if (sp.np == 0) return;
        pdb_database_s ldb;
        ldb.m = db->m;
        ldb.np = sp.np;
        ldb.ps = db->ps;
        const size_t len = static_cast<size_t>(db->ps * db->ps);
        ldb.lu.alloc(db->m * len);
        PDB_CUDA(cudaMemcpyAsync(ldb.lu.get(), db->lu.get(), db->m * len * sizeof(double), cudaMemcpyDeviceToDevice, s));
        ldb.piv.alloc(static_cast<size_t>(db->m * db->ps));
        PDB_CUDA(cudaMemcpyAsync(ldb.piv.get(), db->piv.get(), db->m * db->ps * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        ldb.phi.alloc(static_cast<size_t>(sp.np));
        PDB_CUDA(cudaMemcpyAsync(ldb.phi.get(), db->phi.get() + R.k0 + off, sp.np * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        precond_compressed_shard(sp, ldb, omega, pc, s);
      };
      part(lo, 0, R.pc_lo);
      part(hi, R.kb, R.pc_hi);
    } else {
      if (lo.np > 0) precond_exact(R.a, lo, omega, R.pc_lo, s);
      if (hi.np > 0) precond_exact(R.a, hi, omega, R.pc_hi, s);
    }
    common_setup(R.ps, omega, R.map, s);
    build_inverse(R.map, s);
    // the residual streams the SELL copy: drop the CSR's columns and values
    // (config 5: 40 GB per rank) once the patches are extracted
    if (R.a.nslices > 0 && plan_of(R.a).version == 9) {
      R.a.col = DevBuf<int32_t>();
      R.a.val = DevBuf<double>();
    }
    R.r.alloc(static_cast<size_t>(std::max<int64_t>(R.nl, 1)));
    R.sols.alloc(static_cast<size_t>(std::max<int64_t>(R.np * patch_size, 1)));
    R.init.alloc(static_cast<size_t>(std::max<int64_t>(R.nl, 1)));
    R.init.zero(s);
  }
  sync(s);
}

namespace {

// sweep phases of one rank
void phase_interface(SlabRank& R, const double* b, double* x, cudaStream_t s) {
  const k::SpmvPlan plan = plan_of(R.a);
  k::residual(plan, R.nl, R.a.row_ptr.get(), R.a.col.get(), R.a.val.get(), x, b, R.r.get(), nullptr, s);
  if (R.np > R.kb) patch_stage(R.pc_hi, R.r.get(), nullptr, R.sols.get() + R.kb * R.ps.ps, s);
  if (R.kb == R.np && R.kb > 0) patch_stage(R.pc_lo, R.r.get(), nullptr, R.sols.get(), s);  // no split: everything now
  // partial sums of the DoFs finished above (their patches are all done)
  k::shard_scatter(seg_total(R.up_seg), R.up.get(), R.map.inv_ptr.get(), R.map.inv.get(), R.sols.get(), nullptr, nullptr, R.zup.get(),
                   nullptr, s);
}

void phase_interior(SlabRank& R, double* x, cudaStream_t s) {
  if (R.kb < R.np && R.kb > 0) patch_stage(R.pc_lo, R.r.get(), nullptr, R.sols.get(), s);
  const int64_t nplain = R.n_own - seg_total(R.pin_seg);
  k::shard_scatter(nplain, R.own_plain.get(), R.map.inv_ptr.get(), R.map.inv.get(), R.sols.get(), nullptr,
                   R.omega_w.get(), nullptr, x, s);
}

void phase_lower(SlabRank& R, double* x, cudaStream_t s) {
  const int64_t npin = seg_total(R.pin_seg);
  if (npin == 0) return;
  k::scatter_vals(npin, R.pin.get(), R.zin.get(), R.init.get(), s);
  k::shard_scatter(npin, R.own_pin.get(), R.map.inv_ptr.get(), R.map.inv.get(), R.sols.get(), R.init.get(),
                   R.omega_w.get(), nullptr, x, s);
}

void exchange_nccl(SlabRank& R, const std::vector<Seg>& sends, double* sbuf, const std::vector<Seg>& recvs,
                   double* rbuf, cudaStream_t s) {
  if (sends.empty() && recvs.empty()) return;
  PDB_NCCL_S(ncclGroupStart());
  for (const auto& g : sends) PDB_NCCL_S(ncclSend(sbuf + g.off, static_cast<size_t>(g.cnt), ncclDouble, g.peer, R.comm, s));
  for (const auto& g : recvs) PDB_NCCL_S(ncclRecv(rbuf + g.off, static_cast<size_t>(g.cnt), ncclDouble, g.peer, R.comm, s));
  PDB_NCCL_S(ncclGroupEnd());
}

// emulated group: copy rank r's segment for q into q's receive segment from r
void exchange_local(pdb_slab_s& g, bool partials, cudaStream_t s) {
  for (auto& Rp : g.ranks) {
    SlabRank& R = *Rp;
    const auto& sends = partials ? R.up_seg : R.xs_seg;
    const double* sbuf = partials ? R.zup.get() : R.xsend.get();
    for (const auto& sg : sends) {
      if (g.slot_of(sg.peer) < 0) continue;  // absent rank (emulated subset)
      SlabRank& Q = *g.ranks[static_cast<size_t>(g.slot_of(sg.peer))];
      const auto& recvs = partials ? Q.pin_seg : Q.xr_seg;
      double* rbuf = partials ? Q.zin.get() : Q.xrecv.get();
      bool found = false;
      for (const auto& rg : recvs)
        if (rg.peer == R.rank) {
          require(rg.cnt == sg.cnt, Errc::internal, "slab exchange: segment sizes differ");
          PDB_CUDA(cudaMemcpyAsync(rbuf + rg.off, sbuf + sg.off, sg.cnt * sizeof(double), cudaMemcpyDeviceToDevice, s));
          found = true;
        }
      require(found, Errc::internal, "slab exchange: no matching receive");
    }
  }
}

}  // namespace

// NCCL rank: interface first, exchanges on the side stream.
void slab_relax_rank(SlabRank& R, const double* b, double* x, int64_t sweeps, cudaStream_t s) {
  if (R.nranks > 1) {
    require(R.comm != nullptr, Errc::invalid_argument, "shard has no communicator");
    if (!R.side) {
      PDB_CUDA(cudaStreamCreateWithFlags(&R.side, cudaStreamNonBlocking));
      for (auto& e : R.ev) PDB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  for (int64_t sw = 0; sw < sweeps; ++sw) {
    phase_interface(R, b, x, s);
    if (R.nranks > 1) {
      PDB_CUDA(cudaEventRecord(R.ev[0], s));
      PDB_CUDA(cudaStreamWaitEvent(R.side, R.ev[0], 0));
      exchange_nccl(R, R.up_seg, R.zup.get(), R.pin_seg, R.zin.get(), R.side);
      PDB_CUDA(cudaEventRecord(R.ev[1], R.side));
    }
    phase_interior(R, x, s);  // overlaps the partial-sum exchange
    if (R.nranks > 1) PDB_CUDA(cudaStreamWaitEvent(s, R.ev[1], 0));
    phase_lower(R, x, s);
    const int64_t nxs = seg_total(R.xs_seg);
    if (R.nranks > 1) {
      if (nxs) k::gather_vals(nxs, R.xs.get(), x, R.xsend.get(), s);
      PDB_CUDA(cudaEventRecord(R.ev[2], s));
      PDB_CUDA(cudaStreamWaitEvent(R.side, R.ev[2], 0));
      exchange_nccl(R, R.xs_seg, R.xsend.get(), R.xr_seg, R.xrecv.get(), R.side);
      PDB_CUDA(cudaEventRecord(R.ev[3], R.side));
      PDB_CUDA(cudaStreamWaitEvent(s, R.ev[3], 0));
      const int64_t nxr = seg_total(R.xr_seg);
      if (nxr) k::scatter_vals(nxr, R.xr.get(), R.xrecv.get(), x, s);
    }
  }
  PDB_LAUNCH_CHECK();
}

// Emulated group: W ranks' phases in order, exchanges as device copies.
void slab_relax_group(pdb_slab_s& g, const std::vector<const double*>& b, const std::vector<double*>& x,
                      int64_t sweeps, cudaStream_t s) {
  const size_t W = g.ranks.size();
  for (int64_t sw = 0; sw < sweeps; ++sw) {
    for (size_t r = 0; r < W; ++r) phase_interface(*g.ranks[r], b[r], x[r], s);
    exchange_local(g, true, s);
    for (size_t r = 0; r < W; ++r) phase_interior(*g.ranks[r], x[r], s);
    for (size_t r = 0; r < W; ++r) phase_lower(*g.ranks[r], x[r], s);
    for (size_t r = 0; r < W; ++r) {
      SlabRank& R = *g.ranks[r];
      const int64_t nxs = seg_total(R.xs_seg);
      if (nxs) k::gather_vals(nxs, R.xs.get(), x[r], R.xsend.get(), s);
    }
    exchange_local(g, false, s);
    for (size_t r = 0; r < W; ++r) {
      SlabRank& R = *g.ranks[r];
      const int64_t nxr = seg_total(R.xr_seg);
      if (nxr) k::scatter_vals(nxr, R.xr.get(), R.xrecv.get(), x[r], s);
    }
  }
  PDB_LAUNCH_CHECK();
}

// One local rank's sweep phases alone (exchanges skipped): the per-rank work
// of a sweep, timed on a single GPU for a slice of a larger job.
void slab_relax_one(pdb_slab_s& g, int i, const double* b, double* x, int64_t sweeps, cudaStream_t s) {
  SlabRank& R = *g.ranks[static_cast<size_t>(i)];
  for (int64_t sw = 0; sw < sweeps; ++sw) {
    phase_interface(R, b, x, s);
    phase_interior(R, x, s);
    phase_lower(R, x, s);
    const int64_t nxs = seg_total(R.xs_seg), nxr = seg_total(R.xr_seg);
    if (nxs) k::gather_vals(nxs, R.xs.get(), x, R.xsend.get(), s);
    if (nxr) k::scatter_vals(nxr, R.xr.get(), R.xrecv.get(), x, s);
  }
  PDB_LAUNCH_CHECK();
}

pdb_slab_s* slab_new(int rank, int nranks, bool emulated, const std::vector<int>& ranks) {
  require(nranks >= 1 && rank >= 0 && rank < nranks, Errc::invalid_argument, "rank must be in [0, nranks)");
  auto g = std::make_unique<pdb_slab_s>();
  g->emulated = emulated;
  if (emulated) {
    std::vector<int> rl = ranks;
    if (rl.empty())
      for (int r = 0; r < nranks; ++r) rl.push_back(r);
    g->slot.assign(static_cast<size_t>(nranks), -1);
    for (int r : rl) {
      g->slot[static_cast<size_t>(r)] = static_cast<int>(g->ranks.size());
      g->ranks.push_back(std::make_unique<SlabRank>());
      g->ranks.back()->rank = r;
      g->ranks.back()->nranks = nranks;
    }
  } else {
    g->ranks.push_back(std::make_unique<SlabRank>());
    g->ranks.back()->rank = rank;
    g->ranks.back()->nranks = nranks;
  }
  return g.release();
}

void slab_delete(pdb_slab_s* g) { delete g; }

void slab_attach(pdb_slab_s& g, const unsigned char* id128) {
  require(!g.emulated, Errc::invalid_argument, "an emulated group needs no communicator");
  SlabRank& R = *g.ranks[0];
  ncclUniqueId uid;
  std::memcpy(uid.internal, id128, sizeof(uid.internal));
  PDB_NCCL_S(ncclCommInitRank(&R.comm, R.nranks, uid, R.rank));
}

const SlabRank& slab_rank(const pdb_slab_s& g, int i) {
  require(i >= 0 && i < static_cast<int>(g.ranks.size()), Errc::invalid_argument, "rank index out of range");
  return *g.ranks[static_cast<size_t>(i)];
}

void slab_relax(pdb_slab_s& g, const std::vector<const double*>& b, const std::vector<double*>& x, int64_t sweeps,
                cudaStream_t s) {
  if (g.emulated)
    slab_relax_group(g, b, x, sweeps, s);
  else
    slab_relax_rank(*g.ranks[0], b[0], x[0], sweeps, s);
}

int slab_local_ranks(const pdb_slab_s& g) { return static_cast<int>(g.ranks.size()); }

double slab_upload_seconds(const pdb_slab_s& g) {
  double t = 0.0;
  for (const auto& r : g.ranks) t += r->upload_s;
  return t;
}

SlabInfo slab_info(const pdb_slab_s& g, int i) {
  const SlabRank& R = slab_rank(g, i);
  return SlabInfo{R.rank, R.nranks, R.nl, static_cast<int64_t>(R.rows.size()), R.np, R.k0, R.kb, R.n_own,
                  seg_total(R.up_seg), seg_total(R.pin_seg), seg_total(R.xs_seg), seg_total(R.xr_seg)};
}

void slab_local_dofs(const pdb_slab_s& g, int i, int64_t* out) {
  const SlabRank& R = slab_rank(g, i);
  std::copy(R.gid.begin(), R.gid.end(), out);
}

void slab_owned(const pdb_slab_s& g, int i, int64_t* out) {
  const SlabRank& R = slab_rank(g, i);
  cudaStream_t s = cudaStreamPerThread;
  const int64_t npin = seg_total(R.pin_seg);
  std::vector<int64_t> o;
  if (R.n_own > 0) {
    const std::vector<int32_t> plain = R.own_plain.to_host(s), pinv = R.own_pin.to_host(s);
    for (int64_t k = 0; k < R.n_own - npin; ++k) o.push_back(plain[static_cast<size_t>(k)]);
    for (int64_t k = 0; k < npin; ++k) o.push_back(pinv[static_cast<size_t>(k)]);
  }
  std::sort(o.begin(), o.end());
  std::copy(o.begin(), o.end(), out);
}

int64_t slab_database_size(const pdb_slab_s& g) { return g.m; }

void slab_phi(const pdb_slab_s& g, int i, int64_t* out) {
  const SlabRank& R = slab_rank(g, i);
  require(!R.phi.empty() || R.np == 0, Errc::invalid_argument, "slab has no rank-local database");
  for (int64_t k = 0; k < R.np; ++k) out[k] = R.phi[static_cast<size_t>(k)];
}

void slab_creators(const pdb_slab_s& g, int64_t* out) { std::copy(g.creators.begin(), g.creators.end(), out); }

}  // namespace pdb
