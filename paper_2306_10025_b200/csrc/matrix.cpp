// Device CSR matrices: validation + upload, SpMV (Matrix Market I/O in
// mmio.cpp).  Reference: sparse.hpp:20-39 (CSR invariants).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>

#include "host.hpp"
#include "kernels.hpp"

namespace pdb {

void require_device() {
  static int state = -1;  // -1 unknown, 0 absent, 1 ok
  static std::string why;
  if (state < 0) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
      state = 0;
      why = e != cudaSuccess ? cudaGetErrorString(e) : "no device";
    } else {
      cudaDeviceProp prop;
      int dev = 0;
      cudaGetDevice(&dev);
      cudaGetDeviceProperties(&prop, dev);
      if (prop.major < 10) {
        state = 0;
        why = std::string("device ") + prop.name + " is not sm_100";
      } else {
        state = 1;
        // keep freed stream-ordered scratch cached in the pool instead of
        // returning it to the driver at every synchronisation
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          uint64_t keep = UINT64_MAX;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
      }
    }
  }
  if (state == 0) fail(Errc::internal, "CUDA device unavailable (" + why + "); patchdb-b200 has no CPU path");
}

int num_sms() {  // of the current device (cached per device)
  static int sms_of[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int dummy = 0;
  int& sms = dev < 64 ? sms_of[dev] : dummy;
  if (!sms) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!sms) sms = 148;
  }
  return sms;
}

// SELL-C-sigma (Kreutzer et al., SIAM J. Sci. Comput. 2014) copy of the
// matrix for the v9 residual: rows are sorted by length (descending, stable)
// inside windows of kSellSigma rows and cut into slices of kSellC = 32; a
// slice is stored column-major (entry j of its l-th row at off + 32 j + l),
// so lane l of a warp walks row l and every load of the warp is one
// contiguous 256-byte (values) / 128-byte (columns) span.  Each lane sums its
// row sequentially in CSR order -- no cross-lane reduction, and with
// unfused multiply/add the residual is bitwise the reference spmv's.
bool sell_classes(const HostCsr& h, std::vector<int32_t>& cls, std::vector<int32_t>& tab, std::vector<int32_t>& tstart) {
  const int64_t n = h.n;
  cls.assign(static_cast<size_t>(n), -1);
  tab.clear();
  tstart.assign(1, 0);
  if (n == 0) return false;
  const int64_t nwin = (n + k::kSellSigma - 1) / k::kSellSigma;
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  auto len = [&](int64_t i) { return h.row_ptr[static_cast<size_t>(i + 1)] - h.row_ptr[static_cast<size_t>(i)]; };
  auto par = [&](auto&& body) {
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t)
      pool.emplace_back([&, t] {
        for (int64_t w = nwin * t / T; w < nwin * (t + 1) / T; ++w) body(w);
      });
    for (auto& th : pool) th.join();
  };
  int64_t max_len = 0;
  for (int64_t i = 0; i < n; ++i) max_len = std::max<int64_t>(max_len, len(i));
  if (max_len > 0xFFFF) return false;
  std::vector<uint64_t> hash(static_cast<size_t>(n));
  par([&](int64_t w) {
    const int64_t r0 = w * k::kSellSigma, r1 = std::min(n, r0 + k::kSellSigma);
    for (int64_t i = r0; i < r1; ++i) {
      uint64_t x = 1469598103934665603ull ^ static_cast<uint64_t>(len(i));
      for (int64_t p = h.row_ptr[static_cast<size_t>(i)]; p < h.row_ptr[static_cast<size_t>(i + 1)]; ++p) {
        x ^= static_cast<uint64_t>(static_cast<uint32_t>(h.col[static_cast<size_t>(p)] - static_cast<int32_t>(i)));
        x *= 1099511628211ull;
      }
      hash[static_cast<size_t>(i)] = x;
    }
  });
  auto same = [&](int64_t a, int64_t b) {
    const int64_t la = len(a);
    if (la != len(b)) return false;
    const int32_t* ca = h.col.data() + h.row_ptr[static_cast<size_t>(a)];
    const int32_t* cb = h.col.data() + h.row_ptr[static_cast<size_t>(b)];
    for (int64_t j = 0; j < la; ++j)
      if (ca[j] - static_cast<int32_t>(a) != cb[j] - static_cast<int32_t>(b)) return false;
    return true;
  };
  std::unordered_map<uint64_t, int32_t> pid;
  std::vector<int64_t> rep;
  for (int64_t i = 0; i < n; ++i) {
    auto it = pid.find(hash[static_cast<size_t>(i)]);
    if (it == pid.end()) {
      // a lattice has a handful of patterns; past n/8 of them (or a 4 MB
      // offset table) the rows do not share patterns: explicit columns
      if (static_cast<int64_t>(rep.size()) >= std::max<int64_t>(1, std::min<int64_t>(4096, n / 8)) ||
          tab.size() + static_cast<size_t>(len(i)) > (size_t{1} << 20)) {
        cls.assign(static_cast<size_t>(n), -1);
        tab.clear();
        tstart.assign(1, 0);
        return false;
      }
      it = pid.emplace(hash[static_cast<size_t>(i)], static_cast<int32_t>(rep.size())).first;
      rep.push_back(i);
      const int32_t* c = h.col.data() + h.row_ptr[static_cast<size_t>(i)];
      for (int64_t j = 0; j < len(i); ++j) tab.push_back(c[j] - static_cast<int32_t>(i));
      tstart.push_back(static_cast<int32_t>(tab.size()));
    }
    if (!same(rep[static_cast<size_t>(it->second)], i)) {
      cls.assign(static_cast<size_t>(n), -1);
      tab.clear();
      tstart.assign(1, 0);
      return false;
    }
    cls[static_cast<size_t>(i)] = it->second;
  }
  return true;
}

namespace {

void upload_mirror(MirrorHost& M, const std::vector<int32_t>& tab, const std::vector<int32_t>& tstart, DeviceCsr& d,
                   cudaStream_t s) {
  d.sell_off.alloc(M.soff.size());
  d.sell_off.upload(M.soff.data(), M.soff.size(), s);
  d.sell_row.alloc(M.rows.size());
  d.sell_row.upload(M.rows.data(), M.rows.size(), s);
  d.sell_val.alloc(M.val.size());
  d.sell_val.upload(M.val.data(), M.val.size(), s);
  d.sell_col.alloc(1);
  d.sell_tab.alloc(tab.size());
  d.sell_tab.upload(tab.data(), tab.size(), s);
  d.sell_tstart.alloc(tstart.size());
  d.sell_tstart.upload(tstart.data(), tstart.size(), s);
  d.sell_classes = static_cast<int64_t>(tstart.size()) - 1;
  d.mir_clo.alloc(M.clo.size());
  d.mir_clo.upload(M.clo.data(), M.clo.size(), s);
  d.mir_rbase.alloc(M.rbase.size());
  d.mir_rbase.upload(M.rbase.data(), M.rbase.size(), s);
  d.mir_kslot.alloc(M.kslot.size());
  d.mir_kslot.upload(M.kslot.data(), M.kslot.size(), s);
  d.mir_virtual = M.virtual_rows;
  d.win_slice = M.win_slice;
  d.nslices = M.nslices;
  d.mirror = true;
  sync(s);  // the host vectors go out of scope after the copies
}

}  // namespace

void build_sell(const HostCsr& h, DeviceCsr& d, cudaStream_t s) {
  const int64_t n = h.n;
  if (n == 0 || h.nnz() == 0) return;
  const int64_t nwin = (n + k::kSellSigma - 1) / k::kSellSigma;
  std::vector<int32_t> perm(static_cast<size_t>(n));
  std::vector<int64_t> win_slices(static_cast<size_t>(nwin) + 1, 0);
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  auto len = [&](int64_t i) { return h.row_ptr[static_cast<size_t>(i + 1)] - h.row_ptr[static_cast<size_t>(i)]; };
  auto par = [&](auto&& body) {
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t)
      pool.emplace_back([&, t] {
        for (int64_t w = nwin * t / T; w < nwin * (t + 1) / T; ++w) body(w);
      });
    for (auto& th : pool) th.join();
  };
  // ---- column-pattern classes: used only when every row falls into one
  // (PDB_SELL_CLASSES=0 disables them); then the half-storage layout when
  // its preconditions hold (PDB_SELL_MIRROR=0 disables it)
  std::vector<int32_t> cls, tab, tstart;
  const char* ce = getenv("PDB_SELL_CLASSES");
  const bool classed = !(ce && ce[0] == '0') && sell_classes(h, cls, tab, tstart);
  if (!classed) {
    cls.assign(static_cast<size_t>(n), -1);
    tab.clear();
    tstart.assign(1, 0);
  }
  d.mirror = false;
  d.mir_why = classed ? "" : "rows do not share column patterns";
  if (classed) {
    // opt-in (capacity mode): half the residual bytes, but measured slower
    // than the plain classed copy on B200
    const char* me = getenv("PDB_SELL_MIRROR");
    if (!(me && me[0] == '1')) {
      d.mir_why = "not requested (PDB_SELL_MIRROR=1)";
    } else {
      MirrorHost M;
      if (build_mirror_host(h, cls, tab, tstart, k::kSellSigma, M)) {
        upload_mirror(M, tab, tstart, d, s);
        return;
      }
      d.mir_why = M.why;
    }
  }
  par([&](int64_t w) {
    const int64_t r0 = w * k::kSellSigma, r1 = std::min(n, r0 + k::kSellSigma);
    for (int64_t i = r0; i < r1; ++i) perm[static_cast<size_t>(i)] = static_cast<int32_t>(i);
    std::stable_sort(perm.begin() + r0, perm.begin() + r1, [&](int32_t a, int32_t b) {
      const int64_t la = len(a), lb = len(b);
      if (la != lb) return la > lb;
      return cls[static_cast<size_t>(a)] < cls[static_cast<size_t>(b)];
    });
    win_slices[static_cast<size_t>(w) + 1] = (r1 - r0 + k::kSellC - 1) / k::kSellC;
  });
  for (int64_t w = 0; w < nwin; ++w) win_slices[static_cast<size_t>(w) + 1] += win_slices[static_cast<size_t>(w)];
  const int64_t ns = win_slices.back();
  // slice widths and offsets (slices are numbered window by window)
  std::vector<int64_t> off(static_cast<size_t>(ns) + 1, 0);
  for (int64_t w = 0; w < nwin; ++w) {
    const int64_t r0 = w * k::kSellSigma, r1 = std::min(n, r0 + k::kSellSigma);
    for (int64_t q = 0; q < win_slices[static_cast<size_t>(w) + 1] - win_slices[static_cast<size_t>(w)]; ++q) {
      const int64_t sl = win_slices[static_cast<size_t>(w)] + q;
      const int64_t first = r0 + q * k::kSellC;  // longest row of the slice
      off[static_cast<size_t>(sl) + 1] = off[static_cast<size_t>(sl)] + k::kSellC * len(perm[static_cast<size_t>(first)]);
      (void)r1;
    }
  }
  std::vector<int32_t> rows(static_cast<size_t>(2 * ns * k::kSellC), 0);
  std::vector<double> val(static_cast<size_t>(off.back()), 0.0);
  std::vector<int32_t> col(classed ? 1 : static_cast<size_t>(off.back()), 0);
  par([&](int64_t w) {
    const int64_t r0 = w * k::kSellSigma, r1 = std::min(n, r0 + k::kSellSigma);
    for (int64_t q = 0; q < win_slices[static_cast<size_t>(w) + 1] - win_slices[static_cast<size_t>(w)]; ++q) {
      const int64_t sl = win_slices[static_cast<size_t>(w)] + q;
      const int64_t o = off[static_cast<size_t>(sl)];
      for (int l = 0; l < k::kSellC; ++l) {
        const int64_t at = r0 + q * k::kSellC + l;
        const size_t ri = static_cast<size_t>(2 * (sl * k::kSellC + l));
        if (at >= r1) {
          rows[ri] = -1;
          rows[ri + 1] = 0;
          continue;
        }
        const int32_t row = perm[static_cast<size_t>(at)];
        const int64_t p0 = h.row_ptr[static_cast<size_t>(row)], L = len(row);
        rows[ri] = row;
        rows[ri + 1] = static_cast<int32_t>(classed ? (L | (static_cast<int64_t>(cls[static_cast<size_t>(row)] + 1) << 16)) : L);
        for (int64_t j = 0; j < L; ++j) {
          val[static_cast<size_t>(o + j * k::kSellC + l)] = h.val[static_cast<size_t>(p0 + j)];
          if (!classed) col[static_cast<size_t>(o + j * k::kSellC + l)] = h.col[static_cast<size_t>(p0 + j)];
        }
      }
    }
  });
  d.sell_off.alloc(off.size());
  d.sell_off.upload(off.data(), off.size(), s);
  d.sell_row.alloc(rows.size());
  d.sell_row.upload(rows.data(), rows.size(), s);
  d.sell_val.alloc(val.size());
  d.sell_val.upload(val.data(), val.size(), s);
  d.sell_col.alloc(col.size());
  d.sell_col.upload(col.data(), col.size(), s);
  d.sell_classes = classed ? static_cast<int64_t>(tstart.size()) - 1 : 0;
  if (classed) {
    d.sell_tab.alloc(tab.size());
    d.sell_tab.upload(tab.data(), tab.size(), s);
    d.sell_tstart.alloc(tstart.size());
    d.sell_tstart.upload(tstart.data(), tstart.size(), s);
  }
  d.nslices = ns;
  d.win_slice = win_slices;
  sync(s);
}

// Host -> device copy of a large pageable array: chunks are copied into two
// pinned staging buffers by host threads and DMA'd from there, the copy of
// chunk i + 1 overlapping the transfer of chunk i (the driver's own pageable
// path moves one staging block at a time).  Pinned sources and small arrays
// take cudaMemcpyAsync directly.  Synchronous on return.
void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  constexpr size_t kChunk = size_t{64} << 20;
  if (bytes == 0) return;
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();  // a pageable pointer may leave an error on older drivers
  if (pinned || bytes < 4 * kChunk) {
    PDB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    sync(s);
    return;
  }
  struct Stage {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
  };
  static Stage stage_of[64];  // per device (events belong to one device)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  PDB_CUDA(cudaGetDevice(&dev));
  require(dev < 64, Errc::internal, "device ordinal beyond the per-device caches");
  Stage& st = stage_of[dev];
  for (int b = 0; b < 2; ++b)
    if (!st.buf[b]) {
      PDB_CUDA(cudaMallocHost(&st.buf[b], kChunk));
      PDB_CUDA(cudaEventCreateWithFlags(&st.ev[b], cudaEventDisableTiming));
    }
  const int T = static_cast<int>(std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  size_t i = 0;
  for (size_t off = 0; off < bytes; off += kChunk, ++i) {
    const size_t n = std::min(kChunk, bytes - off);
    const int b = static_cast<int>(i & 1);
    if (i >= 2) PDB_CUDA(cudaEventSynchronize(st.ev[b]));  // its previous transfer is done
    char* buf = static_cast<char*>(st.buf[b]);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t)
      pool.emplace_back([&, t] {
        const size_t a = n * t / T, e = n * (t + 1) / T;
        std::memcpy(buf + a, sp + off + a, e - a);
      });
    for (auto& th : pool) th.join();
    PDB_CUDA(cudaMemcpyAsync(dp + off, buf, n, cudaMemcpyHostToDevice, s));
    PDB_CUDA(cudaEventRecord(st.ev[b], s));
  }
  sync(s);
}

void alloc_csr(Index n, Index nnz, DeviceCsr& d, cudaStream_t s) {
  require_device();
  d.n = n;
  d.nnz = nnz;
  d.row_ptr.alloc(static_cast<size_t>(n + 1));
  // 32 zeroed elements of tail padding: the bulk-copy SpMV widens spans to
  // 16-byte bounds and may read past the last nonzero
  constexpr size_t kPad = 32;
  d.col.alloc(static_cast<size_t>(nnz) + kPad);
  d.val.alloc(static_cast<size_t>(nnz) + kPad);
  PDB_CUDA(cudaMemsetAsync(d.col.get() + nnz, 0, kPad * sizeof(int32_t), s));
  PDB_CUDA(cudaMemsetAsync(d.val.get() + nnz, 0, kPad * sizeof(double), s));
}

void finish_csr(const HostCsr& h, const std::vector<int64_t>& row_ptr, DeviceCsr& d, cudaStream_t s) {
  // warp items of the CSR residual (v5)
  const std::vector<int32_t> part = k::item_partition(d.n, row_ptr.data());
  d.nitems = static_cast<int>(part.size()) - 1;
  d.item_start.alloc(part.size());
  d.item_start.upload(part.data(), part.size(), s);
  std::vector<int64_t> base(part.size());
  for (size_t b = 0; b < part.size(); ++b) base[b] = row_ptr[static_cast<size_t>(part[b])];
  d.item_base.alloc(base.size());
  d.item_base.upload(base.data(), base.size(), s);
  sync(s);
  const char* e = getenv("PDB_SPMV_SELL");
  if (e && std::string(e) == "0") return;
  // the SELL copy is built on the device from the uploaded CSR; the host
  // build stays for the opt-in half storage (PDB_SELL_MIRROR=1) and for A/B
  // runs (PDB_SELL_DEVICE=0) -- the two produce the same arrays
  const char* me = getenv("PDB_SELL_MIRROR");
  const char* de = getenv("PDB_SELL_DEVICE");
  if (!(me && me[0] == '1') && !(de && de[0] == '0')) {
    TraceScope tr("build_sell (device)", s);
    build_sell_device(d, s);
  } else {
    require(h.n == d.n && h.nnz() == d.nnz, Errc::internal, "host build of the SELL copy needs the host CSR");
    TraceScope tr("build_sell (host)", s);
    build_sell(h, d, s);
  }
}

void upload_csr(const HostCsr& h, DeviceCsr& d, cudaStream_t s) {
  alloc_csr(h.n, h.nnz(), d, s);
  h2d_staged(d.row_ptr.get(), h.row_ptr.data(), h.row_ptr.size() * sizeof(int64_t), s);
  h2d_staged(d.col.get(), h.col.data(), h.col.size() * sizeof(int32_t), s);
  h2d_staged(d.val.get(), h.val.data(), h.val.size() * sizeof(double), s);
  finish_csr(h, h.row_ptr, d, s);
}

// Residual plan: the SELL-C-sigma copy by default; PDB_SPMV_VERSION=5 / 2
// selects the CSR warp-item / row-group kernels (A/B, or no SELL copy).
k::SpmvPlan plan_of(const DeviceCsr& a) {
  const char* ver = getenv("PDB_SPMV_VERSION");
  const int v = ver ? atoi(ver) : 9;
  if (v == 9 && a.nslices > 0) {
    k::SpmvPlan p = k::spmv_plan(a.n, a.nnz);
    p.version = 9;
    const char* e = getenv("PDB_SPMV_PER");
    p.entries = e && atoi(e) == 4 ? 4 : 8;  // steps in flight per lane (measured: 8 > 4)
    p.sell_off = a.sell_off.get();
    p.sell_row = a.sell_row.get();
    p.sell_val = a.sell_val.get();
    p.sell_col = a.sell_col.get();
    p.nslices = a.nslices;
    if (a.sell_classes > 0) {
      p.sell_tab = a.sell_tab.get();
      p.sell_tstart = a.sell_tstart.get();
    }
    if (a.mirror) {
      p.mir_clo = a.mir_clo.get();
      p.mir_rbase = a.mir_rbase.get();
      p.mir_kslot = a.mir_kslot.get();
      p.mir_ntab = static_cast<int>(a.sell_tab.size());
      p.mir_ncls = static_cast<int>(a.sell_classes);
      p.mir_nval = static_cast<int64_t>(a.sell_val.size());
    }
    p.blocks = static_cast<int>((a.nslices + 7) / 8);
    return p;
  }
  if (v == 2) return k::spmv_plan(a.n, a.nnz);
  return k::spmv_plan_items(a.n, a.nnz, a.item_start.get(), a.item_base.get(), a.nitems);
}

HostCsr validated_csr(Index n, const int64_t* rp, const int64_t* ci, const double* v) {
  require(n >= 0, Errc::invalid_argument, "negative matrix dimension");
  require(n < (Index{1} << 31), Errc::invalid_argument, "matrix has more than 2^31-1 rows");
  require(rp[0] == 0, Errc::invalid_argument, "row_ptr[0] must be 0");
  HostCsr h;
  h.n = n;
  h.row_ptr.assign(rp, rp + n + 1);
  for (Index i = 0; i < n; ++i)
    require(rp[i + 1] >= rp[i], Errc::invalid_argument, "row_ptr must be nondecreasing");
  const Index nnz = rp[n];
  h.col.resize(static_cast<size_t>(nnz));
  h.val.assign(v, v + nnz);
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  std::vector<int> bad(static_cast<size_t>(T), 0);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      const Index b = n * t / T, e = n * (t + 1) / T;
      for (Index i = b; i < e && !bad[t]; ++i)
        for (Index p = rp[i]; p < rp[i + 1]; ++p) {
          const Index c = ci[p];
          if (c < 0 || c >= n) {
            bad[t] = 1;
            break;
          }
          if (p > rp[i] && ci[p - 1] >= c) {
            bad[t] = 2;
            break;
          }
          if (!std::isfinite(v[p])) {
            bad[t] = 3;
            break;
          }
          h.col[static_cast<size_t>(p)] = static_cast<int32_t>(c);
        }
    });
  for (auto& th : pool) th.join();
  for (int b : bad) {
    if (b == 1) fail(Errc::index_out_of_range, "column index outside matrix");
    if (b == 2) fail(Errc::invalid_argument, "column indices must be strictly increasing within each row");
    if (b == 3) fail(Errc::invalid_argument, "non-finite matrix entry");
  }
  return h;
}

HostCsr download_csr(const DeviceCsr& d, cudaStream_t s) {
  HostCsr h;
  h.n = d.n;
  h.row_ptr = d.row_ptr.to_host(s);
  h.col = d.col.to_host(s);
  h.val = d.val.to_host(s);
  h.col.resize(static_cast<size_t>(d.nnz));  // drop the tail padding
  h.val.resize(static_cast<size_t>(d.nnz));
  return h;
}

void spmv_device(const DeviceCsr& a, const double* x, double* y, cudaStream_t s) {
  const k::SpmvPlan plan = plan_of(a);
  k::spmv(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, y, s);
  PDB_LAUNCH_CHECK();
}

}  // namespace pdb
