// SELL-C-sigma copy of a device-resident CSR matrix, built on the device:
// the same arrays as the host build_sell (matrix.cpp) -- column-pattern
// classes numbered in order of first occurrence, rows sorted stably by
// (length descending, class ascending) inside windows of kSellSigma rows,
// slices of kSellC rows stored column-major -- so the residual that streams
// it is bitwise the same.  Host work is limited to the class table (at most
// 4096 patterns) and the window/slice counts, which depend on n only.
//
//   row hash        FNV-1a of (length, col - row ...), one thread per row
//   patterns        radix sort of (hash, row); a pattern's representative is
//                   its first row; classes numbered by that row
//   verification    every row against its class's offset list (a hash
//                   collision or too many patterns: explicit columns)
//   window sort     radix sort of (window, ~length, class) keys over the
//                   row ids: stable, as std::stable_sort
//   slices          width = length of the slice's first (longest) row,
//                   offsets by an exclusive scan, values (and columns) copied
//                   by one warp per slice (coalesced 256-byte stores)
#include <algorithm>
#include <numeric>

#include <cub/cub.cuh>

#include "host.hpp"
#include "kernels.hpp"

namespace pdb {

namespace {

constexpr int kB = 256;
inline unsigned gridn(int64_t n, int b) { return (unsigned)std::max<int64_t>(1, (n + b - 1) / b); }

__global__ void row_hash_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                uint64_t* __restrict__ hash, int32_t* __restrict__ ids,
                                unsigned long long* __restrict__ max_len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p0 = rp[i], p1 = rp[i + 1];
  uint64_t x = 1469598103934665603ull ^ (uint64_t)(p1 - p0);
  for (int64_t p = p0; p < p1; ++p) {
    x ^= (uint64_t)(uint32_t)(col[p] - (int32_t)i);
    x *= 1099511628211ull;
  }
  hash[i] = x;
  ids[i] = (int32_t)i;
  atomicMax(max_len, (unsigned long long)(p1 - p0));
}

__global__ void heads_kernel(int64_t n, const uint64_t* __restrict__ hs, int32_t* __restrict__ head) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) head[k] = (k == 0 || hs[k] != hs[k - 1]) ? 1 : 0;
}

// seg = inclusive scan of head - 1: the pattern of sorted position k
__global__ void pattern_reps_kernel(int64_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ seg,
                                    const int32_t* __restrict__ rows_sorted, int32_t* __restrict__ rep) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && head[k]) rep[seg[k] - 1] = rows_sorted[k];
}

__global__ void row_class_kernel(int64_t n, const int32_t* __restrict__ seg, const int32_t* __restrict__ rows_sorted,
                                 const int32_t* __restrict__ cls_of_pattern, int32_t* __restrict__ cls) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) cls[rows_sorted[k]] = cls_of_pattern[seg[k] - 1];
}

// every row's offsets equal its class's list (sell_classes' `same`)
__global__ void verify_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const int32_t* __restrict__ cls, const int32_t* __restrict__ tab,
                              const int32_t* __restrict__ tstart, int32_t* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cls[i];
  const int64_t p0 = rp[i], L = rp[i + 1] - p0;
  const int32_t t0 = tstart[c], tl = tstart[c + 1] - t0;
  bool ok = L == tl;
  for (int64_t j = 0; ok && j < L; ++j) ok = col[p0 + j] - (int32_t)i == tab[t0 + j];
  if (!ok) atomicOr(bad, 1);
}

// window-sort key: window (20 bits) | 2^31-1 - length (31 bits) | class + 1 (13 bits)
__global__ void sort_key_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cls,
                                uint64_t* __restrict__ key, int32_t* __restrict__ ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t w = (uint64_t)(i / k::kSellSigma);
  const uint64_t L = (uint64_t)(rp[i + 1] - rp[i]);
  const uint64_t c = cls ? (uint64_t)(cls[i] + 1) : 0;
  key[i] = (w << 44) | ((0x7FFFFFFFull - L) << 13) | c;
  ids[i] = (int32_t)i;
}

// slice sl of window w: rows perm[r0 + q * 32 + l]; width = length of lane 0's row
__global__ void slice_width_kernel(int64_t ns, int64_t n, int64_t nwin, const int64_t* __restrict__ win_slice,
                                   const int32_t* __restrict__ perm, const int64_t* __restrict__ rp,
                                   int64_t* __restrict__ width32) {
  const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= ns) return;
  int64_t lo = 0, hi = nwin - 1;  // window of the slice: win_slice[w] <= sl < win_slice[w + 1]
  while (lo < hi) {
    const int64_t m = (lo + hi + 1) >> 1;
    if (win_slice[m] <= sl) lo = m;
    else hi = m - 1;
  }
  const int64_t first = lo * k::kSellSigma + (sl - win_slice[lo]) * k::kSellC;
  const int32_t row = perm[first];
  width32[sl] = (int64_t)k::kSellC * (rp[row + 1] - rp[row]);
  (void)n;
}

// one warp per slice: descriptors, then entry j of lane l's row at off + 32 j + l
__global__ void slice_fill_kernel(int64_t ns, int64_t n, int64_t nwin, const int64_t* __restrict__ win_slice,
                                  const int32_t* __restrict__ perm, const int64_t* __restrict__ rp,
                                  const int32_t* __restrict__ col, const double* __restrict__ val,
                                  const int32_t* __restrict__ cls, const int64_t* __restrict__ off,
                                  int2* __restrict__ rows, double* __restrict__ sval, int32_t* __restrict__ scol) {
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= ns) return;
  int64_t lo = 0, hi = nwin - 1;
  while (lo < hi) {
    const int64_t m = (lo + hi + 1) >> 1;
    if (win_slice[m] <= sl) lo = m;
    else hi = m - 1;
  }
  const int64_t r1 = std::min<int64_t>(n, (lo + 1) * k::kSellSigma);
  const int64_t at = lo * k::kSellSigma + (sl - win_slice[lo]) * k::kSellC + lane;
  int32_t row = -1;
  int64_t p0 = 0, L = 0;
  if (at < r1) {
    row = perm[at];
    p0 = rp[row];
    L = rp[row + 1] - p0;
    rows[sl * k::kSellC + lane] = make_int2(row, cls ? (int32_t)(L | ((int64_t)(cls[row] + 1) << 16)) : (int32_t)L);
  } else {
    rows[sl * k::kSellC + lane] = make_int2(-1, 0);
  }
  const int64_t o = off[sl], width = (off[sl + 1] - o) / k::kSellC;
  for (int64_t j = 0; j < width; ++j) {
    const bool live = j < L;
    sval[o + j * k::kSellC + lane] = live ? val[p0 + j] : 0.0;
    if (scol) scol[o + j * k::kSellC + lane] = live ? col[p0 + j] : 0;
  }
}

template <typename K, typename V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int end_bit, cudaStream_t s) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit, s);
  Scratch<unsigned char> tmp(bytes, s);
  cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kin, kout, vin, vout, n, 0, end_bit, s);
}

// Column-pattern classes of the device CSR (sell_classes, matrix.cpp): true
// and cls / tab / tstart filled when every row is in one of at most
// min(4096, n/8) patterns with an offset table of at most 2^20 entries.
bool classes_device(const DeviceCsr& d, DevBuf<int32_t>& cls, std::vector<int32_t>& tab, std::vector<int32_t>& tstart,
                    cudaStream_t s) {
  const int64_t n = d.n;
  Scratch<uint64_t> hash(n, s), hs(n, s);
  Scratch<int32_t> ids(n, s), rs(n, s);
  Scratch<unsigned long long> mx(1, s);
  PDB_CUDA(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned long long), s));
  row_hash_kernel<<<gridn(n, kB), kB, 0, s>>>(n, d.row_ptr.get(), d.col.get(), hash.get(), ids.get(), mx.get());
  PDB_LAUNCH_CHECK();
  unsigned long long max_len = 0;
  PDB_CUDA(cudaMemcpyAsync(&max_len, mx.get(), sizeof(max_len), cudaMemcpyDeviceToHost, s));
  sync(s);
  if (max_len > 0xFFFF) return false;
  sort_pairs(hash.get(), hs.get(), ids.get(), rs.get(), n, 64, s);
  Scratch<int32_t> head(n, s), seg(n, s);
  heads_kernel<<<gridn(n, kB), kB, 0, s>>>(n, hs.get(), head.get());
  {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, head.get(), seg.get(), n, s);
    Scratch<unsigned char> tmp(bytes, s);
    cub::DeviceScan::InclusiveSum(tmp.get(), bytes, head.get(), seg.get(), n, s);
  }
  int32_t U = 0;
  PDB_CUDA(cudaMemcpyAsync(&U, seg.get() + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync(s);
  if (U > std::max<int64_t>(1, std::min<int64_t>(4096, n / 8))) return false;
  Scratch<int32_t> rep(U, s);
  pattern_reps_kernel<<<gridn(n, kB), kB, 0, s>>>(n, head.get(), seg.get(), rs.get(), rep.get());
  PDB_LAUNCH_CHECK();
  std::vector<int32_t> reph(static_cast<size_t>(U));
  rep.download(reph.data(), reph.size());
  sync(s);
  // classes in order of first occurrence (the host numbering)
  std::vector<int32_t> order(static_cast<size_t>(U));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return reph[static_cast<size_t>(a)] < reph[static_cast<size_t>(b)]; });
  std::vector<int32_t> cls_of(static_cast<size_t>(U));
  for (int32_t c = 0; c < U; ++c) cls_of[static_cast<size_t>(order[static_cast<size_t>(c)])] = c;
  // offset lists of the representatives, in class order
  std::vector<int64_t> rp_all;  // row_ptr[rep], row_ptr[rep + 1] per class
  tstart.assign(1, 0);
  tab.clear();
  std::vector<int64_t> lo(static_cast<size_t>(U)), len(static_cast<size_t>(U));
  for (int32_t c = 0; c < U; ++c) {
    const int32_t r = reph[static_cast<size_t>(order[static_cast<size_t>(c)])];
    int64_t pr[2];
    PDB_CUDA(cudaMemcpyAsync(pr, d.row_ptr.get() + r, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    sync(s);
    lo[static_cast<size_t>(c)] = pr[0];
    len[static_cast<size_t>(c)] = pr[1] - pr[0];
    if (static_cast<int64_t>(tab.size()) + len[static_cast<size_t>(c)] > (int64_t{1} << 20)) return false;
    std::vector<int32_t> cc(static_cast<size_t>(len[static_cast<size_t>(c)]));
    if (!cc.empty())
      PDB_CUDA(cudaMemcpyAsync(cc.data(), d.col.get() + pr[0], cc.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    sync(s);
    for (int32_t v : cc) tab.push_back(v - r);
    tstart.push_back(static_cast<int32_t>(tab.size()));
  }
  Scratch<int32_t> cop(U, s), dtab(std::max<size_t>(tab.size(), 1), s), dts(tstart.size(), s), bad(1, s);
  cop.upload(cls_of.data(), cls_of.size());
  if (!tab.empty()) dtab.upload(tab.data(), tab.size());
  dts.upload(tstart.data(), tstart.size());
  cls.alloc(static_cast<size_t>(n));
  row_class_kernel<<<gridn(n, kB), kB, 0, s>>>(n, seg.get(), rs.get(), cop.get(), cls.get());
  PDB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int32_t), s));
  verify_kernel<<<gridn(n, kB), kB, 0, s>>>(n, d.row_ptr.get(), d.col.get(), cls.get(), dtab.get(), dts.get(),
                                            bad.get());
  PDB_LAUNCH_CHECK();
  int32_t bh = 0;
  PDB_CUDA(cudaMemcpyAsync(&bh, bad.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync(s);
  return bh == 0;
}

}  // namespace

void build_sell_device(DeviceCsr& d, cudaStream_t s) {
  const int64_t n = d.n;
  if (n == 0 || d.nnz == 0) return;
  require(n < (int64_t{1} << 31) && n / k::kSellSigma < (int64_t{1} << 20), Errc::invalid_argument,
          "matrix too large for the SELL copy");
  DevBuf<int32_t> cls;
  std::vector<int32_t> tab, tstart;
  const char* ce = getenv("PDB_SELL_CLASSES");
  const bool classed = !(ce && ce[0] == '0') && classes_device(d, cls, tab, tstart, s);
  d.mirror = false;
  d.mir_why = classed ? "not requested (PDB_SELL_MIRROR=1)" : "rows do not share column patterns";
  // window sort
  Scratch<uint64_t> key(n, s), ks(n, s);
  Scratch<int32_t> ids(n, s);
  DevBuf<int32_t> perm(static_cast<size_t>(n));
  sort_key_kernel<<<gridn(n, kB), kB, 0, s>>>(n, d.row_ptr.get(), classed ? cls.get() : nullptr, key.get(), ids.get());
  PDB_LAUNCH_CHECK();
  sort_pairs(key.get(), ks.get(), ids.get(), perm.get(), n, 64, s);
  // windows and slices (depend on n only)
  const int64_t nwin = (n + k::kSellSigma - 1) / k::kSellSigma;
  std::vector<int64_t> win_slices(static_cast<size_t>(nwin) + 1, 0);
  for (int64_t w = 0; w < nwin; ++w) {
    const int64_t r0 = w * k::kSellSigma, r1 = std::min(n, r0 + k::kSellSigma);
    win_slices[static_cast<size_t>(w) + 1] = win_slices[static_cast<size_t>(w)] + (r1 - r0 + k::kSellC - 1) / k::kSellC;
  }
  const int64_t ns = win_slices.back();
  Scratch<int64_t> dws(win_slices.size(), s), w32(ns + 1, s);
  dws.upload(win_slices.data(), win_slices.size());
  d.sell_off.alloc(static_cast<size_t>(ns + 1));
  slice_width_kernel<<<gridn(ns, kB), kB, 0, s>>>(ns, n, nwin, dws.get(), perm.get(), d.row_ptr.get(), w32.get());
  PDB_CUDA(cudaMemsetAsync(w32.get() + ns, 0, sizeof(int64_t), s));
  {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, w32.get(), d.sell_off.get(), ns + 1, s);
    Scratch<unsigned char> tmp(bytes, s);
    cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, w32.get(), d.sell_off.get(), ns + 1, s);
  }
  int64_t total = 0;
  PDB_CUDA(cudaMemcpyAsync(&total, d.sell_off.get() + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  sync(s);
  d.sell_row.alloc(static_cast<size_t>(2 * ns * k::kSellC));
  d.sell_val.alloc(static_cast<size_t>(std::max<int64_t>(total, 1)));
  d.sell_col.alloc(classed ? 1 : static_cast<size_t>(std::max<int64_t>(total, 1)));
  slice_fill_kernel<<<gridn(ns * 32, kB), kB, 0, s>>>(
      ns, n, nwin, dws.get(), perm.get(), d.row_ptr.get(), d.col.get(), d.val.get(), classed ? cls.get() : nullptr,
      d.sell_off.get(), reinterpret_cast<int2*>(d.sell_row.get()), d.sell_val.get(), classed ? nullptr : d.sell_col.get());
  PDB_LAUNCH_CHECK();
  d.sell_classes = classed ? static_cast<int64_t>(tstart.size()) - 1 : 0;
  if (classed) {
    d.sell_tab.alloc(std::max<size_t>(tab.size(), 1));
    d.sell_tab.upload(tab.data(), tab.size(), s);
    d.sell_tstart.alloc(tstart.size());
    d.sell_tstart.upload(tstart.data(), tstart.size(), s);
  }
  d.nslices = ns;
  d.win_slice = win_slices;
  sync(s);
}

}  // namespace pdb
