// Patch sets: detection (reference detect_patches patch.cpp:37-90),
// extraction (extract_all patch.cpp:92-99), JSON export (patch.cpp:128-143).
// Host orchestration; the integer work runs in kernels/detect.cu.
#include <algorithm>
#include <fstream>
#include <numeric>

#include <cub/cub.cuh>

#include "host.hpp"
#include "kernels.hpp"

namespace pdb {

namespace {

template <typename T>
void select_flagged(const T* in, const uint8_t* flags, T* out, int64_t n, int64_t& count, cudaStream_t s) {
  Scratch<int64_t> num(1, s);
  size_t bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, bytes, in, flags, out, num.get(), n, s);
  Scratch<unsigned char> tmp(bytes, s);
  cub::DeviceSelect::Flagged(tmp.get(), bytes, in, flags, out, num.get(), n, s);
  PDB_CUDA(cudaMemcpyAsync(&count, num.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  sync(s);
}

}  // namespace

void detect_patches(const DeviceCsr& a, Index ps, pdb_patchset_s& out, cudaStream_t s) {
  require(ps >= 2, Errc::invalid_argument, "patch size must be >= 2");
  require_device();
  const Index n = a.n;
  // temporaries are stream-ordered (Scratch): no device-wide synchronisation per buffer
  Scratch<uint8_t> cand(static_cast<size_t>(std::max<Index>(n, 1)), s);
  Scratch<int32_t> any(1, s);
  PDB_CUDA(cudaMemsetAsync(any.get(), 0, sizeof(int32_t), s));
  k::detect_candidates(n, a.row_ptr.get(), ps, cand.get(), any.get(), s);
  PDB_LAUNCH_CHECK();
  int32_t any_h = 0;
  PDB_CUDA(cudaMemcpyAsync(&any_h, any.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync(s);
  if (!any_h) fail(Errc::no_patches_found, "no row has exactly " + std::to_string(ps) + " stored entries");

  // candidate rows, ascending
  Scratch<int32_t> ids(static_cast<size_t>(n), s);
  k::iota(n, ids.get(), s);
  Scratch<int32_t> rows(static_cast<size_t>(n), s);
  int64_t nc = 0;
  select_flagged(ids.get(), cand.get(), rows.get(), n, nc, s);

  // consistency + hash
  Scratch<uint8_t> consistent(static_cast<size_t>(nc), s);
  Scratch<uint64_t> hash(static_cast<size_t>(nc), s);
  k::detect_consistency(nc, rows.get(), a.row_ptr.get(), a.col.get(), cand.get(), static_cast<int>(ps),
                        consistent.get(), hash.get(), s);
  PDB_LAUNCH_CHECK();
  Scratch<int32_t> crow(static_cast<size_t>(nc), s);
  Scratch<uint64_t> chash(static_cast<size_t>(nc), s);
  int64_t ncc = 0, tmpc = 0;
  select_flagged(rows.get(), consistent.get(), crow.get(), nc, ncc, s);
  select_flagged(hash.get(), consistent.get(), chash.get(), nc, tmpc, s);
  if (ncc == 0) fail(Errc::no_patches_found, "no consistent patch candidates detected");

  // dedupe: sort positions by hash (stable radix sort keeps ascending positions within a run)
  Scratch<int32_t> pos(static_cast<size_t>(ncc), s), pos_sorted(static_cast<size_t>(ncc), s);
  Scratch<uint64_t> hash_sorted(static_cast<size_t>(ncc), s);
  k::iota(ncc, pos.get(), s);
  {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, chash.get(), hash_sorted.get(), pos.get(), pos_sorted.get(),
                                    static_cast<int>(ncc), 0, 64, s);
    Scratch<unsigned char> tmp(bytes, s);
    cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, chash.get(), hash_sorted.get(), pos.get(), pos_sorted.get(),
                                    static_cast<int>(ncc), 0, 64, s);
  }
  Scratch<uint8_t> keep(static_cast<size_t>(ncc), s);
  k::detect_dedupe(ncc, hash_sorted.get(), pos_sorted.get(), crow.get(), a.row_ptr.get(), a.col.get(),
                   static_cast<int>(ps), keep.get(), s);
  PDB_LAUNCH_CHECK();
  Scratch<int32_t> emitted(static_cast<size_t>(ncc), s);
  int64_t np = 0;
  select_flagged(crow.get(), keep.get(), emitted.get(), ncc, np, s);

  // fronts -> std::sort by front with the reference comparator (patch.cpp:82-83).
  // When the fronts are distinct the sorted order is unique, so a device radix
  // sort gives it; only fronts shared by two patches need libstdc++'s own
  // (unstable) std::sort on the host.
  Scratch<int32_t> order(static_cast<size_t>(np), s);
  k::iota(np, order.get(), s);
  DevBuf<int32_t> patches(static_cast<size_t>(np * ps));
  k::gather_patches(np, emitted.get(), order.get(), a.row_ptr.get(), a.col.get(), static_cast<int>(ps),
                    patches.get(), s);
  PDB_LAUNCH_CHECK();
  Scratch<int32_t> fronts(static_cast<size_t>(np), s), fronts_sorted(static_cast<size_t>(np), s),
      order_sorted(static_cast<size_t>(np), s), flags(2, s);
  k::patch_fronts(np, static_cast<int>(ps), patches.get(), fronts.get(), s);
  {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, fronts.get(), fronts_sorted.get(), order.get(),
                                    order_sorted.get(), static_cast<int>(np), 0, 32, s);
    Scratch<unsigned char> tmp(bytes, s);
    cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, fronts.get(), fronts_sorted.get(), order.get(),
                                    order_sorted.get(), static_cast<int>(np), 0, 32, s);
  }
  flags.zero();
  k::front_order(np, fronts_sorted.get(), order_sorted.get(), flags.get(), s);
  PDB_LAUNCH_CHECK();
  int32_t fl[2] = {0, 0};
  PDB_CUDA(cudaMemcpyAsync(fl, flags.get(), sizeof(fl), cudaMemcpyDeviceToHost, s));
  sync(s);
  if (fl[0]) {  // shared fronts: the reference comparator's order, on the host
    std::vector<int32_t> fh(static_cast<size_t>(np));
    fronts.download(fh.data(), fh.size());
    sync(s);
    std::vector<std::pair<int64_t, int32_t>> keyed(static_cast<size_t>(np));
    for (int64_t e = 0; e < np; ++e) keyed[static_cast<size_t>(e)] = {fh[static_cast<size_t>(e)], static_cast<int32_t>(e)};
    std::sort(keyed.begin(), keyed.end(),
              [](const std::pair<int64_t, int32_t>& x, const std::pair<int64_t, int32_t>& y) { return x.first < y.first; });
    bool identity = true;
    std::vector<int32_t> ord(static_cast<size_t>(np));
    for (int64_t e = 0; e < np; ++e) {
      ord[static_cast<size_t>(e)] = keyed[static_cast<size_t>(e)].second;
      identity = identity && ord[static_cast<size_t>(e)] == e;
    }
    if (!identity) {
      order.upload(ord.data(), ord.size());
      k::gather_patches(np, emitted.get(), order.get(), a.row_ptr.get(), a.col.get(), static_cast<int>(ps),
                        patches.get(), s);
      PDB_LAUNCH_CHECK();
    }
  } else if (fl[1]) {
    k::gather_patches(np, emitted.get(), order_sorted.get(), a.row_ptr.get(), a.col.get(), static_cast<int>(ps),
                      patches.get(), s);
    PDB_LAUNCH_CHECK();
  }

  out.n = n;
  out.np = np;
  out.ps = ps;
  out.weights.alloc(static_cast<size_t>(std::max<Index>(n, 1)));
  Scratch<int32_t> cover(static_cast<size_t>(std::max<Index>(n, 1)), s);
  cover.zero();
  k::cover_weights(n, np, static_cast<int>(ps), patches.get(), cover.get(), out.weights.get(), s);
  PDB_LAUNCH_CHECK();
  out.patches = std::move(patches);
  sync(s);
}

void extract_patches(const DeviceCsr& a, const pdb_patchset_s& ps, DevBuf<double>& mats, cudaStream_t s) {
  require(ps.n == a.n, Errc::dimension_mismatch, "patch set does not match the matrix size");
  mats.alloc(static_cast<size_t>(ps.np * ps.ps * ps.ps));
  k::extract(ps.np, nullptr, static_cast<int>(ps.ps), ps.patches.get(), a.row_ptr.get(), a.col.get(), a.val.get(),
             mats.get(), s);
  PDB_LAUNCH_CHECK();
}

std::vector<int64_t> patches_host(const pdb_patchset_s& ps, cudaStream_t s) {
  const std::vector<int32_t> p32 = ps.patches.to_host(s);
  return std::vector<int64_t>(p32.begin(), p32.end());
}

void write_patchset_json(const pdb_patchset_s& ps, const std::string& path, cudaStream_t s) {
  const std::vector<int32_t> p = ps.patches.to_host(s);
  std::ofstream out(path);
  if (!out) fail(Errc::io_error, "cannot open '" + path + "' for writing");
  out << "{\n  \"p_s\": " << ps.ps << ",\n  \"patches\": [";
  for (int64_t k = 0; k < ps.np; ++k) {
    out << (k == 0 ? "\n    [" : ",\n    [");
    for (int64_t i = 0; i < ps.ps; ++i) {
      if (i) out << ", ";
      out << p[static_cast<size_t>(k * ps.ps + i)];
    }
    out << "]";
  }
  out << "\n  ]\n}\n";
  if (!out) fail(Errc::io_error, "error while writing '" + path + "'");
}

}  // namespace pdb
