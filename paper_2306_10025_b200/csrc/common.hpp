// Shared host-side plumbing: error model, CUDA checks, device buffers.
//
// Error model mirrors the reference (errors.hpp:8-39): an exception carrying
// a machine-readable code, mapped to pdb_status at the C-ABI boundary
// (capi.cpp).  CUDA failures become Errc::internal.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

namespace pdb {

using Index = std::int64_t;

enum class Errc {
  invalid_argument = 1,
  dimension_mismatch = 2,
  singular_matrix = 3,
  index_out_of_range = 4,
  duplicate_index = 5,
  parse_error = 6,
  non_square_matrix = 7,
  no_patches_found = 8,
  empty_cluster = 9,
  budget_too_small = 10,
  invalid_degree = 11,
  non_positive_coefficient = 12,
  io_error = 13,
  internal = 14,
};

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

[[noreturn]] inline void fail(Errc code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool cond, Errc code, const char* msg) {
  if (!cond) fail(code, msg);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    fail(Errc::internal, std::string("CUDA error in ") + what + " (" + file + ":" + std::to_string(line) +
                             "): " + cudaGetErrorString(e));
}
#define PDB_CUDA(call) ::pdb::cuda_check((call), #call, __FILE__, __LINE__)
#define PDB_LAUNCH_CHECK() ::pdb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Lazily verifies that a usable sm_100 device is present.  There is no CPU
// fallback: every compute entry point calls this first.
void require_device();

// Owning device allocation (cudaMalloc); movable, not copyable.
template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { alloc(n); }
  ~DevBuf() { reset(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void alloc(std::size_t n) {
    reset();
    if (n == 0) return;
    if (pooled()) {
      // the device's stream-ordered pool (kept, not returned to the driver:
      // require_device sets the release threshold), synchronised so the
      // buffer is usable from any stream at once
      PDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), cudaStreamPerThread));
      PDB_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
    } else {
      PDB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)));
    }
    n_ = n;
  }
  void reset() {
    if (p_) {
      if (pooled()) {
        cudaDeviceSynchronize();  // what cudaFree implies: no stream may still use the buffer
        cudaFreeAsync(p_, cudaStreamPerThread);
      } else {
        cudaFree(p_);
      }
    }
    p_ = nullptr;
    n_ = 0;
  }
  // PDB_DEVBUF_POOL=0: plain cudaMalloc / cudaFree
  static bool pooled() {
    static const bool on = [] {
      const char* e = std::getenv("PDB_DEVBUF_POOL");
      return !(e && e[0] == '0');
    }();
    return on;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  std::size_t bytes() const { return n_ * sizeof(T); }
  void upload(const T* h, std::size_t n, cudaStream_t s) {
    if (n) PDB_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(T* h, std::size_t n, cudaStream_t s) const {
    if (n) PDB_CUDA(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host(cudaStream_t s) const {
    std::vector<T> h(n_);
    download(h.data(), n_, s);
    PDB_CUDA(cudaStreamSynchronize(s));
    return h;
  }
  void zero(cudaStream_t s) {
    if (n_) PDB_CUDA(cudaMemsetAsync(p_, 0, bytes(), s));
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

// Stream-ordered scratch allocation (cudaMallocAsync pool), freed on the same stream.
template <typename T>
class Scratch {
 public:
  Scratch(std::size_t n, cudaStream_t s) : s_(s), n_(n) {
    if (n) PDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
  }
  ~Scratch() {
    if (p_) cudaFreeAsync(p_, s_);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  Scratch(Scratch&& o) noexcept : s_(o.s_), p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* h, std::size_t n) {
    if (n) PDB_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s_));
  }
  void download(T* h, std::size_t n) const {
    if (n) PDB_CUDA(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s_));
  }
  void zero() {
    if (n_) PDB_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s_));
  }

 private:
  cudaStream_t s_;
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

inline cudaStream_t default_stream() { return cudaStreamPerThread; }
inline void sync(cudaStream_t s) { PDB_CUDA(cudaStreamSynchronize(s)); }

// PDB_TRACE=1: wall time of a scope, stream-synchronised at both ends, on stderr.
class TraceScope {
 public:
  // accum_s (optional): the scope's seconds are also added there, traced or not
  TraceScope(const char* name, cudaStream_t s, double* accum_s = nullptr) : name_(name), s_(s), accum_(accum_s) {
    static const bool on = [] {
      const char* e = std::getenv("PDB_TRACE");
      return e && e[0] == '1';
    }();
    on_ = on;
    if (on_ || accum_) {
      cudaStreamSynchronize(s_);
      t0_ = std::chrono::steady_clock::now();
    }
  }
  ~TraceScope() {
    if (!on_ && !accum_) return;
    cudaStreamSynchronize(s_);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
    if (accum_) *accum_ += ms * 1e-3;
    if (on_) std::fprintf(stderr, "[trace] %s %.2f ms\n", name_, ms);
  }
  TraceScope(const TraceScope&) = delete;
  TraceScope& operator=(const TraceScope&) = delete;

 private:
  const char* name_;
  cudaStream_t s_;
  double* accum_ = nullptr;
  bool on_ = false;
  std::chrono::steady_clock::time_point t0_;
};

int num_sms();

// TMA descriptor (a CUtensorMap) of a preconditioner's fragment-ordered inverses, see kernels.hpp.
struct FragTensorMap {
  alignas(64) unsigned char opaque[128];
};

}  // namespace pdb
