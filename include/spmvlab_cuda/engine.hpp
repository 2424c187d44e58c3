// spmvlab_cuda/engine.hpp -- source-compatible C++ drop-in for the reference's algorithm interface
// (/root/reference/proj/include/spmvlab/engine.hpp), forwarding to the C ABI in spmvlab_cuda.h.
//
// Same names and semantics as the reference, in namespace spmvlab::cuda:
//   Algorithm, all_algorithms, algorithm_name, algorithm_from_name   (engine.hpp:30-72)
//   EngineOptions                                                    (engine.hpp:75-79)
//   BuiltFormat build_format(Algorithm, const Triplet&, threads, opt) (engine.hpp:96-122)
//   void run_spmv(Algorithm, const BuiltFormat&, const Vec& x, Vec& y, p, opt)  (engine.hpp:126-148)
//   Vec  run_spmv(Algorithm, const BuiltFormat&, const Vec& x, p, opt)          (engine.hpp:150-156)
//   StorageBreakdown storage_report(const BuiltFormat&)              (engine.hpp:158-160)
//   Error / ErrorKind                                                (types.hpp:47-104)
// `Triplet` is any type with the reference TripletMatrix members (m, n, row_ind, col_ind, data as
// contiguous containers) -- spmvlab::TripletMatrix itself works unchanged.  Calls are synchronous
// like the reference (host vectors in, host vectors out); run_spmv_device() is the stream-ordered
// device-pointer entry point for resident data.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../spmvlab_cuda.h"

namespace spmvlab::cuda {

enum class Algorithm { SeqCrs, ParCrs, Merge, Csb, Csbh, Bcoh, Bcohc, Bcohch, Bcohchp, MergeB, MergeBH };

inline constexpr std::array<Algorithm, 11> all_algorithms = {
    Algorithm::SeqCrs, Algorithm::ParCrs,  Algorithm::Merge,  Algorithm::Csb,
    Algorithm::Csbh,   Algorithm::Bcoh,    Algorithm::Bcohc,  Algorithm::Bcohch,
    Algorithm::Bcohchp, Algorithm::MergeB, Algorithm::MergeBH,
};

inline const char* algorithm_name(Algorithm alg) {
  static const char* names[] = {"crs", "parcrs", "merge", "csb", "csbh", "bcoh",
                                "bcohc", "bcohch", "bcohchp", "mergeb", "mergebh"};
  const int i = static_cast<int>(alg);
  return i >= 0 && i < 11 ? names[i] : "unknown";
}

enum class ErrorKind {
  DimensionMismatch, InvalidArgument, CorruptFormat, Overflow, BadHeader, UnsupportedFormat,
  UnsupportedField, UnsupportedSymmetry, IndexOutOfRange, DuplicateEntry, ParseError, Truncated,
  BadMagic, IoError,
};

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& message) : std::runtime_error(message), kind_(kind) {}
  ErrorKind kind() const noexcept { return kind_; }

 private:
  ErrorKind kind_;
};

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == 0) return;
  const std::string msg = spmvlab_cuda_last_error();
  if (rc < 100) throw Error(static_cast<ErrorKind>(rc - 1), msg);
  throw CudaError("spmvlab_cuda failure " + std::to_string(rc) + ": " + msg);
}

inline void check_cuda(cudaError_t e) {
  if (e != cudaSuccess) throw CudaError(cudaGetErrorString(e));
}

inline Algorithm algorithm_from_name(const std::string& name) {
  for (Algorithm a : all_algorithms)
    if (name == algorithm_name(a)) return a;
  throw Error(ErrorKind::InvalidArgument, "unknown algorithm '" + name + "'");
}

struct EngineOptions {
  std::uint64_t l2_bytes = 512 * 1024;
  std::size_t split_threshold = 0;
  unsigned build_threads = 1;
  bool deterministic = false;  // blocked formats: bitwise-reproducible y (see spmvlab_cuda_options)
  spmvlab_cuda_options c() const { return {l2_bytes, split_threshold, build_threads, deterministic ? 1u : 0u}; }
};

struct StorageArray {
  std::string name;
  std::size_t bytes = 0;
};

struct StorageBreakdown {
  std::string format;
  std::vector<StorageArray> arrays;
  std::size_t bytes(const std::string& name) const {
    std::size_t t = 0;
    for (const auto& a : arrays)
      if (a.name == name) t += a.bytes;
    return t;
  }
  std::size_t total() const {
    std::size_t t = 0;
    for (const auto& a : arrays) t += a.bytes;
    return t;
  }
  std::size_t index_bytes() const { return total() - bytes("data"); }
};

// RAII device buffer.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t bytes) { resize(bytes); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
    }
    return *this;
  }
  ~DeviceBuffer() { reset(); }
  void resize(std::size_t bytes) {
    if (bytes <= n_) return;
    reset();
    check_cuda(cudaMalloc(&p_, bytes ? bytes : 16));
    n_ = bytes;
  }
  void reset() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }

 private:
  void* p_ = nullptr;
  std::size_t n_ = 0;
};

// A device-resident format (the reference's BuiltFormat variant).  Move-only, immutable.
class BuiltFormat {
 public:
  BuiltFormat() = default;
  BuiltFormat(Algorithm alg, spmvlab_cuda_format* f) : alg_(alg), f_(f) { check(spmvlab_cuda_get_format_info(f_, &info_)); }
  BuiltFormat(const BuiltFormat&) = delete;
  BuiltFormat& operator=(const BuiltFormat&) = delete;
  BuiltFormat(BuiltFormat&& o) noexcept { *this = std::move(o); }
  BuiltFormat& operator=(BuiltFormat&& o) noexcept {
    if (this != &o) {
      if (f_) spmvlab_cuda_free_format(f_);
      alg_ = o.alg_;
      f_ = std::exchange(o.f_, nullptr);
      info_ = o.info_;
      x_stage_ = std::move(o.x_stage_);
      y_stage_ = std::move(o.y_stage_);
    }
    return *this;
  }
  ~BuiltFormat() {
    if (f_) spmvlab_cuda_free_format(f_);
  }

  Algorithm algorithm() const { return alg_; }
  const spmvlab_cuda_format* handle() const { return f_; }
  const spmvlab_cuda_format_info& info() const { return info_; }
  std::uint32_t m() const { return info_.m; }
  std::uint32_t n() const { return info_.n; }
  std::uint64_t nnz() const { return info_.nnz; }

  // Host copy of one named array (reference field names; BCOH band_* / off_* tables too).
  template <typename T>
  std::vector<T> download(const std::string& name) const {
    std::uint64_t bytes = 0;
    check(spmvlab_cuda_download_array(f_, name.c_str(), nullptr, 0, &bytes));
    std::vector<T> out(bytes / sizeof(T));
    if (bytes) check(spmvlab_cuda_download_array(f_, name.c_str(), out.data(), bytes, &bytes));
    return out;
  }

  // Staging buffers for host-vector multiplies (allocated once per format).
  double* x_stage() const {
    x_stage_.resize(sizeof(double) * (info_.n ? info_.n : 1));
    return x_stage_.as<double>();
  }
  double* y_stage() const {
    y_stage_.resize(sizeof(double) * (info_.m ? info_.m : 1));
    return y_stage_.as<double>();
  }

 private:
  Algorithm alg_ = Algorithm::Merge;
  spmvlab_cuda_format* f_ = nullptr;
  spmvlab_cuda_format_info info_{};
  mutable DeviceBuffer x_stage_, y_stage_;
};

// Uploads a host triplet and runs `build` on the device COO view.
template <typename Triplet, typename Build>
BuiltFormat build_from_host(Algorithm alg, const Triplet& a, Build&& build) {
  const std::size_t nnz = a.data.size();
  if (a.row_ind.size() != nnz || a.col_ind.size() != nnz)
    throw Error(ErrorKind::InvalidArgument, "triplet arrays must have equal length");
  DeviceBuffer r(4 * nnz), c(4 * nnz), v(8 * nnz);
  if (nnz) {
    check_cuda(cudaMemcpy(r.as<void>(), a.row_ind.data(), 4 * nnz, cudaMemcpyHostToDevice));
    check_cuda(cudaMemcpy(c.as<void>(), a.col_ind.data(), 4 * nnz, cudaMemcpyHostToDevice));
    check_cuda(cudaMemcpy(v.as<void>(), a.data.data(), 8 * nnz, cudaMemcpyHostToDevice));
  }
  const spmvlab_cuda_coo coo{static_cast<std::uint32_t>(a.m), static_cast<std::uint32_t>(a.n), nnz,
                             r.as<std::uint32_t>(), c.as<std::uint32_t>(), v.as<double>()};
  spmvlab_cuda_format* f = nullptr;
  check(build(&coo, &f));
  return BuiltFormat(alg, f);
}

// build_format (inc/engine.hpp:96-122) from a host triplet.
template <typename Triplet>
BuiltFormat build_format(Algorithm alg, const Triplet& a, unsigned threads, const EngineOptions& opt = {}) {
  const spmvlab_cuda_options o = opt.c();
  return build_from_host(alg, a, [&](const spmvlab_cuda_coo* coo, spmvlab_cuda_format** f) {
    return spmvlab_cuda_build_format(static_cast<int>(alg), coo, threads, &o, f, nullptr);
  });
}

// build_csb / build_mergeb / build_bcoh with an explicit block size 2^log2_beta (inc/csb.hpp:51,
// inc/mergeb.hpp:50, inc/bcoh.hpp:194; `threads` = the BCOH band count p).
template <typename Triplet>
BuiltFormat build_format_beta(Algorithm alg, const Triplet& a, unsigned log2_beta, unsigned threads = 1) {
  return build_from_host(alg, a, [&](const spmvlab_cuda_coo* coo, spmvlab_cuda_format** f) {
    return spmvlab_cuda_build_format_beta(static_cast<int>(alg), coo, log2_beta, threads, f, nullptr);
  });
}

// Stream-ordered multiply on device pointers (no synchronisation).
inline void run_spmv_device(Algorithm alg, const BuiltFormat& f, const double* x_dev, std::size_t x_len,
                            double* y_dev, std::size_t y_len, unsigned p, const EngineOptions& opt = {},
                            cudaStream_t stream = nullptr) {
  const spmvlab_cuda_options o = opt.c();
  check(spmvlab_cuda_run_spmv(static_cast<int>(alg), f.handle(), x_dev, x_len, y_dev, y_len, p, &o, stream));
}

// The cfg5 application loop x <- A x (spmvlab_cuda_iterate): x_dev in/out, work_dev n doubles,
// norms_dev NULL or 2 * iters doubles; stream-ordered (graph=true needs a non-default stream).
inline void iterate_device(Algorithm alg, const BuiltFormat& f, double* x_dev, double* work_dev, std::uint32_t iters,
                           unsigned p, bool normalize = false, bool graph = false, double* norms_dev = nullptr,
                           cudaStream_t stream = nullptr) {
  const int flags = (normalize ? SPMVLAB_ITER_NORMALIZE : 0) | (graph ? SPMVLAB_ITER_GRAPH : 0);
  check(spmvlab_cuda_iterate(static_cast<int>(alg), f.handle(), x_dev, work_dev, iters, p, flags, norms_dev, stream));
}

// run_spmv (inc/engine.hpp:126-148): host vectors, y fully overwritten, synchronous.
template <typename Vec>
void run_spmv(Algorithm alg, const BuiltFormat& f, const Vec& x, Vec& y, unsigned p, const EngineOptions& opt = {}) {
  const spmvlab_cuda_options o = opt.c();
  check(spmvlab_cuda_run_spmv_host(static_cast<int>(alg), f.handle(), x.data(), x.size(), y.data(), y.size(), p,
                                   &o, f.x_stage(), f.y_stage(), nullptr));
  check_cuda(cudaStreamSynchronize(nullptr));
}

template <typename Vec>
Vec run_spmv(Algorithm alg, const BuiltFormat& f, const Vec& x, unsigned p, const EngineOptions& opt = {}) {
  Vec y(f.m(), 0.0);
  run_spmv(alg, f, x, y, p, opt);
  return y;
}

// crs_to_triplet / csb_to_triplet / mergeb_to_triplet / bcoh_to_triplet (crs.hpp:94, csb.hpp:103,
// mergeb.hpp:110, bcoh.hpp:379) for any format: a host triplet (any type with the TripletMatrix
// members) in the reference's output order.
template <typename Triplet>
Triplet to_triplet(const BuiltFormat& f) {
  const std::size_t nnz = f.nnz();
  DeviceBuffer r(4 * nnz), c(4 * nnz), v(8 * nnz);
  check(spmvlab_cuda_format_to_triplet(f.handle(), r.as<std::uint32_t>(), c.as<std::uint32_t>(), v.as<double>(),
                                       nullptr));
  Triplet t;
  t.m = f.m();
  t.n = f.n();
  t.row_ind.resize(nnz);
  t.col_ind.resize(nnz);
  t.data.resize(nnz);
  if (nnz) {
    check_cuda(cudaMemcpy(t.row_ind.data(), r.as<void>(), 4 * nnz, cudaMemcpyDeviceToHost));
    check_cuda(cudaMemcpy(t.col_ind.data(), c.as<void>(), 4 * nnz, cudaMemcpyDeviceToHost));
    check_cuda(cudaMemcpy(t.data.data(), v.as<void>(), 8 * nnz, cudaMemcpyDeviceToHost));
  }
  return t;
}

// The CsbWorkItem list spmv_csb builds (spmv_parallel.hpp:202-264), host copy.
inline std::vector<spmvlab_cuda_csb_item> csb_work_items(const BuiltFormat& f, std::size_t split_threshold = 0) {
  std::uint64_t count = 0;
  check(spmvlab_cuda_csb_work_items(f.handle(), split_threshold, nullptr, 0, &count, nullptr));
  std::vector<spmvlab_cuda_csb_item> out(count);
  if (count) {
    DeviceBuffer d(sizeof(spmvlab_cuda_csb_item) * count);
    check(spmvlab_cuda_csb_work_items(f.handle(), split_threshold, d.as<spmvlab_cuda_csb_item>(), count, &count,
                                      nullptr));
    check_cuda(cudaMemcpy(out.data(), d.as<void>(), sizeof(spmvlab_cuda_csb_item) * count, cudaMemcpyDeviceToHost));
  }
  return out;
}

inline StorageBreakdown storage_report(const BuiltFormat& f) {
  spmvlab_cuda_storage_array rows[16];
  std::size_t count = 0;
  check(spmvlab_cuda_storage_report(f.handle(), rows, 16, &count));
  static const char* formats[] = {"crs", "crs", "crs", "csb", "csbh", "bcoh",
                                  "bcohc", "bcohch", "bcohchp", "mergeb", "mergebh"};
  StorageBreakdown out;
  out.format = formats[static_cast<int>(f.algorithm())];
  for (std::size_t i = 0; i < count; ++i) out.arrays.push_back({rows[i].name, static_cast<std::size_t>(rows[i].bytes)});
  return out;
}

}  // namespace spmvlab::cuda
