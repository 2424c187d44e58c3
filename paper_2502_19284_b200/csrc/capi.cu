// capi.cu -- the extern "C" boundary (include/spmvlab_cuda.h) over the sm_100a kernels.
//
// Mirrors the reference's algorithm interface (inc/engine.hpp:84-160): engine_block_size,
// build_format, run_spmv (argument checks of check_spmv_args, inc/spmv_parallel.hpp:90-99, and the
// BCOH band check, :339-341), storage_report.  Errors become return codes (ErrorKind + 1).
#include <atomic>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// select_block_size, inc/block_size.hpp:47-61
static unsigned select_block_size(uint64_t n, unsigned cap, uint64_t l2_bytes) {
  if (n < 1) n = 1;
  const unsigned ceil_log2_n = n <= 1 ? 0 : bit_width64(n - 1);
  unsigned lb = 3 + (ceil_log2_n + 1) / 2;
  while (lb > 1) {
    const uint64_t beta = 1ull << lb;
    if (lb <= cap && 2 * beta * 8 <= l2_bytes / 2) break;
    --lb;
  }
  return lb;
}

// engine_block_size, inc/engine.hpp:84-91
static unsigned engine_log2_beta(int alg, uint32_t n, uint64_t l2_bytes) {
  return select_block_size(n < 1 ? 1 : n, is_bcoh_alg(alg) ? 15u : 16u, l2_bytes);
}

// partition_rows_by_nnz, inc/block_size.hpp:73-102 (host; also used by the BCOH build)
int partition_rows_by_nnz_host(const uint32_t* prefix, uint32_t m, unsigned p, unsigned lb,
                               uint32_t* bounds) {
  if (p < 1) return fail(kInvalidArgument, "thread count must be >= 1");
  const uint64_t nnz = prefix[m];
  const uint32_t beta = 1u << lb;
  const uint32_t block_rows = (uint32_t)(((uint64_t)m + beta - 1) >> lb);
  for (unsigned k = 0; k <= p; ++k) bounds[k] = m;
  bounds[0] = 0;
  uint32_t prev_cut = 0;
  for (unsigned k = 1; k < p; ++k) {
    const uint64_t target = nnz * k;
    uint64_t lo = 0, hi = (uint64_t)m + 1;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if ((uint64_t)prefix[mid] * p < target) lo = mid + 1; else hi = mid;
    }
    uint32_t cut = (uint32_t)((lo + beta / 2) >> lb);
    const uint32_t hic = block_rows >= p ? block_rows - (p - k) : block_rows;
    const uint32_t loc = prev_cut + 1 < hic ? prev_cut + 1 : hic;
    if (cut < loc) cut = loc;
    if (cut > hic) cut = hic;
    const uint64_t b = (uint64_t)cut << lb;
    bounds[k] = b < m ? (uint32_t)b : m;
    prev_cut = cut;
  }
  return kOk;
}

// ---------------------------------------------------------------- instrumentation
static std::atomic<uint64_t> g_launches{0};
void note_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
struct KernelTimer {
  std::mutex mu;
  bool enabled = false;
  std::vector<cudaEvent_t> ev;  // start/stop pairs
  size_t used = 0;              // pairs recorded since the last flush
  double total_ms = 0.0;
  uint64_t launches = 0;
  std::string name;
  static constexpr size_t kPairs = 4096;

  void flush_locked() {
    for (size_t i = 0; i < used; ++i) {
      cudaEventSynchronize(ev[2 * i + 1]);
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]) == cudaSuccess) total_ms += ms;
    }
    used = 0;
  }
};
KernelTimer& timer() {
  static KernelTimer t;
  return t;
}
}  // namespace

void timing_begin(const char* kernel, cudaStream_t s) {
  KernelTimer& t = timer();
  if (!t.enabled) return;
  std::lock_guard<std::mutex> lk(t.mu);
  if (t.ev.empty()) {
    t.ev.resize(2 * KernelTimer::kPairs);
    for (auto& e : t.ev) cudaEventCreate(&e);
  }
  if (t.used == KernelTimer::kPairs) t.flush_locked();
  t.name = kernel;
  cudaEventRecord(t.ev[2 * t.used], s);
}

void timing_end(cudaStream_t s) {
  KernelTimer& t = timer();
  if (!t.enabled) return;
  std::lock_guard<std::mutex> lk(t.mu);
  cudaEventRecord(t.ev[2 * t.used + 1], s);
  ++t.used;
  ++t.launches;
}

bool timing_enable(bool on) {
  KernelTimer& t = timer();
  std::lock_guard<std::mutex> lk(t.mu);
  const bool was = t.enabled;
  t.enabled = on;
  return was;
}

}  // namespace spmvcu

using namespace spmvcu;

// ---------------------------------------------------------------- Format methods

spmvlab_cuda_format::~spmvlab_cuda_format() {
  for (auto& a : arrays)
    if (a.ptr) cudaFree(a.ptr);
  for (auto& kv : scratch) {
    cudaFree(kv.second.carry_row);
    cudaFree(kv.second.carry_val);
  }
}

const spmvlab_cuda_format::Scratch* spmvlab_cuda_format::stream_scratch(cudaStream_t s) const {
  std::lock_guard<std::mutex> lk(scratch_mu);
  auto it = scratch.find(s);
  if (it != scratch.end()) return &it->second;
  Scratch sc;
  const uint64_t n = (uint64_t)merge_tiles + 1;
  if (cudaMalloc(&sc.carry_row, 4 * n) != cudaSuccess || cudaMalloc(&sc.carry_val, 8 * n) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(sc.carry_row);
    return nullptr;
  }
  return &scratch.emplace(s, sc).first->second;
}

DevArray* spmvlab_cuda_format::find(const std::string& name) {
  for (auto& a : arrays)
    if (a.name == name) return &a;
  return nullptr;
}
const DevArray* spmvlab_cuda_format::find(const std::string& name) const {
  for (auto& a : arrays)
    if (a.name == name) return &a;
  return nullptr;
}

void* spmvlab_cuda_format::add(const std::string& name, uint64_t count, uint32_t esz, cudaStream_t s) {
  DevArray a;
  a.name = name;
  a.esz = esz;
  a.bytes = count * esz;
  // Padded so 16-byte-aligned bulk (TMA) copies may over-read up to 3 elements past the end.
  // From the device's stream-ordered pool (kept mapped between builds, so rebuilding a format
  // does not pay the driver's page mapping again); build_format synchronises its stream before
  // returning, so the arrays are then usable from any stream.  Released with cudaFree.
  const uint64_t alloc = ((a.bytes + 15) & ~uint64_t(15)) + 64;
  a.ptr = pool_alloc(alloc, s);
  if (!a.ptr) return nullptr;
  arrays.push_back(a);
  return a.ptr;
}

void spmvlab_cuda_format::drop(const std::string& name) {
  for (size_t i = 0; i < arrays.size(); ++i)
    if (arrays[i].name == name) {
      if (arrays[i].ptr) cudaFree(arrays[i].ptr);
      arrays.erase(arrays.begin() + (long)i);
      return;
    }
}

void spmvlab_cuda_format::set_count(const std::string& name, uint64_t count) {
  if (DevArray* a = find(name)) a->bytes = count * a->esz;
}

// ---------------------------------------------------------------- C ABI

extern "C" {

int spmvlab_cuda_abi_version(void) { return SPMVLAB_CUDA_ABI_VERSION; }

const char* spmvlab_cuda_last_error(void) { return g_last_error.c_str(); }

int spmvlab_cuda_release_pool(void) {
  pool_trim();
  return check_launch("spmvlab_cuda_release_pool");
}

unsigned spmvlab_cuda_select_block_size(uint64_t n, unsigned cap, uint64_t l2_bytes) {
  return select_block_size(n, cap, l2_bytes);
}

int spmvlab_cuda_partition_rows_by_nnz(const uint32_t* prefix, uint32_t m, unsigned p, unsigned lb,
                                       uint32_t* bounds) {
  return partition_rows_by_nnz_host(prefix, m, p, lb, bounds);
}

static int check_coo(int alg, const spmvlab_cuda_coo* a, spmvlab_cuda_format** out) {
  if (!out || !a) return fail(kInvalidArgument, "null argument");
  *out = nullptr;
  if (alg < 0 || alg >= kAlgCount) return fail(kInvalidArgument, "unknown algorithm");
  if ((uint64_t)a->m > (1ull << 31) || (uint64_t)a->n > (1ull << 31))
    return fail(kOverflow, "matrix dimension exceeds the supported index width");
  if (a->nnz > 0xFFFFFFFFull) return fail(kOverflow, "nnz does not fit the 32-bit index type");
  if (a->nnz && (!a->row_ind || !a->col_ind || !a->data)) return fail(kInvalidArgument, "null COO array");
  return kOk;
}

static int build_with_beta(int alg, const spmvlab_cuda_coo* a, unsigned threads, unsigned lb, uint64_t split,
                           bool det, spmvlab_cuda_format** out, void* stream);

int spmvlab_cuda_build_format(int alg, const spmvlab_cuda_coo* a, unsigned threads,
                              const spmvlab_cuda_options* opt, spmvlab_cuda_format** out,
                              void* stream) {
  if (int rc = check_coo(alg, a, out)) return rc;
  const uint64_t l2 = opt ? opt->l2_bytes : 512 * 1024;
  const uint64_t split = opt ? opt->split_threshold : 0;
  const bool det = opt && opt->deterministic;
  return build_with_beta(alg, a, threads, engine_log2_beta(alg, a->n, l2), split, det, out, stream);
}

int spmvlab_cuda_build_format_beta(int alg, const spmvlab_cuda_coo* a, unsigned log2_beta, unsigned threads,
                                   spmvlab_cuda_format** out, void* stream) {
  if (int rc = check_coo(alg, a, out)) return rc;
  if (is_crs_alg(alg)) return fail(kInvalidArgument, "CRS formats take no block size");
  const bool bcoh = !is_csb_alg(alg) && !is_mergeb_alg(alg);
  if (log2_beta < 1 || log2_beta > (bcoh ? 15u : 16u))
    return fail(kInvalidArgument, bcoh ? "block size outside the 15-bit increment cap"
                                       : "block size outside the 16-bit packing cap");
  if (bcoh && threads < 1) return fail(kInvalidArgument, "band count must be >= 1");
  return build_with_beta(alg, a, threads, log2_beta, 0, false, out, stream);
}

static int build_with_beta(int alg, const spmvlab_cuda_coo* a, unsigned threads, unsigned lb, uint64_t split,
                           bool det, spmvlab_cuda_format** out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* f = new (std::nothrow) spmvlab_cuda_format();
  if (!f) return fail(kNoMemory, "host allocation failed");
  f->alg = alg;
  f->deterministic = det && !is_crs_alg(alg);
  f->m = a->m;
  f->n = a->n;
  f->nnz = a->nnz;
  int rc;
  {
    Arena ar(s);
    if (is_crs_alg(alg)) {
      rc = build_crs(*f, *a, ar);
      if (rc == kOk) rc = build_merge_plan(*f, ar);
    } else if (is_csb_alg(alg)) {
      rc = build_csb(*f, *a, lb, alg == kCsbh, split, ar);
    } else if (is_mergeb_alg(alg)) {
      rc = build_mergeb(*f, *a, lb, alg == kMergeBH, ar);
    } else {
      rc = build_bcoh(*f, *a, lb, threads, ar);
    }
    ar.release();
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == kOk) rc = check_launch("build_format");
  }
  if (rc != kOk) {
    if (g_last_error.empty() || rc < 100) {
      switch (rc) {
        case kIndexOutOfRange: g_last_error = "index out of range: entry outside the matrix shape"; break;
        case kDuplicateEntry: g_last_error = "duplicate entry: duplicate (row, col) coordinate"; break;
        case kNoMemory: g_last_error = "device allocation failed"; break;
        default: break;
      }
    }
    delete f;
    return rc;
  }
  *out = f;
  return kOk;
}

int spmvlab_cuda_run_spmv(int alg, const spmvlab_cuda_format* f, const double* x, uint64_t x_len,
                          double* y, uint64_t y_len, unsigned p, const spmvlab_cuda_options* opt,
                          void* stream) {
  if (!f) return fail(kInvalidArgument, "null format");
  if (x_len != f->n)
    return fail(kDimensionMismatch, "x has length " + std::to_string(x_len) + ", matrix has " +
                                        std::to_string(f->n) + " columns");
  if (y_len != f->m)
    return fail(kDimensionMismatch, "y has length " + std::to_string(y_len) + ", matrix has " +
                                        std::to_string(f->m) + " rows");
  if (alg != kSeqCrs && p < 1) return fail(kInvalidArgument, "worker count must be >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  (void)opt;
  switch (alg) {
    case kSeqCrs:
    case kParCrs:
    case kMerge:
      if (!is_crs_alg(f->alg)) return fail(kInvalidArgument, "format is not CRS");
      return alg == kSeqCrs ? spmv_seq_crs(*f, x, y, s)
                            : (alg == kParCrs ? spmv_par_crs(*f, x, y, s) : spmv_merge(*f, x, y, s));
    case kCsb:
    case kCsbh:
      if (!is_csb_alg(f->alg)) return fail(kInvalidArgument, "format is not CSB");
      return spmv_blocked(*f, x, y, s);
    case kMergeB:
    case kMergeBH:
      if (!is_mergeb_alg(f->alg)) return fail(kInvalidArgument, "format is not MergeB");
      return spmv_blocked(*f, x, y, s);
    case kBcoh:
    case kBcohc:
    case kBcohch:
    case kBcohchp:
      if (!is_bcoh_alg(f->alg)) return fail(kInvalidArgument, "format is not BCOH");
      if (p != f->bands)
        return fail(kInvalidArgument, "matrix was built for " + std::to_string(f->bands) +
                                          " bands, multiply requested " + std::to_string(p));
      return spmv_blocked(*f, x, y, s);
    default:
      return fail(kInvalidArgument, "unknown algorithm");
  }
}

int spmvlab_cuda_run_spmv_host(int alg, const spmvlab_cuda_format* f, const double* x_host,
                               uint64_t x_len, double* y_host, uint64_t y_len, unsigned p,
                               const spmvlab_cuda_options* opt, double* x_dev, double* y_dev,
                               void* stream) {
  if (!f) return fail(kInvalidArgument, "null format");
  if (x_len != f->n || y_len != f->m) return spmvlab_cuda_run_spmv(alg, f, x_dev, x_len, y_dev, y_len, p, opt, stream);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (x_len) cudaMemcpyAsync(x_dev, x_host, x_len * sizeof(double), cudaMemcpyHostToDevice, s);
  const int rc = spmvlab_cuda_run_spmv(alg, f, x_dev, x_len, y_dev, y_len, p, opt, stream);
  if (rc) return rc;
  if (y_len) cudaMemcpyAsync(y_host, y_dev, y_len * sizeof(double), cudaMemcpyDeviceToHost, s);
  return check_launch("run_spmv_host");
}

int spmvlab_cuda_iterate(int alg, const spmvlab_cuda_format* f, double* x, double* work, uint32_t iters,
                         unsigned p, int flags, double* norms, void* stream) {
  if (!f) return fail(kInvalidArgument, "null format");
  if (f->m != f->n) return fail(kDimensionMismatch, "iterate needs a square matrix");
  if (f->n && (!x || !work)) return fail(kInvalidArgument, "null x or work buffer");
  if (flags & ~(SPMVLAB_ITER_NORMALIZE | SPMVLAB_ITER_GRAPH)) return fail(kInvalidArgument, "unknown flags");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto mult = [&](const double* xi, double* yi, cudaStream_t st) {
    return spmvlab_cuda_run_spmv(alg, f, xi, f->n, yi, f->m, p, nullptr, st);
  };
  const bool merge_engine = alg == kMerge && is_crs_alg(f->alg);
  if (!(flags & SPMVLAB_ITER_GRAPH) || iters == 0)
    return iterate(*f, mult, x, work, iters, flags, norms, s, merge_engine);
  if (!s) return fail(kInvalidArgument, "graph mode needs a non-default stream");
  // nothing may allocate synchronously inside the capture: create this stream's carry scratch now
  if (alg == kMerge && is_crs_alg(f->alg) && !f->stream_scratch(s))
    return fail(kNoMemory, "device allocation failed (merge carry scratch)");
  const bool timing = timing_enable(false);  // no event brackets inside a capture
  const int rc = iterate(*f, mult, x, work, iters, flags, norms, s, merge_engine);
  timing_enable(timing);
  return rc;
}

int spmvlab_cuda_exchange_alloc(uint64_t bytes, void** dev_ptr, unsigned char ipc_handle[64]) {
  if (!dev_ptr || !ipc_handle) return fail(kInvalidArgument, "null argument");
  *dev_ptr = nullptr;
  if (cudaMalloc(dev_ptr, bytes ? bytes : 8) != cudaSuccess) {
    cudaGetLastError();
    return fail(kNoMemory, "device allocation failed (exchange buffer)");
  }
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, *dev_ptr) != cudaSuccess) {
    cudaFree(*dev_ptr);
    *dev_ptr = nullptr;
    return check_launch("cudaIpcGetMemHandle");
  }
  static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
  std::memcpy(ipc_handle, &h, 64);
  return kOk;
}

int spmvlab_cuda_exchange_open(const unsigned char ipc_handle[64], void** dev_ptr) {
  if (!dev_ptr || !ipc_handle) return fail(kInvalidArgument, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, 64);
  if (cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    *dev_ptr = nullptr;
    return check_launch("cudaIpcOpenMemHandle");
  }
  return kOk;
}

int spmvlab_cuda_exchange_close(void* dev_ptr, int opened) {
  if (!dev_ptr) return kOk;
  if (opened ? cudaIpcCloseMemHandle(dev_ptr) != cudaSuccess : cudaFree(dev_ptr) != cudaSuccess)
    return check_launch("exchange_close");
  return kOk;
}

int spmvlab_cuda_run_spmv_scatter(const spmvlab_cuda_format* f, const double* x, uint64_t x_len, double* y,
                                  uint64_t y_len, double* const* dest, unsigned ndest, uint64_t dest_len,
                                  uint64_t row_offset, void* stream) {
  if (!f) return fail(kInvalidArgument, "null format");
  if (!is_crs_alg(f->alg)) return fail(kInvalidArgument, "format is not CRS");
  if (x_len != f->n || y_len != f->m) return fail(kDimensionMismatch, "x / y length does not match the matrix");
  if (ndest > kMaxRowDest || (ndest && !dest)) return fail(kInvalidArgument, "bad destination list");
  if (ndest && row_offset + f->m > dest_len)
    return fail(kInvalidArgument, "row_offset + m exceeds the destination buffers");
  RowDest d{};
  for (unsigned i = 0; i < ndest; ++i) d.p[i] = dest[i];
  d.n = ndest;
  d.off = row_offset;
  return spmv_merge(*f, x, y, static_cast<cudaStream_t>(stream), &d);
}

int spmvlab_cuda_storage_report(const spmvlab_cuda_format* f, spmvlab_cuda_storage_array* rows,
                                size_t capacity, size_t* count) {
  if (!f) return fail(kInvalidArgument, "null format");
  if (count) *count = (size_t)f->nstorage;
  if (!rows) return kOk;
  for (int i = 0; i < f->nstorage && (size_t)i < capacity; ++i) {
    std::memset(rows[i].name, 0, sizeof(rows[i].name));
    std::strncpy(rows[i].name, f->arrays[i].name.c_str(), sizeof(rows[i].name) - 1);
    rows[i].bytes = f->arrays[i].bytes;
  }
  return kOk;
}

int spmvlab_cuda_get_format_info(const spmvlab_cuda_format* f, spmvlab_cuda_format_info* info) {
  if (!f || !info) return fail(kInvalidArgument, "null argument");
  info->alg = f->alg;
  info->m = f->m;
  info->n = f->n;
  info->nnz = f->nnz;
  info->log2_beta = f->log2_beta;
  info->block_rows = f->block_rows;
  info->block_cols = f->block_cols;
  info->element_level = f->element_level;
  info->block_level = f->block_level;
  info->bands = f->bands;
  info->merge_tiles = f->merge_tiles;
  info->work_items = f->work_items;
  info->merge_ipt = f->merge_ipt;
  info->merge_panels = f->merge_panels;
  info->merge_panel_row_visits = f->merge_panel_row_visits;
  info->merge_hot_slots = f->merge_hot;
  info->merge_hot_share = f->merge_hot_share;
  return kOk;
}

int spmvlab_cuda_format_array(const spmvlab_cuda_format* f, const char* name, const void** dev_ptr,
                              uint64_t* bytes) {
  if (!f || !name) return fail(kInvalidArgument, "null argument");
  const DevArray* a = f->find(name);
  if (!a) return fail(kInvalidArgument, std::string("no array named ") + name);
  if (dev_ptr) *dev_ptr = a->ptr;
  if (bytes) *bytes = a->bytes;
  return kOk;
}

int spmvlab_cuda_download_array(const spmvlab_cuda_format* f, const char* name, void* host_dst,
                                uint64_t capacity, uint64_t* bytes) {
  if (!f || !name) return fail(kInvalidArgument, "null argument");
  const DevArray* a = f->find(name);
  if (!a) return fail(kInvalidArgument, std::string("no array named ") + name);
  if (bytes) *bytes = a->bytes;
  if (!host_dst) return kOk;
  if (capacity < a->bytes) return fail(kInvalidArgument, "host buffer too small");
  if (a->bytes && cudaMemcpy(host_dst, a->ptr, a->bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    return check_launch("download_array");
  return kOk;
}

void spmvlab_cuda_free_format(spmvlab_cuda_format* f) { delete f; }

int spmvlab_cuda_validate(const spmvlab_cuda_coo* a, void* stream) {
  if (!a) return fail(kInvalidArgument, "null argument");
  if ((uint64_t)a->m > (1ull << 31) || (uint64_t)a->n > (1ull << 31))
    return fail(kOverflow, "matrix dimension exceeds the supported index width");
  Arena ar(static_cast<cudaStream_t>(stream));
  const int rc = validate_coo(*a, ar);
  if (rc == kIndexOutOfRange) return fail(rc, "index out of range: entry outside the matrix shape");
  if (rc == kDuplicateEntry) return fail(rc, "duplicate entry: duplicate (row, col) coordinate");
  return rc;
}

int spmvlab_cuda_row_prefix(const spmvlab_cuda_coo* a, uint32_t* prefix, void* stream) {
  if (!a || !prefix || (a->nnz && !a->row_ind)) return fail(kInvalidArgument, "null argument");
  g_last_error.clear();
  Arena ar(static_cast<cudaStream_t>(stream));
  const int rc = row_prefix(*a, prefix, ar);
  if (rc == kIndexOutOfRange) return fail(rc, "index out of range: row outside the matrix shape");
  return rc;
}

int spmvlab_cuda_merge_path_search(const uint32_t* a, uint64_t a_len, const uint32_t* b,
                                   uint64_t b_len, const uint64_t* diags, uint64_t count,
                                   uint64_t* out_i, void* stream) {
  return merge_path_search(a, a_len, b, b_len, diags, count, out_i, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_curve_keys(int kind, const uint32_t* rows, const uint32_t* cols, uint64_t count,
                            unsigned level, uint64_t* keys, void* stream) {
  if (level > 31) return fail(kInvalidArgument, "curve level exceeds 31");
  return curve_keys(kind, rows, cols, count, level, keys, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_sort_pairs(uint64_t* keys, uint32_t* values, uint64_t count, int begin_bit,
                            int end_bit, void* stream) {
  if (begin_bit < 0 || end_bit > 64 || begin_bit > end_bit) return fail(kInvalidArgument, "bad bit range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Arena ar(s);
  uint64_t* k2 = ar.alloc_n<uint64_t>(count);
  uint32_t* v2 = ar.alloc_n<uint32_t>(count);
  if (!k2 || !v2) return fail(kNoMemory, "device allocation failed");
  if (radix_sort_pairs(keys, k2, values, v2, count, begin_bit, end_bit, ar)) {
    cudaMemcpyAsync(keys, k2, count * 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(values, v2, count * 4, cudaMemcpyDeviceToDevice, s);
  }
  ar.release();
  return check_launch("sort_pairs");
}

int spmvlab_cuda_cache_read(const char* path, spmvlab_cuda_coo* a, void* stream) {
  if (!path || !a) return fail(kInvalidArgument, "null argument");
  g_last_error.clear();
  return cache_read(path, a, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_cache_info(const char* path, uint32_t* m, uint32_t* n, uint64_t* nnz) {
  if (!path || !m || !n || !nnz) return fail(kInvalidArgument, "null argument");
  return cache_info(path, m, n, nnz);
}

int spmvlab_cuda_cache_write(const char* path, const spmvlab_cuda_coo* a, void* stream) {
  if (!path || !a) return fail(kInvalidArgument, "null argument");
  return cache_write(path, *a, static_cast<cudaStream_t>(stream));
}

void spmvlab_cuda_free_coo(spmvlab_cuda_coo* a) {
  if (!a) return;
  cudaFree(const_cast<uint32_t*>(a->row_ind));
  cudaFree(const_cast<uint32_t*>(a->col_ind));
  cudaFree(const_cast<double*>(a->data));
  std::memset(a, 0, sizeof(*a));
}

int spmvlab_cuda_read_matrix_market(const char* path, spmvlab_cuda_coo* a, spmvlab_cuda_mm_header* header,
                                    void* stream) {
  if (!path || !a) return fail(kInvalidArgument, "null argument");
  g_last_error.clear();
  return mm_read_device(path, a, header, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_read_matrix_market_host(const char* path, spmvlab_cuda_host_coo* out,
                                         spmvlab_cuda_mm_header* header) {
  if (!path || !out) return fail(kInvalidArgument, "null argument");
  g_last_error.clear();
  return mm_read_host(path, out, header);
}

void spmvlab_cuda_free_host_coo(spmvlab_cuda_host_coo* a) {
  if (!a) return;
  std::free(a->row_ind);
  std::free(a->col_ind);
  std::free(a->data);
  std::memset(a, 0, sizeof(*a));
}

int spmvlab_cuda_load_matrix(const char* path, spmvlab_cuda_coo* a, void* stream) {
  if (!path || !a) return fail(kInvalidArgument, "null argument");
  g_last_error.clear();
  return load_matrix(path, a, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_crs_to_icrs(const spmvlab_cuda_format* crs, spmvlab_cuda_bicrs* out, void* stream) {
  if (!crs || !out) return fail(kInvalidArgument, "null argument");
  if (!is_crs_alg(crs->alg)) return fail(kInvalidArgument, "format is not CRS");
  g_last_error.clear();
  std::memset(out, 0, sizeof(*out));
  return crs_to_icrs(*crs, out, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_triplet_to_bicrs(const spmvlab_cuda_coo* a, const uint32_t* order, spmvlab_cuda_bicrs* out,
                                  void* stream) {
  if (!a || !out || (a->nnz && !order)) return fail(kInvalidArgument, "null argument");
  if ((uint64_t)a->m > (1ull << 31) || (uint64_t)a->n > (1ull << 31))
    return fail(kOverflow, "matrix dimension exceeds the supported index width");
  g_last_error.clear();
  std::memset(out, 0, sizeof(*out));
  return triplet_to_bicrs(*a, order, out, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_bicrs_spmv(const spmvlab_cuda_bicrs* a, const double* x, uint64_t x_len, double* y,
                            uint64_t y_len, uint64_t* stats_host, void* stream) {
  if (!a) return fail(kInvalidArgument, "null argument");
  if (x_len != a->n)
    return fail(kDimensionMismatch, "x has length " + std::to_string(x_len) + ", matrix has " +
                                        std::to_string(a->n) + " columns");
  if (y_len != a->m)
    return fail(kDimensionMismatch, "y has length " + std::to_string(y_len) + ", matrix has " +
                                        std::to_string(a->m) + " rows");
  g_last_error.clear();
  return bicrs_spmv(*a, x, y, stats_host, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_bicrs_to_triplet(const spmvlab_cuda_bicrs* a, uint32_t* rows, uint32_t* cols, void* stream) {
  if (!a || (a->nnz && (!rows || !cols))) return fail(kInvalidArgument, "null argument");
  g_last_error.clear();
  return bicrs_decode_all(*a, rows, cols, nullptr, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_format_to_triplet(const spmvlab_cuda_format* f, uint32_t* rows, uint32_t* cols, double* vals,
                                   void* stream) {
  if (!f || (f->nnz && (!rows || !cols))) return fail(kInvalidArgument, "null argument");
  g_last_error.clear();
  return format_to_triplet(*f, rows, cols, vals, static_cast<cudaStream_t>(stream));
}

int spmvlab_cuda_csb_work_items(const spmvlab_cuda_format* f, uint64_t split_threshold,
                                spmvlab_cuda_csb_item* items, uint64_t capacity, uint64_t* count,
                                void* stream) {
  if (!f || !count) return fail(kInvalidArgument, "null argument");
  if (f->alg != 3 && f->alg != 4) return fail(kInvalidArgument, "format is not CSB");
  g_last_error.clear();
  return csb_work_items(*f, split_threshold, items, capacity, count, static_cast<cudaStream_t>(stream));
}

void spmvlab_cuda_free_bicrs(spmvlab_cuda_bicrs* a) {
  if (!a) return;
  cudaFree(a->col_inc);
  cudaFree(a->row_jump);
  cudaFree(a->data);
  std::memset(a, 0, sizeof(*a));
}

uint64_t spmvlab_cuda_launch_count(void) { return g_launches.load(); }

void spmvlab_cuda_kernel_timing(int enable) {
  KernelTimer& t = timer();
  std::lock_guard<std::mutex> lk(t.mu);
  t.enabled = enable != 0;
}

int spmvlab_cuda_kernel_time(double* total_ms, uint64_t* launches, char* name, size_t cap) {
  KernelTimer& t = timer();
  std::lock_guard<std::mutex> lk(t.mu);
  t.flush_locked();
  if (total_ms) *total_ms = t.total_ms;
  if (launches) *launches = t.launches;
  if (name && cap) {
    std::strncpy(name, t.name.c_str(), cap - 1);
    name[cap - 1] = 0;
  }
  t.total_ms = 0.0;
  t.launches = 0;
  return kOk;
}

int spmvlab_cuda_exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, void* stream) {
  Arena ar(static_cast<cudaStream_t>(stream));
  exclusive_scan_u32(in, out, n, ar);
  ar.release();
  return check_launch("exclusive_scan");
}

}  // extern "C"
