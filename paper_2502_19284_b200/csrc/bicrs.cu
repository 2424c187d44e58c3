// bicrs.cu -- standalone ICRS / BICRS (inc/bicrs.hpp).
//
// Reference: IncrementalRowStorage<Increment> (bicrs.hpp:33-45) -- col_inc (nnz + 1 entries:
// column increments, +n on a row change, a final n), row_jump (the first row, then one row delta
// per row change) and data; ICRS = u32 increments built from CRS order (crs_to_icrs, :120-150),
// BICRS = i64 increments for any element order (triplet_to_bicrs, :154-200).  The reference
// replays the increments sequentially (replay_bicrs, :54-94).  Here both directions are
// data-parallel:
//   build:  increment of element p = f(element p, element p-1); row-change flags + a scan place
//           the row jumps.
//   decode: R_k = inclusive prefix sum of the increments; the number of wraps W_k = R_k div n
//           (the running column R_k - n W_k is in [0, n) exactly when the stream is valid), the
//           column is R_k mod n and the row is the prefix sum of row_jump at W_k.  Every check of
//           the sequential replay becomes a per-element predicate (running column >= 0, at most
//           one wrap per element, rows in range, final wrap present, all row jumps consumed) ->
//           CorruptFormat.
// The multiply adds each product into y with an fp64 reduction (the element order is arbitrary).
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {

extern thread_local std::string g_last_error;

namespace {

// ---------------------------------------------------------------- int64 inclusive scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__global__ void scan_tile_sums(const T* __restrict__ in, uint64_t n, int64_t* __restrict__ sums) {
  __shared__ int64_t ws[kScanThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  int64_t s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t k = base + (uint64_t)i * kScanThreads + threadIdx.x;
    if (k < n) s += (int64_t)in[k];
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

// inclusive scan of one tile given its exclusive offset (offs == nullptr: 0)
template <typename T>
__global__ void scan_tile_apply(const T* __restrict__ in, uint64_t n, const int64_t* __restrict__ offs,
                                int64_t* __restrict__ out) {
  __shared__ int64_t ws[kScanThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t k = base + i;
    v[i] = k < n ? (int64_t)in[k] : 0;
    s += v[i];
  }
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  int64_t incl = s;
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
    if (lane >= (unsigned)off) incl += t;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  int64_t pre = offs ? offs[blockIdx.x] : 0;
  for (unsigned w = 0; w < warp; ++w) pre += ws[w];
  int64_t run = pre + incl - s;
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t k = base + i;
    run += v[i];
    if (k < n) out[k] = run;
  }
}

// out[k] = in[0] + ... + in[k] (int64), any length
template <typename T>
int inclusive_scan_i64(const T* in, uint64_t n, int64_t* out, Arena& ar) {
  cudaStream_t s = ar.stream();
  if (n == 0) return kOk;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    scan_tile_apply<T><<<1, kScanThreads, 0, s>>>(in, n, nullptr, out);
    return check_launch("scan_i64");
  }
  int64_t* sums = ar.alloc_n<int64_t>(tiles);
  int64_t* offs = ar.alloc_n<int64_t>(tiles + 1);
  if (!sums || !offs) return kNoMemory;
  scan_tile_sums<T><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, sums);
  // exclusive offsets = inclusive scan of the sums shifted by one
  cudaMemsetAsync(offs, 0, 8, s);
  if (int rc = inclusive_scan_i64<int64_t>(sums, tiles, offs + 1, ar)) return rc;
  scan_tile_apply<T><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, offs, out);
  return check_launch("scan_i64");
}

// ---------------------------------------------------------------- builds
__global__ void icrs_row_flags(const uint32_t* __restrict__ row_ptr, uint32_t m, uint32_t* __restrict__ start,
                               uint32_t* __restrict__ nonempty) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const uint32_t b = row_ptr[r], e = row_ptr[r + 1];
  nonempty[r] = e > b;
  if (e > b) start[b] = 1u;
}

// crs_to_icrs (bicrs.hpp:120-150): u32 arithmetic, exactly the reference's index_t expressions
__global__ void icrs_incs(const uint32_t* __restrict__ col, const uint32_t* __restrict__ start, uint64_t nnz,
                          uint32_t n, uint32_t* __restrict__ col_inc) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nnz) return;
  if (k == nnz) {
    col_inc[k] = n;
    return;
  }
  const uint32_t c = col[k];
  col_inc[k] = k == 0 ? c : (start[k] ? c - col[k - 1] + n : c - col[k - 1]);
}

__global__ void icrs_rows(const uint32_t* __restrict__ nonempty, const uint32_t* __restrict__ pos, uint32_t m,
                          uint32_t* __restrict__ rows_c) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m && nonempty[r]) rows_c[pos[r]] = r;
}

__global__ void icrs_jumps(const uint32_t* __restrict__ rows_c, uint32_t cnt, uint32_t* __restrict__ row_jump) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) row_jump[i] = i == 0 ? rows_c[0] : rows_c[i] - rows_c[i - 1];
}

__global__ void order_check(const uint32_t* __restrict__ order, uint64_t nnz, uint32_t* __restrict__ seen,
                            uint32_t* __restrict__ err) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const uint32_t id = order[p];
  if (id >= nnz || atomicExch(&seen[id], 1u) != 0u) atomicOr(err, 1u);
}

// triplet_to_bicrs (bicrs.hpp:154-200): signed 64-bit increments
__global__ void bicrs_incs(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cols,
                           const double* __restrict__ vals, const uint32_t* __restrict__ order, uint64_t nnz,
                           uint32_t n, int64_t* __restrict__ col_inc, uint32_t* __restrict__ chg,
                           double* __restrict__ data) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > nnz) return;
  if (p == nnz) {
    col_inc[p] = (int64_t)n;
    return;
  }
  const uint32_t id = order[p];
  const int64_t r = rows[id], c = cols[id];
  data[p] = vals[id];
  if (p == 0) {
    col_inc[0] = c;
    chg[0] = 1u;
    return;
  }
  const uint32_t q = order[p - 1];
  const int64_t pr = rows[q], pc = cols[q];
  const bool change = r != pr;
  col_inc[p] = change ? c - pc + (int64_t)n : c - pc;
  chg[p] = change ? 1u : 0u;
}

__global__ void bicrs_jumps(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ order,
                            const uint32_t* __restrict__ chg, const uint32_t* __restrict__ pos, uint64_t nnz,
                            int64_t* __restrict__ row_jump) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz || !chg[p]) return;
  const int64_t r = rows[order[p]];
  row_jump[pos[p]] = p == 0 ? r : r - (int64_t)rows[order[p - 1]];
}

// ---------------------------------------------------------------- decode (replay_bicrs)
__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  const int64_t q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// Per element k < nnz: W_k, column, row; err bit 1 = corrupt.  Also publishes W_{nnz-1} and W_nnz.
__global__ void bicrs_decode(const int64_t* __restrict__ R, const int64_t* __restrict__ rowp, uint64_t n_jump,
                             uint64_t nnz, uint32_t m, uint32_t n, uint32_t* __restrict__ rows_out,
                             uint32_t* __restrict__ cols_out, uint32_t* __restrict__ err,
                             int64_t* __restrict__ wraps) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nnz) return;
  const int64_t Rk = R[k];
  const int64_t W = floordiv(Rk, (int64_t)n);
  const int64_t Wp = k == 0 ? 0 : floordiv(R[k - 1], (int64_t)n);
  bool bad = Rk < 0 || W < Wp || W > Wp + 1;  // running column < 0, or more than one wrap
  if (k == nnz) {                               // the terminating increment must wrap once
    if (nnz > 0 && W != Wp + 1) bad = true;
    wraps[0] = nnz ? Wp : 0;
    wraps[1] = W;
  } else {
    const bool jump_ok = W >= 0 && (uint64_t)W < n_jump;
    const int64_t row = jump_ok ? rowp[W] : -1;
    if (!jump_ok || row < 0 || row >= (int64_t)m) bad = true;
    if (!bad) {
      if (rows_out) rows_out[k] = (uint32_t)row;
      if (cols_out) cols_out[k] = (uint32_t)(Rk - W * (int64_t)n);
    }
  }
  if (bad) atomicOr(err, 1u);
}

__global__ void bicrs_products(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cols,
                               const double* __restrict__ data, uint64_t nnz, const double* __restrict__ x,
                               double* __restrict__ y) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(y + rows[k], data[k] * x[cols[k]]);
}

int fail_b(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace

int crs_to_icrs(const Format& f, spmvlab_cuda_bicrs* out, cudaStream_t s) {
  const uint64_t nnz = f.nnz;
  const uint32_t m = f.m;
  Arena ar(s);
  uint32_t *col_inc = nullptr, *row_jump = nullptr;
  double* data = nullptr;
  uint32_t* start = ar.alloc_n<uint32_t>(nnz + 1);
  uint32_t* nonempty = ar.alloc_n<uint32_t>((uint64_t)m + 1);
  uint32_t* pos = ar.alloc_n<uint32_t>((uint64_t)m + 1);
  uint32_t* rows_c = ar.alloc_n<uint32_t>((uint64_t)m + 1);
  if (!start || !nonempty || !pos || !rows_c) return kNoMemory;
  cudaMemsetAsync(start, 0, 4 * (nnz + 1), s);
  const uint32_t* rp = f.find("row_ptr")->as<uint32_t>();
  const uint32_t* col = f.find("col_ind")->as<uint32_t>();
  if (m) icrs_row_flags<<<(m + 255) / 256, 256, 0, s>>>(rp, m, start, nonempty);
  exclusive_scan_u32(nonempty, pos, m, ar);
  uint32_t cnt = 0;
  cudaMemcpyAsync(&cnt, pos + m, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (cudaMalloc(&col_inc, 4 * (nnz + 1)) != cudaSuccess || cudaMalloc(&row_jump, 4ull * (cnt ? cnt : 1)) != cudaSuccess ||
      cudaMalloc(&data, 8 * (nnz ? nnz : 1)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(col_inc);
    cudaFree(row_jump);
    return kNoMemory;
  }
  icrs_incs<<<(unsigned)((nnz + 1 + 255) / 256), 256, 0, s>>>(col, start, nnz, f.n, col_inc);
  if (m) icrs_rows<<<(m + 255) / 256, 256, 0, s>>>(nonempty, pos, m, rows_c);
  if (cnt) icrs_jumps<<<(cnt + 255) / 256, 256, 0, s>>>(rows_c, cnt, row_jump);
  if (nnz) cudaMemcpyAsync(data, f.find("data")->ptr, 8 * nnz, cudaMemcpyDeviceToDevice, s);
  ar.release();
  cudaStreamSynchronize(s);
  *out = spmvlab_cuda_bicrs{f.m, f.n, nnz, 0, col_inc, row_jump, cnt, data};
  return check_launch("crs_to_icrs");
}

int triplet_to_bicrs(const spmvlab_cuda_coo& a, const uint32_t* order, spmvlab_cuda_bicrs* out, cudaStream_t s) {
  const uint64_t nnz = a.nnz;
  Arena ar(s);
  uint32_t* seen = ar.alloc_n<uint32_t>(nnz + 1);
  uint32_t* err = ar.alloc_n<uint32_t>(1);
  uint32_t* chg = ar.alloc_n<uint32_t>(nnz + 1);
  uint32_t* pos = ar.alloc_n<uint32_t>(nnz + 1);
  if (!seen || !err || !chg || !pos) return kNoMemory;
  cudaMemsetAsync(seen, 0, 4 * (nnz + 1), s);
  cudaMemsetAsync(err, 0, 4, s);
  if (nnz) order_check<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(order, nnz, seen, err);
  uint32_t herr = 0;
  cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (herr) return fail_b(kInvalidArgument, "element order is not a permutation");
  int64_t *col_inc = nullptr, *row_jump = nullptr;
  double* data = nullptr;
  if (cudaMalloc(&col_inc, 8 * (nnz + 1)) != cudaSuccess || cudaMalloc(&data, 8 * (nnz ? nnz : 1)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(col_inc);
    return kNoMemory;
  }
  bicrs_incs<<<(unsigned)((nnz + 1 + 255) / 256), 256, 0, s>>>(a.row_ind, a.col_ind, a.data, order, nnz, a.n, col_inc,
                                                               chg, data);
  exclusive_scan_u32(chg, pos, nnz, ar);
  uint32_t cnt = 0;
  cudaMemcpyAsync(&cnt, pos + nnz, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (cudaMalloc(&row_jump, 8ull * (cnt ? cnt : 1)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(col_inc);
    cudaFree(data);
    return kNoMemory;
  }
  if (nnz)
    bicrs_jumps<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(a.row_ind, order, chg, pos, nnz, row_jump);
  ar.release();
  cudaStreamSynchronize(s);
  *out = spmvlab_cuda_bicrs{a.m, a.n, nnz, 1, col_inc, row_jump, cnt, data};
  return check_launch("triplet_to_bicrs");
}

// Decodes rows / cols (either may be null) and the replay statistics; CorruptFormat on violation.
int bicrs_decode_all(const spmvlab_cuda_bicrs& b, uint32_t* rows, uint32_t* cols, uint64_t* stats, cudaStream_t s) {
  const uint64_t nnz = b.nnz;
  if (b.n == 0 && nnz) return fail_b(kCorruptFormat, "col_inc must hold nnz + 1 entries");
  if (nnz && b.n_row_jump == 0) return fail_b(kCorruptFormat, "missing first row jump");
  if (nnz == 0) {
    if (stats) stats[0] = stats[1] = 0;
    return kOk;
  }
  Arena ar(s);
  int64_t* R = ar.alloc_n<int64_t>(nnz + 1);
  int64_t* rowp = ar.alloc_n<int64_t>(b.n_row_jump);
  uint32_t* err = ar.alloc_n<uint32_t>(1);
  int64_t* wraps = ar.alloc_n<int64_t>(2);
  if (!R || !rowp || !err || !wraps) return kNoMemory;
  int rc = b.kind == 0 ? inclusive_scan_i64(static_cast<const uint32_t*>(b.col_inc), nnz + 1, R, ar)
                       : inclusive_scan_i64(static_cast<const int64_t*>(b.col_inc), nnz + 1, R, ar);
  if (rc) return rc;
  rc = b.kind == 0 ? inclusive_scan_i64(static_cast<const uint32_t*>(b.row_jump), b.n_row_jump, rowp, ar)
                   : inclusive_scan_i64(static_cast<const int64_t*>(b.row_jump), b.n_row_jump, rowp, ar);
  if (rc) return rc;
  cudaMemsetAsync(err, 0, 4, s);
  bicrs_decode<<<(unsigned)((nnz + 1 + 255) / 256), 256, 0, s>>>(R, rowp, b.n_row_jump, nnz, b.m, b.n, rows, cols,
                                                                  err, wraps);
  uint32_t herr = 0;
  int64_t hw[2] = {0, 0};
  cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hw, wraps, 16, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (int e = check_launch("bicrs_decode")) return e;
  if (herr) return fail_b(kCorruptFormat, "increment replay left the matrix or wrapped more than once");
  if ((uint64_t)hw[0] + 1 != b.n_row_jump)
    return fail_b(kCorruptFormat, "replay consumed the wrong number of row jumps");
  if (stats) {
    stats[0] = (uint64_t)hw[1];  // overflow events: every wrap, the terminating one included
    stats[1] = (uint64_t)hw[0];  // row jumps consumed after the first
  }
  return kOk;
}

int bicrs_spmv(const spmvlab_cuda_bicrs& b, const double* x, double* y, uint64_t* stats, cudaStream_t s) {
  const uint64_t nnz = b.nnz;
  if (b.m) cudaMemsetAsync(y, 0, 8ull * b.m, s);
  if (nnz == 0) return bicrs_decode_all(b, nullptr, nullptr, stats, s);
  uint32_t *rows = nullptr, *cols = nullptr;
  if (cudaMallocAsync(&rows, 4 * nnz, s) != cudaSuccess || cudaMallocAsync(&cols, 4 * nnz, s) != cudaSuccess) {
    cudaGetLastError();
    if (rows) cudaFreeAsync(rows, s);
    return kNoMemory;
  }
  int rc = bicrs_decode_all(b, rows, cols, stats, s);
  if (rc == kOk) {
    bicrs_products<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(rows, cols, b.data, nnz, x, y);
    note_launch();
    rc = check_launch("bicrs_spmv");
  }
  cudaFreeAsync(rows, s);
  cudaFreeAsync(cols, s);
  return rc;
}

}  // namespace spmvcu
