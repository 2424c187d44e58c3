// convert_common.cu -- triplet validation and curve-key generation on the device.
#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
namespace {

__global__ void validate_keys(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cols,
                              uint64_t nnz, uint32_t m, uint32_t n, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ idx, uint32_t* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint32_t r = rows[k], c = cols[k];
    if (r >= m || c >= n) atomicOr(err, 1u);
    keys[k] = ((uint64_t)r << 32) | c;
    idx[k] = 0;
  }
}

__global__ void adjacent_dups(const uint64_t* __restrict__ keys, uint64_t nnz, uint32_t* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; k < nnz; k += stride)
    if (keys[k] == keys[k - 1]) atomicOr(err, 2u);
}

__global__ void curve_keys_kernel(int kind, const uint32_t* __restrict__ rows,
                                  const uint32_t* __restrict__ cols, uint64_t count, unsigned level,
                                  uint64_t* __restrict__ keys) {
  SPMV_HILBERT_TABLES();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
    keys[k] = kind == 0 ? morton_encode(rows[k], cols[k], level) : hilbert_encode_t(rows[k], cols[k], level, s_henc);
}

// row_counts (inc/triplet.hpp:75-80): warp-aggregated increments (entries of one row that meet in
// a warp add once); rows out of range are flagged, not counted.
__global__ void row_count_kernel(const uint32_t* __restrict__ rows, uint64_t nnz, uint32_t m,
                                 uint32_t* __restrict__ counts, uint32_t* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint32_t r = rows[k];
    const unsigned active = __activemask();
    if (r >= m) {
      atomicOr(err, 1u);
      continue;
    }
    const unsigned peers = __match_any_sync(__activemask() & active, r);
    if (lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(counts + r, (unsigned)__popc(peers));
  }
}

}  // namespace

// row_prefix (inc/triplet.hpp:82-87): prefix[0..m] = exclusive prefix sums of the row counts.
int row_prefix(const spmvlab_cuda_coo& a, uint32_t* prefix, Arena& ar) {
  cudaStream_t s = ar.stream();
  cudaMemsetAsync(prefix, 0, 4 * ((uint64_t)a.m + 1), s);
  if (a.nnz) {
    uint32_t* err = ar.alloc_n<uint32_t>(1);
    if (!err) return kNoMemory;
    cudaMemsetAsync(err, 0, 4, s);
    row_count_kernel<<<grid_for(a.nnz, 256), 256, 0, s>>>(a.row_ind, a.nnz, a.m, prefix, err);
    uint32_t herr = 0;
    cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (herr) return kIndexOutOfRange;
  }
  exclusive_scan_u32(prefix, prefix, a.m, ar);
  return check_launch("row_prefix");
}

// validate, inc/triplet.hpp:42-59: range check, then duplicates via sorted (row << 32 | col).
int validate_coo(const spmvlab_cuda_coo& a, Arena& ar) {
  cudaStream_t s = ar.stream();
  const uint64_t nnz = a.nnz;
  if (nnz == 0) return kOk;
  uint64_t* keys = ar.alloc_n<uint64_t>(nnz);
  uint64_t* keys2 = ar.alloc_n<uint64_t>(nnz);
  uint32_t* idx = ar.alloc_n<uint32_t>(nnz);
  uint32_t* idx2 = ar.alloc_n<uint32_t>(nnz);
  uint32_t* err = ar.alloc_n<uint32_t>(1);
  if (!keys || !keys2 || !idx || !idx2 || !err) return kNoMemory;
  cudaMemsetAsync(err, 0, 4, s);
  validate_keys<<<grid_for(nnz, 256), 256, 0, s>>>(a.row_ind, a.col_ind, nnz, a.m, a.n, keys, idx, err);
  uint32_t herr = 0;
  cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (herr & 1u) return kIndexOutOfRange;
  const int bits = (int)bit_width64(a.m ? a.m - 1 : 0) + 32;
  const bool alt = radix_sort_pairs(keys, keys2, idx, idx2, nnz, 0, bits, ar);
  adjacent_dups<<<grid_for(nnz, 256), 256, 0, s>>>(alt ? keys2 : keys, nnz, err);
  cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (herr & 2u) return kDuplicateEntry;
  return check_launch("validate");
}

int curve_keys(int kind, const uint32_t* rows, const uint32_t* cols, uint64_t count, unsigned level,
               uint64_t* keys, cudaStream_t s) {
  if (count == 0) return kOk;
  curve_keys_kernel<<<grid_for(count, 256), 256, 0, s>>>(kind, rows, cols, count, level, keys);
  return check_launch("curve_keys");
}

}  // namespace spmvcu
