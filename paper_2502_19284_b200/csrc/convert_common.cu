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

}  // namespace

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
