// ingest.cu -- SPMVLAB1 triplet cache ingest and export.
//
// Reference: cache_write / cache_read (inc/cache_io.hpp:58-91) stream every 64-bit field through
// an istream 8 bytes at a time and then validate() with a host sort (22 s at R-MAT scale 22).
// Here the three 64-bit streams are read with large sequential reads into two pinned staging
// buffers; while the host reads chunk k+1, chunk k is copied to the device and narrowed there
// (u64 -> u32 indices exactly as static_cast<index_t> does, values as raw bit patterns), and the
// triplet is validated on the device (range check + radix-sorted duplicate check).
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {

extern thread_local std::string g_last_error;

namespace {

constexpr char kMagic[8] = {'S', 'P', 'M', 'V', 'L', 'A', 'B', '1'};
constexpr size_t kChunkElems = size_t(1) << 22;  // 32 MiB of u64 per staging buffer

__global__ void narrow_u64(const uint64_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    out[i] = (uint32_t)in[i];
}

__global__ void widen_u32(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) out[i] = in[i];
}

int fail_io(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

// Streams `count` u64 values from the file into dst (u32: narrowed, u64: copied) on the device.
int stream_field(FILE* f, uint64_t count, void* dst, bool narrow, uint64_t* pinned[2], uint64_t* dstage[2],
                 cudaEvent_t done[2], cudaStream_t s) {
  uint64_t off = 0;
  int b = 0;
  while (off < count) {
    const size_t n = (size_t)std::min<uint64_t>(kChunkElems, count - off);
    cudaEventSynchronize(done[b]);  // staging buffer b free again
    const size_t got = fread(pinned[b], 8, n, f);
    if (got != n) return fail_io(kTruncated, "truncated input: cache stream ended early");
    cudaMemcpyAsync(dstage[b], pinned[b], n * 8, cudaMemcpyHostToDevice, s);
    if (narrow)
      narrow_u64<<<grid_for(n, 256), 256, 0, s>>>(dstage[b], static_cast<uint32_t*>(dst) + off, n);
    else
      cudaMemcpyAsync(static_cast<uint64_t*>(dst) + off, dstage[b], n * 8, cudaMemcpyDeviceToDevice, s);
    cudaEventRecord(done[b], s);
    off += n;
    b ^= 1;
  }
  return kOk;
}

}  // namespace

// Reads and checks the header (cache_io.hpp:70-80).
int read_header(FILE* f, uint64_t& m, uint64_t& n, uint64_t& nnz) {
  char magic[8];
  if (fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0)
    return fail_io(kBadMagic, "bad magic: not a spmvlab cache file");
  uint64_t hdr[3];
  if (fread(hdr, 8, 3, f) != 3) return fail_io(kTruncated, "truncated input: cache stream ended early");
  m = hdr[0];  // little-endian host (x86-64 / aarch64)
  n = hdr[1];
  nnz = hdr[2];
  if (m > (1ull << 31) || n > (1ull << 31))
    return fail_io(kOverflow, "index overflow: matrix dimension exceeds the supported index width");
  if (nnz > 0xFFFFFFFFull) return fail_io(kOverflow, "index overflow: nnz exceeds the 32-bit index type");
  return kOk;
}

int cache_info(const char* path, uint32_t* m, uint32_t* n, uint64_t* nnz) {
  File file;
  file.f = fopen(path, "rb");
  if (!file.f) return fail_io(kIoError, std::string("cannot open ") + path);
  uint64_t mm, nn, k;
  if (int rc = read_header(file.f, mm, nn, k)) return rc;
  *m = (uint32_t)mm;
  *n = (uint32_t)nn;
  *nnz = k;
  return kOk;
}

int cache_read(const char* path, spmvlab_cuda_coo* a, cudaStream_t s) {
  const bool caller_buffers = a->row_ind && a->col_ind && a->data;
  const uint64_t capacity = a->nnz;
  File file;
  file.f = fopen(path, "rb");
  if (!file.f) return fail_io(kIoError, std::string("cannot open ") + path);
  uint64_t m, n, nnz;
  if (int rc = read_header(file.f, m, n, nnz)) return rc;
  uint32_t *rows = nullptr, *cols = nullptr;
  double* vals = nullptr;
  if (caller_buffers) {
    if (capacity < nnz) return fail_io(kInvalidArgument, "caller buffers smaller than the cache's nnz");
    rows = const_cast<uint32_t*>(a->row_ind);
    cols = const_cast<uint32_t*>(a->col_ind);
    vals = const_cast<double*>(a->data);
  } else {
    std::memset(a, 0, sizeof(*a));
    const size_t bytes_idx = (size_t)(nnz ? nnz : 1) * 4, bytes_val = (size_t)(nnz ? nnz : 1) * 8;
    if (cudaMalloc(&rows, bytes_idx) != cudaSuccess || cudaMalloc(&cols, bytes_idx) != cudaSuccess ||
        cudaMalloc(&vals, bytes_val) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(rows);
      cudaFree(cols);
      return fail_io(kNoMemory, "device allocation failed");
    }
  }
  uint64_t* pinned[2] = {nullptr, nullptr};
  uint64_t* dstage[2] = {nullptr, nullptr};
  cudaEvent_t done[2];
  const size_t stage_elems = (size_t)std::min<uint64_t>(kChunkElems, nnz ? nnz : 1);
  int rc = kOk;
  for (int b = 0; b < 2; ++b) {
    cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
    cudaEventRecord(done[b], s);
    if (cudaMallocHost(&pinned[b], stage_elems * 8) != cudaSuccess ||
        cudaMalloc(&dstage[b], stage_elems * 8) != cudaSuccess)
      rc = kNoMemory;
  }
  if (rc == kOk) rc = stream_field(file.f, nnz, rows, true, pinned, dstage, done, s);
  if (rc == kOk) rc = stream_field(file.f, nnz, cols, true, pinned, dstage, done, s);
  if (rc == kOk) rc = stream_field(file.f, nnz, vals, false, pinned, dstage, done, s);
  cudaStreamSynchronize(s);
  for (int b = 0; b < 2; ++b) {
    cudaFreeHost(pinned[b]);
    cudaFree(dstage[b]);
    cudaEventDestroy(done[b]);
  }
  if (rc == kOk) {
    a->m = (uint32_t)m;
    a->n = (uint32_t)n;
    a->nnz = nnz;
    a->row_ind = rows;
    a->col_ind = cols;
    a->data = vals;
    Arena ar(s);
    rc = validate_coo(*a, ar);  // cache_read ends with validate(out) (inc/cache_io.hpp:89)
    ar.release();
    cudaStreamSynchronize(s);
    if (rc == kIndexOutOfRange) g_last_error = "index out of range: entry outside the matrix shape";
    if (rc == kDuplicateEntry) g_last_error = "duplicate entry: duplicate (row, col) coordinate";
  }
  if (rc != kOk) {
    if (rc == kNoMemory && g_last_error.empty()) g_last_error = "allocation failed";
    if (!caller_buffers) {
      cudaFree(rows);
      cudaFree(cols);
      cudaFree(vals);
      std::memset(a, 0, sizeof(*a));
    }
  }
  return rc;
}

int cache_write(const char* path, const spmvlab_cuda_coo& a, cudaStream_t s) {
  File file;
  file.f = fopen(path, "wb");
  if (!file.f) return fail_io(kIoError, std::string("cannot open ") + path);
  const uint64_t hdr[3] = {a.m, a.n, a.nnz};
  if (fwrite(kMagic, 1, 8, file.f) != 8 || fwrite(hdr, 8, 3, file.f) != 3)
    return fail_io(kIoError, "cache write failed");
  const size_t stage = (size_t)std::min<uint64_t>(kChunkElems, a.nnz ? a.nnz : 1);
  uint64_t* dbuf = nullptr;
  uint64_t* hbuf = nullptr;
  if (cudaMalloc(&dbuf, stage * 8) != cudaSuccess || cudaMallocHost(&hbuf, stage * 8) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(dbuf);
    return fail_io(kNoMemory, "allocation failed");
  }
  int rc = kOk;
  for (int field = 0; field < 3 && rc == kOk; ++field) {
    for (uint64_t off = 0; off < a.nnz; off += stage) {
      const size_t n = (size_t)std::min<uint64_t>(stage, a.nnz - off);
      if (field < 2) {
        const uint32_t* src = (field == 0 ? a.row_ind : a.col_ind) + off;
        widen_u32<<<grid_for(n, 256), 256, 0, s>>>(src, dbuf, n);
        cudaMemcpyAsync(hbuf, dbuf, n * 8, cudaMemcpyDeviceToHost, s);
      } else {
        cudaMemcpyAsync(hbuf, a.data + off, n * 8, cudaMemcpyDeviceToHost, s);
      }
      if (cudaStreamSynchronize(s) != cudaSuccess) {
        rc = check_launch("cache_write");
        break;
      }
      if (fwrite(hbuf, 8, n, file.f) != n) {
        rc = fail_io(kIoError, "cache write failed");
        break;
      }
    }
  }
  cudaFree(dbuf);
  cudaFreeHost(hbuf);
  return rc;
}

}  // namespace spmvcu
