// microbench.cu -- diagnostic kernels (dev tool, not product): pure streaming read bandwidth and
// the x-gather floor of CSR SpMV on a given column-index array.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__global__ void stream_read(const double4* __restrict__ p, uint64_t n4, double* out) {
  double acc = 0;
  const uint64_t pf = pol_first();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + i), "l"(pf));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5) out[0] = acc;
}

// gather: sum_k x[col[k]] with coalesced col loads, IPT gathers in flight per thread
template <int IPT>
__global__ void gather_x(const uint32_t* __restrict__ col, uint64_t nnz, const double* __restrict__ x,
                         double* out) {
  double acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < nnz; base += stride * IPT) {
    uint32_t c[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint64_t k = base + i * stride;
      c[i] = k < nnz ? __ldg(col + k) : 0;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) acc += __ldg(x + c[i]);
  }
  if (acc == 1234.5) out[0] = acc;
}

// gather + stream vals, the full "product" phase without any merge logic
template <int IPT>
__global__ void gather_mul(const uint32_t* __restrict__ col, const double* __restrict__ val, uint64_t nnz,
                           const double* __restrict__ x, double* out) {
  double acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < nnz; base += stride * IPT) {
    uint32_t c[IPT];
    double v[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint64_t k = base + i * stride;
      c[i] = k < nnz ? __ldg(col + k) : 0;
      v[i] = k < nnz ? __ldg(val + k) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) acc += v[i] * __ldg(x + c[i]);
  }
  if (acc == 1234.5) out[0] = acc;
}

// tiled: one CTA per contiguous tile of THREADS*IPT elements (the merge kernel's access pattern)
template <int THREADS, int IPT>
__global__ void gather_mul_tiled(const uint32_t* __restrict__ col, const double* __restrict__ val, uint64_t nnz,
                                 const double* __restrict__ x, double* out) {
  const uint64_t base = (uint64_t)blockIdx.x * THREADS * IPT + threadIdx.x;
  uint32_t c[IPT];
  double v[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint64_t k = base + i * THREADS;
    c[i] = k < nnz ? __ldg(col + k) : 0;
    v[i] = k < nnz ? __ldg(val + k) : 0.0;
  }
  double acc = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) acc += v[i] * __ldg(x + c[i]);
  if (acc == 1234.5) out[0] = acc;
}

// tiled with a dependent tile-coordinate load first (the merge kernel's first round trip), then
// optional smem staging + barrier
template <int THREADS, int IPT, bool STAGE>
__global__ void gather_mul_tiled_meta(const uint32_t* __restrict__ col, const double* __restrict__ val,
                                      const uint32_t* __restrict__ starts, uint64_t nnz,
                                      const double* __restrict__ x, double* out) {
  __shared__ double s[THREADS * IPT];
  const uint64_t base = (uint64_t)starts[blockIdx.x] + threadIdx.x;
  uint32_t c[IPT];
  double v[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint64_t k = base + i * THREADS;
    c[i] = k < nnz ? __ldg(col + k) : 0;
    v[i] = k < nnz ? __ldg(val + k) : 0.0;
  }
  double acc = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const double p = v[i] * __ldg(x + c[i]);
    if (STAGE) s[threadIdx.x + i * THREADS] = p; else acc += p;
  }
  if (STAGE) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) acc += s[(threadIdx.x * IPT + i) % (THREADS * IPT)];
  }
  if (acc == 1234.5) out[0] = acc;
}

// warp-private tiles of 32*IPT elements, staged in smem with __syncwarp only
template <int WARPS, int IPT>
__global__ void gather_mul_warp_stage(const uint32_t* __restrict__ col, const double* __restrict__ val,
                                      uint64_t nnz, const double* __restrict__ x, double* out) {
  __shared__ double s[WARPS][32 * IPT];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t base = ((uint64_t)blockIdx.x * WARPS + w) * 32 * IPT + lane;
  uint32_t c[IPT];
  double v[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint64_t k = base + i * 32;
    c[i] = k < nnz ? __ldg(col + k) : 0;
    v[i] = k < nnz ? __ldg(val + k) : 0.0;
  }
#pragma unroll
  for (int i = 0; i < IPT; ++i) s[w][lane + i * 32] = v[i] * __ldg(x + c[i]);
  __syncwarp();
  double acc = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) acc += s[w][lane * IPT + i];
  if (acc == 1234.5) out[0] = acc;
}

extern "C" {
int mb_gather_mul_warp_stage(const uint32_t* col, const double* val, uint64_t nnz, const double* x, double* out,
                             void* s) {
  const unsigned blocks = (unsigned)((nnz + 4 * 224 - 1) / (4 * 224));
  gather_mul_warp_stage<4, 7><<<blocks, 128, 0, (cudaStream_t)s>>>(col, val, nnz, x, out);
  return (int)cudaGetLastError();
}
int mb_gather_mul_tiled_meta(const uint32_t* col, const double* val, const uint32_t* starts, uint64_t nnz,
                             const double* x, double* out, int stage, void* s) {
  const unsigned blocks = (unsigned)((nnz + 895) / 896);
  if (stage)
    gather_mul_tiled_meta<128, 7, true><<<blocks, 128, 0, (cudaStream_t)s>>>(col, val, starts, nnz, x, out);
  else
    gather_mul_tiled_meta<128, 7, false><<<blocks, 128, 0, (cudaStream_t)s>>>(col, val, starts, nnz, x, out);
  return (int)cudaGetLastError();
}
int mb_gather_mul_tiled(const uint32_t* col, const double* val, uint64_t nnz, const double* x, double* out,
                        int threads, void* s) {
  if (threads == 128)
    gather_mul_tiled<128, 7><<<(unsigned)((nnz + 895) / 896), 128, 0, (cudaStream_t)s>>>(col, val, nnz, x, out);
  else
    gather_mul_tiled<256, 7><<<(unsigned)((nnz + 1791) / 1792), 256, 0, (cudaStream_t)s>>>(col, val, nnz, x, out);
  return (int)cudaGetLastError();
}
int mb_stream_read(const void* p, uint64_t bytes, double* out, int blocks, void* s) {
  stream_read<<<blocks, 256, 0, (cudaStream_t)s>>>((const double4*)p, bytes / 32, out);
  return (int)cudaGetLastError();
}
int mb_gather_x(const uint32_t* col, uint64_t nnz, const double* x, double* out, int blocks, void* s) {
  gather_x<8><<<blocks, 256, 0, (cudaStream_t)s>>>(col, nnz, x, out);
  return (int)cudaGetLastError();
}
int mb_gather_mul(const uint32_t* col, const double* val, uint64_t nnz, const double* x, double* out, int blocks,
                  void* s) {
  gather_mul<8><<<blocks, 256, 0, (cudaStream_t)s>>>(col, val, nnz, x, out);
  return (int)cudaGetLastError();
}
}

// blocked: lane l of a warp handles 4 consecutive elements of each 128-element group (one 128-bit
// col load + one 256-bit val load per lane), gathers in lane-blocked order
template <int Q>
__global__ void gather_mul_blocked4(const uint32_t* __restrict__ col, const double* __restrict__ val, uint64_t nnz,
                                    const double* __restrict__ x, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  for (uint64_t g = warp * Q; g * 128 < nnz; g += nwarps * Q) {
    uint4 c[Q];
    double v[Q][4];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const uint64_t k = (g + q) * 128 + 4 * lane;
      if (k + 3 < nnz) {
        c[q] = __ldg(reinterpret_cast<const uint4*>(col + k));
        asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(v[q][0]), "=d"(v[q][1]), "=d"(v[q][2]), "=d"(v[q][3]) : "l"(val + k));
      } else {
        c[q] = make_uint4(0, 0, 0, 0);
        v[q][0] = v[q][1] = v[q][2] = v[q][3] = 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q)
      acc += v[q][0] * __ldg(x + c[q].x) + v[q][1] * __ldg(x + c[q].y) + v[q][2] * __ldg(x + c[q].z) +
             v[q][3] * __ldg(x + c[q].w);
  }
  if (acc == 1234.5) out[0] = acc;
}

extern "C" int mb_gather_mul_blocked4(const uint32_t* col, const double* val, uint64_t nnz, const double* x,
                                      double* out, int blocks, int q, void* s) {
  if (q == 1) gather_mul_blocked4<1><<<blocks, 256, 0, (cudaStream_t)s>>>(col, val, nnz, x, out);
  else gather_mul_blocked4<2><<<blocks, 256, 0, (cudaStream_t)s>>>(col, val, nnz, x, out);
  return (int)cudaGetLastError();
}
