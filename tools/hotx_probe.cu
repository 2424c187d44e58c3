// hotx_probe.cu -- dev tool (not product): does a shared-memory copy of the most-referenced x
// entries relieve merge-CSR's x-gather wall on R-MAT?  The product phase only (sum val*x[col] over
// the cfg2 matrix, lane-blocked passes of 128 as the merge kernel), persistent CTAs:
//   ldg -- every x by LDG (read-only path, L2 evict-last)
//   hot -- col' = 0x80000000 | slot for the H most-referenced columns (a build-time remap), their
//          x values copied into shared memory once per CTA; the rest by LDG
#include <cstdint>
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld4(const uint32_t* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void ldv4(const double* p, uint64_t pol, double v[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ double ldx(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

template <bool HOT>
__device__ __forceinline__ double gx(const double* __restrict__ x, const double* sx, uint32_t c, uint64_t pl) {
  if constexpr (HOT) {
    double v;
    if ((int)c < 0) v = sx[c & 0x7FFFFFFFu];
    else v = ldx(x + c, pl);
    return v;
  } else {
    return ldx(x + c, pl);
  }
}

template <bool HOT, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_probe(const uint32_t* __restrict__ col,
                                                            const double* __restrict__ val, uint64_t passes,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ xh, uint32_t H,
                                                            double* out, int contig) {
  extern __shared__ __align__(16) double sx[];
  if constexpr (HOT) {
    for (uint32_t i = threadIdx.x; i < H / 2; i += blockDim.x)
      reinterpret_cast<double2*>(sx)[i] = reinterpret_cast<const double2*>(xh)[i];
    __syncthreads();
  }
  const unsigned lane = threadIdx.x & 31;
  const uint64_t pf = pol_first(), pl = pol_last();
  uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  if (contig) {  // warp w: passes [w * P / nw, (w + 1) * P / nw), two adjacent passes per step
    const uint64_t lo = w0 * passes / nw, hi = (w0 + 1) * passes / nw;
    for (uint64_t q = lo; q < hi; q += 2) {
      const uint64_t k0 = q * 128 + 4 * lane, k1 = (q + 1 < hi ? q + 1 : q) * 128 + 4 * lane;
      const uint4 c0 = ld4(col + k0, pf), c1 = ld4(col + k1, pf);
      double v0[4], v1[4];
      ldv4(val + k0, pf, v0);
      ldv4(val + k1, pf, v1);
      const double a0 = v0[0] * gx<HOT>(x, sx, c0.x, pl) + v0[1] * gx<HOT>(x, sx, c0.y, pl) +
                        v0[2] * gx<HOT>(x, sx, c0.z, pl) + v0[3] * gx<HOT>(x, sx, c0.w, pl);
      const double a1 = v1[0] * gx<HOT>(x, sx, c1.x, pl) + v1[1] * gx<HOT>(x, sx, c1.y, pl) +
                        v1[2] * gx<HOT>(x, sx, c1.z, pl) + v1[3] * gx<HOT>(x, sx, c1.w, pl);
      acc += a0 + (q + 1 < hi ? a1 : 0.0);
    }
    w0 = passes;
  }
  uint64_t p = w0;
  for (; p + nw < passes; p += 2 * nw) {
    const uint64_t k0 = p * 128 + 4 * lane, k1 = (p + nw) * 128 + 4 * lane;
    const uint4 c0 = ld4(col + k0, pf), c1 = ld4(col + k1, pf);
    double v0[4], v1[4];
    ldv4(val + k0, pf, v0);
    ldv4(val + k1, pf, v1);
    const double a0 = v0[0] * gx<HOT>(x, sx, c0.x, pl) + v0[1] * gx<HOT>(x, sx, c0.y, pl) +
                      v0[2] * gx<HOT>(x, sx, c0.z, pl) + v0[3] * gx<HOT>(x, sx, c0.w, pl);
    const double a1 = v1[0] * gx<HOT>(x, sx, c1.x, pl) + v1[1] * gx<HOT>(x, sx, c1.y, pl) +
                      v1[2] * gx<HOT>(x, sx, c1.z, pl) + v1[3] * gx<HOT>(x, sx, c1.w, pl);
    acc += a0 + a1;
  }
  for (; p < passes; p += nw) {
    const uint64_t k = p * 128 + 4 * lane;
    const uint4 c = ld4(col + k, pf);
    double v[4];
    ldv4(val + k, pf, v);
    acc += v[0] * gx<HOT>(x, sx, c.x, pl) + v[1] * gx<HOT>(x, sx, c.y, pl) + v[2] * gx<HOT>(x, sx, c.z, pl) +
           v[3] * gx<HOT>(x, sx, c.w, pl);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}

template <bool HOT, int WARPS, int MINB>
static int run(const uint32_t* col, const double* val, uint64_t passes, const double* x, const double* xh, uint32_t H,
               double* out, cudaStream_t st, int contig) {
  const int smem = HOT ? (int)(H * 8) : 0;
  if (HOT) cudaFuncSetAttribute(k_probe<HOT, WARPS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_probe<HOT, WARPS, MINB><<<148 * MINB, WARPS * 32, smem, st>>>(col, val, passes, x, xh, H, out, contig);
  return (int)cudaGetLastError();
}

// shape: 0 = 8 warps x 6 CTAs, 1 = 24 warps x 2 CTAs, 2 = 32 warps x 1 CTA, 3 = 16 warps x 3 CTAs,
//        4 = 16 warps x 2 CTAs
extern "C" int hp_run(int hot, int contig, int shape, const uint32_t* col, const double* val, uint64_t passes, const double* x,
                      const double* xh, uint32_t H, double* out, cudaStream_t st) {
#define S(h, w, b, id) \
  if (hot == h && shape == id) return run<h, w, b>(col, val, passes, x, xh, H, out, st, contig);
  S(0, 8, 6, 0) S(0, 24, 2, 1) S(0, 32, 1, 2) S(0, 16, 3, 3) S(0, 16, 2, 4)
  S(1, 8, 6, 0) S(1, 24, 2, 1) S(1, 32, 1, 2) S(1, 16, 3, 3) S(1, 16, 2, 4)
#undef S
  return -1;
}

// ---- cluster variant: a cluster of CL CTAs shares one hot copy of CL * Hl slots in distributed
// shared memory; slot s lives in CTA (s % CL) at local index s / CL (remote reads through mapa)
template <int CL>
__device__ __forceinline__ double gxc(const double* __restrict__ x, double* const* peers, uint32_t c, uint64_t pl) {
  double v;
  if ((int)c < 0) {
    const uint32_t s = c & 0x7FFFFFFFu;
    v = peers[s % CL][s / CL];
  } else {
    v = ldx(x + c, pl);
  }
  return v;
}

template <int CL>
__global__ void __launch_bounds__(1024, 1) k_cluster(const uint32_t* __restrict__ col, const double* __restrict__ val,
                                                     uint64_t passes, const double* __restrict__ x,
                                                     const double* __restrict__ xh, uint32_t H, double* out,
                                                     int contig) {
  extern __shared__ __align__(16) double sx[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const uint32_t Hl = (H + CL - 1) / CL;
  for (uint32_t i = threadIdx.x; i < Hl; i += blockDim.x) {
    const uint32_t s = i * CL + rank;
    sx[i] = s < H ? xh[s] : 0.0;
  }
  double* peers[CL];
#pragma unroll
  for (int r = 0; r < CL; ++r) peers[r] = cl.map_shared_rank(sx, r);
  cl.sync();
  const unsigned lane = threadIdx.x & 31;
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  const uint64_t lo = contig ? w0 * passes / nw : w0, hi = contig ? (w0 + 1) * passes / nw : passes;
  const uint64_t step = contig ? 1 : nw;
  for (uint64_t q = lo; q < hi; q += step) {
    const uint64_t k = q * 128 + 4 * lane;
    const uint4 c = ld4(col + k, pf);
    double v[4];
    ldv4(val + k, pf, v);
    acc += v[0] * gxc<CL>(x, peers, c.x, pl) + v[1] * gxc<CL>(x, peers, c.y, pl) + v[2] * gxc<CL>(x, peers, c.z, pl) +
           v[3] * gxc<CL>(x, peers, c.w, pl);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane == 0) atomicAdd(out, acc);
  cl.sync();  // peers' shared memory must outlive every remote read
}

extern "C" int hp_cluster(int CL, int contig, const uint32_t* col, const double* val, uint64_t passes, const double* x,
                          const double* xh, uint32_t H, double* out, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 / CL * CL);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = (size_t)((H + CL - 1) / CL) * 8;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define CLU(n)                                                                                                   \
  if (CL == n) {                                                                                                 \
    cudaFuncSetAttribute(k_cluster<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes); \
    cudaLaunchKernelEx(&cfg, k_cluster<n>, col, val, passes, x, xh, H, out, contig);                            \
    return (int)cudaGetLastError();                                                                              \
  }
  CLU(1) CLU(2) CLU(4)
#undef CLU
  return -1;
}
