// gather4_probe.cu -- dev tool (not product): can TMA move merge-CSR's x gathers off the L1 data
// pipe?  Three ways to form sum_k val[k] * x[col[k]] over the cfg2 matrix, each warp walking
// passes of 128 consecutive nonzeros (lane l owns 4l..4l+3, the merge kernel's layout):
//   ldg     -- 128-bit col / 256-bit val loads, x by LDG (the shipped kernel's product phase)
//   gather4 -- x viewed as rows of R doubles; each lane issues ONE cp.async.bulk.tensor
//              tile::gather4 for its 4 columns (4 rows of R*8 bytes) into a per-warp smem ring of S
//              stages, completion on one mbarrier per stage; values read back with LDS
//   bulk16  -- one 16-byte cp.async.bulk (non-tensor) per nonzero into the ring
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

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
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
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
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int r0, int r1,
                                        int r2, int r3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(su32(dst)),
      "l"(tm), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk16(void* dst, const void* src, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 16, [%2], %3;" ::"r"(
          su32(dst)),
      "l"(src), "r"(su32(bar)), "l"(pol)
      : "memory");
}

// ---- baseline: LDG gathers, lane-blocked, two passes in flight
__global__ void __launch_bounds__(256) k_ldg(const uint32_t* __restrict__ col, const double* __restrict__ val,
                                             uint64_t passes, const double* __restrict__ x, double* out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  for (uint64_t p = w0; p < passes; p += nw) {
    const uint64_t k = p * 128 + 4 * lane;
    const uint4 c = ld4(col + k, pf);
    double v[4];
    ldv4(val + k, pf, v);
    acc += v[0] * ldx(x + c.x, pl) + v[1] * ldx(x + c.y, pl) + v[2] * ldx(x + c.z, pl) + v[3] * ldx(x + c.w, pl);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}

// ---- TMA gather4: per warp a ring of S stages of 32 slots x (4 rows x R doubles)
template <int R, int S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_gather4(const uint32_t* __restrict__ col,
                                                        const double* __restrict__ val, uint64_t passes,
                                                        const __grid_constant__ CUtensorMap tm, double* out) {
  constexpr int SLOT = 4 * R * 8;         // bytes per lane per stage
  constexpr int STAGE = 32 * SLOT;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[WARPS][S];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* ring = sm + (size_t)w * S * STAGE;
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t nw = (uint64_t)gridDim.x * WARPS;
  const uint64_t w0 = (uint64_t)blockIdx.x * WARPS + w;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t cm[S];  // c mod R of the lane's 4 columns, per stage (8 bits each)
  auto issue = [&](uint64_t p, int s) {
    const uint4 c = ld4(col + p * 128 + 4 * lane, pf);
    cm[s] = (c.x % R) | ((c.y % R) << 8) | ((c.z % R) << 16) | ((c.w % R) << 24);
    if (lane == 0) mbar_expect(&bars[w][s], STAGE);
    __syncwarp();
    gather4(ring + s * STAGE + lane * SLOT, &tm, &bars[w][s], 0, c.x / R, c.y / R, c.z / R, c.w / R, pl);
  };
  uint64_t p = w0;
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (p + (uint64_t)s * nw < passes) issue(p + (uint64_t)s * nw, s);
  double acc = 0;
  uint32_t ph = 0;
  while (p < passes) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (p < passes) {
        double v[4];
        ldv4(val + p * 128 + 4 * lane, pf, v);
        mbar_wait(&bars[w][s], ph);
        const double* slot = reinterpret_cast<const double*>(ring + s * STAGE + lane * SLOT);
        double xv[4] = {0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned k = (u + lane) & 3;  // rotate rows across lanes: spread the banks
          const double t = slot[k * R + ((cm[s] >> (8 * k)) & 0xFF)];
          xv[0] = k == 0 ? t : xv[0];
          xv[1] = k == 1 ? t : xv[1];
          xv[2] = k == 2 ? t : xv[2];
          xv[3] = k == 3 ? t : xv[3];
        }
        acc += v[0] * xv[0] + v[1] * xv[1] + v[2] * xv[2] + v[3] * xv[3];
        __syncwarp();
        const uint64_t pn = p + (uint64_t)S * nw;
        if (pn < passes) issue(pn, s);
        p += nw;
      }
    }
    ph ^= 1u;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}

// ---- bulk16: one 16-byte cp.async.bulk per nonzero (the aligned pair holding x[c])
template <int S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_bulk16(const uint32_t* __restrict__ col,
                                                       const double* __restrict__ val, uint64_t passes,
                                                       const double* __restrict__ x, double* out) {
  constexpr int STAGE = 128 * 16;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[WARPS][S];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* ring = sm + (size_t)w * S * STAGE;
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t nw = (uint64_t)gridDim.x * WARPS;
  const uint64_t w0 = (uint64_t)blockIdx.x * WARPS + w;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t cm[S];
  auto issue = [&](uint64_t p, int s) {
    const uint4 c = ld4(col + p * 128 + 4 * lane, pf);
    cm[s] = (c.x & 1) | ((c.y & 1) << 1) | ((c.z & 1) << 2) | ((c.w & 1) << 3);
    if (lane == 0) mbar_expect(&bars[w][s], STAGE);
    __syncwarp();
    uint8_t* d = ring + s * STAGE + lane * 64;
    bulk16(d, x + (c.x & ~1u), &bars[w][s], pl);
    bulk16(d + 16, x + (c.y & ~1u), &bars[w][s], pl);
    bulk16(d + 32, x + (c.z & ~1u), &bars[w][s], pl);
    bulk16(d + 48, x + (c.w & ~1u), &bars[w][s], pl);
  };
  uint64_t p = w0;
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (p + (uint64_t)s * nw < passes) issue(p + (uint64_t)s * nw, s);
  double acc = 0;
  uint32_t ph = 0;
  while (p < passes) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (p < passes) {
        double v[4];
        ldv4(val + p * 128 + 4 * lane, pf, v);
        mbar_wait(&bars[w][s], ph);
        const double* slot = reinterpret_cast<const double*>(ring + s * STAGE + lane * 64);
        double xv[4] = {0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned k = (u + lane) & 3;
          const double t = slot[k * 2 + ((cm[s] >> k) & 1)];
          xv[0] = k == 0 ? t : xv[0];
          xv[1] = k == 1 ? t : xv[1];
          xv[2] = k == 2 ? t : xv[2];
          xv[3] = k == 3 ? t : xv[3];
        }
        acc += v[0] * xv[0] + v[1] * xv[1] + v[2] * xv[2] + v[3] * xv[3];
        __syncwarp();
        const uint64_t pn = p + (uint64_t)S * nw;
        if (pn < passes) issue(pn, s);
        p += nw;
      }
    }
    ph ^= 1u;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}


// ---- hybrid A: every K-th pass of a warp through TMA gather4 (ring of S stages, issued S TMA
// passes ahead), the others through LDG -- the TMA unit and the LSU are separate paths to the L2
template <int S, int WARPS, int K>
__global__ void __launch_bounds__(WARPS * 32) k_hyb_pass(const uint32_t* __restrict__ col,
                                                         const double* __restrict__ val, uint64_t passes,
                                                         const double* __restrict__ x,
                                                         const __grid_constant__ CUtensorMap tm, double* out) {
  constexpr int SLOT = 128, STAGE = 32 * SLOT;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[WARPS][S];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* ring = sm + (size_t)w * S * STAGE;
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t nw = (uint64_t)gridDim.x * WARPS;
  const uint64_t w0 = (uint64_t)blockIdx.x * WARPS + w;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t cm[S];
  auto issue = [&](uint64_t p, int s) {
    const uint4 c = ld4(col + p * 128 + 4 * lane, pf);
    cm[s] = (c.x & 3) | ((c.y & 3) << 8) | ((c.z & 3) << 16) | ((c.w & 3) << 24);
    if (lane == 0) mbar_expect(&bars[w][s], STAGE);
    __syncwarp();
    gather4(ring + s * STAGE + lane * SLOT, &tm, &bars[w][s], 0, c.x >> 2, c.y >> 2, c.z >> 2, c.w >> 2, pl);
  };
  // pass i of this warp = w0 + i * nw; TMA passes are i % K == 0
  const uint64_t stride_group = (uint64_t)S * K * nw;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const uint64_t p = w0 + (uint64_t)(s * K) * nw;
    if (p < passes) issue(p, s);
  }
  double acc = 0;
  uint32_t ph = 0;
  for (uint64_t g = w0; g < passes; g += stride_group) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint64_t p = g + (uint64_t)(s * K + k) * nw;
        if (p < passes) {
          double v[4];
          ldv4(val + p * 128 + 4 * lane, pf, v);
          if (k == 0) {
            mbar_wait(&bars[w][s], ph);
            const double* slot = reinterpret_cast<const double*>(ring + s * STAGE + lane * SLOT);
            double xv[4] = {0, 0, 0, 0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const unsigned q = (u + lane) & 3;
              const double t = slot[q * 4 + ((cm[s] >> (8 * q)) & 0xFF)];
              xv[0] = q == 0 ? t : xv[0];
              xv[1] = q == 1 ? t : xv[1];
              xv[2] = q == 2 ? t : xv[2];
              xv[3] = q == 3 ? t : xv[3];
            }
            acc += v[0] * xv[0] + v[1] * xv[1] + v[2] * xv[2] + v[3] * xv[3];
            __syncwarp();
            const uint64_t pn = p + stride_group;
            if (pn < passes) issue(pn, s);
          } else {
            const uint4 c = ld4(col + p * 128 + 4 * lane, pf);
            acc += v[0] * ldx(x + c.x, pl) + v[1] * ldx(x + c.y, pl) + v[2] * ldx(x + c.z, pl) +
                   v[3] * ldx(x + c.w, pl);
          }
        }
      }
    }
    ph ^= 1u;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}

// ---- hybrid B: in every pass lanes < T take their 4 x values from a TMA gather4 issued S passes
// ahead, lanes >= T gather with LDG
template <int S, int WARPS, int T>
__global__ void __launch_bounds__(WARPS * 32) k_hyb_lane(const uint32_t* __restrict__ col,
                                                         const double* __restrict__ val, uint64_t passes,
                                                         const double* __restrict__ x,
                                                         const __grid_constant__ CUtensorMap tm, double* out) {
  constexpr int SLOT = 128, STAGE = T * SLOT;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[WARPS][S];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* ring = sm + (size_t)w * S * STAGE;
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t nw = (uint64_t)gridDim.x * WARPS;
  const uint64_t w0 = (uint64_t)blockIdx.x * WARPS + w;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t cm[S];
  auto issue = [&](uint64_t p, int s) {
    if (lane == 0) mbar_expect(&bars[w][s], STAGE);
    __syncwarp();
    if (lane < T) {
      const uint4 c = ld4(col + p * 128 + 4 * lane, pf);
      cm[s] = (c.x & 3) | ((c.y & 3) << 8) | ((c.z & 3) << 16) | ((c.w & 3) << 24);
      gather4(ring + s * STAGE + lane * SLOT, &tm, &bars[w][s], 0, c.x >> 2, c.y >> 2, c.z >> 2, c.w >> 2, pl);
    }
  };
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const uint64_t p = w0 + (uint64_t)s * nw;
    if (p < passes) issue(p, s);
  }
  double acc = 0;
  uint32_t ph = 0;
  uint64_t p = w0;
  while (p < passes) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (p < passes) {
        double v[4];
        ldv4(val + p * 128 + 4 * lane, pf, v);
        double xv[4];
        if (lane >= T) {
          const uint4 c = ld4(col + p * 128 + 4 * lane, pf);
          xv[0] = ldx(x + c.x, pl);
          xv[1] = ldx(x + c.y, pl);
          xv[2] = ldx(x + c.z, pl);
          xv[3] = ldx(x + c.w, pl);
        }
        mbar_wait(&bars[w][s], ph);
        if (lane < T) {
          const double* slot = reinterpret_cast<const double*>(ring + s * STAGE + lane * SLOT);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned q = (u + lane) & 3;
            const double t = slot[q * 4 + ((cm[s] >> (8 * q)) & 0xFF)];
            xv[0] = q == 0 ? t : xv[0];
            xv[1] = q == 1 ? t : xv[1];
            xv[2] = q == 2 ? t : xv[2];
            xv[3] = q == 3 ? t : xv[3];
          }
        }
        acc += v[0] * xv[0] + v[1] * xv[1] + v[2] * xv[2] + v[3] * xv[3];
        __syncwarp();
        const uint64_t pn = p + (uint64_t)S * nw;
        if (pn < passes) issue(pn, s);
        p += nw;
      }
    }
    ph ^= 1u;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encode() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = (EncodeTiled)p;
  }
  return fn;
}

static int make_map(CUtensorMap* tm, const double* x, uint64_t n, int R) {
  cuuint64_t dims[2] = {(cuuint64_t)R, (cuuint64_t)(n / R)};
  cuuint64_t strides[1] = {(cuuint64_t)R * 8};
  cuuint32_t box[2] = {(cuuint32_t)R, 1u};
  cuuint32_t es[2] = {1, 1};
  return (int)encode()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)x, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

extern "C" int gp_hyb(const uint32_t* col, const double* val, uint64_t passes, const double* x, uint64_t n,
                      double* out, int blocks, int kind, int S, int W, int K, cudaStream_t st) {
  CUtensorMap tm;
  if (make_map(&tm, x, n, 4)) return 999;
#define HP(s, w, k)                                                                                \
  if (kind == 0 && S == s && W == w && K == k) {                                                    \
    const int smem = w * s * 32 * 128;                                                             \
    cudaFuncSetAttribute(k_hyb_pass<s, w, k>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  \
    k_hyb_pass<s, w, k><<<blocks, w * 32, smem, st>>>(col, val, passes, x, tm, out);              \
    return (int)cudaGetLastError();                                                                \
  }
#define HL(s, w, t)                                                                                \
  if (kind == 1 && S == s && W == w && K == t) {                                                    \
    const int smem = w * s * t * 128;                                                              \
    cudaFuncSetAttribute(k_hyb_lane<s, w, t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  \
    k_hyb_lane<s, w, t><<<blocks, w * 32, smem, st>>>(col, val, passes, x, tm, out);              \
    return (int)cudaGetLastError();                                                                \
  }
  HP(2, 8, 2) HP(2, 8, 3) HP(2, 8, 4) HP(3, 8, 3) HP(2, 4, 3) HP(2, 8, 6)
  HL(2, 8, 8) HL(2, 8, 12) HL(2, 8, 16) HL(3, 8, 12) HL(4, 8, 8) HL(4, 8, 12) HL(2, 4, 12)
#undef HP
#undef HL
  return -1;
}

template <int R, int S, int WARPS>
static int run_g4(const uint32_t* col, const double* val, uint64_t passes, const double* x, uint64_t n,
                  double* out, int blocks, int boxrows, int l2promo, cudaStream_t st) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)R, (cuuint64_t)(n / R)};
  cuuint64_t strides[1] = {(cuuint64_t)R * 8};
  cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)boxrows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)x, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        l2promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                     : (l2promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_128B),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 1000 + (int)r;
  const int smem = WARPS * S * 32 * 4 * R * 8;
  cudaFuncSetAttribute(k_gather4<R, S, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_gather4<R, S, WARPS><<<blocks, WARPS * 32, smem, st>>>(col, val, passes, tm, out);
  return (int)cudaGetLastError();
}

extern "C" int gp_ldg(const uint32_t* col, const double* val, uint64_t passes, const double* x, double* out,
                      int blocks, cudaStream_t st) {
  k_ldg<<<blocks, 256, 0, st>>>(col, val, passes, x, out);
  return (int)cudaGetLastError();
}

// variant: R in {2,4}, S in {2,4,8}, WARPS in {4,8}
extern "C" int gp_gather4(const uint32_t* col, const double* val, uint64_t passes, const double* x, uint64_t n,
                          double* out, int blocks, int R, int S, int WARPS, int boxrows, int l2promo, cudaStream_t st) {
#define G4(r, s, w) \
  if (R == r && S == s && WARPS == w) return run_g4<r, s, w>(col, val, passes, x, n, out, blocks, boxrows, l2promo, st);
  G4(4, 2, 4) G4(4, 4, 4) G4(4, 8, 4) G4(4, 2, 8) G4(4, 4, 8) G4(2, 4, 4) G4(2, 8, 4) G4(2, 4, 8) G4(2, 8, 8)
  G4(4, 3, 8) G4(2, 6, 8)
#undef G4
  return -1;
}

extern "C" int gp_bulk16(const uint32_t* col, const double* val, uint64_t passes, const double* x, double* out,
                         int blocks, int S, int WARPS, cudaStream_t st) {
#define B16(s, w)                                                                             \
  if (S == s && WARPS == w) {                                                                 \
    const int smem = w * s * 128 * 16;                                                        \
    cudaFuncSetAttribute(k_bulk16<s, w>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    k_bulk16<s, w><<<blocks, w * 32, smem, st>>>(col, val, passes, x, out);                  \
    return (int)cudaGetLastError();                                                           \
  }
  B16(4, 4) B16(8, 4) B16(4, 8) B16(8, 8)
#undef B16
  return -1;
}
