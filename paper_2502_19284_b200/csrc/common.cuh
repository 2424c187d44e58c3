// common.cuh -- shared device helpers for the spmvlab B200 (sm_100a) kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spmvcu {

// ---------------------------------------------------------------- error codes (C ABI)
// 0 ok; 1 + spmvlab::ErrorKind ordinal (inc/types.hpp:47-62); >= 100 CUDA / internal.
enum Status : int {
  kOk = 0,
  kDimensionMismatch = 1,
  kInvalidArgument = 2,
  kCorruptFormat = 3,
  kOverflow = 4,
  kBadHeader = 5,
  kUnsupportedFormat = 6,
  kUnsupportedField = 7,
  kUnsupportedSymmetry = 8,
  kIndexOutOfRange = 9,
  kDuplicateEntry = 10,
  kParseError = 11,
  kTruncated = 12,
  kBadMagic = 13,
  kIoError = 14,
  kCudaError = 100,
  kNoMemory = 101,
};

// Algorithm ordinals, inc/engine.hpp:30-42.
enum Alg : int {
  kSeqCrs = 0, kParCrs, kMerge, kCsb, kCsbh, kBcoh, kBcohc, kBcohch, kBcohchp, kMergeB, kMergeBH,
  kAlgCount
};

inline bool is_crs_alg(int a) { return a == kSeqCrs || a == kParCrs || a == kMerge; }
inline bool is_csb_alg(int a) { return a == kCsb || a == kCsbh; }
inline bool is_mergeb_alg(int a) { return a == kMergeB || a == kMergeBH; }
inline bool is_bcoh_alg(int a) { return a >= kBcoh && a <= kBcohchp; }

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------- cache-hinted loads
// Streaming (read-once) loads of the matrix arrays: no L1 allocation, and an L2 evict-first cache
// policy so the x vector stays L2-resident while A streams past it.  x gathers use the read-only
// path with an evict-last policy.  (sm_100 accepts .L2::evict_* only on 256-bit loads, so the
// priorities are expressed as createpolicy cache-hint operands.)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ld_stream4(const uint32_t* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// x-gather flavours (experiments): 0 nc+L2 evict_last, 1 nc no-L1-allocate, 2 plain, 3 .cg
template <int MODE>
__device__ __forceinline__ double ld_xm(const double* p, uint64_t pol) {
  double v;
  if constexpr (MODE == 0) {
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  } else if constexpr (MODE == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  } else if constexpr (MODE == 2) {
    v = *p;
  } else {
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  }
  return v;
}

// ---------------------------------------------------------------- curves (inc/curves.hpp)
// Hilbert orientation state: bit0 = swapped, bit1 = flipped (HilbertOrientation,
// curves.hpp:60-103).  position(): x = col bit, y = row bit, flip, swap, pos = 3x ^ y.
__host__ __device__ __forceinline__ unsigned hil_position(unsigned st, unsigned rbit, unsigned cbit) {
  unsigned x = cbit ^ ((st >> 1) & 1u), y = rbit ^ ((st >> 1) & 1u);
  if (st & 1u) { unsigned t = x; x = y; y = t; }
  return (3u * x) ^ y;
}
__host__ __device__ __forceinline__ unsigned hil_child(unsigned st, unsigned pos) {
  return pos == 0 ? st ^ 1u : (pos == 3 ? st ^ 3u : st);
}
__host__ __device__ __forceinline__ void hil_cell(unsigned st, unsigned pos, unsigned& rbit, unsigned& cbit) {
  unsigned x = (pos >> 1) & 1u;                 // rx = {0,0,1,1}
  unsigned y = (pos ^ (pos >> 1)) & 1u;         // ry = {0,1,1,0}
  if (st & 2u) { x ^= 1u; y ^= 1u; }
  if (st & 1u) { unsigned t = x; x = y; y = t; }
  rbit = y;
  cbit = x;
}

// hilbert_encode (curves.hpp:133-143), two bits of (row, col) per step.  A 4-state automaton;
// the state/position transition is a 16-entry table packed into two 32-bit words.
__host__ __device__ __forceinline__ uint64_t hilbert_encode(uint32_t row, uint32_t col, unsigned level) {
  unsigned st = 0;
  uint64_t v = 0;
  for (int b = (int)level - 1; b >= 0; --b) {
    const unsigned pos = hil_position(st, (row >> b) & 1u, (col >> b) & 1u);
    v = (v << 2) | pos;
    st = hil_child(st, pos);
  }
  return v;
}
__host__ __device__ __forceinline__ void hilbert_decode(uint64_t d, unsigned level, uint32_t& row, uint32_t& col) {
  unsigned st = 0;
  uint32_t r = 0, c = 0;
  for (int b = (int)level - 1; b >= 0; --b) {
    const unsigned pos = (unsigned)((d >> (2 * b)) & 3u);
    unsigned rb, cb;
    hil_cell(st, pos, rb, cb);
    r |= rb << b;
    c |= cb << b;
    st = hil_child(st, pos);
  }
  row = r;
  col = c;
}

// Table-driven Hilbert coding, 4 bits of row and column per step: enc[state << 8 | r4 << 4 | c4] =
// (8 output bits | next state << 8), dec[state << 8 | 4 digits] = (r4 | c4 << 4 | next << 8).
// The tables are the 1-bit automaton above composed four times; a CTA builds them in shared memory
// (hil_tables_init, then __syncthreads) -- 6 table steps instead of 22-26 automaton steps.
__device__ __forceinline__ void hil_tables_init(uint16_t* enc, uint16_t* dec) {
  for (unsigned i = threadIdx.x; i < 1024; i += blockDim.x) {
    const unsigned st0 = i >> 8, v = i & 255u;
    unsigned st = st0, out = 0;
    for (int b = 3; b >= 0; --b) {
      const unsigned pos = hil_position(st, (v >> (4 + b)) & 1u, (v >> b) & 1u);
      out = (out << 2) | pos;
      st = hil_child(st, pos);
    }
    enc[i] = (uint16_t)(out | (st << 8));
    st = st0;
    unsigned r = 0, c = 0;
    for (int b = 3; b >= 0; --b) {
      const unsigned pos = (v >> (2 * b)) & 3u;
      unsigned rb, cb;
      hil_cell(st, pos, rb, cb);
      r |= rb << b;
      c |= cb << b;
      st = hil_child(st, pos);
    }
    dec[i] = (uint16_t)(r | (c << 4) | (st << 8));
  }
}
__device__ __forceinline__ uint64_t hilbert_encode_t(uint32_t row, uint32_t col, unsigned level,
                                                     const uint16_t* enc) {
  unsigned st = 0;
  uint64_t v = 0;
  int b = (int)level - 1;
  for (; b >= 0 && ((b + 1) & 3); --b) {  // leading level % 4 bits one at a time
    const unsigned pos = hil_position(st, (row >> b) & 1u, (col >> b) & 1u);
    v = (v << 2) | pos;
    st = hil_child(st, pos);
  }
  for (; b >= 3; b -= 4) {
    const unsigned e = enc[(st << 8) | (((row >> (b - 3)) & 15u) << 4) | ((col >> (b - 3)) & 15u)];
    v = (v << 8) | (e & 255u);
    st = e >> 8;
  }
  return v;
}
__device__ __forceinline__ void hilbert_decode_t(uint64_t d, unsigned level, uint32_t& row, uint32_t& col,
                                                 const uint16_t* dec) {
  unsigned st = 0;
  uint32_t r = 0, c = 0;
  int b = (int)level - 1;
  for (; b >= 0 && ((b + 1) & 3); --b) {
    const unsigned pos = (unsigned)((d >> (2 * b)) & 3u);
    unsigned rb, cb;
    hil_cell(st, pos, rb, cb);
    r |= rb << b;
    c |= cb << b;
    st = hil_child(st, pos);
  }
  for (; b >= 3; b -= 4) {
    const unsigned e = dec[(st << 8) | (unsigned)((d >> (2 * (b - 3))) & 255u)];
    r |= (e & 15u) << (b - 3);
    c |= ((e >> 4) & 15u) << (b - 3);
    st = e >> 8;
  }
  row = r;
  col = c;
}

// Declares and builds the CTA's Hilbert tables (s_henc / s_hdec); must run before any early return.
#define SPMV_HILBERT_TABLES()                        \
  __shared__ uint16_t s_henc[1024], s_hdec[1024];    \
  hil_tables_init(s_henc, s_hdec);                   \
  __syncthreads()

// morton_encode (curves.hpp:107-117): row bit above column bit, by magic-number spreading.
__host__ __device__ __forceinline__ uint64_t spread_bits(uint32_t v) {
  uint64_t x = v;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}
__host__ __device__ __forceinline__ uint32_t compact_bits(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return (uint32_t)x;
}
__host__ __device__ __forceinline__ uint64_t morton_encode(uint32_t row, uint32_t col, unsigned level) {
  const uint32_t mask = level >= 32 ? 0xFFFFFFFFu : ((1u << level) - 1u);
  return (spread_bits(row & mask) << 1) | spread_bits(col & mask);
}

__host__ __device__ __forceinline__ unsigned bit_width64(uint64_t v) {
#ifdef __CUDA_ARCH__
  return v ? 64u - (unsigned)__clzll((long long)v) : 0u;
#else
  return v ? 64u - (unsigned)__builtin_clzll(v) : 0u;
#endif
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// ---------------------------------------------------------------- TMA bulk copies + mbarrier
// 1-D bulk copies (cp.async.bulk, no tensor map) global -> shared, completion counted in bytes on
// an mbarrier.  Addresses and sizes must be multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}

}  // namespace spmvcu
