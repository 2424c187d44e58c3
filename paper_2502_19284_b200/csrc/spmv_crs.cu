// spmv_crs.cu -- the CRS engines: sequential CRS, ParCRS and merge-path CRS (sm_100a).
//
//  * SeqCrs (spmv_crs_seq, inc/crs.hpp:43-57): one thread per row summing in storage order with
//    explicitly rounded multiply and add (no FMA contraction), so y is BITWISE equal to the
//    reference's sequential kernel.
//  * ParCrs (spmv_parcrs, inc/spmv_parallel.hpp:106-125): rows claimed by sub-warp groups whose
//    width is the next power of two >= the mean row length (2 on heavy-tailed row lengths); lanes
//    stride the row, shuffle-reduce; rows above a length threshold get one CTA each.
//  * Merge (spmv_merge, inc/spmv_parallel.hpp:130-160): the merge path over (row_ptr[1..m],
//    0..nnz-1) is cut into equal tiles at build time (merge_partition: one diagonal search per
//    tile boundary, spmv_parallel.hpp:47-86).  Each tile leaves one (row, partial) carry-out and a
//    fix-up kernel adds the carries of rows spanning tiles in tile order (deterministic; the
//    sequential carry loop of spmv_parallel.hpp:157-159).  The tile kernel
//    (merge_spmv_vec_kernel, 256 threads, 32 * {32,16,8} items per warp tile by matrix size) walks
//    the tile's nonzeros in lane-blocked passes of 128 -- each lane loads 4 consecutive col_ind /
//    data entries with one 128-bit and one 256-bit load, gathers and multiplies in registers (two
//    passes in flight); row ends of the pass are scattered to the element they close through a
//    128-entry shared map, each lane walks its 4 products, one warp segmented scan joins the
//    lanes.  Kernel and fix-up are launched with programmatic stream serialization (the next grid
//    is resident while the previous drains; griddepcontrol.wait before any memory access).
//    With a hot-x plan (a column-skewed matrix, build_hot_columns) the tile kernel is instead the
//    persistent merge_hot_kernel: one 1,024-thread CTA per SM keeps x at the most referenced
//    columns in shared memory and walks 8-wide, software-pipelined passes of 256 elements.
//    Superseded designs and what they measured at cfg2 are listed in DESIGN.md section 4 (shared-
//    memory / warp-staged / shuffle-only tiles, a persistent TMA bulk-copy ring, TMA gather4 x
//    fetches, a distributed-shared-memory hot copy); the floor for an LSU-gather kernel is the
//    L1TEX wavefront rate of the x gathers (one per gathered line).
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
extern thread_local std::string g_last_error;
namespace {

// The first nlong CTAs each own one long row: all threads form the rounded products of the next
// 2048-element chunk in shared memory while thread 0 adds the current chunk in storage order
// (double buffered), so the sum is the reference's left-to-right chain.  The other CTAs run one
// thread per short row with 8 products in flight ahead of the sequential adds.
constexpr int kSeqThreads = 256;
constexpr int kSeqChunk = 2048;

__global__ void __launch_bounds__(kSeqThreads) seq_crs_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, uint32_t m, const uint32_t* __restrict__ long_rows,
    uint32_t nlong, uint32_t lim) {
  if (blockIdx.x < nlong) {
    __shared__ double prod[2][kSeqChunk];
    const uint32_t r = long_rows[blockIdx.x];
    const uint32_t b = row_ptr[r], e = row_ptr[r + 1];
    const uint32_t nch = (e - b + kSeqChunk - 1) / kSeqChunk;
    auto fill = [&](uint32_t c) {
      const uint32_t base = b + c * kSeqChunk;
#pragma unroll
      for (int u = 0; u < kSeqChunk / kSeqThreads; ++u) {
        const uint32_t k = base + u * kSeqThreads + threadIdx.x;
        if (k < e) prod[c & 1][u * kSeqThreads + threadIdx.x] = __dmul_rn(__ldg(val + k), __ldg(x + __ldg(col + k)));
      }
    };
    fill(0);
    __syncthreads();
    double sum = 0.0;
    for (uint32_t c = 0; c < nch; ++c) {
      if (c + 1 < nch) fill(c + 1);
      if (threadIdx.x == 0) {
        const uint32_t cnt = min((uint32_t)kSeqChunk, e - b - c * kSeqChunk);
        const double* p = prod[c & 1];
#pragma unroll 16
        for (uint32_t i = 0; i < cnt; ++i) sum = __dadd_rn(sum, p[i]);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) y[r] = sum;
    return;
  }
  const uint32_t i = (blockIdx.x - nlong) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t b = row_ptr[i], e = row_ptr[i + 1];
  if (e - b > lim) return;  // owned by a long-row CTA
  double sum = 0.0;
  uint32_t k = b;
  for (; k + 8 <= e; k += 8) {
    double p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = __dmul_rn(__ldg(val + k + u), __ldg(x + __ldg(col + k + u)));
#pragma unroll
    for (int u = 0; u < 8; ++u) sum = __dadd_rn(sum, p[u]);
  }
  for (; k < e; ++k) sum = __dadd_rn(sum, __dmul_rn(__ldg(val + k), __ldg(x + __ldg(col + k))));
  y[i] = sum;
}

// The first nlong CTAs each sum one long row (4 independent strided partials per thread, then a
// CTA reduction); the remaining CTAs run the sub-warp groups over all other rows.
template <int G>
__global__ void __launch_bounds__(256) par_crs_kernel(const uint32_t* __restrict__ row_ptr,
                                                      const uint32_t* __restrict__ col,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ x,
                                                      double* __restrict__ y, uint32_t m,
                                                      const uint32_t* __restrict__ long_rows, uint32_t nlong,
                                                      uint32_t lim) {
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const unsigned lane = threadIdx.x & 31u;
  if (blockIdx.x < nlong) {
    __shared__ double part[8];
    const uint32_t r = long_rows[blockIdx.x];
    const uint32_t b = row_ptr[r], e = row_ptr[r + 1];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    uint32_t k = b + threadIdx.x;
    for (; k + 768 < e; k += 1024) {
      s0 += ld_stream(val + k, pf) * ld_x(x + ld_stream(col + k, pf), pl);
      s1 += ld_stream(val + k + 256, pf) * ld_x(x + ld_stream(col + k + 256, pf), pl);
      s2 += ld_stream(val + k + 512, pf) * ld_x(x + ld_stream(col + k + 512, pf), pl);
      s3 += ld_stream(val + k + 768, pf) * ld_x(x + ld_stream(col + k + 768, pf), pl);
    }
    for (; k < e; k += 256) s0 += ld_stream(val + k, pf) * ld_x(x + ld_stream(col + k, pf), pl);
    double s = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
    if (lane == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += part[w];
      y[r] = t;
    }
    return;
  }
  const uint64_t gid = (uint64_t)(blockIdx.x - nlong) * blockDim.x + threadIdx.x;
  const uint32_t sub = threadIdx.x & (G - 1);
  const uint64_t group = gid / G;
  const uint64_t ngroups = (uint64_t)(gridDim.x - nlong) * blockDim.x / G;
  const unsigned gmask = (G == 32) ? 0xFFFFFFFFu : (((1u << G) - 1u) << (lane & ~(unsigned)(G - 1)));
  for (uint64_t r = group; r < m; r += ngroups) {
    const uint32_t b = row_ptr[r], e = row_ptr[r + 1];
    if (e - b > lim) continue;  // group-uniform: a long-row CTA owns it
    double s = 0.0;
    for (uint32_t k = b + sub; k < e; k += G) s += ld_stream(val + k, pf) * ld_x(x + ld_stream(col + k, pf), pl);
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(gmask, s, off, G);
    if (sub == 0) y[r] = s;
  }
}

// ---------------------------------------------------------------- lane-blocked vector variant

// 4 consecutive nonzeros of a 128-element pass per lane, loaded with one 128-bit col_ind load and
// one 256-bit data load (sm_100 ld.global.v4.f64); the products never leave registers.  Elements
// outside [j0, j1) are masked (the tile's merge-path element range is not 4-aligned).
// x[c], or its shared-memory copy: with a hot-x plan the column index of the most referenced
// columns carries 0x80000000 | slot (merge_hot_col) and sx holds x at those columns.
template <bool HOT, bool NA = false>
__device__ __forceinline__ double gather_x(const double* __restrict__ x, const double* sx, uint32_t c, uint64_t pl) {
  if constexpr (HOT) {
    double v;
    if ((int)c < 0) v = sx[c & 0x7FFFFFFFu];
    else v = ld_xm<1>(x + c, pl);  // no L1 allocation: the L1 left beside the hot copy keeps its
                                   // lines for gathers in flight (default allocate / plain / .cg:
                                   // 271 / 271 / 265 vs 265 us at cfg2)
    return v;
  } else {  // (NA: no column skew, the L1 keeps no x worth reusing -- merge_x_noalloc)
    return NA ? ld_xm<1>(x + c, pl) : ld_x(x + c, pl);
  }
}

template <bool NA>
__device__ __forceinline__ void vec_products(const uint32_t* __restrict__ col, const double* __restrict__ val,
                                             const double* __restrict__ x, uint32_t k, uint32_t j0, uint32_t j1,
                                             uint64_t pf, uint64_t pl, double p[4]) {
  if (k >= j0 && k + 3 < j1) {
    const uint4 c = ld_stream4(col + k, pf);
    double v0, v1, v2, v3;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "l"(val + k), "l"(pf));
    p[0] = v0 * gather_x<false, NA>(x, nullptr, c.x, pl);
    p[1] = v1 * gather_x<false, NA>(x, nullptr, c.y, pl);
    p[2] = v2 * gather_x<false, NA>(x, nullptr, c.z, pl);
    p[3] = v3 * gather_x<false, NA>(x, nullptr, c.w, pl);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t e = k + u;
      p[u] = (e >= j0 && e < j1) ? ld_stream(val + e, pf) * gather_x<false, NA>(x, nullptr, ld_stream(col + e, pf), pl)
                                   : 0.0;
    }
  }
}

// One 128-element pass of a warp tile.  Row ends falling in the pass are read 32 at a time from
// row_ptr and scattered to the element they close (smap: element -> row + 1); each lane
// then walks its 4 products in registers, stores rows that close inside the lane, and the lane
// tails are combined by one warp segmented scan (carry = the open row's running sum).
// ACC (column panels after the first): finished rows are added to y (the earlier panels' sums)
// instead of stored; rows with no entries in the panel are left alone unless they must also be
// scattered to the peers (the last panel of the fused exchange stores every row's final value).
// (SCATTER: the peers receive the tile's finished rows in one coalesced copy at the tile end --
// push_rows -- instead of one remote store per row per peer as the row closes)
// A doubly-compressed ACC panel walks local rows: local row r is global row rows[r].
template <bool SCATTER, bool ACC, bool LAST>
__device__ __forceinline__ void put_row_m(double* y, const uint32_t* __restrict__ rows, const RowDest& d, uint32_t r,
                                          double v) {
  if constexpr (ACC) {
    if (rows) r = __ldg(rows + r);
    v += y[r];
  }
  put_row<false, LAST>(y, d, r, v);
}

// Row ends of one pass, read 32 at a time from row_ptr and scattered to the element that closes the
// row (smap: element - base -> row + 1); empty rows (and rows whose elements precede the tile) are
// stored right away.
template <bool SCATTER, bool ACC, bool LAST>
__device__ __forceinline__ void row_ends(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ rows,
                                         double* __restrict__ y, uint32_t* smap, uint32_t base, uint32_t pend,
                                         uint32_t j0, uint32_t r1, uint32_t& rp, uint32_t& prevE, unsigned lane,
                                         const RowDest& dest) {
  while (rp < r1) {
    const uint32_t idx = rp + lane;
    const bool have = idx < r1;
    const uint32_t E = have ? __ldg(row_ptr + idx + 1) : 0xFFFFFFFFu;
    uint32_t S = __shfl_up_sync(0xFFFFFFFFu, E, 1);
    if (lane == 0) S = prevE;
    const bool in = have && E <= pend;
    if (in) {
      if (E == S || E <= j0) {  // empty, or elements precede the tile
        if (!ACC) put_row_m<SCATTER, ACC, LAST>(y, rows, dest, idx, 0.0);
      }
      else smap[E - 1 - base] = idx + 1u;   // closes at element E - 1 of this pass
    }
    const unsigned inmask = __ballot_sync(0xFFFFFFFFu, in);
    const int nin = __popc(inmask);
    if (nin) prevE = __shfl_sync(0xFFFFFFFFu, E, nin - 1);
    rp += (uint32_t)nin;
    if (nin < 32) break;
  }
}

// Each lane walks its 4 products in registers (rows closing inside the lane are stored), the lane
// tails are combined by one warp segmented scan (carry = the open row's running sum).
// ACC (column panels after the first): finished rows are added to y (the earlier panels' sums)
// instead of stored; rows with no entries in the panel are left alone unless they must also be
// scattered to the peers (the last panel of the fused exchange stores every row's final value).
// (SCATTER: the peers receive the tile's finished rows in one coalesced copy at the tile end --
// push_rows -- instead of one remote store per row per peer as the row closes)
// A doubly-compressed ACC panel walks local rows: local row r is global row rows[r].
template <bool SCATTER, bool ACC, bool LAST>
__device__ __forceinline__ void pass_reduce(const uint32_t* __restrict__ rows, double* __restrict__ y,
                                            const uint32_t* smap, uint32_t rp0, const double p[4], double& carry,
                                            unsigned lane, const RowDest& dest) {
  __syncwarp();
  // Row ids only grow along the tile, so entries written by earlier passes (row + 1 <= rp0) read as
  // "no row end" and the map is never cleared (saves a 512-byte shared store per pass).
  const uint4 m4 = *reinterpret_cast<const uint4*>(smap + 4 * lane);
  const int rid[4] = {m4.x > rp0 ? (int)(m4.x - 1u) : -1, m4.y > rp0 ? (int)(m4.y - 1u) : -1,
                      m4.z > rp0 ? (int)(m4.z - 1u) : -1, m4.w > rp0 ? (int)(m4.w - 1u) : -1};
  double run = 0.0, first_val = 0.0;
  int first_row = -1;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    run += p[u];
    if (rid[u] >= 0) {
      if (first_row < 0) {
        first_row = rid[u];
        first_val = run;
      } else {
        put_row_m<SCATTER, ACC, LAST>(y, rows, dest, rid[u], run);
      }
      run = 0.0;
    }
  }
  const unsigned heads = __ballot_sync(0xFFFFFFFFu, first_row >= 0);
  const unsigned le = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int seg = heads & le ? 31 - __clz(heads & le) : 0;
  // (a data-dependent depth -- log2 of the longest segment -- measured slower: 313 vs 292 us)
  // (skipping levels no segment needs -- runs of the uniform non-head mask -- measured 293 vs 291)
  double v = run;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double ov = __shfl_up_sync(0xFFFFFFFFu, v, off);
    if ((int)lane - off >= seg) v += ov;
  }
  double ex = __shfl_up_sync(0xFFFFFFFFu, v, 1);
  if (lane == 0) ex = 0.0;
  if (first_row >= 0)
    put_row_m<SCATTER, ACC, LAST>(y, rows, dest, first_row,
                                  first_val + ex + ((heads & ((1u << lane) - 1u)) ? 0.0 : carry));
  const double v31 = __shfl_sync(0xFFFFFFFFu, v, 31);
  carry = heads ? v31 : carry + v31;
  __syncwarp();
}

// One 128-element pass of a warp tile: its row ends, then the reduction.
template <bool SCATTER, bool ACC, bool LAST>
__device__ __forceinline__ void vec_pass(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ rows,
                                         double* __restrict__ y, uint32_t* smap, uint32_t base, uint32_t j0,
                                         uint32_t j1, uint32_t r1, uint32_t& rp, uint32_t& prevE, const double p[4],
                                         double& carry, unsigned lane, const RowDest& dest) {
  const uint32_t rp0 = rp;  // map entries <= rp0 are stale (rows closed by earlier passes) or unset
  row_ends<SCATTER, ACC, LAST>(row_ptr, rows, y, smap, base, min(base + 128u, j1), j0, r1, rp, prevE, lane, dest);
  pass_reduce<SCATTER, ACC, LAST>(rows, y, smap, rp0, p, carry, lane, dest);
}

// The fused exchange: rows [lo, hi) of y, just finished by this warp, copied to every peer's buffer
// at the shard's row offset -- coalesced 8-byte stores per lane, one contiguous run per peer.
__device__ __forceinline__ void push_rows(const double* y, const RowDest& d, uint32_t lo, uint32_t hi,
                                          unsigned lane) {
  for (uint32_t r = lo + lane; r < hi; r += 32) {
    const double v = y[r];
    for (unsigned i = 0; i < d.n; ++i) d.p[i][d.off + r] = v;
  }
}

// Merge-path tiles of 32 * IPT items per warp, the tile's elements walked in lane-blocked passes of
// 128 with two passes' loads and gathers in flight.  No product staging: shared memory holds only
// the 128-entry row map.  LAST: the final (or only) column panel -- its stores of y are final and
// leave the L2 with evict-first; earlier panels' partial sums are re-read by the next panel.
// passes in flight per warp (loads and gathers of kMergeNP * 128 elements issued together; 3 passes
// at 5 CTAs / SM measured 316 vs 289 us at cfg2, 4 spill)
constexpr int kMergeNP = 2;

// One warp tile t: the merge path's items [tile_row/nnz[t], tile_row/nnz[t + 1]).
template <bool SCATTER, bool ACC, bool LAST, bool NA>
__device__ __forceinline__ void merge_tile(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ rows,
                                           const uint32_t* __restrict__ col, const double* __restrict__ val,
                                           const double* __restrict__ x, double* __restrict__ y,
                                           const uint32_t* __restrict__ tile_row,
                                           const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
                                           double* __restrict__ carry_val, uint32_t t, uint32_t* smap,
                                           unsigned lane, const RowDest& dest) {
  *reinterpret_cast<uint4*>(smap + 4 * lane) = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const uint32_t j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
  // (a fractional evict-last share for x larger than the L2 measured within 1 % on cfg3-5)
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  uint32_t rp = r0;
  uint32_t prevE = __ldg(row_ptr + r0);
  double carry = 0.0;
  bool more = true;
  __syncwarp();
  for (uint32_t base = j0 & ~3u; more; base += 128u * kMergeNP) {
    double p[kMergeNP][4];
#pragma unroll
    for (int i = 0; i < kMergeNP; ++i)
      vec_products<NA>(col, val, x, base + 128u * i + 4 * lane, j0, j1, pf, pl, p[i]);
#pragma unroll
    for (int i = 0; i < kMergeNP; ++i) {
      if (i > 0 && !(base + 128u * i < j1 || rp < r1)) {
        more = false;
        break;
      }
      vec_pass<SCATTER, ACC, LAST>(row_ptr, rows, y, smap, base + 128u * i, j0, j1, r1, rp, prevE, p[i], carry,
                                   lane, dest);
    }
    if (!(base + 128u * kMergeNP < j1 || rp < r1)) more = false;
  }
  if (lane == 0) {
    carry_row[t] = r1;
    carry_val[t] = carry;
  }
  if constexpr (SCATTER) {
    // rows final in this tile: [r0 + 1, r1), and row r0 too in tile 0 (every other tile's first
    // row receives the previous tiles' carries in the fix-up, which pushes it)
    __syncwarp();
    push_rows(y, dest, t == 0 ? r0 : r0 + 1u, r1, lane);
  }
  __syncwarp();
}

// ---------------------------------------------------------------- persistent 8-wide tiles
// The persistent kernels walk a tile in passes of 256 elements, 8 consecutive ones per lane: one
// 256-bit col_ind load and two 256-bit data loads (L2 evict-first as an instruction qualifier --
// no policy register), one row-map round trip and one warp segmented scan per 256 elements (half
// the merge instructions per element of the 4-wide passes).  Software pipelined: col_ind of the
// next pass is loaded one pass ahead, and the row window (row_ptr of the next 32 rows) is loaded
// with the pass's data and x gathers, so a pass costs about one memory latency instead of three
// in series (col -> x, then row_ptr).
struct Cols8 {
  uint32_t c[8];
};

__device__ __forceinline__ Cols8 cols8(const uint32_t* __restrict__ col, uint32_t k, uint32_t j0, uint32_t j1) {
  Cols8 r;
  if (k >= j0 && k + 7 < j1) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.c[0]), "=r"(r.c[1]), "=r"(r.c[2]), "=r"(r.c[3]), "=r"(r.c[4]), "=r"(r.c[5]),
                   "=r"(r.c[6]), "=r"(r.c[7])
                 : "l"(col + k));
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) r.c[u] = (k + u >= j0 && k + u < j1) ? __ldg(col + k + u) : 0u;
  }
  return r;
}

__device__ __forceinline__ void ld_val4(const double* p, double v[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

template <bool HOT>
__device__ __forceinline__ void products8(const double* __restrict__ val, const double* __restrict__ x,
                                          const double* sx, const Cols8& c, uint32_t k, uint32_t j0, uint32_t j1,
                                          uint64_t pl, double p[8]) {
  if (k >= j0 && k + 7 < j1) {
    double v[8];
    ld_val4(val + k, v);
    ld_val4(val + k + 4, v + 4);
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = v[u] * gather_x<HOT>(x, sx, c.c[u], pl);
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t e = k + u;
      p[u] = (e >= j0 && e < j1) ? __ldg(val + e) * gather_x<HOT>(x, sx, c.c[u], pl) : 0.0;
    }
  }
}

// y stores of the persistent kernels: the default L2 policy, so that a caller reading y right after
// the multiply (the iterated loop's norm pass) finds it in the L2 (evict-first measured no faster
// for the multiply alone)
__device__ __forceinline__ void st_y(double* y, uint32_t r, double v, uint64_t) { y[r] = v; }

// The rescaled loop's mass inside the persistent kernel (spmv_merge_norms, NORMS): sum of y = sum of
// the products, per lane; sigma = a factor on the products (the loop's drift correction, 1 unless
// the stored vector's scale left [2^-256, 2^256]).  (The residual sum |y_r - u_r| in here too --
// u_r fetched with the row window, shuffled to the lane that finalises the row -- measured slower
// than the loop's separate pass: cfg2 346 vs 302 us per iteration.)
struct TileNorms {
  double mass, sigma;
};

template <bool SCATTER>
__device__ __forceinline__ void row_ends8(const uint32_t* __restrict__ row_ptr, double* __restrict__ y,
                                          uint16_t* smap, uint32_t r0, uint32_t base, uint32_t pend, uint32_t j0,
                                          uint32_t r1,
                                          uint32_t& rp, uint32_t& prevE, uint32_t& wb, uint32_t& wE, uint32_t& wS0,
                                          unsigned lane, uint64_t ps) {
  while (rp < r1) {
    const uint32_t idx = wb + lane;
    uint32_t S = __shfl_up_sync(0xFFFFFFFFu, wE, 1);
    if (lane == 0) S = wS0;
    const bool in = idx >= rp && idx < r1 && wE <= pend;
    if (in && (wE == S || wE <= j0)) st_y(y, idx, 0.0, ps);  // empty, or elements precede the tile
    else if (in) smap[wE - 1 - base] = (uint16_t)(idx - r0 + 1u);  // closes at element wE - 1 of the pass
    const unsigned inmask = __ballot_sync(0xFFFFFFFFu, in);
    if (inmask) {
      prevE = __shfl_sync(0xFFFFFFFFu, wE, 31 - __clz(inmask));
      rp += (uint32_t)__popc(inmask);
    }
    if (rp < wb + 32u || rp >= r1) break;
    wb = rp;  // every row of the window closed: the next 32
    wS0 = prevE;
    wE = wb + lane < r1 ? __ldg(row_ptr + wb + 1 + lane) : 0xFFFFFFFFu;
  }
}

// (the row map holds row - r0 + 1 as 16 bits: a tile spans at most 65535 rows, build_merge_plan)
__device__ __forceinline__ void reduce8(double* __restrict__ y, const uint16_t* smap, uint32_t r0, uint32_t rp0,
                                        const double p[8], double& carry, unsigned lane, uint64_t ps) {
  __syncwarp();
  const uint4 mq = *reinterpret_cast<const uint4*>(smap + 8 * lane);
  const uint32_t mm[8] = {mq.x & 0xFFFFu, mq.x >> 16, mq.y & 0xFFFFu, mq.y >> 16,
                          mq.z & 0xFFFFu, mq.z >> 16, mq.w & 0xFFFFu, mq.w >> 16};
  const uint32_t stale = rp0 - r0;  // entries <= stale: rows closed by earlier passes, or unset
  double run = 0.0, first_val = 0.0;
  int first_row = -1;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    run += p[u];
    const bool end = mm[u] > stale;
    if (end && first_row >= 0) st_y(y, r0 + mm[u] - 1u, run, ps);
    if (end && first_row < 0) {
      first_row = (int)(r0 + mm[u] - 1u);
      first_val = run;
    }
    run = end ? 0.0 : run;
  }
  const unsigned heads = __ballot_sync(0xFFFFFFFFu, first_row >= 0);
  const unsigned le = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int seg = heads & le ? 31 - __clz(heads & le) : 0;
  double v = run;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double ov = __shfl_up_sync(0xFFFFFFFFu, v, off);
    v += ((int)lane - off >= seg) ? ov : 0.0;
  }
  double ex = __shfl_up_sync(0xFFFFFFFFu, v, 1);
  if (lane == 0) ex = 0.0;
  if (first_row >= 0)
    st_y(y, (uint32_t)first_row, first_val + ex + ((heads & ((1u << lane) - 1u)) ? 0.0 : carry), ps);
  const double v31 = __shfl_sync(0xFFFFFFFFu, v, 31);
  carry = heads ? v31 : carry + v31;
  __syncwarp();
}

template <bool HOT, bool SCATTER, bool NORMS>
__device__ __forceinline__ void merge_tile8(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                                            const double* __restrict__ val, const double* __restrict__ x,
                                            const double* sx, double* __restrict__ y,
                                            const uint32_t* __restrict__ tile_row,
                                            const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
                                            double* __restrict__ carry_val, uint32_t t, uint16_t* smap,
                                            unsigned lane, const RowDest& dest, uint64_t pl, uint64_t ps,
                                            TileNorms& nm) {
  *reinterpret_cast<uint4*>(smap + 8 * lane) = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const uint32_t j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
  uint32_t rp = r0;
  uint32_t prevE = __ldg(row_ptr + r0);
  double carry = 0.0;
  uint32_t base = j0 & ~7u;
  Cols8 cn = cols8(col, base + 8 * lane, j0, j1);
  __syncwarp();
  while (base < j1 || rp < r1) {
    uint32_t wb = rp, wS0 = prevE;
    uint32_t wE = rp + lane < r1 ? __ldg(row_ptr + rp + 1 + lane) : 0xFFFFFFFFu;
    double p[8];
    products8<HOT>(val, x, sx, cn, base + 8 * lane, j0, j1, pl, p);
    cn = cols8(col, base + 256u + 8 * lane, j0, j1);
    if constexpr (NORMS) {
#pragma unroll
      for (int u = 0; u < 8; ++u) p[u] *= nm.sigma;
      nm.mass += ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
    }
    const uint32_t rp0 = rp;
    row_ends8<SCATTER>(row_ptr, y, smap, r0, base, min(base + 256u, j1), j0, r1, rp, prevE, wb, wE, wS0, lane, ps);
    reduce8(y, smap, r0, rp0, p, carry, lane, ps);
    base += 256u;
  }
  if (lane == 0) {
    carry_row[t] = r1;
    carry_val[t] = carry;
  }
  if constexpr (SCATTER) {
    // rows final in this tile: [r0 + 1, r1), and row r0 too in tile 0 (every other tile's first
    // row receives the previous tiles' carries in the fix-up, which pushes it)
    __syncwarp();
    push_rows(y, dest, t == 0 ? r0 : r0 + 1u, r1, lane);
  }
  __syncwarp();
}

template <int IPT, int WARPS, bool SCATTER, bool ACC, bool LAST, bool NA>
__global__ void __launch_bounds__(WARPS * 32, (kMergeNP > 2 ? 40 : 48) / WARPS) merge_spmv_vec_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ rows, const uint32_t* __restrict__ col,
    const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const uint32_t* __restrict__ tile_row,
    const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
    double* __restrict__ carry_val, uint32_t tiles, const __grid_constant__ RowDest dest) {
  __shared__ __align__(16) uint32_t s_map_all[WARPS][128];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t t = blockIdx.x * WARPS + warp;
  // programmatic dependent launch: resident early, but no memory access before the previous
  // kernel of the stream has completed; the fix-up behind may be launched right away
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (t >= tiles) return;
  merge_tile<SCATTER, ACC, LAST, NA>(row_ptr, rows, col, val, x, y, tile_row, tile_nnz, carry_row, carry_val, t,
                                     s_map_all[warp], lane, dest);
}

// Hot-x variant (R-MAT-like column skew; plan built by build_hot_columns): one persistent CTA of
// kHotWarps warps per SM.  The CTA first copies x at the plan's hot columns (merge_hot_cols, the
// most referenced ones) into shared memory; its warps then walk tiles t = warp id, + grid warps,
// ... with those columns read from shared memory (LDS: a few bank wavefronts per warp instead of
// one L2 sector per lane) and the rest gathered from the L2 without L1 allocation (the L1 left
// beside the hot copy holds the gathers in flight).  NORMS (the rescaled loop without norms): the
// products are scaled by the loop's drift factor and summed per CTA for the mass.
template <bool HOT, bool SCATTER, bool NORMS = false>
__global__ void __launch_bounds__(kHotWarps * 32, 1) merge_hot_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const uint32_t* __restrict__ tile_row,
    const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row, double* __restrict__ carry_val,
    uint32_t tiles, const uint32_t* __restrict__ hot_cols, uint32_t nhot, const __grid_constant__ RowDest dest,
    double* __restrict__ cpart, const double* __restrict__ sigma) {
  extern __shared__ __align__(16) double s_hot[];
  __shared__ __align__(16) uint16_t s_map_all[kHotWarps][256];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const uint64_t pl = policy_evict_last(), ps = policy_evict_first();
  if constexpr (HOT) {
    for (uint32_t i = threadIdx.x; i < nhot; i += kHotWarps * 32) s_hot[i] = ld_x(x + __ldg(hot_cols + i), pl);
    __syncthreads();
  }
  TileNorms nm{0.0, NORMS ? *sigma : 1.0};
  for (uint32_t t = blockIdx.x * kHotWarps + warp; t < tiles; t += gridDim.x * kHotWarps)
    merge_tile8<HOT, SCATTER, NORMS>(row_ptr, col, val, x, s_hot, y, tile_row, tile_nnz, carry_row, carry_val, t,
                                     s_map_all[warp], lane, dest, pl, ps, nm);
  if constexpr (NORMS) {  // this CTA's mass: lanes by xor tree, then warps in order
    __shared__ double s_m[kHotWarps];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nm.mass += __shfl_xor_sync(0xFFFFFFFFu, nm.mass, off);
    if (lane == 0) s_m[warp] = nm.mass;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int w = 0; w < kHotWarps; ++w) b += s_m[w];
      cpart[blockIdx.x] = b;
    }
  }
}

// ---------------------------------------------------------------- carry fix-up

// One lane per tile, 32 tiles per warp.  Runs of equal carry rows are summed with a warp segmented
// scan; the tail lane of a run that starts and ends inside the chunk adds it to y.  A run that
// starts in the chunk and continues past it is finished by the whole warp sweeping the following
// carries 32 at a time.  Runs that started in an earlier chunk are left to that chunk's warp.
// Deterministic (fixed reduction order) and O(run / 32) dependent steps for the longest rows.
// (rows: the panel's compressed row ids, or null; m: the panel's row count)
template <bool SCATTER, bool LAST>
__device__ __forceinline__ void fixup_runs(const uint32_t* __restrict__ carry_row, const double* __restrict__ carry_val,
                                           uint32_t tiles, double* __restrict__ y, uint32_t m,
                                           const uint32_t* __restrict__ rows, const RowDest& dest) {
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u;
  if (base >= tiles) return;
  const uint32_t t = base + lane;
  const uint32_t r = t < tiles ? carry_row[t] : 0xFFFFFFFFu;
  double v = t < tiles ? carry_val[t] : 0.0;
  uint32_t prow = __shfl_up_sync(0xFFFFFFFFu, r, 1);
  if (lane == 0) prow = base > 0 ? carry_row[base - 1] : ~r;
  const unsigned heads = __ballot_sync(0xFFFFFFFFu, r != prow);
  const unsigned le = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int seg = 31 - __clz((heads | 1u) & le);
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double o = __shfl_up_sync(0xFFFFFFFFu, v, off);
    if ((int)lane - off >= seg) v += o;
  }
  const bool started_here = (heads >> seg) & 1u;
  const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
  if (tail && lane != 31 && started_here && r < m) {
    const uint32_t g = rows ? rows[r] : r;
    put_row<SCATTER, LAST>(y, dest, g, y[g] + v);
  }
  // the chunk's last run: finish it here if it started here
  const uint32_t r31 = __shfl_sync(0xFFFFFFFFu, r, 31);
  const bool own31 = __shfl_sync(0xFFFFFFFFu, started_here, 31);
  if (!own31 || r31 >= m) return;
  double total = __shfl_sync(0xFFFFFFFFu, v, 31);
  for (uint32_t nb = base + 32; nb < tiles; nb += 32) {
    const uint32_t u = nb + lane;
    const bool in = u < tiles && carry_row[u] == r31;
    const unsigned match = __ballot_sync(0xFFFFFFFFu, in);
    const unsigned runlen = match == 0xFFFFFFFFu ? 32u : (unsigned)(__ffs(~match) - 1);
    double w = lane < runlen ? carry_val[u] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) w += __shfl_xor_sync(0xFFFFFFFFu, w, off);
    total += w;
    if (runlen < 32) break;
  }
  if (lane == 0) {
    const uint32_t g = rows ? rows[r31] : r31;
    put_row<SCATTER, LAST>(y, dest, g, y[g] + total);
  }
}

template <bool SCATTER, bool LAST>
__global__ void merge_fixup_kernel(const uint32_t* __restrict__ carry_row,
                                   const double* __restrict__ carry_val, uint32_t tiles,
                                   double* __restrict__ y, uint32_t m, const uint32_t* __restrict__ rows,
                                   const __grid_constant__ RowDest dest) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  fixup_runs<SCATTER, LAST>(carry_row, carry_val, tiles, y, m, rows, dest);
}

// The carry fix-up of spmv_merge_norms: merge_fixup_kernel's work (no peers, final y), then the
// last block to finish (ticket) sums the tile kernel's per-CTA masses in a fixed order and updates
// the loop state as iter_pass_kernel does for a rescaled iteration without norms (iterate.cu).
__global__ void __launch_bounds__(256) merge_fixup_norms_kernel(const uint32_t* __restrict__ carry_row,
                                                                const double* __restrict__ carry_val, uint32_t tiles,
                                                                double* __restrict__ y, uint32_t m, IterScratch* sc,
                                                                uint32_t nparts) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  fixup_runs<false, true>(carry_row, carry_val, tiles, y, m, nullptr, RowDest{});
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || threadIdx.x >= 32) return;
  __threadfence();
  const unsigned lane = threadIdx.x;
  double tm = 0.0;
  for (uint32_t i = lane; i < nparts; i += 32) tm += __ldcg(sc->cpart + i);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tm += __shfl_xor_sync(0xFFFFFFFFu, tm, off);
  if (lane == 0) {
    // y = sigma A u_k and x_k = s_k u_k: mass_k = sum A x_k = (s_k / sigma) sum y; x_{k+1} = A x_k /
    // mass_k = y / sum y, so the stored vector stays y and s_{k+1} = 1 / sum y -- if that leaves
    // [2^-256, 2^256] the next multiply scales its products by it (sigma), which brings the next
    // stored vector back to unit scale
    const double sigma = sc->pscale, sk = sc->scale;
    sc->pair[0] = 0.0;
    sc->pair[1] = sk / sigma * tm;
    const double nxt = 1.0 / tm;
    sc->scale = nxt;
    sc->pscale = (fabs(nxt) >= 0x1p-256 && fabs(nxt) <= 0x1p256) ? 1.0 : nxt;
    sc->ticket = 0;
    sc->iter += 1;
  }
}

// ---------------------------------------------------------------- launchers

using Scratch = Format::Scratch;

// Launch with programmatic stream serialization: the kernel may be scheduled while the previous
// kernel of the stream drains (it waits with griddepcontrol.wait before touching memory).
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned threads, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Panel k of a column-panelled format (k = 0 and one panel: the plain CRS arrays), then its carry
// fix-up.  The fix-up of panel k runs before panel k + 1's kernel (stream order; PDL waits for full
// completion), so the accumulating panels read final sums.
template <int IPT, bool SCATTER, bool ACC, bool LAST>
void launch_merge_panel(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s,
                        const RowDest& dest, uint32_t k) {
  constexpr int WARPS = kMergeThreads / 32;
  const uint32_t t0 = f.panel_tile_off[k], tiles = f.panel_tile_off[k + 1] - t0, o = t0 + k;
  if (tiles == 0) return;
  const bool pan = f.merge_panels > 1;
  const uint32_t* rp = pan ? f.find("merge_panel_row_ptr")->as<uint32_t>() + f.panel_rp_off[k]
                           : f.find("row_ptr")->as<uint32_t>();
  const uint32_t* rows = k > 0 && f.panel_rows_off[k] != 0xFFFFFFFFu
                             ? f.find("merge_panel_rows")->as<uint32_t>() + f.panel_rows_off[k]
                             : nullptr;
  const uint32_t* col = f.find(pan ? "merge_panel_col" : "col_ind")->as<uint32_t>();
  const double* val = f.find(pan ? "merge_panel_data" : "data")->as<double>();
  const uint32_t* trow = f.find("merge_tile_row")->as<uint32_t>() + o;
  const uint32_t* tnnz = f.find("merge_tile_nnz")->as<uint32_t>() + o;
  if (f.merge_x_noalloc)
    launch_pdl(merge_spmv_vec_kernel<IPT, WARPS, SCATTER, ACC, LAST, true>, (tiles + WARPS - 1) / WARPS,
               kMergeThreads, s, rp, rows, col, val, x, y, trow, tnnz, sc->carry_row + t0, sc->carry_val + t0, tiles,
               dest);
  else
    launch_pdl(merge_spmv_vec_kernel<IPT, WARPS, SCATTER, ACC, LAST, false>, (tiles + WARPS - 1) / WARPS,
               kMergeThreads, s, rp, rows, col, val, x, y, trow, tnnz, sc->carry_row + t0, sc->carry_val + t0, tiles,
               dest);
  launch_pdl(merge_fixup_kernel<SCATTER, LAST>, (tiles + 255) / 256, 256, s, sc->carry_row + t0,
             (const double*)(sc->carry_val + t0), tiles, y, f.panel_nrows[k], rows, dest);
}

// The tile kernels' own peer push (SCATTER): the single panel, or panel 0 of a panelled multiply
// run last (launch_merge_panels_scatter).
// The persistent plan (one panel only; with or without hot x): merge_hot_kernel, then the carry fix-up.
template <bool HOT, bool SCATTER>
void launch_merge_persistent(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s,
                             const RowDest& dest) {
  if (HOT)
    once_per_device([] {
      cudaFuncSetAttribute(merge_hot_kernel<HOT, SCATTER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kHotMaxSlots * 8);
    });
  const uint32_t tiles = f.merge_tiles;
  const uint32_t* rp = f.find("row_ptr")->as<uint32_t>();
  const uint32_t* col = f.find(HOT ? "merge_hot_col" : "col_ind")->as<uint32_t>();
  const double* val = f.find("data")->as<double>();
  const uint32_t* hot = HOT ? f.find("merge_hot_cols")->as<uint32_t>() : nullptr;
  const uint32_t* trow = f.find("merge_tile_row")->as<uint32_t>();
  const uint32_t* tnnz = f.find("merge_tile_nnz")->as<uint32_t>();
  const unsigned grid = std::min<uint32_t>(kNumSMs, (tiles + kHotWarps - 1) / kHotWarps);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kHotWarps * 32);
  cfg.dynamicSmemBytes = HOT ? (size_t)f.merge_hot * 8 : 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, merge_hot_kernel<HOT, SCATTER>, rp, col, val, x, y, trow, tnnz, sc->carry_row,
                     sc->carry_val, tiles, hot, HOT ? f.merge_hot : 0u, dest, (double*)nullptr,
                     (const double*)nullptr);
  launch_pdl(merge_fixup_kernel<SCATTER, true>, (tiles + 255) / 256, 256, s, sc->carry_row,
             (const double*)sc->carry_val, tiles, y, f.m, (const uint32_t*)nullptr, dest);
}

// A column-panelled multiply with row destinations (the fused multi-GPU exchange): y is cleared,
// the panels k >= 1 accumulate first, and panel 0 -- the one walking every row, on R-MAT the bulk
// of the entries -- runs LAST, accumulating, with each warp tile copying the rows it finished to the
// peers as it ends (rows with no entries in panel 0 are already final, and so pushed too; the carry
// fix-up pushes the rest), so the exchange overlaps the largest panel's compute instead of following
// all of it.  The panel sums are added in the order 1, ..., K-1, 0 here (0, 1, ..., K-1 without
// destinations): the two results agree within the summation tolerance, not bitwise.
template <int IPT>
void launch_merge_panels_scatter(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s,
                                 const RowDest& dest) {
  cudaMemsetAsync(y, 0, sizeof(double) * f.m, s);
  for (uint32_t k = 1; k < f.merge_panels; ++k) {
    launch_merge_panel<IPT, false, true, false>(f, x, y, sc, s, dest, k);
    if (f.panel_tile_off[k + 1] > f.panel_tile_off[k]) note_launch(2);
  }
  launch_merge_panel<IPT, true, true, true>(f, x, y, sc, s, dest, 0);
  if (f.panel_tile_off[1] > f.panel_tile_off[0]) note_launch(2);
}

template <int IPT>
void launch_merge_ipt(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s,
                      const RowDest& dest, uint32_t k) {
  const bool last = k + 1 == f.merge_panels;
  if (k == 0 && last) {
    if (dest.n) launch_merge_panel<IPT, true, false, true>(f, x, y, sc, s, dest, k);
    else launch_merge_panel<IPT, false, false, true>(f, x, y, sc, s, dest, k);
  } else if (k == 0) {
    launch_merge_panel<IPT, false, false, false>(f, x, y, sc, s, dest, k);
  } else if (!last) {
    launch_merge_panel<IPT, false, true, false>(f, x, y, sc, s, dest, k);
  } else {
    launch_merge_panel<IPT, false, true, true>(f, x, y, sc, s, dest, k);
  }
}

}  // namespace

bool merge_norms_supported(const Format& f) { return f.merge_persist && f.merge_hot && f.m == f.n; }

int spmv_merge_norms(const Format& f, const double* u, double* y, cudaStream_t s, IterScratch* sc) {
  if (!merge_norms_supported(f)) return kInvalidArgument;
  const Scratch* cs = f.stream_scratch(s);
  if (!cs) {
    g_last_error = "device allocation failed (merge carry scratch)";
    return kNoMemory;
  }
  once_per_device([] {
    cudaFuncSetAttribute(merge_hot_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kHotMaxSlots * 8);
  });
  const uint32_t tiles = f.merge_tiles;
  const unsigned grid = std::min<uint32_t>(kNumSMs, (tiles + kHotWarps - 1) / kHotWarps);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kHotWarps * 32);
  cfg.dynamicSmemBytes = (size_t)f.merge_hot * 8;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  timing_begin("merge_hot_kernel", s);
  cudaLaunchKernelEx(&cfg, merge_hot_kernel<true, false, true>, f.find("row_ptr")->as<uint32_t>(),
                     (const uint32_t*)f.find("merge_hot_col")->as<uint32_t>(), (const double*)f.find("data")->as<double>(),
                     u, y, (const uint32_t*)f.find("merge_tile_row")->as<uint32_t>(),
                     (const uint32_t*)f.find("merge_tile_nnz")->as<uint32_t>(), cs->carry_row, cs->carry_val, tiles,
                     (const uint32_t*)f.find("merge_hot_cols")->as<uint32_t>(), f.merge_hot, RowDest{}, sc->cpart,
                     (const double*)&sc->pscale);
  launch_pdl(merge_fixup_norms_kernel, (tiles + 255) / 256, 256, s, (const uint32_t*)cs->carry_row,
             (const double*)cs->carry_val, tiles, y, f.m, sc, grid);
  note_launch(2);
  timing_end(s);
  return check_launch("spmv_merge_norms");
}

int spmv_seq_crs(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.m == 0) return kOk;
  const DevArray* lra = f.find("par_long_rows");
  const uint32_t* lr = lra ? lra->as<uint32_t>() : nullptr;
  const uint32_t nl = lr ? f.par_long : 0, lim = lr ? f.par_lim : 0xFFFFFFFFu;
  timing_begin("seq_crs_kernel", s);
  seq_crs_kernel<<<(f.m + kSeqThreads - 1) / kSeqThreads + nl, kSeqThreads, 0, s>>>(
      f.find("row_ptr")->as<uint32_t>(), f.find("col_ind")->as<uint32_t>(), f.find("data")->as<double>(), x, y,
      f.m, lr, nl, lim);
  timing_end(s);
  note_launch();
  return check_launch("spmv_seq_crs");
}

int spmv_par_crs(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.m == 0) return kOk;
  const uint32_t* rp = f.find("row_ptr")->as<uint32_t>();
  const uint32_t* ci = f.find("col_ind")->as<uint32_t>();
  const double* d = f.find("data")->as<double>();
  const unsigned blocks = grid_for((uint64_t)f.m * f.par_group, 256, kNumSMs * 8) + f.par_long;
  const DevArray* lra = f.find("par_long_rows");
  const uint32_t* lr = lra ? lra->as<uint32_t>() : nullptr;
  const uint32_t nl = lr ? f.par_long : 0, lim = lr ? f.par_lim : 0xFFFFFFFFu;
  note_launch();
  timing_begin("par_crs_kernel", s);
  switch (f.par_group) {
    case 2: par_crs_kernel<2><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m, lr, nl, lim); break;
    case 4: par_crs_kernel<4><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m, lr, nl, lim); break;
    case 8: par_crs_kernel<8><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m, lr, nl, lim); break;
    case 16: par_crs_kernel<16><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m, lr, nl, lim); break;
    default: par_crs_kernel<32><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m, lr, nl, lim); break;
  }
  timing_end(s);
  return check_launch("spmv_par_crs");
}

bool merge_shape_supported(int threads, int ipt) {
  return threads == kMergeThreads && (ipt == 8 || ipt == 16 || ipt == 32);
}

// One multiply: every panel's tile kernel + carry fix-up.  The timed region (kernel timing, for the
// roofline) spans all of them, from the first tile kernel to the last fix-up.
int spmv_merge(const Format& f, const double* x, double* y, cudaStream_t s, const RowDest* dest_in) {
  if (f.merge_tiles == 0) return kOk;
  RowDest dest{};
  if (dest_in) {
    dest = *dest_in;
    if (dest.n > kMaxRowDest) {
      g_last_error = "too many row destinations";
      return kInvalidArgument;
    }
  }
  if (!merge_shape_supported((int)f.merge_threads, (int)f.merge_ipt)) {
    g_last_error = "merge tile shape not instantiated";
    return kInvalidArgument;
  }
  const Scratch* sc = f.stream_scratch(s);
  if (!sc) {
    g_last_error = "device allocation failed (merge carry scratch)";
    return kNoMemory;
  }
  if (f.merge_persist) {
    timing_begin("merge_hot_kernel", s);
    // (the same kernel without hot x -- x gathers only, more L1 for them -- measured slower than
    // merge_spmv_vec_kernel: cfg2 307 vs 292 us, cfg3 unpanelled 1059 vs 998 us)
    if (dest.n) launch_merge_persistent<true, true>(f, x, y, sc, s, dest);
    else launch_merge_persistent<true, false>(f, x, y, sc, s, dest);
    note_launch(2);
    timing_end(s);
    return check_launch("spmv_merge");
  }
  timing_begin("merge_spmv_vec_kernel", s);
  if (dest.n && f.merge_panels > 1) {
    switch (f.merge_ipt) {
      case 8: launch_merge_panels_scatter<8>(f, x, y, sc, s, dest); break;
      case 16: launch_merge_panels_scatter<16>(f, x, y, sc, s, dest); break;
      default: launch_merge_panels_scatter<32>(f, x, y, sc, s, dest); break;
    }
    timing_end(s);
    return check_launch("spmv_merge");
  }
  for (uint32_t k = 0; k < f.merge_panels; ++k) {
    switch (f.merge_ipt) {
      case 8: launch_merge_ipt<8>(f, x, y, sc, s, dest, k); break;
      case 16: launch_merge_ipt<16>(f, x, y, sc, s, dest, k); break;
      default: launch_merge_ipt<32>(f, x, y, sc, s, dest, k); break;
    }
    if (f.panel_tile_off[k + 1] > f.panel_tile_off[k]) note_launch(2);
  }
  timing_end(s);
  return check_launch("spmv_merge");
}

}  // namespace spmvcu
