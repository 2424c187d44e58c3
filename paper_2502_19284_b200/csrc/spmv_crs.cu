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
//    sequential carry loop of spmv_parallel.hpp:157-159).  Five tile kernels:
//      - kVariantVector (default, 256 threads, 32 * {32,16,8} items per warp tile by matrix size):
//        the tile's nonzeros in lane-blocked passes of 128 -- each lane loads 4 consecutive
//        col_ind / data entries with one 128-bit and one 256-bit load, gathers and multiplies in
//        registers (two passes in flight); row ends of the pass are scattered to the element they
//        close through a 128-entry shared map, each lane walks its 4 products, one warp segmented
//        scan joins the lanes.  No product staging.  Kernel and fix-up are launched with
//        programmatic stream serialization (the next grid is resident while the previous drains;
//        griddepcontrol.wait before any memory access): 291 -> 287 us per multiply at cfg2.
//        Folding the fix-up
//        into the kernel measured slower: a look-back spin on the previous tile's carry 407 us, a
//        last-arrival counter per spanning row (fence + atomic at each tile end) 356 us -- the
//        tile-end latency holds warp slots this latency-bound kernel needs.
//      - kVariantWarpStage (256 x 7): one tile of 32*IPT items per WARP in warp-private
//        shared memory, warp synchronisation only: coalesced streaming loads of row ends /
//        col_ind / data (all IPT in flight per lane), IPT x gathers in flight, products staged,
//        lane start points by scattering row ends to their owners + shuffle suffix-minimum,
//        per-lane merge walk of IPT items (odd IPT: bank-conflict free), warp segmented scan,
//        completed rows stored straight to y.  cfg2: 330 us.
//      - kVariantSmem: the same with one CTA-wide tile per CTA (CTA barriers).  cfg2: 355 us.
//      - kVariantShuffle: one tile per warp and no shared memory: coalesced 32-element groups,
//        row-start mask by OR-reduction, shuffle segmented scan.  cfg2: 388 us (warp shuffles
//        occupy the same L1 data pipe as the x gathers).
//      - kVariantTma: persistent CTAs fed by TMA bulk copies (cp.async.bulk + mbarrier ring).
//        cfg2: 427 us (fewer resident CTAs leave the x-gather latency exposed).
//    The floor for all of them on R-MAT s22 is the x-gather rate (tools/microbench).
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

// ---------------------------------------------------------------- shuffle variant (default)

// Consumes every row end (rows rp.. < r1) with end E <= jlim, 32 per batch: the lane holding row r
// writes y[r] = (sum of the row's products in the group [j, jlim), fetched from the tail lane of
// its segment, 0 if it has none) + carry for rp0, the row in progress at the group start.
// Sets `any` if a row end was consumed and `last_end` to the end of the last one.
__device__ __forceinline__ void consume_row_ends(const uint32_t* __restrict__ row_ptr, double* __restrict__ y,
                                                 uint32_t& rp, uint32_t r1, uint32_t j, uint32_t jlim,
                                                 double s, double carry, bool& any, uint32_t& last_end,
                                                 unsigned lane) {
  const uint32_t rp0 = rp;
  uint32_t prev_last = j;  // end of the row preceding the batch (any value <= j for the first batch)
  while (rp < r1) {
    const uint32_t r = rp + lane;
    const bool have = r < r1;
    const uint32_t E = have ? __ldg(row_ptr + r + 1) : 0xFFFFFFFFu;
    const bool in = have && E <= jlim;
    const unsigned inmask = __ballot_sync(0xFFFFFFFFu, in);
    uint32_t prevE = __shfl_up_sync(0xFFFFFFFFu, E, 1);
    if (lane == 0) prevE = prev_last;
    const bool has = E > max(prevE, j);  // row r owns elements inside this group
    const int pos = (int)E - 1 - (int)j;  // its tail lane
    double v = __shfl_sync(0xFFFFFFFFu, s, (in && has) ? pos : 0);
    if (!has) v = 0.0;
    if (r == rp0) v += carry;
    if (in) y[r] = v;
    const int nin = __popc(inmask);
    if (nin) {
      last_end = __shfl_sync(0xFFFFFFFFu, E, nin - 1);
      prev_last = last_end;
      any = true;
      rp += (uint32_t)nin;
    }
    if (nin < 32) break;
  }
}

template <int U, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) merge_spmv_shfl_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const uint32_t* __restrict__ tile_row,
    const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
    double* __restrict__ carry_val, uint32_t tiles) {
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t t = blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t >= tiles) return;
  const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const uint32_t j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  uint32_t rp = r0;    // first row whose end has not been consumed by this tile
  double carry = 0.0;  // this tile's partial sum of row rp
  for (uint32_t jb = j0; jb < j1; jb += 32 * U) {
    double p[U];
    uint32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = jb + 32 * u + lane;
      const bool ok = k < j1;
      c[u] = ok ? ld_stream(col + k, pf) : 0u;
      p[u] = ok ? ld_stream(val + k, pf) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = jb + 32 * u + lane;
      if (k < j1) p[u] *= ld_x(x + c[u], pl);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = jb + 32 * u;
      if (j >= j1) break;
      const uint32_t jend = min(j + 32u, j1);  // group covers elements [j, jend)
      // row-start mask of the group: a row starting at element j + b sets bit b (bit 0 always)
      unsigned heads = 1u;
      {
        uint32_t q = rp;
        while (q < r1) {
          const uint32_t r = q + lane;
          const uint32_t E = r < r1 ? __ldg(row_ptr + r + 1) : 0xFFFFFFFFu;
          const bool in = r < r1 && E < jend;
          heads |= __reduce_or_sync(0xFFFFFFFFu, in && E >= j ? (1u << (E - j)) : 0u);
          const int nin = __popc(__ballot_sync(0xFFFFFFFFu, r < r1 && E <= jend));
          q += (uint32_t)nin;
          if (nin < 32) break;
        }
      }
      // inclusive segmented scan of the products
      double s = p[u];
      const int seg = 31 - __clz(heads & (lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u)));
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double o = __shfl_up_sync(0xFFFFFFFFu, s, off);
        if ((int)lane - off >= seg) s += o;
      }
      bool any = false;
      uint32_t last_end = 0;
      consume_row_ends(row_ptr, y, rp, r1, j, jend, s, carry, any, last_end, lane);
      const double s_last = __shfl_sync(0xFFFFFFFFu, s, (int)(jend - 1 - j));
      if (!any) carry += s_last;                       // the whole group lies inside row rp
      else carry = (last_end >= jend) ? 0.0 : s_last;  // partial of the row begun in this group
    }
  }
  // rows of this tile ending exactly at j1, and empty rows, after the last nonzero
  bool any = false;
  uint32_t last_end = 0;
  consume_row_ends(row_ptr, y, rp, r1, j1, j1, 0.0, carry, any, last_end, lane);
  if (lane == 0) {
    carry_row[t] = r1;
    carry_val[t] = any ? 0.0 : carry;  // this tile's partial of row r1
  }
}

// ---------------------------------------------------------------- shared-memory variant

// Segmented-scan operator on (has_row_end, value): (f1,v1) + (f2,v2) = (f1|f2, f2 ? v2 : v1+v2).
struct Seg {
  double v;
  int f;
};
__device__ __forceinline__ Seg seg_combine(Seg a, Seg b) { return {b.f ? b.v : a.v + b.v, a.f | b.f}; }

template <int THREADS>
struct MergeScratch {
  int first[THREADS];  // first row end consumed by each thread (or nrows)
  int wmin[THREADS / 32];
  double wv[THREADS / 32];
  int wf[THREADS / 32];
};

// Merges one staged tile.  srow[0..nrows): row ends row_ptr[r0+1..r1]; sbuf[0..nnzs): products;
// writes the y values of the tile's rows to sbuf[nnzs .. nnzs+nrows) and returns the tile's
// partial sum of row r1.  Called by all THREADS threads; ends with __syncthreads.
template <int THREADS, int IPT>
__device__ __forceinline__ double merge_tile(const uint32_t* srow, double* sbuf, int nrows, int nnzs,
                                             uint32_t j0, MergeScratch<THREADS>& sc) {
  constexpr int WARPS = THREADS / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int len = nrows + nnzs;
  // Row end ri is consumed at path diagonal ri + (row_end - j0), i.e. by thread diag / IPT; each
  // thread starts at the first row end owned by a thread >= it (suffix minimum).
  sc.first[tid] = nrows;
  __syncthreads();
  for (int ri = tid; ri < nrows; ri += THREADS) {
    const int own = (ri + (int)(srow[ri] - j0)) / IPT;
    const int prev = ri == 0 ? -1 : (ri - 1 + (int)(srow[ri - 1] - j0)) / IPT;
    if (own != prev) sc.first[own] = ri;
  }
  __syncthreads();
  int mn = sc.first[tid];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_down_sync(0xFFFFFFFFu, mn, off);
    if (lane + off < 32) mn = min(mn, o);
  }
  if (lane == 0) sc.wmin[warp] = mn;
  __syncthreads();
#pragma unroll
  for (int w = warp + 1; w < WARPS; ++w) mn = min(mn, sc.wmin[w]);

  const int diag = min(tid * IPT, len);
  int ri = mn, ji = diag - mn;
  const int dend = min(diag + IPT, len);
  double run = 0.0, first_val = 0.0;
  int first_row = -1;
  uint32_t next_end = ri < nrows ? srow[ri] : 0xFFFFFFFFu;
  for (int d = diag; d < dend; ++d) {
    if (ri < nrows && (ji >= nnzs || next_end <= j0 + (uint32_t)ji)) {
      if (first_row < 0) { first_row = ri; first_val = run; }
      else sbuf[nnzs + ri] = run;
      run = 0.0;
      ++ri;
      next_end = ri < nrows ? srow[ri] : 0xFFFFFFFFu;
    } else {
      run += sbuf[ji];
      ++ji;
    }
  }
  Seg inc{run, first_row >= 0 ? 1 : 0};
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Seg o;
    o.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, off);
    o.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, off);
    if (lane >= off) inc = seg_combine(o, inc);
  }
  if (lane == 31) { sc.wv[warp] = inc.v; sc.wf[warp] = inc.f; }
  __syncthreads();
  Seg wpre{0.0, 0}, all{0.0, 0};
#pragma unroll
  for (int w = 0; w < WARPS; ++w) {
    const Seg sw{sc.wv[w], sc.wf[w]};
    if (w < warp) wpre = seg_combine(wpre, sw);
    all = seg_combine(all, sw);
  }
  Seg excl;
  excl.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, 1);
  excl.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, 1);
  if (lane == 0) excl = Seg{0.0, 0};
  excl = seg_combine(wpre, excl);
  if (first_row >= 0) sbuf[nnzs + first_row] = first_val + excl.v;
  __syncthreads();
  return all.v;
}

template <int THREADS, int IPT>
__global__ void __launch_bounds__(THREADS, 4) merge_spmv_smem_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const uint32_t* __restrict__ tile_row,
    const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
    double* __restrict__ carry_val) {
  constexpr int TILE = THREADS * IPT;
  __shared__ uint32_t s_rowend[TILE];
  __shared__ double s_buf[TILE];  // [0, nnzs): products; [nnzs, nnzs + nrows): y of the tile's rows
  __shared__ MergeScratch<THREADS> sc;
  const int tid = threadIdx.x;
  const uint32_t t = blockIdx.x;
  const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const uint32_t j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
  const int nrows = (int)(r1 - r0), nnzs = (int)(j1 - j0);
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  {
    uint32_t rv[IPT], cv[IPT];
    double vv[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = tid + i * THREADS;
      rv[i] = k < nrows ? ld_stream(row_ptr + r0 + 1 + k, pf) : 0u;
      cv[i] = k < nnzs ? ld_stream(col + j0 + k, pf) : 0u;
      vv[i] = k < nnzs ? ld_stream(val + j0 + k, pf) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = tid + i * THREADS;
      if (k < nnzs) vv[i] *= ld_x(x + cv[i], pl);
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = tid + i * THREADS;
      if (k < nrows) s_rowend[k] = rv[i];
      if (k < nnzs) s_buf[k] = vv[i];
    }
  }
  __syncthreads();
  const double carry = merge_tile<THREADS, IPT>(s_rowend, s_buf, nrows, nnzs, j0, sc);
  if (tid == 0) {
    carry_row[t] = r1;
    carry_val[t] = carry;
  }
  for (int k = tid; k < nrows; k += THREADS) y[r0 + k] = s_buf[nnzs + k];
}

// ---------------------------------------------------------------- warp-staged variant

// One merge-path tile of 32*IPT items per warp, staged in warp-private shared memory (warp
// synchronisation only; the warps of an SM drift freely through load / gather / merge phases).
// Two shared-memory operations per nonzero (striped product store, blocked product load); each
// lane's starting path point comes from scattering row ends to their owning lanes plus a
// shuffle suffix-minimum; rows completed by a lane are stored straight to y.
// Register budget: IPT <= 7 fits 40 registers (48 warps per SM); larger tiles need ~64.
template <int IPT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, (IPT <= 7 ? 48 : 32) / WARPS) merge_spmv_wstage_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const uint32_t* __restrict__ tile_row,
    const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
    double* __restrict__ carry_val, uint32_t tiles) {
  constexpr int TILE = 32 * IPT;
  __shared__ uint32_t s_row_all[WARPS][TILE];
  __shared__ double s_buf_all[WARPS][TILE];
  __shared__ int s_first_all[WARPS][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t t = blockIdx.x * WARPS + warp;
  if (t >= tiles) return;
  uint32_t* srow = s_row_all[warp];
  double* sbuf = s_buf_all[warp];
  int* sfirst = s_first_all[warp];
  const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const uint32_t j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
  const int nrows = (int)(r1 - r0), nnzs = (int)(j1 - j0);
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  {
    uint32_t rv[IPT], cv[IPT];
    double vv[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = lane + i * 32;
      rv[i] = k < nrows ? ld_stream(row_ptr + r0 + 1 + k, pf) : 0u;
      cv[i] = k < nnzs ? ld_stream(col + j0 + k, pf) : 0u;
      vv[i] = k < nnzs ? ld_stream(val + j0 + k, pf) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = lane + i * 32;
      if (k < nnzs) vv[i] *= ld_x(x + cv[i], pl);
    }
    sfirst[lane] = nrows;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = lane + i * 32;
      if (k < nrows) srow[k] = rv[i];
      if (k < nnzs) sbuf[k] = vv[i];
    }
    __syncwarp();
    // row end k is consumed at path diagonal k + (end - j0): owner lane = diagonal / IPT
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = lane + i * 32;
      if (k < nrows) {
        const int own = (k + (int)(rv[i] - j0)) / IPT;
        const int prev = k == 0 ? -1 : (k - 1 + (int)(srow[k - 1] - j0)) / IPT;
        if (own != prev) sfirst[own] = k;
      }
    }
  }
  __syncwarp();
  int mn = sfirst[lane];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_down_sync(0xFFFFFFFFu, mn, off);
    if (lane + off < 32) mn = min(mn, o);
  }
  const int len = nrows + nnzs;
  const int diag = min(lane * IPT, len);
  int ri = mn, ji = diag - mn;
  const int dend = min(diag + IPT, len);
  double run = 0.0, first_val = 0.0;
  int first_row = -1;
  uint32_t next_end = ri < nrows ? srow[ri] : 0xFFFFFFFFu;
  for (int d = diag; d < dend; ++d) {
    if (ri < nrows && (ji >= nnzs || next_end <= j0 + (uint32_t)ji)) {
      if (first_row < 0) { first_row = ri; first_val = run; }
      else y[r0 + ri] = run;
      run = 0.0;
      ++ri;
      next_end = ri < nrows ? srow[ri] : 0xFFFFFFFFu;
    } else {
      run += sbuf[ji];
      ++ji;
    }
  }
  // Warp segmented scan of the lane tails; a lane that completed a row starts a new segment (its
  // tail follows its last row end).  Segment starts come from one ballot, so only the values are
  // shuffled: v = sum of tails from the segment start through this lane.
  const unsigned heads = __ballot_sync(0xFFFFFFFFu, first_row >= 0);
  const unsigned le = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int seg = heads & le ? 31 - __clz(heads & le) : 0;
  double v = run;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double ov = __shfl_up_sync(0xFFFFFFFFu, v, off);
    if (lane - off >= seg) v += ov;
  }
  double ex = __shfl_up_sync(0xFFFFFFFFu, v, 1);
  if (lane == 0) ex = 0.0;
  if (first_row >= 0) y[r0 + first_row] = first_val + ex;
  if (lane == 31) {
    carry_row[t] = r1;
    carry_val[t] = v;
  }
}

// ---------------------------------------------------------------- lane-blocked vector variant

// 4 consecutive nonzeros of a 128-element pass per lane, loaded with one 128-bit col_ind load and
// one 256-bit data load (sm_100 ld.global.v4.f64); the products never leave registers.  Elements
// outside [j0, j1) are masked (the tile's merge-path element range is not 4-aligned).
// x gathers of the vector kernel; -DSPMV_XG_CG makes them L2-only (.cg): 384 vs 292 us at cfg2,
// the 13 % L1 hit rate of R-MAT's hot columns is worth keeping.
__device__ __forceinline__ double ld_xg(const double* p, uint64_t pol) {
#ifdef SPMV_XG_CG
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
#elif defined(SPMV_XG_L1_EVICT_LAST)  // measured 299 vs 292 us
  double v;
  asm volatile("ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
#else
  return ld_x(p, pol);
#endif
}

__device__ __forceinline__ void vec_products(const uint32_t* __restrict__ col, const double* __restrict__ val,
                                             const double* __restrict__ x, uint32_t k, uint32_t j0, uint32_t j1,
                                             uint64_t pf, uint64_t pl, double p[4]) {
  if (k >= j0 && k + 3 < j1) {
    const uint4 c = ld_stream4(col + k, pf);
    double v0, v1, v2, v3;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "l"(val + k), "l"(pf));
    p[0] = v0 * ld_xg(x + c.x, pl);
    p[1] = v1 * ld_xg(x + c.y, pl);
    p[2] = v2 * ld_xg(x + c.z, pl);
    p[3] = v3 * ld_xg(x + c.w, pl);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t e = k + u;
      p[u] = (e >= j0 && e < j1) ? ld_stream(val + e, pf) * ld_x(x + ld_stream(col + e, pf), pl) : 0.0;
    }
  }
}

// Split form for software pipelining: the col_ind quad of a later pass is loaded early
// (vec_cols) so its x gathers issue as soon as that pass starts (vec_products_c).
__device__ __forceinline__ uint4 vec_cols(const uint32_t* __restrict__ col, uint32_t k, uint32_t j0, uint32_t j1,
                                          uint64_t pf) {
  return (k >= j0 && k + 3 < j1) ? ld_stream4(col + k, pf) : make_uint4(0u, 0u, 0u, 0u);
}
__device__ __forceinline__ void vec_products_c(const uint32_t* __restrict__ col, const double* __restrict__ val,
                                               const double* __restrict__ x, uint32_t k, uint32_t j0, uint32_t j1,
                                               uint64_t pf, uint64_t pl, uint4 c, double p[4]) {
  if (k >= j0 && k + 3 < j1) {
    double v0, v1, v2, v3;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "l"(val + k), "l"(pf));
    p[0] = v0 * ld_x(x + c.x, pl);
    p[1] = v1 * ld_x(x + c.y, pl);
    p[2] = v2 * ld_x(x + c.z, pl);
    p[3] = v3 * ld_x(x + c.w, pl);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t e = k + u;
      p[u] = (e >= j0 && e < j1) ? ld_stream(val + e, pf) * ld_x(x + ld_stream(col + e, pf), pl) : 0.0;
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
template <bool SCATTER, bool ACC>
__device__ __forceinline__ void put_row_m(double* y, const RowDest& d, uint32_t r, double v) {
  if constexpr (ACC) v += y[r];
  put_row<SCATTER>(y, d, r, v);
}

template <bool SCATTER, bool ACC>
__device__ __forceinline__ void vec_pass(const uint32_t* __restrict__ row_ptr, double* __restrict__ y, uint32_t* smap,
                                         uint32_t base, uint32_t j0, uint32_t j1, uint32_t r1, uint32_t& rp,
                                         uint32_t& prevE, const double p[4], double& carry, unsigned lane,
                                         const RowDest& dest) {
  const uint32_t pend = min(base + 128u, j1);
  const uint32_t rp0 = rp;  // map entries <= rp0 are stale (rows closed by earlier passes) or unset
  while (rp < r1) {
    const uint32_t idx = rp + lane;
    const bool have = idx < r1;
    const uint32_t E = have ? __ldg(row_ptr + idx + 1) : 0xFFFFFFFFu;
    uint32_t S = __shfl_up_sync(0xFFFFFFFFu, E, 1);
    if (lane == 0) S = prevE;
    const bool in = have && E <= pend;
    if (in) {
      if (E == S || E <= j0) {  // empty, or elements precede the tile
        if (!ACC || SCATTER) put_row_m<SCATTER, ACC>(y, dest, idx, 0.0);
      }
      else smap[E - 1 - base] = idx + 1u;   // closes at element E - 1 of this pass
    }
    const unsigned inmask = __ballot_sync(0xFFFFFFFFu, in);
    const int nin = __popc(inmask);
    if (nin) prevE = __shfl_sync(0xFFFFFFFFu, E, nin - 1);
    rp += (uint32_t)nin;
    if (nin < 32) break;
  }
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
        put_row_m<SCATTER, ACC>(y, dest, rid[u], run);
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
    put_row_m<SCATTER, ACC>(y, dest, first_row, first_val + ex + ((heads & ((1u << lane) - 1u)) ? 0.0 : carry));
  const double v31 = __shfl_sync(0xFFFFFFFFu, v, 31);
  carry = heads ? v31 : carry + v31;
  __syncwarp();
}

// Merge-path tiles of 32 * IPT items per warp (the same partition and carry fix-up as the other
// variants), the tile's elements walked in lane-blocked passes of 128 with two passes' loads and
// gathers in flight.  No product staging: shared memory holds only the 128-entry row map.
template <int IPT, int WARPS, int NP, bool SCATTER, bool ACC>
__global__ void __launch_bounds__(WARPS * 32, (NP == 1 ? 40 : 48) / WARPS) merge_spmv_vec_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
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
  uint32_t* smap = s_map_all[warp];
  *reinterpret_cast<uint4*>(smap + 4 * lane) = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const uint32_t j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
  // (a fractional evict-last share for x larger than the L2 measured within 1 % on cfg3-5)
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  uint32_t rp = r0;
  uint32_t prevE = __ldg(row_ptr + r0);
  double carry = 0.0;
  bool more = true;
  uint4 cn[NP];  // NP == 1 selects the col_ind-prefetching form: next pass's quad loaded early
  if (NP == 1) cn[0] = vec_cols(col, (j0 & ~3u) + 4 * lane, j0, j1, pf);
  for (uint32_t base = j0 & ~3u; more; base += 128u * (NP == 1 ? 2 : NP)) {
    constexpr int NPP = NP == 1 ? 2 : NP;
    double p[NPP][4];
    if constexpr (NP == 1) {
      const uint4 cb = vec_cols(col, base + 128u + 4 * lane, j0, j1, pf);
      vec_products_c(col, val, x, base + 4 * lane, j0, j1, pf, pl, cn[0], p[0]);
      cn[0] = vec_cols(col, base + 256u + 4 * lane, j0, j1, pf);
      vec_products_c(col, val, x, base + 128u + 4 * lane, j0, j1, pf, pl, cb, p[1]);
    } else {
#pragma unroll
      for (int i = 0; i < NP; ++i) vec_products(col, val, x, base + 128u * i + 4 * lane, j0, j1, pf, pl, p[i]);
    }
#pragma unroll
    for (int i = 0; i < NPP; ++i) {
      if (i > 0 && !(base + 128u * i < j1 || rp < r1)) {
        more = false;
        break;
      }
      vec_pass<SCATTER, ACC>(row_ptr, y, smap, base + 128u * i, j0, j1, r1, rp, prevE, p[i], carry, lane, dest);
    }
    if (!(base + 128u * NPP < j1 || rp < r1)) more = false;
  }
  if (lane == 0) {
    carry_row[t] = r1;
    carry_val[t] = carry;
  }
}

// ---------------------------------------------------------------- TMA variant

template <int THREADS, int IPT, int STAGES>
struct MergeTmaCfg {
  static constexpr int TILE = THREADS * IPT;
  static constexpr int CAP = TILE + 8;                 // elements per buffer (alignment slack)
  static constexpr int VAL_OFF = 0;                    // double[CAP]
  static constexpr int COL_OFF = VAL_OFF + 8 * CAP;    // uint32[CAP]
  static constexpr int ROW_OFF = COL_OFF + 4 * CAP;    // uint32[CAP]
  static constexpr int STAGE_BYTES = ((ROW_OFF + 4 * CAP) + 127) / 128 * 128;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 32 * STAGES + 128;
};

template <int THREADS, int IPT, int STAGES>
__global__ void __launch_bounds__(THREADS, 2) merge_spmv_tma_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const uint32_t* __restrict__ tile_row,
    const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
    double* __restrict__ carry_val, uint32_t tiles) {
  using Cfg = MergeTmaCfg<THREADS, IPT, STAGES>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint4* meta = reinterpret_cast<uint4*>(bars + STAGES);  // (r0, r1, j0, j1) per stage
  __shared__ MergeScratch<THREADS> sc;
  const int tid = threadIdx.x;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();

  auto issue = [&](uint32_t t, int s) {
    const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1], j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
    meta[s] = make_uint4(r0, r1, j0, j1);
    uint8_t* buf = smem + s * Cfg::STAGE_BYTES;
    const uint32_t ja = j0 & ~3u, jb = (j1 + 3u) & ~3u;
    const uint32_t ra = (r0 + 1u) & ~3u, rb = (r1 + 1u + 3u) & ~3u;
    const uint32_t nb_col = (jb - ja) * 4u, nb_val = (jb - ja) * 8u, nb_row = (rb - ra) * 4u;
    mbar_arrive_expect_tx(&bars[s], nb_col + nb_val + nb_row);
    if (nb_val) {
      bulk_g2s(buf + Cfg::VAL_OFF, val + ja, nb_val, &bars[s], pf);
      bulk_g2s(buf + Cfg::COL_OFF, col + ja, nb_col, &bars[s], pf);
    }
    if (nb_row) bulk_g2s(buf + Cfg::ROW_OFF, row_ptr + ra, nb_row, &bars[s], pf);
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) {
      const uint32_t t = blockIdx.x + s * gridDim.x;
      if (t < tiles) issue(t, s);
    }
  int it = 0;
  for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    const int s = it % STAGES;
    mbar_wait(&bars[s], (uint32_t)((it / STAGES) & 1));
    const uint4 mt = meta[s];
    const uint32_t r0 = mt.x, r1 = mt.y, j0 = mt.z, j1 = mt.w;
    const int nrows = (int)(r1 - r0), nnzs = (int)(j1 - j0);
    uint8_t* buf = smem + s * Cfg::STAGE_BYTES;
    double* sval = reinterpret_cast<double*>(buf + Cfg::VAL_OFF) + (j0 & 3u);
    const uint32_t* scol = reinterpret_cast<const uint32_t*>(buf + Cfg::COL_OFF) + (j0 & 3u);
    const uint32_t* srow = reinterpret_cast<const uint32_t*>(buf + Cfg::ROW_OFF) + ((r0 + 1u) & 3u);
    double xv[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = tid + i * THREADS;
      xv[i] = k < nnzs ? ld_x(x + scol[k], pl) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int k = tid + i * THREADS;
      if (k < nnzs) sval[k] *= xv[i];
    }
    __syncthreads();
    const double carry = merge_tile<THREADS, IPT>(srow, sval, nrows, nnzs, j0, sc);
    if (tid == 0) {
      carry_row[t] = r1;
      carry_val[t] = carry;
    }
    for (int k = tid; k < nrows; k += THREADS) y[r0 + k] = sval[nnzs + k];
    __syncthreads();  // stage s free again
    if (tid == 0) {
      const uint32_t tn = t + STAGES * gridDim.x;
      if (tn < tiles) {
        fence_proxy_async();
        issue(tn, s);
      }
    }
  }
}

// ---------------------------------------------------------------- carry fix-up

// One lane per tile, 32 tiles per warp.  Runs of equal carry rows are summed with a warp segmented
// scan; the tail lane of a run that starts and ends inside the chunk adds it to y.  A run that
// starts in the chunk and continues past it is finished by the whole warp sweeping the following
// carries 32 at a time.  Runs that started in an earlier chunk are left to that chunk's warp.
// Deterministic (fixed reduction order) and O(run / 32) dependent steps for the longest rows.
template <bool SCATTER>
__global__ void merge_fixup_kernel(const uint32_t* __restrict__ carry_row,
                                   const double* __restrict__ carry_val, uint32_t tiles,
                                   double* __restrict__ y, uint32_t m, const __grid_constant__ RowDest dest) {
  const unsigned lane = threadIdx.x & 31u;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
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
  if (tail && lane != 31 && started_here && r < m) put_row<SCATTER>(y, dest, r, y[r] + v);
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
  if (lane == 0) put_row<SCATTER>(y, dest, r31, y[r31] + total);
}

// ---------------------------------------------------------------- launchers

#define MERGE_ARGS                                                                                          \
  f.find("row_ptr")->as<uint32_t>(), f.find("col_ind")->as<uint32_t>(), f.find("data")->as<double>(), x, y, \
      f.find("merge_tile_row")->as<uint32_t>(), f.find("merge_tile_nnz")->as<uint32_t>(), sc->carry_row,    \
      sc->carry_val

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

template <int THREADS, int IPT>
void launch_merge_shfl(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s) {
  constexpr int WARPS = THREADS / 32;
  merge_spmv_shfl_kernel<IPT, WARPS><<<(f.merge_tiles + WARPS - 1) / WARPS, THREADS, 0, s>>>(MERGE_ARGS,
                                                                                             f.merge_tiles);
}

template <int THREADS, int IPT>
void launch_merge_wstage(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s) {
  constexpr int WARPS = THREADS / 32;
  merge_spmv_wstage_kernel<IPT, WARPS><<<(f.merge_tiles + WARPS - 1) / WARPS, THREADS, 0, s>>>(MERGE_ARGS,
                                                                                               f.merge_tiles);
}

// Panel k of a column-panelled format (k = 0 and one panel: the plain CRS arrays).  The fix-up of
// panel k runs before panel k + 1's kernel (stream order; PDL waits for full completion), so the
// accumulating panels read final sums.
template <int THREADS, int IPT, int NP>
void launch_merge_vec(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s,
                      const RowDest& dest, uint32_t k) {
  constexpr int WARPS = THREADS / 32;
  const uint32_t t0 = f.panel_tile_off[k], tiles = f.panel_tile_off[k + 1] - t0, o = t0 + k;
  if (tiles == 0) return;
  const unsigned grid = (tiles + WARPS - 1) / WARPS;
  const bool pan = f.merge_panels > 1;
  const uint32_t* rp = pan ? f.find("merge_panel_row_ptr")->as<uint32_t>() + (uint64_t)k * f.m
                           : f.find("row_ptr")->as<uint32_t>();
  const uint32_t* col = f.find(pan ? "merge_panel_col" : "col_ind")->as<uint32_t>();
  const double* val = f.find(pan ? "merge_panel_data" : "data")->as<double>();
  const uint32_t* trow = f.find("merge_tile_row")->as<uint32_t>() + o;
  const uint32_t* tnnz = f.find("merge_tile_nnz")->as<uint32_t>() + o;
#define MERGE_VEC_ARGS rp, col, val, x, y, trow, tnnz, sc->carry_row + t0, sc->carry_val + t0, tiles, dest
  const bool scatter = dest.n && k + 1 == f.merge_panels;
  if (k == 0) {
    if (scatter) launch_pdl(merge_spmv_vec_kernel<IPT, WARPS, NP, true, false>, grid, THREADS, s, MERGE_VEC_ARGS);
    else launch_pdl(merge_spmv_vec_kernel<IPT, WARPS, NP, false, false>, grid, THREADS, s, MERGE_VEC_ARGS);
  } else {
    if (scatter) launch_pdl(merge_spmv_vec_kernel<IPT, WARPS, NP, true, true>, grid, THREADS, s, MERGE_VEC_ARGS);
    else launch_pdl(merge_spmv_vec_kernel<IPT, WARPS, NP, false, true>, grid, THREADS, s, MERGE_VEC_ARGS);
  }
#undef MERGE_VEC_ARGS
}

template <int THREADS, int IPT>
void launch_merge_smem(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s) {
  merge_spmv_smem_kernel<THREADS, IPT><<<f.merge_tiles, THREADS, 0, s>>>(MERGE_ARGS);
}

template <int THREADS, int IPT, int STAGES>
void launch_merge_tma(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s) {
  using Cfg = MergeTmaCfg<THREADS, IPT, STAGES>;
  auto kern = merge_spmv_tma_kernel<THREADS, IPT, STAGES>;
  once_per_device([] {
    cudaFuncSetAttribute(merge_spmv_tma_kernel<THREADS, IPT, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM);
  });
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, Cfg::SMEM);
  const int grid_per_sm = occ > 0 ? occ : 1;
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t grid = std::min<uint32_t>(f.merge_tiles, (uint32_t)(sms * grid_per_sm));
  kern<<<grid, THREADS, Cfg::SMEM, s>>>(MERGE_ARGS, f.merge_tiles);
}

}  // namespace

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

// Instantiated merge tile shapes (merge_shapes.inc): (threads per CTA, items per thread, variant).
bool merge_shape_supported(int threads, int ipt, int variant) {
#define SPMV_MERGE_SHAPE(T, I, V) if (threads == T && ipt == I && variant == V) return true;
#include "merge_shapes.inc"
#undef SPMV_MERGE_SHAPE
  return false;
}

uint32_t merge_tile_items(int threads, int ipt, int variant) {
  const bool per_warp = variant == kVariantShuffle || variant == kVariantWarpStage || variant == kVariantVector ||
                        variant == kVariantVector3;
  return (uint32_t)((per_warp ? 32 : threads) * ipt);
}

static const char* merge_kernel_name(int variant) {
  switch (variant) {
    case kVariantVector:
    case kVariantVector3: return "merge_spmv_vec_kernel";
    case kVariantShuffle: return "merge_spmv_shfl_kernel";
    case kVariantWarpStage: return "merge_spmv_wstage_kernel";
    case kVariantTma: return "merge_spmv_tma_kernel";
    default: return "merge_spmv_smem_kernel";
  }
}

template <int T, int I, int V>
static void launch_merge_shape(const Format& f, const double* x, double* y, const Scratch* sc, cudaStream_t s,
                               const RowDest& dest, uint32_t k) {
  if constexpr (V == kVariantShuffle) launch_merge_shfl<T, I>(f, x, y, sc, s);
  else if constexpr (V == kVariantWarpStage) launch_merge_wstage<T, I>(f, x, y, sc, s);
  else if constexpr (V == kVariantVector) launch_merge_vec<T, I, 2>(f, x, y, sc, s, dest, k);
  else if constexpr (V == kVariantVector3) launch_merge_vec<T, I, 1>(f, x, y, sc, s, dest, k);  // col prefetch
  else if constexpr (V == kVariantSmem) launch_merge_smem<T, I>(f, x, y, sc, s);
  else launch_merge_tma<T, I, 2>(f, x, y, sc, s);
}

int spmv_merge(const Format& f, const double* x, double* y, cudaStream_t s, const RowDest* dest_in) {
  if (f.merge_tiles == 0) return kOk;
  const int threads = (int)f.merge_threads, ipt = (int)f.merge_ipt, variant = (int)f.merge_variant;
  RowDest dest{};
  if (dest_in) {
    dest = *dest_in;
    if (dest.n > kMaxRowDest) {
      g_last_error = "too many row destinations";
      return kInvalidArgument;
    }
    if (dest.n && variant != kVariantVector && variant != kVariantVector3) {
      g_last_error = "row scatter needs the vector merge kernel";
      return kInvalidArgument;
    }
  }
  const Scratch* sc = f.stream_scratch(s);
  if (!sc) {
    g_last_error = "device allocation failed (merge carry scratch)";
    return kNoMemory;
  }
  const bool vec = variant == kVariantVector || variant == kVariantVector3;
  // with column panels the timed region spans every panel's kernel and the fix-ups between them
  timing_begin(merge_kernel_name(variant), s);
  for (uint32_t k = 0; k < f.merge_panels; ++k) {
    bool launched = false;
#define SPMV_MERGE_SHAPE(T, I, V)                              \
  if (!launched && threads == T && ipt == I && variant == V) { \
    launch_merge_shape<T, I, V>(f, x, y, sc, s, dest, k);      \
    launched = true;                                           \
  }
#include "merge_shapes.inc"
#undef SPMV_MERGE_SHAPE
    if (k + 1 == f.merge_panels) timing_end(s);
    if (!launched) {
      g_last_error = "merge tile shape not instantiated";
      return kInvalidArgument;
    }
    note_launch(2);
    const uint32_t t0 = f.panel_tile_off[k], tiles = f.panel_tile_off[k + 1] - t0;
    const uint32_t* crow = sc->carry_row + t0;
    const double* cval = sc->carry_val + t0;
    const unsigned fgrid = (tiles + 255) / 256;
    if (tiles == 0) continue;
    if (dest.n && k + 1 == f.merge_panels)
      launch_pdl(merge_fixup_kernel<true>, fgrid, 256, s, crow, cval, tiles, y, f.m, dest);
    else if (vec)
      launch_pdl(merge_fixup_kernel<false>, fgrid, 256, s, crow, cval, tiles, y, f.m, dest);
    else
      merge_fixup_kernel<false><<<fgrid, 256, 0, s>>>(crow, cval, tiles, y, f.m, dest);
  }
  return check_launch("spmv_merge");
}

}  // namespace spmvcu
