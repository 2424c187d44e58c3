// blocked.cu -- the CSB / MergeB / BCOH multiplies on the device (sm_100a).
//
// Reference engines: spmv_csb (inc/spmv_parallel.hpp:202-331), spmv_bcoh (:336-350, replaying
// bcoh_for_each_block / bcoh_for_each_element, inc/bcoh.hpp:115-187) and spmv_mergeb (:355-402).
// All three walk an element stream that is grouped by sparse block, with in-block coordinates
// either packed (row << 16 | col) or ICRS-compressed (u16 column increments that overflow at beta
// into a u16 row jump).  On the GPU the block level is replaced by the absolute block table built
// with the format (the BICRS / Hilbert-pointer decode pre-pass) and the stream is cut into chunks
// of <= 256 elements that never cross a block.  One warp multiplies one chunk 32 elements at a
// time: coalesced loads of the in-block indices and values, x gathers through the read-only path,
// ICRS decoded with two warp prefix sums (in_col = S mod beta, row changes = S / beta, the row
// jumps of the new rows summed with a second scan), a warp segmented reduction over runs of equal
// rows, and one fp64 reduction into y per run (y is cleared first, as the reference engines clear
// their output rows, spmv_parallel.hpp:277-281 and :344-345).  (A lane-blocked form -- 4
// consecutive elements per lane, 128-bit index / 256-bit data loads, one ICRS scan and one
// segmented scan per 128 elements -- measured slower on R-MAT s22: BCOH 532 vs 462, BCOHC 411 vs
// 337, MergeB 423 vs 334 us: rows end almost every element there, and the per-lane fp64
// reductions of lane-strided rows coalesce worse than the 32 consecutive rows of a warp step.)
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {

extern thread_local std::string g_last_error;

namespace {

// Warp-wide in-block coordinate decoder of one chunk, 32 elements per step: packed (row << 16 |
// col) or ICRS, whose running state (column sum S, row count R, in-block row IR, next row jump
// rjn) starts from the chunk's precomputed state.
template <bool ICRS>
struct ChunkCoords {
  uint32_t S = 0, IR = 0, rjn = 0;
  int R = -1;

  __device__ __forceinline__ void start(const uint4* __restrict__ ch_state, uint64_t c) {
    if (ICRS) {
      const uint4 st = ch_state[c];
      S = st.x;
      R = (int)st.y;
      IR = st.z;
      rjn = st.w;
    }
  }

  __device__ __forceinline__ void step(const uint32_t* __restrict__ packed, const uint16_t* __restrict__ col_inc,
                                       const uint16_t* __restrict__ row_jump, uint32_t k, bool valid,
                                       unsigned lane, unsigned lb, uint64_t pf, uint32_t& ir, uint32_t& ic) {
    if (!ICRS) {
      const uint32_t pk = valid ? ld_stream(packed + k, pf) : 0u;
      ir = pk >> 16;
      ic = pk & 0xFFFFu;
    } else {
      uint32_t inc = valid ? (uint32_t)__ldg(col_inc + k) : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, off);
        if ((int)lane >= off) inc += t;
      }
      const uint32_t Sk = S + inc;
      const int r = (int)(Sk >> lb);
      ic = Sk & ((1u << lb) - 1u);
      const int r_last = __shfl_sync(0xFFFFFFFFu, r, 31);
      const int nnew = r_last - R;
      uint32_t jv = (int)lane < nnew ? (uint32_t)__ldg(row_jump + rjn + lane) : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, jv, off);
        if ((int)lane >= off) jv += t;
      }
      const int idx = r - R - 1;
      const uint32_t cum = __shfl_sync(0xFFFFFFFFu, jv, idx > 0 ? idx : 0);
      ir = idx >= 0 ? IR + cum : IR;
      S = __shfl_sync(0xFFFFFFFFu, Sk, 31);
      IR = __shfl_sync(0xFFFFFFFFu, ir, 31);
      R = r_last;
      rjn += (uint32_t)nnew;
    }
  }
};

template <bool ICRS>
__global__ void __launch_bounds__(256) blocked_spmv_kernel(
    const uint32_t* __restrict__ packed, const uint16_t* __restrict__ col_inc,
    const uint16_t* __restrict__ row_jump, const double* __restrict__ data,
    const uint32_t* __restrict__ ch_begin, const uint32_t* __restrict__ ch_blk,
    const uint4* __restrict__ ch_state, const uint2* __restrict__ blk_rc, const uint32_t* __restrict__ ord,
    uint32_t nchunks, unsigned lb, const double* __restrict__ x, double* __restrict__ y) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  for (uint64_t q = gw; q < nchunks; q += nw) {
    const uint32_t c = ord ? ord[q] : (uint32_t)q;  // column-panel schedule (x > L2) or storage order
    const uint32_t e0 = ch_begin[c], e1 = ch_begin[c + 1];
    const uint2 rc = blk_rc[ch_blk[c]];
    const uint32_t rbase = rc.x << lb, cbase = rc.y << lb;
    ChunkCoords<ICRS> cur;
    cur.start(ch_state, c);
    for (uint32_t base = e0; base < e1; base += 32) {
      const uint32_t k = base + lane;
      const bool valid = k < e1;
      uint32_t ir, ic;
      cur.step(packed, col_inc, row_jump, k, valid, lane, lb, pf, ir, ic);
      double v = valid ? ld_stream(data + k, pf) * ld_x(x + cbase + ic, pl) : 0.0;
      const uint32_t row = valid ? rbase + ir : 0xFFFFFFFFu;
      // warp segmented sum over runs of equal rows
      const uint32_t prow = __shfl_up_sync(0xFFFFFFFFu, row, 1);
      const unsigned heads = __ballot_sync(0xFFFFFFFFu, lane == 0 || prow != row);
      // (skipping the scan when every lane is its own row measured slower for the packed formats)
      const int seg_start = 31 - __clz(heads & (lt | (1u << lane)));
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double t = __shfl_up_sync(0xFFFFFFFFu, v, off);
        if ((int)lane - off >= seg_start) v += t;
      }
      const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
      if (tail && valid) atomicAdd(y + row, v);
    }
  }
}

// Block-row window kernel for the curve-ordered formats (CSB, CSBH, MergeBH, BCOHCH, BCOHCHP; the
// chunks listed by block row, through chunk_order where the storage interleaves block rows): one
// CTA per window item -- a run of chunks inside one block row -- accumulates into a beta-row y window in
// shared memory (shared fp64 adds, conflicts rare), then stores the window to y (item owns the
// whole block row) or adds its nonzero entries (block row split into several items).  Replaces
// one global fp64 reduction per element by one shared-memory add; the role of the reference's
// per-task temporary vectors (spmv_parallel.hpp:218-274, 311-330).
constexpr int kWinThreads = 1024;

__global__ void __launch_bounds__(kWinThreads) window_spmv_kernel(
    const uint32_t* __restrict__ packed, const double* __restrict__ data,
    const uint32_t* __restrict__ ch_begin, const uint32_t* __restrict__ ch_blk,
    const uint2* __restrict__ blk_rc, const uint32_t* __restrict__ item_chunk,
    const uint32_t* __restrict__ item_br, const uint32_t* __restrict__ item_whole,
    const uint32_t* __restrict__ ord, unsigned lb, uint32_t m, const double* __restrict__ x,
    double* __restrict__ y) {
  extern __shared__ double win[];
  const uint32_t item = blockIdx.x;
  const uint32_t c0 = item_chunk[item], c1 = item_chunk[item + 1];
  const uint32_t beta = 1u << lb;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t i = threadIdx.x; i < beta; i += blockDim.x) win[i] = 0.0;
  __syncthreads();
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  constexpr int U = 8;  // 8 x 32 = one full chunk in flight per warp
  for (uint32_t q = c0 + warp; q < c1; q += nwarps) {
    const uint32_t c = ord ? ord[q] : q;  // chunks in (panel, block row) order, or storage order
    const uint32_t e0 = ch_begin[c], e1 = ch_begin[c + 1];
    const uint32_t cbase = blk_rc[ch_blk[c]].y << lb;
    for (uint32_t base = e0; base < e1; base += 32 * U) {
      uint32_t pk[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = base + 32 * u + lane;
        pk[u] = k < e1 ? ld_stream(packed + k, pf) : 0u;
        v[u] = k < e1 ? ld_stream(data + k, pf) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = base + 32 * u + lane;
        if (k < e1) v[u] *= ld_x(x + cbase + (pk[u] & 0xFFFFu), pl);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = base + 32 * u + lane;
        // shared fp64 adds are CAS loops: merge runs of equal rows inside the warp first so that
        // no two lanes of one instruction hit the same word (row-sorted blocks have long runs)
        const uint32_t row = k < e1 ? pk[u] >> 16 : 0xFFFFFFFFu;
        const uint32_t prow = __shfl_up_sync(0xFFFFFFFFu, row, 1);
        const unsigned heads = __ballot_sync(0xFFFFFFFFu, lane == 0 || prow != row);
        double w = v[u];
        if (heads != 0xFFFFFFFFu) {
          const int seg_start = 31 - __clz(heads & ((2u << lane) - 1u));
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(0xFFFFFFFFu, w, off);
            if ((int)lane - off >= seg_start) w += t;
          }
        }
        const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
        if (tail && k < e1) atomicAdd(&win[row], w);
      }
    }
  }
  __syncthreads();
  const uint32_t rbase = item_br[item] << lb;
  const uint32_t rows = min(beta, m - rbase);
  const bool whole = item_whole[item] != 0;
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double w = win[i];
    if (whole) y[rbase + i] = w;
    else if (w != 0.0) atomicAdd(y + rbase + i, w);
  }
}

// Deterministic window kernel (deterministic builds, every blocked format): one CTA per window
// item; an item owning its whole block row stores its rows (the reference's exclusive rows,
// spmv_parallel.hpp:311-350), a block row split over several items gets one partial window per
// item, summed in item order by det_combine.  No atomics inside the CTA either: every warp owns the window rows of
// one hash bucket (32 buckets), and each batch of up to 128 elements per warp is exchanged through
// shared memory so that warp b receives exactly the products of bucket b's rows -- per-warp bucket
// counts (match_any ranks), a CTA scan to bucket-major offsets, a scatter of (row, product) into the
// stage -- then warp b adds its list into its rows with plain loads and stores (equal rows inside
// one 32-element step combined first, in lane order).  Every order is fixed, so y is the same bits
// every run.  The price is the exchange: cfg2 CSB 1.69 ms against 0.64 ms for the CAS window
// kernel (barrier waits and match_any; ncu r02).
constexpr int kWbWarps = 32;
constexpr int kWbPer = 128;                    // elements per warp per batch
constexpr int kWbStage = kWbWarps * kWbPer;    // 4096 staged (row, product) pairs
constexpr int kWbCntPitch = 33;                // [warp][bucket] counts, padded against bank conflicts

__host__ __device__ constexpr size_t wb_smem_bytes(unsigned lb) {
  return (sizeof(double) << lb) + kWbStage * (sizeof(double) + sizeof(uint16_t)) +
         sizeof(uint32_t) * (kWbWarps * kWbCntPitch + 2 * kWbWarps + 2);
}

__device__ __forceinline__ uint32_t wb_bucket(uint32_t r) { return (r * 0x9E3779B1u) >> 27; }

template <bool ICRS>
__global__ void __launch_bounds__(kWbWarps * 32, 1) window_det_kernel(
    const uint32_t* __restrict__ packed, const uint16_t* __restrict__ col_inc, const uint16_t* __restrict__ row_jump,
    const double* __restrict__ data, const uint32_t* __restrict__ ch_begin, const uint32_t* __restrict__ ch_blk,
    const uint4* __restrict__ ch_state, const uint2* __restrict__ blk_rc, const uint32_t* __restrict__ item_chunk,
    const uint32_t* __restrict__ item_br, const uint32_t* __restrict__ item_slot, double* __restrict__ partials,
    const uint32_t* __restrict__ ord, unsigned lb, uint32_t m, const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(16) uint8_t wb_smem[];
  const uint32_t beta = 1u << lb;
  double* win = reinterpret_cast<double*>(wb_smem);
  double* sval = win + beta;
  uint16_t* srow = reinterpret_cast<uint16_t*>(sval + kWbStage);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(srow + kWbStage);
  uint32_t* bstart = cnt + kWbWarps * kWbCntPitch;  // [32 + 1]
  uint32_t* btot = bstart + kWbWarps + 1;           // [32]
  const uint32_t item = blockIdx.x;
  const uint32_t c0 = item_chunk[item], c1 = item_chunk[item + 1];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t i = threadIdx.x; i < beta; i += blockDim.x) win[i] = 0.0;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  // this warp's chunk stream: q = c0 + warp, c0 + warp + 32, ...
  uint32_t q = c0 + warp, e = 0, e1 = 0, cbase = 0;
  ChunkCoords<ICRS> cur;
  auto open_chunk = [&]() {
    if (q < c1) {
      const uint32_t c = ord ? ord[q] : q;
      e = ch_begin[c];
      e1 = ch_begin[c + 1];
      cbase = blk_rc[ch_blk[c]].y << lb;
      cur = ChunkCoords<ICRS>();
      cur.start(ch_state, c);
    }
  };
  open_chunk();
  __syncthreads();
  bool more = true;
  while (more) {
    const bool have = q < c1;
    const uint32_t bend = have ? min(e + (uint32_t)kWbPer, e1) : e;
    uint32_t rw[4], rk[4], bk[4], cl[4];
    double pv[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t k = e + 32u * u + lane;
      ok[u] = have && k < bend;
      uint32_t ir = 0, ic = 0;
      if (__any_sync(0xFFFFFFFFu, ok[u])) cur.step(packed, col_inc, row_jump, k, ok[u], lane, lb, pf, ir, ic);
      pv[u] = ok[u] ? ld_stream(data + k, pf) : 0.0;
      rw[u] = ir;
      cl[u] = ic;
      bk[u] = wb_bucket(rw[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ok[u]) pv[u] *= ld_x(x + cbase + cl[u], pl);
    // per-warp bucket counts and ranks
    cnt[warp * kWbCntPitch + lane] = 0u;
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned act = __ballot_sync(0xFFFFFFFFu, ok[u]);
      uint32_t base = 0u, mm = 0u;
      if (ok[u]) {
        mm = __match_any_sync(act, bk[u]);
        base = cnt[warp * kWbCntPitch + bk[u]];
      }
      __syncwarp();
      if (ok[u]) {
        rk[u] = base + __popc(mm & lt);
        if ((mm & lt) == 0u) cnt[warp * kWbCntPitch + bk[u]] = base + __popc(mm);
      }
      __syncwarp();
    }
    __syncthreads();
    // bucket-major exclusive offsets: warp b scans bucket b's counts over the 32 warps
    {
      const uint32_t v = cnt[lane * kWbCntPitch + warp];
      uint32_t inc = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, off);
        if ((int)lane >= off) inc += t;
      }
      if (lane == 31) btot[warp] = inc;
      __syncthreads();
      if (warp == 0) {
        const uint32_t tv = btot[lane];
        uint32_t ti = tv;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, ti, off);
          if ((int)lane >= off) ti += t;
        }
        bstart[lane] = ti - tv;
        if (lane == 31) bstart[32] = ti;
      }
      __syncthreads();
      cnt[lane * kWbCntPitch + warp] = bstart[warp] + inc - v;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ok[u]) {
        const uint32_t pos = cnt[warp * kWbCntPitch + bk[u]] + rk[u];
        srow[pos] = (uint16_t)rw[u];
        sval[pos] = pv[u];
      }
    __syncthreads();
    // warp `warp` owns bucket `warp`: add its list into its window rows
    const uint32_t beg = bstart[warp], end = bstart[warp + 1];
    for (uint32_t j0 = beg; j0 < end; j0 += 32) {
      const uint32_t j = j0 + lane;
      const bool in = j < end;
      const uint32_t r = in ? srow[j] : 0x10000u + lane;
      double v = in ? sval[j] : 0.0;
      const unsigned mm = __match_any_sync(0xFFFFFFFFu, r);
      if (__any_sync(0xFFFFFFFFu, (mm & (mm - 1u)) != 0u)) {  // equal rows in this step: lane-order sums
        double s = 0.0;
        for (int t = 0; t < 32; ++t) {
          const double vt = __shfl_sync(0xFFFFFFFFu, v, t);
          if ((mm >> t) & 1u) s += vt;
        }
        v = s;
      }
      if (in && (mm & lt) == 0u) win[r] += v;
      __syncwarp();
    }
    // advance this warp's stream
    if (have) {
      e = bend;
      if (e >= e1) {
        q += kWbWarps;
        open_chunk();
      }
    }
    more = __syncthreads_or(q < c1) != 0;
  }
  // an item owning its whole block row stores it; a split one fills its partial slot
  const uint32_t rbase = item_br[item] << lb;
  const uint32_t rows = min(beta, m - rbase);
  const uint32_t slot = item_slot[item];
  double* dst = slot == 0xFFFFFFFFu ? y + rbase : partials + ((uint64_t)slot << lb);
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) dst[i] = win[i];
}

// y rows of the split block rows: the partial windows of their items, added in item order.
__global__ void det_combine(const double* __restrict__ partials, const uint32_t* __restrict__ split_br,
                            const uint32_t* __restrict__ split_first, uint32_t nsplit, unsigned lb, uint32_t m,
                            double* __restrict__ y) {
  const uint32_t beta = 1u << lb;
  const uint64_t total = (uint64_t)nsplit << lb;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
    const uint32_t b = (uint32_t)(g >> lb), i = (uint32_t)(g & (beta - 1));
    const uint64_t row = ((uint64_t)split_br[b] << lb) + i;
    if (row >= m) continue;
    double s = 0.0;
    for (uint32_t q = split_first[b]; q < split_first[b + 1]; ++q) s += partials[((uint64_t)q << lb) + i];
    y[row] = s;
  }
}

// csb_/mergeb_/bcoh_to_triplet (csb.hpp:103-120, mergeb.hpp:110-127, bcoh.hpp:379-392): the
// multiply's chunk walk with the coordinates stored instead of multiplied, at storage positions.
template <bool ICRS>
__global__ void __launch_bounds__(256) blocked_decode_kernel(
    const uint32_t* __restrict__ packed, const uint16_t* __restrict__ col_inc,
    const uint16_t* __restrict__ row_jump, const uint32_t* __restrict__ ch_begin,
    const uint32_t* __restrict__ ch_blk, const uint4* __restrict__ ch_state, const uint2* __restrict__ blk_rc,
    uint32_t nchunks, unsigned lb, uint32_t* __restrict__ rows, uint32_t* __restrict__ cols) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pf = policy_evict_first();
  for (uint64_t c = gw; c < nchunks; c += nw) {
    const uint32_t e0 = ch_begin[c], e1 = ch_begin[c + 1];
    const uint2 rc = blk_rc[ch_blk[c]];
    ChunkCoords<ICRS> cur;
    cur.start(ch_state, c);
    for (uint32_t base = e0; base < e1; base += 32) {
      const uint32_t k = base + lane;
      const bool valid = k < e1;
      uint32_t ir, ic;
      cur.step(packed, col_inc, row_jump, k, valid, lane, lb, pf, ir, ic);
      if (valid) {
        rows[k] = (rc.x << lb) + ir;
        cols[k] = (rc.y << lb) + ic;
      }
    }
  }
}

// crs_to_triplet (crs.hpp:94-105): one warp per row writes the row index over its range.
__global__ void __launch_bounds__(256) crs_rows_kernel(const uint32_t* __restrict__ row_ptr, uint32_t m,
                                                       uint32_t* __restrict__ rows) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = gw; i < m; i += nw)
    for (uint32_t k = row_ptr[i] + lane; k < row_ptr[i + 1]; k += 32) rows[k] = (uint32_t)i;
}

}  // namespace

int format_to_triplet(const Format& f, uint32_t* rows, uint32_t* cols, double* vals, cudaStream_t s) {
  if (f.nnz == 0) return 0;
  if (vals) cudaMemcpyAsync(vals, f.find("data")->ptr, 8 * f.nnz, cudaMemcpyDeviceToDevice, s);
  if (f.alg <= 2) {
    cudaMemcpyAsync(cols, f.find("col_ind")->ptr, 4 * f.nnz, cudaMemcpyDeviceToDevice, s);
    crs_rows_kernel<<<grid_for((uint64_t)f.m * 32, 256), 256, 0, s>>>(f.find("row_ptr")->as<uint32_t>(), f.m, rows);
    note_launch();
    return check_launch("format_to_triplet(crs)");
  }
  const DevArray* cb = f.find("chunk_begin");
  const uint32_t nchunks = (uint32_t)(cb->count() - 1);
  const unsigned blocks = grid_for((uint64_t)nchunks * 32, 256);
  const DevArray* pk = f.find("packed");
  note_launch();
  if (f.alg == kBcoh)  // ICRS in-block stream; every BCOH variant lists both col_inc and packed
    blocked_decode_kernel<true><<<blocks, 256, 0, s>>>(
        nullptr, f.find("col_inc")->as<uint16_t>(), f.find("row_jump")->as<uint16_t>(), cb->as<uint32_t>(),
        f.find("chunk_blk")->as<uint32_t>(), f.find("chunk_state")->as<uint4>(), f.find("blk_rc")->as<uint2>(),
        nchunks, f.log2_beta, rows, cols);
  else
    blocked_decode_kernel<false><<<blocks, 256, 0, s>>>(
        pk->as<uint32_t>(), nullptr, nullptr, cb->as<uint32_t>(), f.find("chunk_blk")->as<uint32_t>(), nullptr,
        f.find("blk_rc")->as<uint2>(), nchunks, f.log2_beta, rows, cols);
  return check_launch("format_to_triplet(blocked)");
}

int spmv_blocked(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.m) cudaMemsetAsync(y, 0, sizeof(double) * f.m, s);
  if (f.work_items == 0) return check_launch("spmv_blocked");
  const bool icrs = f.alg == kBcoh;
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (const DevArray* items = f.find("win_item_chunk")) {
    const uint32_t nitems = (uint32_t)(items->count() - 1);
    const uint32_t* ord = f.find("chunk_order") ? f.find("chunk_order")->as<uint32_t>() : nullptr;
    note_launch();
    if (f.deterministic) {
      const size_t smem = wb_smem_bytes(f.log2_beta);
      once_per_device([] {
        cudaFuncSetAttribute(window_det_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(window_det_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      });
      const DevArray* pk = f.find("packed");
      const uint32_t* slot = f.find("det_item_slot")->as<uint32_t>();
      double* part = f.find("det_partials")->as<double>();
      const uint32_t nsplit = (uint32_t)f.find("det_split_br")->count();
      timing_begin("window_det_kernel", s);
      if (icrs)
        window_det_kernel<true><<<nitems, kWbWarps * 32, smem, s>>>(
            nullptr, f.find("col_inc")->as<uint16_t>(), f.find("row_jump")->as<uint16_t>(), f.find("data")->as<double>(),
            f.find("chunk_begin")->as<uint32_t>(), f.find("chunk_blk")->as<uint32_t>(),
            f.find("chunk_state")->as<uint4>(), f.find("blk_rc")->as<uint2>(), items->as<uint32_t>(),
            f.find("win_item_br")->as<uint32_t>(), slot, part, ord, f.log2_beta, f.m, x, y);
      else
        window_det_kernel<false><<<nitems, kWbWarps * 32, smem, s>>>(
            pk->as<uint32_t>(), nullptr, nullptr, f.find("data")->as<double>(), f.find("chunk_begin")->as<uint32_t>(),
            f.find("chunk_blk")->as<uint32_t>(), nullptr, f.find("blk_rc")->as<uint2>(), items->as<uint32_t>(),
            f.find("win_item_br")->as<uint32_t>(), slot, part, ord, f.log2_beta, f.m, x, y);
      if (nsplit) {
        det_combine<<<grid_for((uint64_t)nsplit << f.log2_beta, 256), 256, 0, s>>>(
            part, f.find("det_split_br")->as<uint32_t>(), f.find("det_split_first")->as<uint32_t>(), nsplit,
            f.log2_beta, f.m, y);
        note_launch();
      }
      timing_end(s);
      return check_launch("spmv_blocked(deterministic window)");
    }
    const size_t smem = sizeof(double) << f.log2_beta;
    once_per_device(
        [] { cudaFuncSetAttribute(window_spmv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); });
    timing_begin("window_spmv_kernel", s);
    window_spmv_kernel<<<nitems, kWinThreads, smem, s>>>(
        f.find("packed")->as<uint32_t>(), f.find("data")->as<double>(), f.find("chunk_begin")->as<uint32_t>(),
        f.find("chunk_blk")->as<uint32_t>(), f.find("blk_rc")->as<uint2>(), items->as<uint32_t>(),
        f.find("win_item_br")->as<uint32_t>(), f.find("win_item_whole")->as<uint32_t>(), ord, f.log2_beta, f.m, x, y);
    timing_end(s);
    return check_launch("spmv_blocked(window)");
  }
  const uint64_t warps_needed = f.work_items;
  const unsigned blocks = (unsigned)std::min<uint64_t>((warps_needed + 7) / 8, (uint64_t)sms * 8);
  const DevArray* pk = f.find("packed");
  const DevArray* ci = f.find("col_inc");
  const DevArray* rj = f.find("row_jump");
  const DevArray* cs = f.find("chunk_state");
  const DevArray* co = f.find("chunk_order");
  const uint32_t* ord = co ? co->as<uint32_t>() : nullptr;
  note_launch();
  timing_begin(icrs ? "blocked_spmv_kernel<icrs>" : "blocked_spmv_kernel<packed>", s);
  if (icrs)
    blocked_spmv_kernel<true><<<blocks, 256, 0, s>>>(
        nullptr, ci->as<uint16_t>(), rj->as<uint16_t>(), f.find("data")->as<double>(),
        f.find("chunk_begin")->as<uint32_t>(), f.find("chunk_blk")->as<uint32_t>(), cs->as<uint4>(),
        f.find("blk_rc")->as<uint2>(), ord, f.work_items, f.log2_beta, x, y);
  else
    blocked_spmv_kernel<false><<<blocks, 256, 0, s>>>(
        pk->as<uint32_t>(), nullptr, nullptr, f.find("data")->as<double>(), f.find("chunk_begin")->as<uint32_t>(),
        f.find("chunk_blk")->as<uint32_t>(), nullptr, f.find("blk_rc")->as<uint2>(), ord, f.work_items, f.log2_beta,
        x, y);
  timing_end(s);
  return check_launch("spmv_blocked");
}

}  // namespace spmvcu
