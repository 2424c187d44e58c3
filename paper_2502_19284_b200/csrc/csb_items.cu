// csb_items.cu -- the reference's CSB work-item list, built on the device.
//
// Reference: spmv_csb (inc/spmv_parallel.hpp:202-264) builds, on every multiply, one item per
// block row with <= threshold nonzeros (temp_slot -1: the item owns the row), and for a heavier
// row a greedy run of cell chunks of <= threshold nonzeros plus, for every cell above the
// threshold, the quadrant leaves of split_block_range (:178-193, quadrant_boundaries
// curves.hpp:185-211); every item of a split row takes the next temp slot.  Our CSB multiply
// uses its own build-time chunk plan (blocked.cu), so this list is an on-demand product for
// callers that schedule the reference's items themselves; it is bit-identical to the
// reference's list.
//
// Device formulation (one CTA per block row, cells in tiles of 256):
//   * the greedy chunking is a serial scan of a tile's cell counts by one thread, out of shared
//     memory;
//   * quadrant leaves are data-parallel: the in-block elements are sorted by their curve rank
//     (2 bits per level, the Hilbert digits already threaded through the orientation), so the
//     quadtree node of depth d holding an element is the rank's top 2d bits and its elements are
//     contiguous.  Element i starts a leaf iff the deepest node holding both i-1 and i (depth =
//     common rank prefix) has more than `threshold` elements -- then it and all its ancestors
//     are split, and i-1, i land in different children; otherwise their common leaf is that node
//     or an ancestor.  The node's extent is two binary searches over the sorted ranks.
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {

extern thread_local std::string g_last_error;

namespace {

constexpr int kItemThreads = 256;

struct ItemCtx {
  const uint32_t* blk_ptr;
  const uint32_t* packed;
  spmvlab_cuda_csb_item* items;  // nullptr: count only
  uint32_t* row_count;           // items per block row (count pass)
  uint32_t* row_slots;           // temp slots per block row (count pass)
  const uint32_t* row_base;      // exclusive scan of row_count (emit pass)
  const uint32_t* slot_base;     // exclusive scan of row_slots (emit pass)
  uint32_t block_cols, lb;
  uint64_t threshold;
  int hilbert;
};

__device__ __forceinline__ uint64_t rank_of(uint32_t pk, unsigned lb, int hilbert, const uint16_t* henc) {
  const uint32_t r = pk >> 16, c = pk & 0xFFFFu;
  return hilbert ? hilbert_encode_t(r, c, lb, henc) : morton_encode(r, c, lb);
}

// first index in [lo, hi) whose rank is >= key
__device__ __forceinline__ uint32_t rank_lower_bound(const uint32_t* packed, uint32_t lo, uint32_t hi, uint64_t key,
                                                     unsigned lb, int hilbert, const uint16_t* henc) {
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (rank_of(packed[mid], lb, hilbert, henc) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// split_block_range (spmv_parallel.hpp:178-193) over cell elements [b, e), e - b > threshold:
// counts the leaves (returned, identical in every thread) and, when emitting, writes leaf k at
// out[k] with temp slot slot0 + k.
__device__ uint32_t cell_leaves(const ItemCtx& c, uint32_t br, uint32_t cell, uint32_t b, uint32_t e,
                                spmvlab_cuda_csb_item* out, int32_t slot0, const uint16_t* henc,
                                uint32_t* s_warp) {
  const unsigned lb = c.lb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t total = 0;
  for (uint32_t base = b; base < e; base += kItemThreads) {
    const uint32_t i = base + threadIdx.x;
    uint32_t flag = 0;
    if (i < e) {
      if (i == b) {
        flag = 1;
      } else {
        const uint64_t ki = rank_of(c.packed[i], lb, c.hilbert, henc);
        const uint64_t kp = rank_of(c.packed[i - 1], lb, c.hilbert, henc);
        // depth of the deepest common node: common prefix in 2-bit digits of the 2*lb-bit ranks
        const unsigned common = (unsigned)(__clzll((long long)(ki ^ kp)) - (64 - 2 * (int)lb)) >> 1;
        const unsigned shift = 2 * (lb - common);
        const uint64_t node_lo = (ki >> shift) << shift, node_hi = node_lo + (1ull << shift);
        const uint32_t lo = rank_lower_bound(c.packed, b, i - 1, node_lo, lb, c.hilbert, henc);
        const uint32_t hi = rank_lower_bound(c.packed, i + 1, e, node_hi, lb, c.hilbert, henc);
        flag = (uint64_t)(hi - lo) > c.threshold;
      }
    }
    // CTA-wide exclusive scan of the start flags
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, flag);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    uint32_t before = 0, tile = 0;
    for (int w = 0; w < kItemThreads / 32; ++w) {
      const uint32_t t = s_warp[w];
      before += w < warp ? t : 0;
      tile += t;
    }
    __syncthreads();
    if (flag && out) {
      const uint32_t k = total + before + __popc(bal & ((1u << lane) - 1u));
      out[k].block_row = br;
      out[k].cell_begin = cell;
      out[k].cell_end = cell + 1;
      out[k].temp_slot = slot0 + (int32_t)k;
      out[k].elem_begin = i;
      if (k) out[k - 1].elem_end = i;
    }
    total += tile;
  }
  if (out && threadIdx.x == 0) out[total - 1].elem_end = e;
  return total;
}

template <bool EMIT>
__global__ void __launch_bounds__(kItemThreads) csb_items_kernel(const ItemCtx c) {
  SPMV_HILBERT_TABLES();
  __shared__ uint32_t s_ptr[kItemThreads + 1];
  __shared__ uint32_t s_leaf[kItemThreads];   // leaves of an over-threshold cell of the tile
  __shared__ uint32_t s_first[kItemThreads];  // its first item (row-local index)
  __shared__ uint32_t s_ofl[kItemThreads];    // the tile's over-threshold cells, ascending
  __shared__ uint32_t s_nofl, s_warp[kItemThreads / 32];
  const uint32_t br = blockIdx.x;
  const uint32_t bcs = c.block_cols;
  const uint64_t row_cell = (uint64_t)br * bcs;
  const uint32_t rb = c.blk_ptr[row_cell], re = c.blk_ptr[row_cell + bcs];
  spmvlab_cuda_csb_item* row_out = EMIT ? c.items + c.row_base[br] : nullptr;
  if (re == rb || (uint64_t)(re - rb) <= c.threshold) {
    if (threadIdx.x == 0) {
      if (!EMIT) {
        c.row_count[br] = re != rb;
        c.row_slots[br] = 0;
      } else if (re != rb) {
        row_out[0] = spmvlab_cuda_csb_item{br, 0, bcs, -1, rb, re};
      }
    }
    return;
  }
  const int32_t slot0 = EMIT ? (int32_t)c.slot_base[br] : 0;
  // serial greedy state (thread 0 only), spmv_parallel.hpp:224-259
  uint32_t chunk_first = 0, nitems = 0;
  uint64_t chunk_count = 0;
  for (uint32_t t0 = 0; t0 < bcs; t0 += kItemThreads) {
    const uint32_t tn = min((uint32_t)kItemThreads, bcs - t0);
    for (uint32_t j = threadIdx.x; j <= tn; j += kItemThreads) s_ptr[j] = c.blk_ptr[row_cell + t0 + j];
    if (threadIdx.x == 0) s_nofl = 0;
    __syncthreads();
    {
      const uint32_t j = threadIdx.x;
      const bool over = j < tn && (uint64_t)(s_ptr[j + 1] - s_ptr[j]) > c.threshold;
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, over);
      if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = __popc(bal);
      __syncthreads();
      uint32_t before = 0;
      for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) before += s_warp[w];
      if (over) s_ofl[before + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = j;
      if (threadIdx.x == kItemThreads - 1) s_nofl = before + __popc(bal);
      __syncthreads();
    }
    const uint32_t nofl = s_nofl;
    for (uint32_t q = 0; q < nofl; ++q) {
      const uint32_t j = s_ofl[q];
      const uint32_t n = cell_leaves(c, br, t0 + j, s_ptr[j], s_ptr[j + 1], nullptr, 0, s_henc, s_warp);
      if (threadIdx.x == 0) s_leaf[j] = n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (uint32_t j = 0; j < tn; ++j) {
        const uint32_t cell = t0 + j;
        const uint64_t cnt = s_ptr[j + 1] - s_ptr[j];
        if (cnt > c.threshold) {
          if (chunk_count) {  // flush_chunk(c)
            if (EMIT) row_out[nitems] = spmvlab_cuda_csb_item{br, chunk_first, cell, slot0 + (int32_t)nitems,
                                                               c.blk_ptr[row_cell + chunk_first], s_ptr[j]};
            ++nitems;
            chunk_count = 0;
          }
          s_first[j] = nitems;
          nitems += s_leaf[j];
          chunk_first = cell + 1;
          continue;
        }
        if (chunk_count == 0) chunk_first = cell;
        if (chunk_count + cnt > c.threshold) {
          if (chunk_count) {
            if (EMIT) row_out[nitems] = spmvlab_cuda_csb_item{br, chunk_first, cell, slot0 + (int32_t)nitems,
                                                               c.blk_ptr[row_cell + chunk_first], s_ptr[j]};
            ++nitems;
            chunk_count = 0;
          }
          chunk_first = cell;
        }
        chunk_count += cnt;
      }
    }
    __syncthreads();
    if (EMIT) {
      for (uint32_t q = 0; q < nofl; ++q) {
        const uint32_t j = s_ofl[q];
        const uint32_t k0 = s_first[j];
        cell_leaves(c, br, t0 + j, s_ptr[j], s_ptr[j + 1], row_out + k0, slot0 + (int32_t)k0, s_henc, s_warp);
      }
    }
    __syncthreads();  // s_ptr / s_ofl are rewritten by the next tile
  }
  if (threadIdx.x == 0) {
    if (chunk_count) {  // flush_chunk(block_cols)
      if (EMIT) row_out[nitems] = spmvlab_cuda_csb_item{br, chunk_first, bcs, slot0 + (int32_t)nitems,
                                                         c.blk_ptr[row_cell + chunk_first], re};
      ++nitems;
    }
    if (!EMIT) {
      c.row_count[br] = nitems;
      c.row_slots[br] = nitems;
    }
  }
}

}  // namespace

int csb_work_items(const Format& f, uint64_t split_threshold, spmvlab_cuda_csb_item* items, uint64_t capacity,
                   uint64_t* count, cudaStream_t s) {
  const uint32_t brs = f.block_rows;
  ItemCtx c{};
  c.blk_ptr = f.find("blk_ptr")->as<uint32_t>();
  c.packed = f.find("packed")->as<uint32_t>();
  c.block_cols = f.block_cols;
  c.lb = f.log2_beta;
  c.threshold = split_threshold ? split_threshold : 2ull << f.log2_beta;
  c.hilbert = f.alg == 4;
  *count = 0;
  if (brs == 0 || f.nnz == 0) return 0;
  Arena ar(s);
  c.row_count = ar.alloc_n<uint32_t>((uint64_t)brs + 1);
  c.row_slots = ar.alloc_n<uint32_t>((uint64_t)brs + 1);
  uint32_t* row_base = ar.alloc_n<uint32_t>((uint64_t)brs + 1);
  uint32_t* slot_base = ar.alloc_n<uint32_t>((uint64_t)brs + 1);
  if (!c.row_count || !c.row_slots || !row_base || !slot_base) return kNoMemory;
  csb_items_kernel<false><<<brs, kItemThreads, 0, s>>>(c);
  exclusive_scan_u32(c.row_count, row_base, brs, ar);
  exclusive_scan_u32(c.row_slots, slot_base, brs, ar);
  note_launch(3);
  uint32_t total = 0;
  cudaMemcpyAsync(&total, row_base + brs, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (int rc = check_launch("csb_work_items")) return rc;
  *count = total;
  if (!items) return 0;
  if (capacity < total) {
    g_last_error = "item buffer holds " + std::to_string(capacity) + " items, the list has " + std::to_string(total);
    return kInvalidArgument;
  }
  c.items = items;
  c.row_base = row_base;
  c.slot_base = slot_base;
  csb_items_kernel<true><<<brs, kItemThreads, 0, s>>>(c);
  note_launch();
  cudaStreamSynchronize(s);
  return check_launch("csb_work_items");
}

}  // namespace spmvcu
