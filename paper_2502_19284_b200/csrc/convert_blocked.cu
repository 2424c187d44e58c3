// convert_blocked.cu -- COO -> CSB / CSBH, MergeB / MergeBH and the BCOH family on the device.
//
// Reference conversions (two-step "sort then populate"):
//   build_csb    inc/csb.hpp:51-100     sort (br, bc, Morton|Hilbert rank in block); blk_ptr over
//                                       the dense cell grid; packed = in_row << 16 | in_col
//   build_mergeb inc/mergeb.hpp:50-108  sort (br, bc, in_row, in_col) | (br, bc, Hilbert rank);
//                                       block runs become a CRS over nonempty blocks
//   build_bcoh   inc/bcoh.hpp:194-376   bands = partition_rows_by_nnz; sort (band, Hilbert(block),
//                                       in_row, in_col) | (band, Hilbert(element)); per-band ICRS or
//                                       packed in-block data, BICRS block jumps or a Hilbert
//                                       pointer array over the band's cells
// B200 design: every ordering is ONE unique 64-bit key per entry (so the radix-sorted order is
// the reference's comparator order), the value rides through the sort as payload, and every
// sequential "populate" loop becomes flag + prefix-sum + scatter passes over the sorted keys.
// The same passes also emit the multiply's plan: an absolute (block row, block col, first
// element) table per nonempty block (the decode pre-pass of the BICRS / Hilbert-pointer block
// level) and a chunk table of <= kChunk elements per chunk, never crossing a block.
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {

extern thread_local std::string g_last_error;
int partition_rows_by_nnz_host(const uint32_t* prefix, uint32_t m, unsigned p, unsigned lb, uint32_t* bounds);

namespace {

enum Kind : int { kCsbZ = 0, kCsbH, kMbRow, kMbH, kBcohRow, kBcohH };

struct Geom {
  int kind;
  unsigned lb;
  uint32_t mask;
  int bcbits;            // CSB / MergeB block-column field width
  unsigned block_level;  // BCOH
  unsigned element_level;
  uint32_t m, n, block_cols;
  unsigned p;            // BCOH bands
};

__device__ __forceinline__ bool is_bcoh_kind(int k) { return k >= kBcohRow; }

__device__ __forceinline__ uint64_t make_key(const Geom& g, uint32_t r, uint32_t c, uint32_t band,
                                             const uint16_t* henc) {
  const uint32_t br = r >> g.lb, bc = c >> g.lb, ir = r & g.mask, ic = c & g.mask;
  const unsigned lb2 = 2 * g.lb;
  switch (g.kind) {
    case kCsbZ:
      return ((uint64_t)br << (g.bcbits + lb2)) | ((uint64_t)bc << lb2) | morton_encode(ir, ic, g.lb);
    case kCsbH:
    case kMbH:
      return ((uint64_t)br << (g.bcbits + lb2)) | ((uint64_t)bc << lb2) | hilbert_encode_t(ir, ic, g.lb, henc);
    case kMbRow:
      return ((uint64_t)br << (g.bcbits + lb2)) | ((uint64_t)bc << lb2) | ((uint64_t)ir << g.lb) | ic;
    case kBcohRow:
      return ((uint64_t)band << (2 * g.element_level)) |
             (hilbert_encode_t(br, bc, g.block_level, henc) << lb2) | ((uint64_t)ir << g.lb) | ic;
    default:  // kBcohH
      return ((uint64_t)band << (2 * g.element_level)) | hilbert_encode_t(r, c, g.element_level, henc);
  }
}

struct Coords {
  uint32_t br, bc, ir, ic, band;
};

__device__ __forceinline__ Coords decode_key(const Geom& g, uint64_t key, const uint16_t* hdec) {
  Coords o;
  const unsigned lb2 = 2 * g.lb;
  o.band = 0;
  if (!is_bcoh_kind(g.kind)) {
    o.br = (uint32_t)(key >> (g.bcbits + lb2));
    o.bc = (uint32_t)((key >> lb2) & ((1ull << g.bcbits) - 1ull));
    const uint64_t rank = key & ((1ull << lb2) - 1ull);
    if (g.kind == kCsbZ) {
      o.ir = compact_bits(rank >> 1);
      o.ic = compact_bits(rank);
    } else if (g.kind == kMbRow) {
      o.ir = (uint32_t)(rank >> g.lb);
      o.ic = (uint32_t)(rank & g.mask);
    } else {
      hilbert_decode_t(rank, g.lb, o.ir, o.ic, hdec);
    }
  } else {
    const unsigned el2 = 2 * g.element_level;
    o.band = (uint32_t)(el2 >= 64 ? 0 : (key >> el2));
    const uint64_t low = el2 >= 64 ? key : (key & ((1ull << el2) - 1ull));
    if (g.kind == kBcohRow) {
      hilbert_decode_t(low >> lb2, g.block_level, o.br, o.bc, hdec);
      o.ir = (uint32_t)((low >> g.lb) & g.mask);
      o.ic = (uint32_t)(low & g.mask);
    } else {
      uint32_t r, c;
      hilbert_decode_t(low, g.element_level, r, c, hdec);
      o.br = r >> g.lb;
      o.bc = c >> g.lb;
      o.ir = r & g.mask;
      o.ic = c & g.mask;
    }
  }
  return o;
}

__device__ __forceinline__ uint32_t band_of(const uint32_t* bounds, unsigned p, uint32_t row) {
  unsigned lo = 0, hi = p + 1;  // upper_bound(bounds, row) - 1 (inc/bcoh.hpp:224-227)
  while (lo < hi) {
    const unsigned mid = (lo + hi) >> 1;
    if (bounds[mid] <= row) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

__global__ void blk_keys(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cols,
                         const double* __restrict__ vals, uint64_t nnz, Geom g,
                         const uint32_t* __restrict__ bounds, uint64_t* __restrict__ keys,
                         uint64_t* __restrict__ payload, uint32_t* err) {
  SPMV_HILBERT_TABLES();
  extern __shared__ uint32_t s_bounds[];
  const bool bcoh = is_bcoh_kind(g.kind);
  if (bcoh)
    for (unsigned i = threadIdx.x; i <= g.p; i += blockDim.x) s_bounds[i] = bounds[i];
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint32_t r = rows[k], c = cols[k];
    if (r >= g.m || c >= g.n) {
      atomicOr(err, 1u);
      keys[k] = 0;
      payload[k] = 0;
      continue;
    }
    keys[k] = make_key(g, r, c, bcoh ? band_of(s_bounds, g.p, r) : 0u, s_henc);
    payload[k] = (uint64_t)__double_as_longlong(vals[k]);
  }
}

// Sorted keys -> in-block data, block-start flags, ICRS row-change flags and increments, cell
// histogram, duplicate detection.
__global__ void blk_populate(const uint64_t* __restrict__ skeys, const uint64_t* __restrict__ svals,
                             uint64_t nnz, Geom g, uint32_t* __restrict__ packed,
                             double* __restrict__ data, uint16_t* __restrict__ col_inc,
                             uint32_t* __restrict__ blk_flag, uint32_t* __restrict__ rj_flag,
                             uint32_t* __restrict__ cell_counts, uint32_t* err) {
  SPMV_HILBERT_TABLES();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t beta = 1u << g.lb;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint64_t key = skeys[k];
    const Coords c = decode_key(g, key, s_hdec);
    const bool first = k == 0;
    const uint64_t pkey = first ? 0 : skeys[k - 1];
    if (!first && pkey == key) atomicOr(err, 2u);
    const bool new_block = first || (pkey >> (2 * g.lb)) != (key >> (2 * g.lb));
    blk_flag[k] = new_block ? 1u : 0u;
    if (packed) packed[k] = (c.ir << 16) | c.ic;
    data[k] = __longlong_as_double((long long)svals[k]);
    if (col_inc) {
      uint32_t inc, rjf;
      if (new_block) {
        inc = c.ic;
        rjf = 1;
      } else {
        const Coords pc = decode_key(g, pkey, s_hdec);
        if (c.ir == pc.ir) {
          inc = c.ic - pc.ic;
          rjf = 0;
        } else {
          inc = c.ic - pc.ic + beta;
          rjf = 1;
        }
      }
      col_inc[k] = (uint16_t)inc;
      rj_flag[k] = rjf;
    }
    if (cell_counts) {
      const uint32_t cell = c.br * g.block_cols + c.bc;
      const unsigned active = __activemask();
      const unsigned peers = __match_any_sync(active, cell);
      if (lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&cell_counts[cell], (unsigned)__popc(peers));
    }
  }
}

// Block table (and ICRS row jumps) from the flags and their exclusive scans.
__global__ void blk_table(const uint64_t* __restrict__ skeys, uint64_t nnz, Geom g,
                          const uint32_t* __restrict__ blk_flag, const uint32_t* __restrict__ blk_scan,
                          const uint32_t* __restrict__ rj_flag, const uint32_t* __restrict__ rj_scan,
                          uint32_t* __restrict__ blk_begin, uint2* __restrict__ blk_rc,
                          uint32_t* __restrict__ blk_band, uint32_t* __restrict__ blk_rj,
                          uint16_t* __restrict__ row_jump) {
  SPMV_HILBERT_TABLES();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const bool nb = blk_flag[k] != 0;
    const bool rj = rj_flag && rj_flag[k] != 0;
    if (!nb && !rj) continue;
    const Coords c = decode_key(g, skeys[k], s_hdec);
    if (nb) {
      const uint32_t b = blk_scan[k];
      blk_begin[b] = (uint32_t)k;
      blk_rc[b] = make_uint2(c.br, c.bc);
      if (blk_band) blk_band[b] = c.band;
      if (blk_rj) blk_rj[b] = rj_scan[k];
    }
    if (rj) {
      uint32_t v = c.ir;
      if (!nb) v = c.ir - decode_key(g, skeys[k - 1], s_hdec).ir;
      row_jump[rj_scan[k]] = (uint16_t)v;
    }
  }
}

__global__ void mergeb_arrays(const uint2* __restrict__ blk_rc, uint32_t nblk, uint32_t* __restrict__ blk_col_ind,
                              uint32_t* __restrict__ row_counts) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const uint2 rc = blk_rc[b];
  blk_col_ind[b] = rc.y;
  atomicAdd(&row_counts[rc.x], 1u);
}

// BICRS block level (inc/bcoh.hpp:329-350): block_nnz, col_jump_block, row-jump flags.
__global__ void bicrs_blocks(const uint32_t* __restrict__ blk_begin, const uint2* __restrict__ blk_rc,
                             const uint32_t* __restrict__ blk_band, uint32_t nblk, uint32_t block_cols,
                             uint32_t* __restrict__ block_nnz, int16_t* __restrict__ col_jump_block,
                             uint32_t* __restrict__ rjb_flag) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  block_nnz[b] = blk_begin[b + 1] - blk_begin[b];
  const uint2 rc = blk_rc[b];
  const bool first = b == 0 || blk_band[b - 1] != blk_band[b];
  int16_t cj;
  uint32_t f;
  if (first) {
    cj = (int16_t)rc.y;
    f = 1;
  } else {
    const uint2 pr = blk_rc[b - 1];
    if (rc.x == pr.x) {
      cj = (int16_t)(uint16_t)((int64_t)rc.y - (int64_t)pr.y);
      f = 0;
    } else {
      cj = (int16_t)(uint16_t)((int64_t)rc.y - (int64_t)pr.y + block_cols);
      f = 1;
    }
  }
  col_jump_block[b] = cj;
  rjb_flag[b] = f;
}

__global__ void bicrs_row_jumps(const uint2* __restrict__ blk_rc, const uint32_t* __restrict__ blk_band,
                                uint32_t nblk, const uint32_t* __restrict__ rjb_flag,
                                const uint32_t* __restrict__ rjb_scan, const uint32_t* __restrict__ band_fbr,
                                int16_t* __restrict__ row_jump_block) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk || !rjb_flag[b]) return;
  const bool first = b == 0 || blk_band[b - 1] != blk_band[b];
  const uint32_t br = blk_rc[b].x;
  const int64_t v = first ? (int64_t)br - (int64_t)band_fbr[blk_band[b]] : (int64_t)br - (int64_t)blk_rc[b - 1].x;
  row_jump_block[rjb_scan[b]] = (int16_t)(uint16_t)v;
}

// Hilbert-pointer block level (inc/bcoh.hpp:351-366): the cells of every band rectangle keyed by
// (band, Hilbert(br, bc) at block_level), i.e. the order of hilbert_rect_walk.
__global__ void hptr_cell_keys(uint64_t total_cells, unsigned p, const uint64_t* __restrict__ cell_off,
                               const uint32_t* __restrict__ band_fbr, uint32_t block_cols,
                               unsigned block_level, uint64_t* __restrict__ keys,
                               uint32_t* __restrict__ cell_id) {
  SPMV_HILBERT_TABLES();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t gidx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gidx < total_cells; gidx += stride) {
    unsigned lo = 0, hi = p;  // band = last b with cell_off[b] <= gidx
    while (lo < hi) {
      const unsigned mid = (lo + hi + 1) >> 1;
      if (cell_off[mid] <= gidx) lo = mid; else hi = mid - 1;
    }
    const uint64_t local = gidx - cell_off[lo];
    const uint32_t br = band_fbr[lo] + (uint32_t)(local / block_cols);
    const uint32_t bc = (uint32_t)(local % block_cols);
    keys[gidx] = ((uint64_t)lo << (2 * block_level)) | hilbert_encode_t(br, bc, block_level, s_henc);
    cell_id[gidx] = br * block_cols + bc;
  }
}

__global__ void hptr_counts(const uint32_t* __restrict__ sorted_cell, uint64_t total_cells,
                            const uint32_t* __restrict__ cell_counts, uint32_t* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total_cells; c += stride)
    counts[c] = cell_counts[sorted_cell[c]];
}

__global__ void hptr_fill(const uint32_t* __restrict__ excl, uint64_t total_cells, unsigned p,
                          const uint64_t* __restrict__ cell_off, uint32_t* __restrict__ blk_ptr) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total_cells + p; c += stride) {
    if (c < p) {
      blk_ptr[cell_off[c] + c] = 0;  // leading zero of band c
      continue;
    }
    const uint64_t gidx = c - p;
    unsigned lo = 0, hi = p;
    while (lo < hi) {
      const unsigned mid = (lo + hi + 1) >> 1;
      if (cell_off[mid] <= gidx) lo = mid; else hi = mid - 1;
    }
    blk_ptr[gidx + lo + 1] = excl[gidx + 1] - excl[cell_off[lo]];
  }
}

// Per-band offsets into the element, block and row-jump streams (lower bounds over sorted data).
__global__ void band_offsets(const uint64_t* __restrict__ skeys, uint64_t nnz, unsigned el2, unsigned p,
                             const uint32_t* __restrict__ blk_band, uint32_t nblk,
                             const uint32_t* __restrict__ rj_scan, const uint32_t* __restrict__ rjb_scan,
                             uint64_t* __restrict__ off_elem, uint64_t* __restrict__ off_block,
                             uint64_t* __restrict__ off_rj, uint64_t* __restrict__ off_rjb) {
  const unsigned b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > p) return;
  uint64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((skeys[mid] >> el2) < b) lo = mid + 1; else hi = mid;
  }
  off_elem[b] = lo;
  off_rj[b] = rj_scan ? rj_scan[lo] : 0;
  uint64_t blo = 0, bhi = nblk;
  while (blo < bhi) {
    const uint64_t mid = (blo + bhi) >> 1;
    if (blk_band[mid] < b) blo = mid + 1; else bhi = mid;
  }
  off_block[b] = blo;
  off_rjb[b] = rjb_scan ? rjb_scan[blo] : 0;
}

// partition_rows_by_nnz only needs its greedy row rounded to the nearest block-row boundary,
// cut = (r* + beta/2) >> lb: i.e. which "rounding cell" [c*beta - beta/2, (c+1)*beta - beta/2)
// holds r*.  Deciding that needs prefix[] only at the rows just before each cell end, so two
// counters per cell suffice -- the cell total and the count of its last row -- accumulated in
// shared memory (a few thousand cells) instead of one global atomic per entry into m counters.
constexpr uint32_t kMaxRoundCells = 6144;

__global__ void round_cell_hist(const uint32_t* __restrict__ rows, uint64_t nnz, uint32_t m, unsigned lb,
                                uint32_t cells, uint32_t* __restrict__ total, uint32_t* __restrict__ last) {
  __shared__ uint32_t s_tot[kMaxRoundCells], s_last[kMaxRoundCells];
  for (uint32_t i = threadIdx.x; i < cells; i += blockDim.x) s_tot[i] = s_last[i] = 0;
  __syncthreads();
  const uint32_t half = 1u << (lb - 1), bmask = (1u << lb) - 1u;
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = 0; base < nnz; base += stride) {
    const uint64_t k = base + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = k < nnz;
    const uint32_t r = valid ? rows[k] : 0u;
    const bool ok = valid && r < m;
    const uint32_t c = (uint32_t)(((uint64_t)r + half) >> lb);
    const uint32_t c0 = __shfl_sync(0xFFFFFFFFu, c, 0);
    if (__all_sync(0xFFFFFFFFu, ok && c == c0)) {
      if (lane == 0) atomicAdd(&s_tot[c0], 32u);
    } else if (ok) {
      atomicAdd(&s_tot[c], 1u);
    }
    if (ok && ((r + half + 1u) & bmask) == 0u) atomicAdd(&s_last[c], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < cells; i += blockDim.x) {
    if (s_tot[i]) atomicAdd(&total[i], s_tot[i]);
    if (s_last[i]) atomicAdd(&last[i], s_last[i]);
  }
}

__global__ void greedy_rows(const uint32_t* __restrict__ prefix, uint32_t m, unsigned p, uint32_t* out) {
  const unsigned k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (k >= p) return;
  const uint64_t target = (uint64_t)prefix[m] * k;
  uint64_t lo = 0, hi = (uint64_t)m + 1;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((uint64_t)prefix[mid] * p < target) lo = mid + 1; else hi = mid;
  }
  out[k - 1] = (uint32_t)lo;
}

__global__ void row_hist(const uint32_t* __restrict__ rows, uint64_t nnz, uint32_t m, uint32_t* counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint32_t r = rows[k];
    if (r < m) atomicAdd(&counts[r], 1u);
  }
}

// Chunk plan: <= chunk elements per chunk, never crossing a block.  For ICRS the chunk also
// records the decoder state before its first element: S (running col_inc sum within the block),
// R (row changes so far, -1 at a block start) and IR (current in-block row).
__global__ void chunk_count(const uint32_t* __restrict__ blk_begin, uint32_t nblk, uint32_t chunk,
                            uint32_t* __restrict__ nch) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  nch[b] = (blk_begin[b + 1] - blk_begin[b] + chunk - 1) / chunk;
}

__global__ void chunk_fill(const uint32_t* __restrict__ blk_begin, uint32_t nblk, uint32_t chunk,
                           const uint32_t* __restrict__ ch_off, const uint64_t* __restrict__ skeys, Geom g,
                           const uint32_t* __restrict__ rj_flag, const uint32_t* __restrict__ rj_scan,
                           const uint32_t* __restrict__ blk_rj, uint32_t* __restrict__ ch_begin,
                           uint32_t* __restrict__ ch_blk, uint4* __restrict__ ch_state) {
  SPMV_HILBERT_TABLES();
  // one thread per chunk (a block of 580k elements has 2k+ chunks): its block by binary search
  // over the blocks' chunk offsets
  const uint32_t nchunks = ch_off[nblk];
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  uint32_t lo = 0, hi = nblk - 1;  // last b with ch_off[b] <= c
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (ch_off[mid] <= c) lo = mid; else hi = mid - 1;
  }
  const uint32_t b = lo;
  const uint32_t e0 = blk_begin[b];
  {
    const uint32_t e = e0 + (c - ch_off[b]) * chunk;
    ch_begin[c] = e;
    ch_blk[c] = b;
    if (ch_state) {
      if (e == e0) {
        ch_state[c] = make_uint4(0u, 0xFFFFFFFFu, 0u, blk_rj[b]);
      } else {
        const Coords pc = decode_key(g, skeys[e - 1], s_hdec);
        const uint32_t rjpos = rj_scan[e - 1] + rj_flag[e - 1] - 1;
        const uint32_t R = rjpos - blk_rj[b];
        ch_state[c] = make_uint4(pc.ic + (R << g.lb), R, pc.ir, rjpos + 1);
      }
    }
  }
}

__device__ __forceinline__ uint32_t win_br(const uint32_t* ord, const uint32_t* ch_blk, const uint2* blk_rc,
                                           uint32_t q) {
  return blk_rc[ch_blk[ord ? ord[q] : q]].x;
}
__device__ __forceinline__ uint32_t win_panel(const uint32_t* ord, const uint32_t* ch_blk, const uint2* blk_rc,
                                              uint32_t q, unsigned lb, uint32_t panels, uint32_t width) {
  if (panels <= 1) return 0u;
  return min(panels - 1, (uint32_t)(((uint64_t)blk_rc[ch_blk[ord ? ord[q] : q]].y << lb) / width));
}

// Window-item plan over the chunk sequence q -> chunk ord[q] (identity when ord is null): items
// start at every (panel, block row) change and every per_item-th position, so an item never
// crosses a block row or a panel.  head bit 1: an item starts; bit 2: a block row starts.
__global__ void win_heads(const uint32_t* __restrict__ ord, const uint32_t* __restrict__ ch_blk,
                          const uint2* __restrict__ blk_rc, uint32_t nchunks, uint32_t per_item, unsigned lb,
                          uint32_t panels, uint32_t width, uint32_t* __restrict__ head) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nchunks) return;
  const bool row_start = q == 0 || win_br(ord, ch_blk, blk_rc, q) != win_br(ord, ch_blk, blk_rc, q - 1) ||
                         win_panel(ord, ch_blk, blk_rc, q, lb, panels, width) !=
                             win_panel(ord, ch_blk, blk_rc, q - 1, lb, panels, width);
  head[q] = row_start ? 3u : (q % per_item == 0 ? 1u : 0u);
}

__global__ void win_flag(const uint32_t* __restrict__ head, uint32_t nchunks, uint32_t* __restrict__ flag) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nchunks) flag[c] = head[c] != 0u;
}

// item_whole: the item covers its block row entirely (one panel, one item) -> stores its window.
__global__ void win_fill(const uint32_t* __restrict__ head, const uint32_t* __restrict__ scan,
                         const uint32_t* __restrict__ ord, const uint32_t* __restrict__ ch_blk,
                         const uint2* __restrict__ blk_rc, uint32_t nchunks, uint32_t panels,
                         uint32_t* __restrict__ item_chunk, uint32_t* __restrict__ item_br,
                         uint32_t* __restrict__ item_whole) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nchunks || !head[q]) return;
  const uint32_t i = scan[q];
  uint32_t e = q + 1;
  while (e < nchunks && !head[e]) ++e;
  item_chunk[i] = q;
  item_br[i] = win_br(ord, ch_blk, blk_rc, q);
  item_whole[i] = panels <= 1 && (head[q] & 2u) && (e == nchunks || (head[e] & 2u)) ? 1u : 0u;
}

// Schedule key of a chunk: (column panel of its block, block row); panel = first column / width.
__global__ void sched_keys(const uint32_t* __restrict__ ch_blk, const uint2* __restrict__ blk_rc,
                           uint32_t nchunks, unsigned lb, uint32_t panels, uint32_t width, int brbits,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const uint2 rc = blk_rc[ch_blk[c]];
  const uint32_t panel = panels > 1 ? min(panels - 1, (uint32_t)(((uint64_t)rc.y << lb) / width)) : 0u;
  keys[c] = ((uint64_t)panel << brbits) | rc.x;
  vals[c] = c;
}

int d2h_u32(const uint32_t* dev, uint32_t* host, cudaStream_t s) {
  cudaMemcpyAsync(host, dev, 4, cudaMemcpyDeviceToHost, s);
  return cudaStreamSynchronize(s) == cudaSuccess ? kOk : check_launch("d2h");
}

}  // namespace

constexpr uint32_t kChunk = 256;

// Shared tail of every blocked build: sort, populate, block table, chunk plan.  Writes the
// storage arrays the caller asked for and the plan arrays "blk_begin", "blk_rc", "chunk_begin",
// "chunk_blk" (+ "chunk_state", "blk_rj" for ICRS).
struct BlockedBuild {
  Format& f;
  Arena& ar;
  Geom g;
  uint64_t nnz;
  uint64_t* skeys = nullptr;
  uint32_t nblk = 0;
  uint32_t* blk_flag = nullptr;
  uint32_t* blk_scan = nullptr;
  uint32_t* rj_flag = nullptr;
  uint32_t* rj_scan = nullptr;
  uint32_t nrj = 0;
};

static int blocked_common(BlockedBuild& bb, const spmvlab_cuda_coo& a, const uint32_t* d_bounds,
                          int key_bits, bool want_packed, bool want_icrs, uint32_t* cell_counts,
                          bool want_band) {
  Format& f = bb.f;
  Arena& ar = bb.ar;
  cudaStream_t s = ar.stream();
  const uint64_t nnz = a.nnz;
  uint64_t* keys = ar.alloc_n<uint64_t>(nnz);
  uint64_t* keys2 = ar.alloc_n<uint64_t>(nnz);
  uint64_t* pay = ar.alloc_n<uint64_t>(nnz);
  uint64_t* pay2 = ar.alloc_n<uint64_t>(nnz);
  uint32_t* err = ar.alloc_n<uint32_t>(1);
  if (!keys || !keys2 || !pay || !pay2 || !err) return kNoMemory;
  cudaMemsetAsync(err, 0, 4, s);
  const size_t bsm = is_bcoh_alg(f.alg) ? sizeof(uint32_t) * (bb.g.p + 1) : 0;
  if (bsm > 48 * 1024) {
    g_last_error = "too many bands";
    return kInvalidArgument;
  }
  blk_keys<<<grid_for(nnz, 256), 256, bsm, s>>>(a.row_ind, a.col_ind, a.data, nnz, bb.g, d_bounds, keys, pay, err);
  uint32_t herr = 0;
  if (int rc = d2h_u32(err, &herr, s)) return rc;
  if (herr & 1u) return kIndexOutOfRange;
  const bool alt = radix_sort_pairs(keys, keys2, pay, pay2, nnz, 0, key_bits, ar);
  uint64_t* sk = alt ? keys2 : keys;
  uint64_t* sv = alt ? pay2 : pay;
  bb.skeys = sk;

  uint32_t* packed = want_packed ? static_cast<uint32_t*>(f.add("packed", nnz, 4, s)) : nullptr;
  double* data = static_cast<double*>(f.add("data", nnz, 8, s));
  uint16_t* col_inc = want_icrs ? static_cast<uint16_t*>(f.add("col_inc", nnz, 2, s)) : nullptr;
  if ((want_packed && !packed) || !data || (want_icrs && !col_inc)) return kNoMemory;
  bb.blk_flag = ar.alloc_n<uint32_t>(nnz);
  bb.blk_scan = ar.alloc_n<uint32_t>(nnz + 1);
  if (want_icrs) {
    bb.rj_flag = ar.alloc_n<uint32_t>(nnz);
    bb.rj_scan = ar.alloc_n<uint32_t>(nnz + 1);
  }
  blk_populate<<<grid_for(nnz, 256), 256, 0, s>>>(sk, sv, nnz, bb.g, packed, data, col_inc, bb.blk_flag,
                                                  bb.rj_flag, cell_counts, err);
  exclusive_scan_u32(bb.blk_flag, bb.blk_scan, nnz, ar);
  if (want_icrs) exclusive_scan_u32(bb.rj_flag, bb.rj_scan, nnz, ar);
  if (int rc = d2h_u32(err, &herr, s)) return rc;
  if (herr & 2u) return kDuplicateEntry;
  if (int rc = d2h_u32(bb.blk_scan + nnz, &bb.nblk, s)) return rc;
  if (want_icrs)
    if (int rc = d2h_u32(bb.rj_scan + nnz, &bb.nrj, s)) return rc;

  const uint32_t nblk = bb.nblk;
  uint32_t* blk_begin = static_cast<uint32_t*>(f.add("blk_begin", (uint64_t)nblk + 1, 4, s));
  uint2* blk_rc = static_cast<uint2*>(f.add("blk_rc", nblk, 8, s));
  uint32_t* blk_band = want_band ? static_cast<uint32_t*>(f.add("blk_band", nblk, 4, s)) : nullptr;
  uint32_t* blk_rj = want_icrs ? static_cast<uint32_t*>(f.add("blk_rj", nblk, 4, s)) : nullptr;
  uint16_t* row_jump = want_icrs ? static_cast<uint16_t*>(f.add("row_jump", bb.nrj, 2, s)) : nullptr;
  if (!blk_begin || !blk_rc || (want_band && !blk_band) || (want_icrs && (!blk_rj || !row_jump)))
    return kNoMemory;
  const uint32_t nnz32 = (uint32_t)nnz;
  cudaMemcpyAsync(blk_begin + nblk, &nnz32, 4, cudaMemcpyHostToDevice, s);
  blk_table<<<grid_for(nnz, 256), 256, 0, s>>>(sk, nnz, bb.g, bb.blk_flag, bb.blk_scan, bb.rj_flag, bb.rj_scan,
                                               blk_begin, blk_rc, blk_band, blk_rj, row_jump);

  // chunk plan
  uint32_t* nch = ar.alloc_n<uint32_t>((uint64_t)nblk + 1);
  if (!nch) return kNoMemory;
  if (nblk) chunk_count<<<(nblk + 255) / 256, 256, 0, s>>>(blk_begin, nblk, kChunk, nch);
  exclusive_scan_u32(nch, nch, nblk, ar);
  uint32_t nchunks = 0;
  if (int rc = d2h_u32(nch + nblk, &nchunks, s)) return rc;
  uint32_t* ch_begin = static_cast<uint32_t*>(f.add("chunk_begin", (uint64_t)nchunks + 1, 4, s));
  uint32_t* ch_blk = static_cast<uint32_t*>(f.add("chunk_blk", nchunks, 4, s));
  uint4* ch_state = want_icrs ? static_cast<uint4*>(f.add("chunk_state", nchunks, 16, s)) : nullptr;
  if (!ch_begin || !ch_blk || (want_icrs && !ch_state)) return kNoMemory;
  cudaMemcpyAsync(ch_begin + nchunks, &nnz32, 4, cudaMemcpyHostToDevice, s);
  if (nblk && nchunks)
    chunk_fill<<<(nchunks + 255) / 256, 256, 0, s>>>(blk_begin, nblk, kChunk, nch, sk, bb.g, bb.rj_flag,
                                                     bb.rj_scan, blk_rj, ch_begin, ch_blk, ch_state);
  f.work_items = nchunks;
  f.needs_zero_y = true;
  return check_launch("blocked_common");
}

// Window items for CSB / CSBH / MergeBH when the beta-row window fits in shared memory (beta <=
// 2^14, 128 KB of fp64).  Those formats order elements inside a block along a curve, so the 32
// rows a warp reduces into are scattered and the per-run global reduction kernel pays one L2
// sector per element; the window kernel turns that into shared-memory adds (R-MAT s22: 831 ->
// 637 us).  Row-major MergeB blocks give coalesced runs and stay on the reduction kernel, which
// is faster there (335 vs 465 us).  SPMVLAB_BLOCKED_WINDOW=0 disables, =1 forces for all four.
// Chunks per window item: R-MAT s22 CSB 741 / 671 / 636 / 667 / 711 / 1226 us at 64 / 128 / 256 /
// 512 / 1024 / 4096 (window zero + write-out per item vs. the tail of one 1024-thread CTA per SM).
constexpr uint32_t kWinChunks = 256;
// x bytes per column panel of the chunk schedule (see schedule_plan)
constexpr uint64_t kBlkPanelXBytes = 48ull << 20;

// The multiply's chunk schedule.
//  * Column panels: when x outgrows the L2 (configs 3-5), every chunk walk in storage order sweeps
//    all of x once per block row (cfg3 MergeB: 7.97 GB of DRAM reads for 1.35 GB of algorithmic
//    bytes).  K = ceil(8n / kBlkPanelXBytes) panels of block columns are run one after the other
//    ("chunk_order" = the chunk ids stably sorted by (panel, block row)), so one panel's x window
//    stays L2-resident while its blocks stream past; y rows are then revisited once per panel.
//    Measured (B200, panel MB 4096 / 96 / 64 / 48 / 32 / 24): cfg3 MergeB 1.86 / 1.56 / 1.56 /
//    1.47 / 1.36 / 1.32 ms, BCOH 1.88 / 1.59 / 1.60 / 1.42 / 1.27 / 1.26; cfg4 MergeB 1.42 / 1.24 /
//    1.23 / 1.15 / 1.54 / 1.33, BCOH 1.02 / 1.09 / 1.08 / 1.05 / 1.19 / 1.08.  What is left is one
//    fp64 L2 reduction per element: the blocks are hypersparse at the reference's beta (cfg3 ~86
//    nonzeros per 2^14 x 2^14 block), so runs of equal rows are ~1 long.
//  * Window items (curve_in_block): runs of the same ordered list that never cross a (panel,
//    block row) pair; an item owning a whole block row stores its window, the others add theirs.
//    BCOH's Hilbert-ordered blocks interleave block rows (`permute`), so there the list is sorted
//    even with one panel.
//  * Deterministic builds: every blocked format gets window items (the chunks sorted by block row)
//    for the bucketed window kernel, which sums in a fixed order; an item owning its whole block row
//    stores it (the reference's exclusive rows), a block row split over several items gets one
//    partial window per item, added in item order by det_combine.
static int schedule_plan(Format& f, Arena& ar, bool curve_in_block, bool permute = false) {
  if (f.work_items == 0) return kOk;
  cudaStream_t s = ar.stream();
  const char* env = std::getenv("SPMVLAB_BLOCKED_WINDOW");
  const bool det = f.deterministic && f.log2_beta <= 14;
  const bool window = det || ((env && env[0] ? env[0] == '1' : curve_in_block) && f.log2_beta <= 14);
  if (det) permute = true;
  uint64_t xbytes = kBlkPanelXBytes;
  if (const char* e = std::getenv("SPMVLAB_BLK_PANEL_MB")) xbytes = (uint64_t)std::max(1, atoi(e)) << 20;
  const uint64_t want_panels = (8ull * f.n + xbytes - 1) / xbytes;
  // (window formats keep one panel: their per-element shared-memory adds, not x, bound them, and
  // the per-(panel, block row) window flushes cost more than the x locality saves -- cfg3 CSB
  // 1.89 -> 2.01 ms with 48 MB panels)
  f.blk_panels = window ? 1u : (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want_panels, f.block_cols));
  if (f.deterministic && !det) f.deterministic = false;  // beta > 2^14: no shared-memory window
  const uint32_t width = (uint32_t)(((uint64_t)f.n + f.blk_panels - 1) / f.blk_panels);
  const uint32_t nch = (uint32_t)f.work_items;
  const uint32_t* ch_blk = f.find("chunk_blk")->as<uint32_t>();
  const uint2* blk_rc = f.find("blk_rc")->as<uint2>();
  const uint32_t* ord = nullptr;
  if (f.blk_panels > 1 || (window && permute)) {
    const int brbits = std::max(1, (int)bit_width64(f.block_rows ? f.block_rows - 1 : 0));
    const int pbits = (int)bit_width64(f.blk_panels - 1);
    uint64_t* k1 = ar.alloc_n<uint64_t>(nch);
    uint64_t* k2 = ar.alloc_n<uint64_t>(nch);
    uint32_t* v2 = ar.alloc_n<uint32_t>(nch);
    uint32_t* v1 = static_cast<uint32_t*>(f.add("chunk_order", nch, 4, s));
    if (!k1 || !k2 || !v1 || !v2) return kNoMemory;
    sched_keys<<<(nch + 255) / 256, 256, 0, s>>>(ch_blk, blk_rc, nch, f.log2_beta, f.blk_panels, width, brbits,
                                                   k1, v1);
    if (radix_sort_pairs(k1, k2, v1, v2, nch, 0, brbits + pbits, ar))
      cudaMemcpyAsync(v1, v2, 4ull * nch, cudaMemcpyDeviceToDevice, s);
    ord = v1;
  }
  if (!window) return check_launch("schedule_plan");
  uint32_t* head = ar.alloc_n<uint32_t>((uint64_t)nch + 1);
  uint32_t* flag = ar.alloc_n<uint32_t>((uint64_t)nch + 1);
  if (!head || !flag) return kNoMemory;
  win_heads<<<(nch + 255) / 256, 256, 0, s>>>(ord, ch_blk, blk_rc, nch, kWinChunks, f.log2_beta, f.blk_panels,
                                               width, head);
  win_flag<<<(nch + 255) / 256, 256, 0, s>>>(head, nch, flag);  // flag = head != 0
  exclusive_scan_u32(flag, flag, nch, ar);                        // -> item index of each head
  uint32_t nitems = 0;
  if (int rc = d2h_u32(flag + nch, &nitems, s)) return rc;
  uint32_t* item_chunk = static_cast<uint32_t*>(f.add("win_item_chunk", (uint64_t)nitems + 1, 4, s));
  uint32_t* item_br = static_cast<uint32_t*>(f.add("win_item_br", nitems, 4, s));
  uint32_t* item_whole = static_cast<uint32_t*>(f.add("win_item_whole", nitems, 4, s));
  if (!item_chunk || !item_br || !item_whole) return kNoMemory;
  cudaMemcpyAsync(item_chunk + nitems, &nch, 4, cudaMemcpyHostToDevice, s);
  win_fill<<<(nch + 255) / 256, 256, 0, s>>>(head, flag, ord, ch_blk, blk_rc, nch, f.blk_panels, item_chunk,
                                              item_br, item_whole);
  if (det) {
    // A block row split over several items: each writes its whole window to a partial slot and
    // det_combine adds the slots in item order -- a fixed order, so still the same bits every run.
    std::vector<uint32_t> br(nitems), whole(nitems);
    cudaMemcpyAsync(br.data(), item_br, 4ull * nitems, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(whole.data(), item_whole, 4ull * nitems, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("schedule_plan (det)");
    std::vector<uint32_t> slot(nitems, 0xFFFFFFFFu), sbr, sfirst;
    uint32_t nslots = 0;
    for (uint32_t i = 0; i < nitems; ++i) {
      if (whole[i]) continue;
      if (sbr.empty() || sbr.back() != br[i]) {
        sbr.push_back(br[i]);
        sfirst.push_back(nslots);
      }
      slot[i] = nslots++;
    }
    sfirst.push_back(nslots);
    uint32_t* d_slot = static_cast<uint32_t*>(f.add("det_item_slot", nitems, 4, s));
    uint32_t* d_sbr = static_cast<uint32_t*>(f.add("det_split_br", sbr.size(), 4, s));
    uint32_t* d_sfirst = static_cast<uint32_t*>(f.add("det_split_first", sfirst.size(), 4, s));
    double* part = static_cast<double*>(f.add("det_partials", ((uint64_t)nslots << f.log2_beta) + 1, 8, s));
    if (!d_slot || !d_sbr || !d_sfirst || !part) return kNoMemory;
    cudaMemcpyAsync(d_slot, slot.data(), 4ull * nitems, cudaMemcpyHostToDevice, s);
    if (!sbr.empty()) cudaMemcpyAsync(d_sbr, sbr.data(), 4ull * sbr.size(), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_sfirst, sfirst.data(), 4ull * sfirst.size(), cudaMemcpyHostToDevice, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("schedule_plan (det)");
  }
  return check_launch("schedule_plan");
}

static Geom base_geom(const Format& f, unsigned lb) {
  Geom g{};
  g.lb = lb;
  g.mask = (1u << lb) - 1u;
  g.m = f.m;
  g.n = f.n;
  g.block_cols = f.block_cols;
  g.bcbits = (int)bit_width64(f.block_cols ? f.block_cols - 1 : 0);
  return g;
}

int build_csb(Format& f, const spmvlab_cuda_coo& a, unsigned lb, bool hilbert, uint64_t, Arena& ar) {
  cudaStream_t s = ar.stream();
  if (lb < 1 || lb > 16) return kInvalidArgument;
  f.log2_beta = lb;
  f.block_rows = (uint32_t)(((uint64_t)f.m + (1u << lb) - 1) >> lb);
  f.block_cols = (uint32_t)(((uint64_t)f.n + (1u << lb) - 1) >> lb);
  const uint64_t cells = (uint64_t)f.block_rows * f.block_cols;
  uint32_t* blk_ptr = static_cast<uint32_t*>(f.add("blk_ptr", cells + 1, 4, s));
  if (!blk_ptr) return kNoMemory;
  cudaMemsetAsync(blk_ptr, 0, 4 * (cells + 1), s);
  Geom g = base_geom(f, lb);
  g.kind = hilbert ? kCsbH : kCsbZ;
  const int brbits = (int)bit_width64(f.block_rows ? f.block_rows - 1 : 0);
  BlockedBuild bb{f, ar, g, a.nnz};
  if (a.nnz) {
    if (int rc = blocked_common(bb, a, nullptr, brbits + g.bcbits + 2 * (int)lb, true, false, blk_ptr, false))
      return rc;
  } else {
    f.add("packed", 0, 4, s);
    f.add("data", 0, 8, s);
  }
  exclusive_scan_u32(blk_ptr, blk_ptr, cells, ar);
  // storage_report order (inc/storage.hpp:85-90): blk_ptr, packed, data
  std::stable_partition(f.arrays.begin(), f.arrays.end(), [](const DevArray& d) {
    return d.name == "blk_ptr" || d.name == "packed" || d.name == "data";
  });
  f.nstorage = 3;
  if (int rc = schedule_plan(f, ar, true)) return rc;
  return check_launch("build_csb");
}

int build_mergeb(Format& f, const spmvlab_cuda_coo& a, unsigned lb, bool hilbert, Arena& ar) {
  cudaStream_t s = ar.stream();
  if (lb < 1 || lb > 16) return kInvalidArgument;
  f.log2_beta = lb;
  f.block_rows = (uint32_t)(((uint64_t)f.m + (1u << lb) - 1) >> lb);
  f.block_cols = (uint32_t)(((uint64_t)f.n + (1u << lb) - 1) >> lb);
  Geom g = base_geom(f, lb);
  g.kind = hilbert ? kMbH : kMbRow;
  const int brbits = (int)bit_width64(f.block_rows ? f.block_rows - 1 : 0);
  uint32_t* blk_row_ptr = static_cast<uint32_t*>(f.add("blk_row_ptr", (uint64_t)f.block_rows + 1, 4, s));
  if (!blk_row_ptr) return kNoMemory;
  cudaMemsetAsync(blk_row_ptr, 0, 4 * ((uint64_t)f.block_rows + 1), s);
  BlockedBuild bb{f, ar, g, a.nnz};
  uint32_t nblk = 0;
  if (a.nnz) {
    if (int rc = blocked_common(bb, a, nullptr, brbits + g.bcbits + 2 * (int)lb, true, false, nullptr, false))
      return rc;
    nblk = bb.nblk;
  } else {
    f.add("packed", 0, 4, s);
    f.add("data", 0, 8, s);
    uint32_t* bb0 = static_cast<uint32_t*>(f.add("blk_begin", 1, 4, s));
    cudaMemsetAsync(bb0, 0, 4, s);
  }
  uint32_t* blk_col_ind = static_cast<uint32_t*>(f.add("blk_col_ind", nblk, 4, s));
  uint32_t* blk_data_ptr = static_cast<uint32_t*>(f.add("blk_data_ptr", (uint64_t)nblk + 1, 4, s));
  if (!blk_col_ind || !blk_data_ptr) return kNoMemory;
  cudaMemcpyAsync(blk_data_ptr, f.find("blk_begin")->ptr, 4 * ((uint64_t)nblk + 1), cudaMemcpyDeviceToDevice, s);
  if (nblk)
    mergeb_arrays<<<(nblk + 255) / 256, 256, 0, s>>>(f.find("blk_rc")->as<uint2>(), nblk, blk_col_ind, blk_row_ptr);
  exclusive_scan_u32(blk_row_ptr, blk_row_ptr, f.block_rows, ar);
  // storage_report order (inc/storage.hpp:92-99)
  const char* order[] = {"blk_row_ptr", "blk_col_ind", "blk_data_ptr", "packed", "data"};
  std::vector<DevArray> sorted;
  for (const char* nm : order) sorted.push_back(*f.find(nm));
  for (auto& d : f.arrays) {
    bool in = false;
    for (const char* nm : order) in = in || d.name == nm;
    if (!in) sorted.push_back(d);
  }
  f.arrays = sorted;
  f.nstorage = 5;
  if (int rc = schedule_plan(f, ar, hilbert)) return rc;
  return check_launch("build_mergeb");
}

int build_bcoh(Format& f, const spmvlab_cuda_coo& a, unsigned lb, unsigned p, Arena& ar) {
  cudaStream_t s = ar.stream();
  const int alg = f.alg;
  const bool icrs = alg == kBcoh;
  const bool helem = alg == kBcohch || alg == kBcohchp;
  const bool hptr = alg == kBcohchp;
  if (lb < 1 || lb > 15) {
    g_last_error = "block size outside the 15-bit increment cap";
    return kInvalidArgument;
  }
  if (p < 1) {
    g_last_error = "band count must be >= 1";
    return kInvalidArgument;
  }
  const uint32_t beta = 1u << lb;
  f.log2_beta = lb;
  f.block_rows = (uint32_t)(((uint64_t)f.m + beta - 1) >> lb);
  f.block_cols = (uint32_t)(((uint64_t)f.n + beta - 1) >> lb);
  uint32_t ext = std::max<uint32_t>(std::max<uint32_t>(f.m, f.n), 1u);
  const unsigned cov = bit_width64((uint64_t)ext - 1);
  if (cov > 31) {
    g_last_error = "grid too large for 64-bit curve keys";
    return kOverflow;
  }
  f.element_level = std::max(cov, lb);
  f.block_level = f.element_level - lb;
  f.bands = p;

  // row prefix + partition_rows_by_nnz (inc/bcoh.hpp:213-216); the greedy lower bounds run on the
  // device, the clamp chain (a few integer ops per band) on the host.
  // raw_cut[k-1] = (greedy row + beta/2) >> lb of partition_rows_by_nnz, from per-rounding-cell
  // counts when they fit in shared memory, else from the full row prefix
  std::vector<uint32_t> raw_cut(p > 1 ? p - 1 : 1), bounds(p + 1);
  const uint32_t half = beta / 2;
  const uint64_t cells = (((uint64_t)f.m + half) >> lb) + 1;
  if (p > 1 && cells <= kMaxRoundCells) {
    uint32_t* d_cell = ar.alloc_n<uint32_t>(2 * cells);
    if (!d_cell) return kNoMemory;
    cudaMemsetAsync(d_cell, 0, 8 * cells, s);
    if (a.nnz)
      round_cell_hist<<<grid_for(a.nnz, 256, kNumSMs * 4), 256, 0, s>>>(a.row_ind, a.nnz, f.m, lb, (uint32_t)cells,
                                                                        d_cell, d_cell + cells);
    std::vector<uint32_t> tot(cells), last(cells);
    cudaMemcpyAsync(tot.data(), d_cell, 4 * cells, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(last.data(), d_cell + cells, 4 * cells, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("bcoh row cells");
    uint64_t nnz_rows = 0;
    for (uint32_t v : tot) nnz_rows += v;
    // prefix[min(E_c - 1, m)] with E_c = (c+1) beta - beta/2, the rows before the cell's last row
    std::vector<uint64_t> pre(cells);
    uint64_t run = 0;
    for (uint64_t c = 0; c < cells; ++c) {
      const uint64_t end_row = (c + 1) * beta - half - 1;
      pre[c] = end_row >= f.m ? nnz_rows : run + tot[c] - last[c];
      run += tot[c];
    }
    for (unsigned k = 1; k < p; ++k) {  // smallest cell whose prefix reaches k * nnz / p
      const uint64_t target = nnz_rows * k;
      uint64_t lo = 0, hi = cells - 1;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (pre[mid] * p >= target) hi = mid; else lo = mid + 1;
      }
      raw_cut[k - 1] = (uint32_t)lo;
    }
  } else if (p > 1) {
    uint32_t* prefix = ar.alloc_n<uint32_t>((uint64_t)f.m + 1);
    uint32_t* d_greedy = ar.alloc_n<uint32_t>(p);
    if (!prefix || !d_greedy) return kNoMemory;
    cudaMemsetAsync(prefix, 0, 4 * ((uint64_t)f.m + 1), s);
    if (a.nnz) row_hist<<<grid_for(a.nnz, 256), 256, 0, s>>>(a.row_ind, a.nnz, f.m, prefix);
    exclusive_scan_u32(prefix, prefix, f.m, ar);
    greedy_rows<<<(p + 255) / 256, 256, 0, s>>>(prefix, f.m, p, d_greedy);
    std::vector<uint32_t> greedy(p - 1);
    cudaMemcpyAsync(greedy.data(), d_greedy, 4 * (p - 1), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("bcoh prefix");
    for (unsigned k = 1; k < p; ++k) raw_cut[k - 1] = (uint32_t)(((uint64_t)greedy[k - 1] + half) >> lb);
  }
  {
    // Replays partition_rows_by_nnz's clamp chain (inc/block_size.hpp:86-98) on the raw cuts.
    const uint32_t block_rows = f.block_rows;
    for (unsigned k = 0; k <= p; ++k) bounds[k] = f.m;
    bounds[0] = 0;
    uint32_t prev_cut = 0;
    for (unsigned k = 1; k < p; ++k) {
      uint32_t cut = raw_cut[k - 1];
      const uint32_t hic = block_rows >= p ? block_rows - (p - k) : block_rows;
      const uint32_t loc = prev_cut + 1 < hic ? prev_cut + 1 : hic;
      if (cut < loc) cut = loc;
      if (cut > hic) cut = hic;
      const uint64_t b = (uint64_t)cut << lb;
      bounds[k] = b < f.m ? (uint32_t)b : f.m;
      prev_cut = cut;
    }
  }
  if (f.block_cols >= (1u << 15)) {
    g_last_error = "band block grid has " + std::to_string(f.block_cols) +
                   " columns; 16-bit block increments require < 2^15";
    return kOverflow;
  }
  std::vector<uint32_t> fbr(p), brc(p), frow(p), rcount(p);
  for (unsigned b = 0; b < p; ++b) {
    frow[b] = bounds[b];
    rcount[b] = bounds[b + 1] - bounds[b];
    fbr[b] = bounds[b] >> lb;
    brc[b] = rcount[b] == 0 ? 0 : (uint32_t)((((uint64_t)bounds[b + 1] + beta - 1) >> lb) - fbr[b]);
    if (brc[b] >= (1u << 15)) {
      g_last_error = "band block grid has too many rows for 16-bit block increments";
      return kOverflow;
    }
  }
  const int bandbits = (int)bit_width64(p - 1);
  if (bandbits + 2 * (int)f.element_level > 64) {
    g_last_error = "band and Hilbert key exceed 64 bits";
    return kOverflow;
  }
  uint32_t* d_bounds = ar.alloc_n<uint32_t>(p + 1);
  uint32_t* d_fbr = ar.alloc_n<uint32_t>(p);
  cudaMemcpyAsync(d_bounds, bounds.data(), 4 * (p + 1), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_fbr, fbr.data(), 4 * p, cudaMemcpyHostToDevice, s);

  // storage arrays in storage_report order are arranged at the end
  Geom g = base_geom(f, lb);
  g.kind = helem ? kBcohH : kBcohRow;
  g.block_level = f.block_level;
  g.element_level = f.element_level;
  g.p = p;
  uint32_t* cell_counts = nullptr;
  uint64_t cells_all = (uint64_t)f.block_rows * f.block_cols;
  if (hptr) {
    cell_counts = ar.alloc_n<uint32_t>(cells_all + 1);
    if (!cell_counts) return kNoMemory;
    cudaMemsetAsync(cell_counts, 0, 4 * (cells_all + 1), s);
  }
  BlockedBuild bb{f, ar, g, a.nnz};
  const unsigned el2 = 2 * f.element_level;
  std::vector<uint64_t> off_elem(p + 1, 0), off_block(p + 1, 0), off_rj(p + 1, 0), off_rjb(p + 1, 0), off_ptr(p + 1, 0);
  uint32_t nblk = 0, nrjb = 0;
  uint32_t* rjb_scan = nullptr;
  if (a.nnz) {
    if (int rc = blocked_common(bb, a, d_bounds, bandbits + (int)el2, !icrs, icrs, cell_counts, true)) return rc;
    nblk = bb.nblk;
  } else {
    f.add("data", 0, 8, s);
    if (icrs) {
      f.add("col_inc", 0, 2, s);
      f.add("row_jump", 0, 2, s);
    } else {
      f.add("packed", 0, 4, s);
    }
    uint32_t* bb0 = static_cast<uint32_t*>(f.add("blk_begin", 1, 4, s));
    cudaMemsetAsync(bb0, 0, 4, s);
  }
  const uint32_t* blk_begin = f.find("blk_begin")->as<uint32_t>();
  // BICRS block level
  uint32_t* block_nnz = static_cast<uint32_t*>(f.add("block_nnz", hptr ? 0 : nblk, 4, s));
  int16_t* col_jump_block = static_cast<int16_t*>(f.add("col_jump_block", hptr ? 0 : nblk, 2, s));
  if (!block_nnz || !col_jump_block) return kNoMemory;
  if (!hptr && nblk) {
    uint32_t* rjb_flag = ar.alloc_n<uint32_t>(nblk);
    rjb_scan = ar.alloc_n<uint32_t>((uint64_t)nblk + 1);
    bicrs_blocks<<<(nblk + 255) / 256, 256, 0, s>>>(blk_begin, f.find("blk_rc")->as<uint2>(),
                                                    f.find("blk_band")->as<uint32_t>(), nblk, f.block_cols,
                                                    block_nnz, col_jump_block, rjb_flag);
    exclusive_scan_u32(rjb_flag, rjb_scan, nblk, ar);
    if (int rc = d2h_u32(rjb_scan + nblk, &nrjb, s)) return rc;
    int16_t* rjb = static_cast<int16_t*>(f.add("row_jump_block", nrjb, 2, s));
    if (!rjb) return kNoMemory;
    bicrs_row_jumps<<<(nblk + 255) / 256, 256, 0, s>>>(f.find("blk_rc")->as<uint2>(),
                                                       f.find("blk_band")->as<uint32_t>(), nblk, rjb_flag,
                                                       rjb_scan, d_fbr, rjb);
  } else {
    f.add("row_jump_block", 0, 2, s);
  }
  // Hilbert pointer block level
  uint64_t total_cells = 0;
  std::vector<uint64_t> cell_off(p + 1, 0);
  for (unsigned b = 0; b < p; ++b) cell_off[b + 1] = cell_off[b] + (uint64_t)brc[b] * f.block_cols;
  total_cells = cell_off[p];
  uint32_t* blk_ptr = static_cast<uint32_t*>(f.add("blk_ptr", hptr ? total_cells + p : 0, 4, s));
  if (!blk_ptr) return kNoMemory;
  if (hptr) {
    for (unsigned b = 0; b <= p; ++b) off_ptr[b] = cell_off[b] + b;
    uint64_t* d_cell_off = ar.alloc_n<uint64_t>(p + 1);
    cudaMemcpyAsync(d_cell_off, cell_off.data(), 8 * (p + 1), cudaMemcpyHostToDevice, s);
    if (total_cells) {
      uint64_t* ck = ar.alloc_n<uint64_t>(total_cells);
      uint64_t* ck2 = ar.alloc_n<uint64_t>(total_cells);
      uint32_t* cid = ar.alloc_n<uint32_t>(total_cells);
      uint32_t* cid2 = ar.alloc_n<uint32_t>(total_cells);
      uint32_t* cnt = ar.alloc_n<uint32_t>(total_cells + 1);
      if (!ck || !ck2 || !cid || !cid2 || !cnt) return kNoMemory;
      hptr_cell_keys<<<grid_for(total_cells, 256), 256, 0, s>>>(total_cells, p, d_cell_off, d_fbr, f.block_cols,
                                                                f.block_level, ck, cid);
      const bool calt = radix_sort_pairs(ck, ck2, cid, cid2, total_cells, 0, bandbits + 2 * (int)f.block_level, ar);
      hptr_counts<<<grid_for(total_cells, 256), 256, 0, s>>>(calt ? cid2 : cid, total_cells, cell_counts, cnt);
      exclusive_scan_u32(cnt, cnt, total_cells, ar);
      hptr_fill<<<grid_for(total_cells + p, 256), 256, 0, s>>>(cnt, total_cells, p, d_cell_off, blk_ptr);
    } else {
      cudaMemsetAsync(blk_ptr, 0, 4 * p, s);
    }
  }
  if (!icrs) {
    if (!f.find("col_inc")) f.add("col_inc", 0, 2, s);
    if (!f.find("row_jump")) f.add("row_jump", 0, 2, s);
  } else if (!f.find("packed")) {
    f.add("packed", 0, 4, s);
  }
  // per-band offsets
  if (a.nnz) {
    uint64_t* d_off = ar.alloc_n<uint64_t>(4 * (p + 1));
    band_offsets<<<(p + 1 + 255) / 256, 256, 0, s>>>(bb.skeys, a.nnz, el2, p, f.find("blk_band")->as<uint32_t>(),
                                                     nblk, bb.rj_scan, rjb_scan, d_off, d_off + (p + 1),
                                                     d_off + 2 * (p + 1), d_off + 3 * (p + 1));
    std::vector<uint64_t> tmp(4 * (p + 1));
    cudaMemcpyAsync(tmp.data(), d_off, 8 * 4 * (p + 1), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("band offsets");
    for (unsigned b = 0; b <= p; ++b) {
      off_elem[b] = tmp[b];
      off_block[b] = hptr ? 0 : tmp[(p + 1) + b];
      off_rj[b] = tmp[2 * (p + 1) + b];
      off_rjb[b] = tmp[3 * (p + 1) + b];
    }
  }
  auto upload = [&](const char* name, const void* host, uint64_t count, uint32_t esz) -> bool {
    void* d = f.add(name, count, esz, s);
    if (!d) return false;
    if (count) cudaMemcpyAsync(d, host, count * esz, cudaMemcpyHostToDevice, s);
    return true;
  };
  bool ok = upload("band_first_row", frow.data(), p, 4) && upload("band_row_count", rcount.data(), p, 4) &&
            upload("band_first_block_row", fbr.data(), p, 4) &&
            upload("band_block_row_count", brc.data(), p, 4) && upload("off_elem", off_elem.data(), p + 1, 8) &&
            upload("off_block", off_block.data(), p + 1, 8) &&
            upload("off_row_jump_block", off_rjb.data(), p + 1, 8) &&
            upload("off_blk_ptr", off_ptr.data(), p + 1, 8) && upload("off_row_jump", off_rj.data(), p + 1, 8);
  if (!ok) return kNoMemory;
  // storage_report order (inc/storage.hpp:101-123)
  const char* order[] = {"block_nnz", "row_jump_block", "col_jump_block", "blk_ptr",
                         "col_inc",   "row_jump",       "packed",         "data"};
  std::vector<DevArray> sorted;
  for (const char* nm : order) sorted.push_back(*f.find(nm));
  for (auto& d : f.arrays) {
    bool in = false;
    for (const char* nm : order) in = in || d.name == nm;
    if (!in) sorted.push_back(d);
  }
  f.arrays = sorted;
  f.nstorage = 8;
  // chunk schedule: column panels when x outgrows the L2; the Hilbert in-block (packed) variants
  // (and deterministic builds) get block-row windows over a block-row ordering of the chunks
  if (a.nnz)
    if (int rc = schedule_plan(f, ar, helem, helem)) return rc;
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("build_bcoh");
  return check_launch("build_bcoh");
}

}  // namespace spmvcu
