// spmv_crs.cu -- the CRS engines: sequential CRS, ParCRS and merge-path CRS (sm_100a).
//
//  * SeqCrs (spmv_crs_seq, inc/crs.hpp:43-57): one thread per row summing in storage order with
//    explicitly rounded multiply and add (no FMA contraction), so y is BITWISE equal to the
//    reference's sequential kernel.
//  * ParCrs (spmv_parcrs, inc/spmv_parallel.hpp:106-125): rows claimed by sub-warp groups whose
//    width is the next power of two >= the mean row length; lanes stride the row, shuffle-reduce.
//  * Merge (spmv_merge, inc/spmv_parallel.hpp:130-160): the merge path over (row_ptr[1..m],
//    0..nnz-1) is cut into equal tiles of kMergeTile items at build time (merge_partition); each CTA
//    stages its tile's products val*x[col] and row ends in shared memory, every thread walks
//    kMergeIpt items of its own sub-path (per-thread diagonal search in shared memory), partial
//    rows are combined by a block-wide segmented scan, y for the tile's rows is written with
//    coalesced stores, and each tile leaves one (row, value) carry-out.  A fix-up kernel adds the
//    carries of rows that span tiles, in tile order (deterministic).
#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
namespace {

__global__ void seq_crs_kernel(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ x,
                               double* __restrict__ y, uint32_t m) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double sum = 0.0;
  const uint32_t e = row_ptr[i + 1];
  for (uint32_t k = row_ptr[i]; k < e; ++k) sum = __dadd_rn(sum, __dmul_rn(val[k], x[col[k]]));
  y[i] = sum;
}

template <int G>
__global__ void __launch_bounds__(256) par_crs_kernel(const uint32_t* __restrict__ row_ptr,
                                                      const uint32_t* __restrict__ col,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ x,
                                                      double* __restrict__ y, uint32_t m) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t sub = threadIdx.x & (G - 1);
  const uint64_t group = gid / G;
  const uint64_t ngroups = (uint64_t)gridDim.x * blockDim.x / G;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned gmask = (G == 32) ? 0xFFFFFFFFu : (((1u << G) - 1u) << (lane & ~(unsigned)(G - 1)));
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  for (uint64_t r = group; r < m; r += ngroups) {
    const uint32_t b = row_ptr[r], e = row_ptr[r + 1];
    double s = 0.0;
    for (uint32_t k = b + sub; k < e; k += G) s += ld_stream(val + k, pf) * ld_x(x + ld_stream(col + k, pf), pl);
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(gmask, s, off, G);
    if (sub == 0) y[r] = s;
  }
}

// Segmented-scan operator on (has_row_end, value): (f1,v1) + (f2,v2) = (f1|f2, f2 ? v2 : v1+v2).
struct Seg {
  double v;
  int f;
};
__device__ __forceinline__ Seg seg_combine(Seg a, Seg b) { return {b.f ? b.v : a.v + b.v, a.f | b.f}; }

template <int THREADS, int IPT>
__global__ void __launch_bounds__(THREADS, 4) merge_spmv_kernel(
    const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const uint32_t* __restrict__ tile_row,
    const uint32_t* __restrict__ tile_nnz, uint32_t* __restrict__ carry_row,
    double* __restrict__ carry_val, uint32_t m) {
  constexpr int TILE = THREADS * IPT;
  constexpr int WARPS = THREADS / 32;
  __shared__ uint32_t s_rowend[TILE];
  __shared__ double s_buf[TILE];  // [0, nnzs): products; [nnzs, nnzs + nrows): y of the tile's rows
  __shared__ double s_wv[WARPS];
  __shared__ int s_wf[WARPS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t t = blockIdx.x;
  const uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const uint32_t j0 = tile_nnz[t], j1 = tile_nnz[t + 1];
  const int nrows = (int)(r1 - r0), nnzs = (int)(j1 - j0);

  // Stage: row ends of rows r0..r1-1 and the products of entries j0..j1-1 (coalesced, streaming).
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  for (int k = tid; k < nrows; k += THREADS) s_rowend[k] = ld_stream(row_ptr + r0 + 1 + k, pf);
#pragma unroll 4
  for (int k = tid; k < nnzs; k += THREADS) {
    const uint32_t c = ld_stream(col + j0 + k, pf);
    s_buf[k] = ld_stream(val + j0 + k, pf) * ld_x(x + c, pl);
  }
  __syncthreads();

  // Per-thread sub-path: diagonal search inside the tile (ties consume row ends).
  const int len = nrows + nnzs;
  const int diag = min(tid * IPT, len);
  int lo = max(0, diag - nnzs), hi = min(diag, nrows);
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_rowend[mid - 1] <= j0 + (uint32_t)(diag - mid)) lo = mid; else hi = mid - 1;
  }
  int ri = lo, ji = diag - lo;
  const int dend = min(diag + IPT, len);
  double run = 0.0, first_val = 0.0;
  int first_row = -1;
  for (int d = diag; d < dend; ++d) {
    if (ri < nrows && (ji >= nnzs || s_rowend[ri] <= j0 + (uint32_t)ji)) {
      if (first_row < 0) { first_row = ri; first_val = run; }
      else s_buf[nnzs + ri] = run;
      run = 0.0;
      ++ri;
    } else {
      run += s_buf[ji];
      ++ji;
    }
  }

  // Block-wide inclusive segmented scan of (has_row_end, tail value).
  Seg me{run, first_row >= 0 ? 1 : 0};
  Seg inc = me;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Seg o;
    o.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, off);
    o.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, off);
    if (lane >= off) inc = seg_combine(o, inc);
  }
  if (lane == 31) { s_wv[warp] = inc.v; s_wf[warp] = inc.f; }
  __syncthreads();
  Seg wpre{0.0, 0};
  for (int w = 0; w < warp; ++w) wpre = seg_combine(wpre, Seg{s_wv[w], s_wf[w]});
  Seg excl;
  excl.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, 1);
  excl.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, 1);
  if (lane == 0) excl = Seg{0.0, 0};
  excl = seg_combine(wpre, excl);
  if (first_row >= 0) s_buf[nnzs + first_row] = first_val + excl.v;
  if (tid == THREADS - 1) {
    const Seg all = seg_combine(wpre, inc);
    carry_row[t] = r1;
    carry_val[t] = all.v;
  }
  __syncthreads();
  for (int k = tid; k < nrows; k += THREADS) y[r0 + k] = s_buf[nnzs + k];
}

// Rows spanning tiles: the head tile of each run of equal carry rows sums the run in tile order.
__global__ void merge_fixup_kernel(const uint32_t* __restrict__ carry_row,
                                   const double* __restrict__ carry_val, uint32_t tiles,
                                   double* __restrict__ y, uint32_t m) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tiles) return;
  const uint32_t r = carry_row[t];
  if (r >= m) return;
  if (t > 0 && carry_row[t - 1] == r) return;
  double s = carry_val[t];
  for (uint32_t u = t + 1; u < tiles && carry_row[u] == r; ++u) s += carry_val[u];
  y[r] += s;
}

}  // namespace

int spmv_seq_crs(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.m == 0) return kOk;
  seq_crs_kernel<<<(f.m + 127) / 128, 128, 0, s>>>(f.find("row_ptr")->as<uint32_t>(),
                                                   f.find("col_ind")->as<uint32_t>(),
                                                   f.find("data")->as<double>(), x, y, f.m);
  return check_launch("spmv_seq_crs");
}

int spmv_par_crs(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.m == 0) return kOk;
  const uint32_t* rp = f.find("row_ptr")->as<uint32_t>();
  const uint32_t* ci = f.find("col_ind")->as<uint32_t>();
  const double* d = f.find("data")->as<double>();
  const unsigned blocks = grid_for((uint64_t)f.m * f.par_group, 256, kNumSMs * 8);
  switch (f.par_group) {
    case 2: par_crs_kernel<2><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    case 4: par_crs_kernel<4><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    case 8: par_crs_kernel<8><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    case 16: par_crs_kernel<16><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    default: par_crs_kernel<32><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
  }
  return check_launch("spmv_par_crs");
}

int spmv_merge(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.merge_tiles == 0) return kOk;
  const uint32_t* crow = f.find("merge_carry_row")->as<uint32_t>();
  merge_spmv_kernel<kMergeThreads, kMergeIpt><<<f.merge_tiles, kMergeThreads, 0, s>>>(
      f.find("row_ptr")->as<uint32_t>(), f.find("col_ind")->as<uint32_t>(), f.find("data")->as<double>(),
      x, y, f.find("merge_tile_row")->as<uint32_t>(), f.find("merge_tile_nnz")->as<uint32_t>(),
      f.find("merge_carry_row")->as<uint32_t>(), f.find("merge_carry_val")->as<double>(), f.m);
  merge_fixup_kernel<<<(f.merge_tiles + 255) / 256, 256, 0, s>>>(
      crow, f.find("merge_carry_val")->as<double>(), f.merge_tiles, y, f.m);
  return check_launch("spmv_merge");
}

}  // namespace spmvcu
