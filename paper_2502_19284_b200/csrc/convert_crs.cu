// convert_crs.cu -- COO -> CRS (triplet_to_crs, inc/crs.hpp:67-91) and the merge-path tile plan.
//
// Reference: sort a permutation by (row, col) with a comparator, count rows, partial_sum, gather.
// Here: one 64-bit key (row << colbits | col) per entry, LSD radix sort of (key, entry index) over
// exactly bit_width(m-1) + bit_width(n-1) bits, then one populate pass that derives col_ind from
// the key, gathers data through the permutation and histograms rows (warp-aggregated atomics over
// the sorted, hence run-grouped, rows), and a decoupled look-back scan for row_ptr.  Keys are
// unique, so the order -- and every output array -- is bit-identical to the reference's.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
namespace {

__global__ void crs_keys(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cols,
                         const double* __restrict__ vals, uint64_t nnz, uint32_t m, uint32_t n,
                         int colbits, uint64_t* __restrict__ keys, uint64_t* __restrict__ payload,
                         uint32_t* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint32_t r = rows[k], c = cols[k];
    if (r >= m || c >= n) atomicOr(err, 1u);
    keys[k] = ((uint64_t)r << colbits) | c;
    payload[k] = __double_as_longlong(vals[k]);
  }
}

__global__ void crs_populate(const uint64_t* __restrict__ skeys, const uint64_t* __restrict__ svals,
                             uint64_t nnz, int colbits,
                             uint32_t* __restrict__ col_ind, double* __restrict__ data,
                             uint32_t* __restrict__ counts, uint32_t* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t cmask = (colbits >= 64) ? ~0ull : ((1ull << colbits) - 1);
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint64_t key = skeys[k];
    const uint32_t row = (uint32_t)(key >> colbits);
    col_ind[k] = (uint32_t)(key & cmask);
    data[k] = __longlong_as_double((long long)svals[k]);
    if (k > 0 && skeys[k - 1] == key) atomicOr(err, 2u);
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, row);
    if (lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&counts[row], (unsigned)__popc(peers));
  }
}

// One merge-path diagonal per tile boundary (diagonal_search, spmv_parallel.hpp:47-69, with
// A = row_ptr[1..m], B = 0..nnz-1).
__global__ void merge_partition(const uint32_t* __restrict__ row_ptr, uint32_t m, uint64_t nnz,
                                uint32_t tiles, uint32_t tile_items, uint32_t* __restrict__ trow,
                                uint32_t* __restrict__ tnnz) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > tiles) return;
  const uint64_t total = (uint64_t)m + nnz;
  const uint64_t dt = (uint64_t)t * tile_items;
  const uint64_t diag = dt < total ? dt : total;
  uint64_t lo = diag > nnz ? diag - nnz : 0;
  uint64_t hi = diag < m ? diag : m;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;
    if ((uint64_t)row_ptr[mid] <= diag - mid) lo = mid; else hi = mid - 1;
  }
  trow[t] = (uint32_t)lo;
  tnnz[t] = (uint32_t)(diag - lo);
}

__global__ void merge_path_search_kernel(const uint32_t* __restrict__ a, uint64_t a_len,
                                         const uint32_t* __restrict__ b,
                                         uint64_t b_len, const uint64_t* __restrict__ diags,
                                         uint64_t count, uint64_t* __restrict__ out_i) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const uint64_t diag = diags[k];
  uint64_t lo = diag > b_len ? diag - b_len : 0;
  uint64_t hi = diag < a_len ? diag : a_len;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;
    const uint64_t j = diag - mid;
    const uint64_t bj = b ? (uint64_t)b[j < b_len ? j : 0] : j;
    const bool pred = j >= b_len || !(bj < (uint64_t)a[mid - 1]);
    if (pred) lo = mid; else hi = mid - 1;
  }
  out_i[k] = lo;
}

__global__ void long_row_flags(const uint32_t* __restrict__ row_ptr, uint32_t m, uint32_t lim,
                               uint32_t* __restrict__ flag) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m) flag[r] = row_ptr[r + 1] - row_ptr[r] > lim;
}

__global__ void long_row_fill(const uint32_t* __restrict__ row_ptr, uint32_t m, uint32_t lim,
                              const uint32_t* __restrict__ scan, uint32_t* __restrict__ out) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m && row_ptr[r + 1] - row_ptr[r] > lim) out[scan[r]] = r;
}

}  // namespace

int build_crs(Format& f, const spmvlab_cuda_coo& a, Arena& ar) {
  cudaStream_t s = ar.stream();
  const uint64_t nnz = a.nnz;
  uint32_t* row_ptr = static_cast<uint32_t*>(f.add("row_ptr", (uint64_t)a.m + 1, 4, s));
  uint32_t* col_ind = static_cast<uint32_t*>(f.add("col_ind", nnz, 4, s));
  double* data = static_cast<double*>(f.add("data", nnz, 8, s));
  f.nstorage = 3;
  if (!row_ptr || !col_ind || !data) return kNoMemory;
  cudaMemsetAsync(row_ptr, 0, sizeof(uint32_t) * ((uint64_t)a.m + 1), s);
  if (nnz == 0) return check_launch("build_crs");

  const int colbits = (int)bit_width64(a.n > 0 ? a.n - 1 : 0);
  const int rowbits = (int)bit_width64(a.m > 0 ? a.m - 1 : 0);
  uint64_t* keys = ar.alloc_n<uint64_t>(nnz);
  uint64_t* keys2 = ar.alloc_n<uint64_t>(nnz);
  uint64_t* pay = ar.alloc_n<uint64_t>(nnz);
  uint64_t* pay2 = ar.alloc_n<uint64_t>(nnz);
  uint32_t* err = ar.alloc_n<uint32_t>(1);
  if (!keys || !keys2 || !pay || !pay2 || !err) return kNoMemory;
  cudaMemsetAsync(err, 0, 4, s);
  crs_keys<<<grid_for(nnz, 256), 256, 0, s>>>(a.row_ind, a.col_ind, a.data, nnz, a.m, a.n, colbits, keys,
                                              pay, err);
  const bool alt = radix_sort_pairs(keys, keys2, pay, pay2, nnz, 0, colbits + rowbits, ar);
  const uint64_t* sk = alt ? keys2 : keys;
  const uint64_t* sp = alt ? pay2 : pay;
  crs_populate<<<grid_for(nnz, 256), 256, 0, s>>>(sk, sp, nnz, colbits, col_ind, data, row_ptr, err);
  exclusive_scan_u32(row_ptr, row_ptr, a.m, ar);
  uint32_t herr = 0;
  cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("build_crs");
  if (herr & 1u) return kIndexOutOfRange;
  if (herr & 2u) return kDuplicateEntry;
  return check_launch("build_crs");
}

int build_merge_plan(Format& f, Arena& ar) {
  cudaStream_t s = ar.stream();
  const uint64_t total = (uint64_t)f.m + f.nnz;
  int th = kMergeThreads, ipt = kMergeIpt, var = kMergeVariant;
  // tile size: the largest of 32 / 16 / 8 items per lane that still leaves >= 4 warp tiles per
  // resident warp slot (148 SMs x 48 warps), so small matrices keep every SM busy
  const uint64_t slots = 4ull * kNumSMs * 48;
  ipt = total >= slots * 32 * 32 ? 32 : (total >= slots * 32 * 16 ? 16 : 8);
  if (const char* e = getenv("SPMVLAB_MERGE_CFG")) {  // developer override "threads,ipt,variant"
    int a = 0, b = 0, c = 0;
    if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && merge_shape_supported(a, b, c)) {
      th = a;
      ipt = b;
      var = c;
    }
  }
  f.merge_threads = th;
  f.merge_ipt = ipt;
  f.merge_variant = var;
  const uint32_t tile_items = merge_tile_items(th, ipt, var);
  const uint64_t tiles = (total + tile_items - 1) / tile_items;
  f.merge_tiles = (uint32_t)tiles;
  uint32_t* trow = static_cast<uint32_t*>(f.add("merge_tile_row", tiles + 1, 4, s));
  uint32_t* tnnz = static_cast<uint32_t*>(f.add("merge_tile_nnz", tiles + 1, 4, s));
  if (!trow || !tnnz) return kNoMemory;
  // carry scratch is per stream (Format::stream_scratch); pre-create the build stream's
  if (!f.stream_scratch(s)) return kNoMemory;
  merge_partition<<<(unsigned)((tiles + 1 + 255) / 256), 256, 0, s>>>(
      f.find("row_ptr")->as<uint32_t>(), f.m, f.nnz, (uint32_t)tiles, tile_items, trow, tnnz);
  // ParCRS sub-warp width: next power of two >= mean row length, clamped to [2, 32]; rows longer
  // than kParLongIters * width get one CTA each.  On heavy-tailed row lengths (more than 0.1 % of
  // the rows are "long") many narrow groups plus the per-row CTAs win instead: width 2, CTAs above
  // 64 nonzeros (R-MAT s22: 1061 -> 492 us; uniform ER / Laplacian rows keep the mean rule).
  const double mean = f.m ? (double)f.nnz / f.m : 0.0;
  uint32_t g = 2;
  while (g < 32 && g < mean) g <<= 1;
  uint32_t lim = kParLongIters * g;
  const char* eg = getenv("SPMVLAB_PARCRS_G");  // developer overrides
  const char* el = getenv("SPMVLAB_PARCRS_LIM");
  uint32_t* flag = ar.alloc_n<uint32_t>((uint64_t)f.m + 1);
  if (!flag) return kNoMemory;
  uint32_t nlong = 0;
  auto count_long = [&](uint32_t l) -> int {
    if (f.m) long_row_flags<<<(f.m + 255) / 256, 256, 0, s>>>(f.find("row_ptr")->as<uint32_t>(), f.m, l, flag);
    exclusive_scan_u32(flag, flag, f.m, ar);
    cudaMemcpyAsync(&nlong, flag + f.m, 4, cudaMemcpyDeviceToHost, s);
    return cudaStreamSynchronize(s) != cudaSuccess ? check_launch("build_merge_plan") : kOk;
  };
  if (int rc = count_long(lim)) return rc;
  if (!eg && !el && (uint64_t)nlong * 1000 > f.m && g > 2) {
    g = 2;
    lim = 2 * kParLongIters;
    if (int rc = count_long(lim)) return rc;
  }
  if (eg || el) {
    if (eg) {
      const int v = atoi(eg);
      if (v == 2 || v == 4 || v == 8 || v == 16 || v == 32) g = (uint32_t)v;
    }
    lim = el ? (uint32_t)std::max(1, atoi(el)) : kParLongIters * g;
    if (int rc = count_long(lim)) return rc;
  }
  f.par_group = g;
  f.par_lim = lim;
  uint32_t* lr = static_cast<uint32_t*>(f.add("par_long_rows", nlong, 4, s));
  if (nlong && !lr) return kNoMemory;
  if (nlong)
    long_row_fill<<<(f.m + 255) / 256, 256, 0, s>>>(f.find("row_ptr")->as<uint32_t>(), f.m, lim, flag, lr);
  f.par_long = nlong;
  return check_launch("build_merge_plan");
}

int merge_path_search(const uint32_t* a, uint64_t a_len, const uint32_t* b, uint64_t b_len, const uint64_t* diags,
                      uint64_t count, uint64_t* out_i, cudaStream_t s) {
  if (count == 0) return kOk;
  merge_path_search_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(a, a_len, b, b_len, diags, count, out_i);
  return check_launch("merge_path_search");
}

}  // namespace spmvcu
