// convert_crs.cu -- COO -> CRS (triplet_to_crs, inc/crs.hpp:67-91) and the merge-path tile plan.
//
// Reference: sort a permutation by (row, col) with a comparator, count rows, partial_sum, gather.
// Here: one 64-bit key (row << colbits | col) per entry, LSD radix sort of (key, entry index) over
// exactly bit_width(m-1) + bit_width(n-1) bits, then one populate pass that derives col_ind from
// the key, gathers data through the permutation and histograms rows (warp-aggregated atomics over
// the sorted, hence run-grouped, rows), and a decoupled look-back scan for row_ptr.  Keys are
// unique, so the order -- and every output array -- is bit-identical to the reference's.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
extern thread_local std::string g_last_error;
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
// row_ptr may be a panel's slice of the stacked panel row pointer (first entry `base`); the tile
// coordinates are then absolute element indices into the panel arrays.
__global__ void merge_partition(const uint32_t* __restrict__ row_ptr, uint32_t m, uint64_t nnz,
                                uint32_t tiles, uint32_t tile_items, uint32_t* __restrict__ trow,
                                uint32_t* __restrict__ tnnz, uint32_t base = 0) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > tiles) return;
  const uint64_t total = (uint64_t)m + nnz;
  const uint64_t dt = (uint64_t)t * tile_items;
  const uint64_t diag = dt < total ? dt : total;
  uint64_t lo = diag > nnz ? diag - nnz : 0;
  uint64_t hi = diag < m ? diag : m;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;
    if ((uint64_t)(row_ptr[mid] - base) <= diag - mid) lo = mid; else hi = mid - 1;
  }
  trow[t] = (uint32_t)lo;
  tnnz[t] = base + (uint32_t)(diag - lo);
}

// ---- column panels (merge-CSR when x exceeds the L2): panel k holds the entries with column in
// [k*W, (k+1)*W), rows in CRS order, stored as the CRS of the K*m-row stacked matrix
// [A_0; A_1; ...].  Columns are sorted inside a CRS row, so a row's panel split points are binary
// searches in its col_ind slice.
__device__ __forceinline__ uint32_t row_lower_bound(const uint32_t* __restrict__ col, uint32_t b, uint32_t e,
                                                    uint64_t v) {
  while (b < e) {
    const uint32_t mid = b + (e - b) / 2;
    if ((uint64_t)col[mid] < v) b = mid + 1; else e = mid;
  }
  return b;
}

// Panel k holds the columns [cut[k], cut[k+1]) (cut[0] = 0, cut[K] = n).
struct PanelCuts {
  uint32_t c[kMaxMergePanels + 1];
};
__device__ __forceinline__ uint32_t panel_of(const PanelCuts& pc, uint32_t panels, uint32_t col) {
  uint32_t k = 0;
  while (k + 1 < panels && col >= pc.c[k + 1]) ++k;
  return k;
}

__global__ void panel_counts(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, uint32_t m,
                             uint32_t panels, const __grid_constant__ PanelCuts pc, uint32_t* __restrict__ cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += stride) {
    const uint32_t b = row_ptr[r], e = row_ptr[r + 1];
    uint32_t prev = b;
    for (uint32_t k = 1; k < panels; ++k) {
      const uint32_t sp = row_lower_bound(col, prev, e, (uint64_t)pc.c[k]);
      cnt[(uint64_t)(k - 1) * m + r] = sp - prev;
      prev = sp;
    }
    cnt[(uint64_t)(panels - 1) * m + r] = e - prev;
  }
}

// Element i of row r in panel k goes to prp[k*m + r] + (i - first element of row r in panel k), that
// first element being a binary search of the panel's first column in the row's col_ind slice.
// One warp per 1024 consecutive elements (coalesced reads; K sequential write streams); an
// element's row is a binary search of row_ptr between the rows of the chunk's first and last
// elements, so rows of 10^6 entries (cfg3) are spread over many warps.
__device__ __forceinline__ uint32_t row_of(const uint32_t* __restrict__ row_ptr, uint32_t lo, uint32_t hi,
                                           uint32_t i) {
  // largest r in [lo, hi] with row_ptr[r] <= i
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo + 1) / 2;
    if (row_ptr[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void panel_fill(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                           const double* __restrict__ val, uint32_t m, uint64_t nnz, uint32_t panels,
                           const __grid_constant__ PanelCuts pc, const uint32_t* __restrict__ prp,
                           uint32_t* __restrict__ pcol,
                           double* __restrict__ pval) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t e0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 1024; e0 < nnz;
       e0 += wstride * 1024) {
    const uint32_t e1 = (uint32_t)(e0 + 1024 < nnz ? e0 + 1024 : nnz);
    uint32_t r_lo = 0, r_hi = 0;
    if (lane == 0) r_lo = row_of(row_ptr, 0, m - 1, (uint32_t)e0);
    if (lane == 1) r_hi = row_of(row_ptr, 0, m - 1, e1 - 1);
    r_lo = __shfl_sync(0xFFFFFFFFu, r_lo, 0);
    r_hi = __shfl_sync(0xFFFFFFFFu, r_hi, 1);
    for (uint32_t i = (uint32_t)e0 + lane; i < e1; i += 32) {
      const uint32_t r = row_of(row_ptr, r_lo, r_hi, i);
      const uint32_t c = col[i];
      const uint32_t k = panel_of(pc, panels, c);
      const uint32_t first = k ? row_lower_bound(col, row_ptr[r], i, (uint64_t)pc.c[k]) : row_ptr[r];
      const uint32_t o = prp[(uint64_t)k * m + r] + (i - first);
      pcol[o] = c;
      pval[o] = val[i];
    }
  }
}

// Panels k >= 1 that are sparse in rows are doubly compressed: only the rows with entries in the
// panel.  flag[j] (j = (k-1) m + r) marks them, pos = its exclusive scan.  meta[k] = (offset of the
// panel's row pointer in the concatenated pointer array, offset of its row ids, pos at the panel's
// first row, 1 if compressed): a compressed panel's row pointer entry i and row id i go to
// (meta.x + i, meta.y + i) with i = pos[j] - meta.z; full panels are copied separately.
__global__ void panel_row_flags(const uint32_t* __restrict__ prp, uint32_t m, uint32_t panels,
                                uint32_t* __restrict__ flag) {
  const uint64_t total = (uint64_t)(panels - 1) * m;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride) {
    const uint64_t g = j + m;  // row r of panel k = j / m + 1 in the stacked pointer
    flag[j] = prp[g + 1] > prp[g] ? 1u : 0u;
  }
}

__global__ void panel_row_fill(const uint32_t* __restrict__ prp, const uint32_t* __restrict__ flag,
                               const uint32_t* __restrict__ pos, uint32_t m, uint32_t panels,
                               const uint4* __restrict__ meta, uint32_t* __restrict__ crp,
                               uint32_t* __restrict__ rows) {
  const uint64_t total = (uint64_t)(panels - 1) * m;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride) {
    if (!flag[j]) continue;
    const uint32_t k = (uint32_t)(j / m) + 1, r = (uint32_t)(j % m);
    const uint4 mk = meta[k];
    if (!mk.w) continue;  // full panel
    const uint32_t i = pos[j] - mk.z;
    rows[mk.y + i] = r;
    crp[mk.x + i] = prp[j + m];
  }
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
  int ipt = kMergeIpt;
  // tile size: the largest of 32 / 16 / 8 items per lane that still leaves >= 4 warp tiles per
  // resident warp slot (148 SMs x 48 warps), so small matrices keep every SM busy
  const uint64_t slots = 4ull * kNumSMs * 48;
  ipt = total >= slots * 32 * 32 ? 32 : (total >= slots * 32 * 16 ? 16 : 8);
  if (const char* e = getenv("SPMVLAB_MERGE_IPT")) {  // developer / test override: 8, 16 or 32
    const int v = atoi(e);
    if (merge_shape_supported(kMergeThreads, v)) ipt = v;
  }
  f.merge_threads = kMergeThreads;
  f.merge_ipt = ipt;
  uint32_t tile_items = 32u * (uint32_t)ipt;
  // Column panels for the merge engine when x outgrows the L2 (beyond ~L2 the x
  // gathers become DRAM sectors): K = ceil(8n / kPanelXBytes), at most kMaxMergePanels, so each
  // panel's x window stays L2-resident while its slice of A streams past.
  uint32_t panels = 1;
  if (f.alg == kMerge && f.nnz > 0) {
    const uint64_t xb = 8ull * f.n;
    panels = (uint32_t)std::min<uint64_t>(kAutoMergePanels, (xb + kPanelXBytes - 1) / kPanelXBytes);
    if (const char* e = getenv("SPMVLAB_MERGE_PANELS")) panels = (uint32_t)std::max(1, std::min(atoi(e), kMaxMergePanels));
    if ((uint64_t)panels * f.m + 1 > 0xFFFFFFFFull || f.n < panels) panels = 1;
  }
  std::vector<uint32_t> pbase(panels + 1, 0);   // first element of each panel in the panel arrays
  std::vector<uint32_t> nrows(panels, f.m);     // rows the panel's merge path walks
  std::vector<uint32_t> rp_off(panels, 0), rows_off(panels, 0);
  if (panels > 1) {
    // The panels are an L2 optimisation: if their arrays do not fit, build without them.
    const uint64_t rows = (uint64_t)panels * f.m;
    uint32_t* prp = ar.alloc_n<uint32_t>(rows + 1);
    uint32_t* flag = ar.alloc_n<uint32_t>((uint64_t)(panels - 1) * f.m + 1);
    uint32_t* pos = ar.alloc_n<uint32_t>((uint64_t)(panels - 1) * f.m + 1);
    uint32_t* p_col = static_cast<uint32_t*>(f.add("merge_panel_col", f.nnz, 4, s));
    double* p_val = static_cast<double*>(f.add("merge_panel_data", f.nnz, 8, s));
    if (!prp || !flag || !pos || !p_col || !p_val) {
      cudaGetLastError();
      f.drop("merge_panel_col");
      f.drop("merge_panel_data");
      panels = 1;
    } else {
      // uniform column ranges; SPMVLAB_MERGE_PANEL_CUTS="c1,c2,..." (developer) sets the inner cuts
      PanelCuts pc{};
      const uint32_t width = (f.n + panels - 1) / panels;
      for (uint32_t k = 0; k <= panels; ++k) pc.c[k] = (uint32_t)std::min<uint64_t>((uint64_t)k * width, f.n);
      if (const char* e = getenv("SPMVLAB_MERGE_PANEL_CUTS")) {
        uint32_t k = 1;
        for (const char* q = e; *q && k < panels; ++k) {
          pc.c[k] = (uint32_t)std::min<unsigned long>(strtoul(q, nullptr, 10), f.n);
          while (*q && *q != ',') ++q;
          if (*q == ',') ++q;
        }
        for (k = 1; k < panels; ++k) pc.c[k] = std::max(pc.c[k], pc.c[k - 1]);
      }
      f.merge_panel_cuts.assign(pc.c, pc.c + panels + 1);
      const uint32_t* rp = f.find("row_ptr")->as<uint32_t>();
      const uint32_t* col = f.find("col_ind")->as<uint32_t>();
      panel_counts<<<grid_for(f.m, 256), 256, 0, s>>>(rp, col, f.m, panels, pc, prp);
      exclusive_scan_u32(prp, prp, rows, ar);
      panel_fill<<<grid_for((f.nnz + 1023) / 1024 * 32, 256), 256, 0, s>>>(
          rp, col, f.find("data")->as<double>(), f.m, f.nnz, panels, pc, prp, p_col, p_val);
      const uint64_t nflag = (uint64_t)(panels - 1) * f.m;
      panel_row_flags<<<grid_for(nflag, 256), 256, 0, s>>>(prp, f.m, panels, flag);
      exclusive_scan_u32(flag, pos, nflag, ar);
      std::vector<uint32_t> pcut(panels, 0);  // pos at each panel start (k >= 1), + the total
      for (uint32_t k = 0; k <= panels; ++k)
        cudaMemcpyAsync(&pbase[k], prp + (uint64_t)k * f.m, 4, cudaMemcpyDeviceToHost, s);
      for (uint32_t k = 1; k < panels; ++k)
        cudaMemcpyAsync(&pcut[k - 1], pos + (uint64_t)(k - 1) * f.m, 4, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(&pcut[panels - 1], pos + nflag, 4, cudaMemcpyDeviceToHost, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("build_merge_plan (panels)");
      // a panel with entries in more than half of the rows keeps a full row pointer (no row-id
      // indirection: cfg4 K = 2, 97 % of the rows in panel 1, 685 -> 647 us)
      std::vector<uint4> meta(panels, make_uint4(0, 0, 0, 0));
      uint64_t ptr_len = (uint64_t)f.m + 1, nr = 0;
      f.merge_panel_row_visits = pcut[panels - 1];
      for (uint32_t k = 1; k < panels; ++k) {
        const uint32_t rk = pcut[k] - pcut[k - 1];
        const bool comp = (uint64_t)rk * 2 <= f.m;
        meta[k] = make_uint4((uint32_t)ptr_len, (uint32_t)nr, pcut[k - 1], comp ? 1u : 0u);
        nrows[k] = comp ? rk : f.m;
        rp_off[k] = (uint32_t)ptr_len;
        rows_off[k] = comp ? (uint32_t)nr : 0xFFFFFFFFu;
        ptr_len += (uint64_t)nrows[k] + 1;
        if (comp) nr += rk;
      }
      uint32_t* crp = static_cast<uint32_t*>(f.add("merge_panel_row_ptr", ptr_len, 4, s));
      uint32_t* prow = static_cast<uint32_t*>(f.add("merge_panel_rows", nr, 4, s));
      uint4* dmeta = reinterpret_cast<uint4*>(ar.alloc_n<uint32_t>(4ull * panels));
      if (!crp || !prow || !dmeta || ptr_len > 0xFFFFFFFFull) {
        cudaGetLastError();
        for (const char* nm : {"merge_panel_col", "merge_panel_data", "merge_panel_row_ptr", "merge_panel_rows"})
          f.drop(nm);
        panels = 1;
      } else {
        cudaMemcpyAsync(dmeta, meta.data(), sizeof(uint4) * panels, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(crp, prp, 4ull * (f.m + 1), cudaMemcpyDeviceToDevice, s);  // panel 0: every row
        panel_row_fill<<<grid_for(nflag, 256), 256, 0, s>>>(prp, flag, pos, f.m, panels, dmeta, crp, prow);
        for (uint32_t k = 1; k < panels; ++k) {
          if (meta[k].w)  // the end entry of a compressed pointer
            cudaMemcpyAsync(crp + rp_off[k] + nrows[k], prp + (uint64_t)(k + 1) * f.m, 4, cudaMemcpyDeviceToDevice, s);
          else            // a full panel: its slice of the stacked pointer
            cudaMemcpyAsync(crp + rp_off[k], prp + (uint64_t)k * f.m, 4ull * (f.m + 1), cudaMemcpyDeviceToDevice, s);
        }
        if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("build_merge_plan (panel rows)");
      }
    }
  }
  if (panels == 1) {
    f.merge_panel_row_visits = 0;
    pbase.assign(2, 0);
    pbase[1] = (uint32_t)f.nnz;
    nrows.assign(1, f.m);
    rp_off.assign(1, 0);
    rows_off.assign(1, 0);
  }
  f.merge_hot = 0;
  f.merge_hot_share = 0.0;
  f.merge_persist = false;
  f.merge_x_noalloc = false;
  if (f.alg == kMerge) {  // the column skew, and on one panel the hot-x plan
    if (int rc = build_hot_columns(f, ar, panels == 1)) return rc;
  }
  if (panels == 1 && f.alg == kMerge) {
    f.merge_persist = f.merge_hot > 0;
    if (f.merge_persist) {
      // equal merge-path shares, kHotTilesPerWarp per warp of the persistent grid
      uint64_t per = (uint64_t)kNumSMs * kHotWarps * kHotTilesPerWarp;
      if (const char* e = getenv("SPMVLAB_MERGE_HOT_TILES")) per = (uint64_t)kNumSMs * kHotWarps * std::max(1, atoi(e));
      // (at most 65535 items: the tile kernel's row map stores row - first row in 16 bits)
      tile_items = (uint32_t)std::min<uint64_t>(65535, std::max<uint64_t>(128, (total + per - 1) / per));
    }
  }
  f.merge_panels = panels;
  f.merge_panel_width = panels > 1 ? (f.n + panels - 1) / panels : f.n;
  f.panel_nrows = nrows;
  f.panel_rp_off = rp_off;
  f.panel_rows_off = rows_off;
  f.panel_tile_off.assign(panels + 1, 0);
  for (uint32_t k = 0; k < panels; ++k) {
    const uint64_t tk = ((uint64_t)nrows[k] + (pbase[k + 1] - pbase[k]) + tile_items - 1) / tile_items;
    f.panel_tile_off[k + 1] = f.panel_tile_off[k] + (uint32_t)tk;
  }
  const uint64_t tiles = f.panel_tile_off[panels];
  f.merge_tiles = (uint32_t)tiles;
  // one extra coordinate per panel (each panel's tile list has tiles_k + 1 boundaries)
  uint32_t* trow = static_cast<uint32_t*>(f.add("merge_tile_row", tiles + panels, 4, s));
  uint32_t* tnnz = static_cast<uint32_t*>(f.add("merge_tile_nnz", tiles + panels, 4, s));
  if (!trow || !tnnz) return kNoMemory;
  // carry scratch is per stream (Format::stream_scratch); pre-create the build stream's
  if (!f.stream_scratch(s)) return kNoMemory;
  const uint32_t* crp = panels > 1 ? f.find("merge_panel_row_ptr")->as<uint32_t>() : f.find("row_ptr")->as<uint32_t>();
  for (uint32_t k = 0; k < panels; ++k) {
    const uint32_t tk = f.panel_tile_off[k + 1] - f.panel_tile_off[k];
    const uint32_t o = f.panel_tile_off[k] + k;
    merge_partition<<<(unsigned)((tk + 1 + 255) / 256), 256, 0, s>>>(
        crp + rp_off[k], nrows[k], (uint64_t)(pbase[k + 1] - pbase[k]), tk, tile_items, trow + o, tnnz + o,
        pbase[k]);
  }
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

// ---- hot-x plan of the merge engine (B200 design, no reference counterpart: a power-law column
// distribution -- R-MAT -- sends a large share of the x gathers to few columns).  Per-column
// reference counts are taken over a sample of col_ind -- every kHotSample-th run of 32 consecutive
// entries (all entries below 2^24 nonzeros) -- and scaled by the sampling stride.  Columns whose
// count is at least T, T the smallest count (>= kHotMinRefs) that keeps them within kHotMaxSlots,
// get a shared-memory slot in column order; the plan copy merge_hot_col of col_ind marks their
// entries 0x80000000 | slot.  Kept only when they cover kHotMinShare of the (sampled) entries.
// (Counting every entry took 0.75 ms at cfg2 -- 65 M atomics, most on a few hot columns.)
constexpr uint32_t kHotSample = 8;
constexpr uint64_t kHotSampleFrom = 1ull << 24;

namespace {
__global__ void col_ref_counts(const uint32_t* __restrict__ col, uint64_t nnz, uint32_t stride_runs,
                               uint32_t* __restrict__ cnt) {
  const uint64_t runs = (nnz + 31) / 32;
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * stride_runs < runs; w += nw) {
    const uint64_t k = w * stride_runs * 32 + lane;
    if (k < nnz) atomicAdd(cnt + col[k], 1u);
  }
}

constexpr uint32_t kRefBins = 65536;  // counts clamped to kRefBins - 1

__global__ void ref_count_hist(const uint32_t* __restrict__ cnt, uint32_t n, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[1024];
  for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t c = cnt[i];
    if (c < 1024) atomicAdd(&sh[c], 1u);
    else atomicAdd(hist + min(c, kRefBins - 1), 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
}

__global__ void hot_flags(const uint32_t* __restrict__ cnt, uint32_t n, uint32_t thr, uint32_t* __restrict__ flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = cnt[i] >= thr;
}

// hot column list, and colmap[c] = the plan's index of column c (0x80000000 | slot, or c)
__global__ void hot_fill(const uint32_t* __restrict__ cnt, uint32_t n, uint32_t thr, const uint32_t* __restrict__ slot,
                         uint32_t* __restrict__ hot_cols, uint32_t* __restrict__ colmap) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool hot = cnt[i] >= thr;
  if (hot) hot_cols[slot[i]] = i;
  colmap[i] = hot ? (0x80000000u | slot[i]) : i;
}

__global__ void hot_remap(const uint32_t* __restrict__ col, uint64_t nnz, const uint32_t* __restrict__ colmap,
                          uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) out[k] = colmap[col[k]];
}
}  // namespace

int build_hot_columns(Format& f, Arena& ar, bool adopt) {
  cudaStream_t s = ar.stream();
  f.merge_hot = 0;
  f.merge_x_noalloc = false;
  if (f.nnz == 0 || f.n == 0 || f.n > 0x7FFFFFFFu) return kOk;
  const uint32_t* col = f.find("col_ind")->as<uint32_t>();
  uint32_t* cnt = ar.alloc_n<uint32_t>((uint64_t)f.n + 1);
  uint32_t* hist = ar.alloc_n<uint32_t>(kRefBins);
  if (!cnt || !hist) return kNoMemory;
  cudaMemsetAsync(cnt, 0, 4ull * f.n, s);
  cudaMemsetAsync(hist, 0, 4ull * kRefBins, s);
  const uint32_t samp = f.nnz >= kHotSampleFrom ? kHotSample : 1u;
  col_ref_counts<<<grid_for((f.nnz + samp - 1) / samp, 256), 256, 0, s>>>(col, f.nnz, samp, cnt);
  ref_count_hist<<<grid_for(f.n, 256, kNumSMs * 4), 256, 0, s>>>(cnt, f.n, hist);
  std::vector<uint32_t> h(kRefBins);
  cudaMemcpyAsync(h.data(), hist, 4ull * kRefBins, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("build_hot_columns");
  const uint32_t min_cnt = (kHotMinRefs + samp - 1) / samp;  // counts are of the sample
  auto select = [&](uint32_t cap, uint64_t& take, uint64_t& refs, uint32_t& thr) {
    take = refs = 0;
    thr = 0;
    for (uint32_t c = kRefBins - 1; c >= min_cnt; --c) {
      if (take + h[c] > cap) break;
      take += h[c];
      refs += (uint64_t)c * h[c] * samp;
      if (h[c]) thr = c;
    }
    return thr != 0 && take != 0 && (double)refs >= kHotMinShare * (double)f.nnz;
  };
  uint64_t take = 0, refs = 0;
  uint32_t thr = 0;
  // No column skew (the most referenced kHotMaxSlots columns cover under kHotMinShare of the
  // entries): the merge kernels gather x without L1 allocation (cfg3 / cfg4: -3 / -2 %; on R-MAT the
  // L1 holds the hot columns: without allocation cfg2 292 -> 389 us, cfg5 +1 %).
  f.merge_x_noalloc = !select(kHotMaxSlots, take, refs, thr);
  uint32_t cap = adopt ? kHotMaxSlots : 0;
  if (const char* e = getenv("SPMVLAB_MERGE_HOT_SLOTS")) cap = (uint32_t)std::max(0, std::min(atoi(e), (int)kHotMaxSlots));
  if (const char* e = getenv("SPMVLAB_MERGE_HOT")) if (atoi(e) == 0) cap = 0;
  if (!adopt || cap == 0 || !select(cap, take, refs, thr)) return check_launch("build_hot_columns");
  uint32_t* flag = ar.alloc_n<uint32_t>((uint64_t)f.n + 1);
  uint32_t* colmap = ar.alloc_n<uint32_t>((uint64_t)f.n);
  uint32_t* hc = static_cast<uint32_t*>(f.add("merge_hot_col", f.nnz, 4, s));
  uint32_t* hl = static_cast<uint32_t*>(f.add("merge_hot_cols", take, 4, s));
  if (!flag || !colmap || !hc || !hl) {  // the hot-x plan is an optimisation: build without it
    cudaGetLastError();
    f.drop("merge_hot_col");
    f.drop("merge_hot_cols");
    return kOk;
  }
  hot_flags<<<grid_for(f.n, 256, 1u << 30), 256, 0, s>>>(cnt, f.n, thr, flag);
  exclusive_scan_u32(flag, flag, f.n, ar);
  hot_fill<<<grid_for(f.n, 256, 1u << 30), 256, 0, s>>>(cnt, f.n, thr, flag, hl, colmap);
  hot_remap<<<grid_for(f.nnz, 256), 256, 0, s>>>(col, f.nnz, colmap, hc);
  uint32_t total = 0;
  cudaMemcpyAsync(&total, flag + f.n, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("build_hot_columns");
  if (total != take) {
    g_last_error = "hot-x plan: column count mismatch";
    return kCudaError;
  }
  f.merge_hot = (uint32_t)take;
  f.merge_hot_share = (double)refs / (double)f.nnz;
  return check_launch("build_hot_columns");
}

int merge_path_search(const uint32_t* a, uint64_t a_len, const uint32_t* b, uint64_t b_len, const uint64_t* diags,
                      uint64_t count, uint64_t* out_i, cudaStream_t s) {
  if (count == 0) return kOk;
  merge_path_search_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(a, a_len, b, b_len, diags, count, out_i);
  return check_launch("merge_path_search");
}

}  // namespace spmvcu
