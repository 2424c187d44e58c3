// spmv_crs.cu -- the CRS engines: sequential CRS, ParCRS and merge-path CRS (sm_100a).
//
//  * SeqCrs (spmv_crs_seq, inc/crs.hpp:43-57): one thread per row summing in storage order with
//    explicitly rounded multiply and add (no FMA contraction), so y is BITWISE equal to the
//    reference's sequential kernel.
//  * ParCrs (spmv_parcrs, inc/spmv_parallel.hpp:106-125): rows claimed by sub-warp groups whose
//    width is the next power of two >= the mean row length; lanes stride the row, shuffle-reduce.
//  * Merge (spmv_merge, inc/spmv_parallel.hpp:130-160): the merge path over (row_ptr[1..m],
//    0..nnz-1) is cut into equal tiles of THREADS*IPT items at build time (merge_partition, one
//    diagonal search per tile boundary).  Per tile a CTA stages the row ends and the products
//    val*x[col] in shared memory (coalesced streaming loads, or TMA bulk copies in the persistent
//    variant), then every thread merges IPT consecutive path items.  Each thread's starting path
//    point comes from scattering the row ends to the threads that consume them (no per-thread
//    binary search), rows that cross threads are combined by a block-wide segmented scan, the y
//    values of the tile's rows are written with coalesced stores, and the tile leaves one
//    (row, partial) carry-out.  A fix-up kernel adds the carries of rows spanning tiles in tile
//    order (deterministic; mirrors the sequential carry loop at spmv_parallel.hpp:157-159).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
extern thread_local std::string g_last_error;
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

template <int THREADS>
struct MergeScratch {
  int first[THREADS];  // first row end consumed by each thread (or nrows)
  int wmin[THREADS / 32];
  double wv[THREADS / 32];
  int wf[THREADS / 32];
};

// Merges one staged tile.  srow[0..nrows): row ends row_ptr[r0+1..r1]; sbuf[0..nnzs): products;
// writes the y values of the tile's rows to sbuf[nnzs .. nnzs+nrows) and returns (in *carry) the
// tile's partial sum of row r1.  Must be called by all THREADS threads; ends with __syncthreads.
template <int THREADS, int IPT>
__device__ __forceinline__ double merge_tile(const uint32_t* srow, double* sbuf, int nrows, int nnzs,
                                             uint32_t j0, MergeScratch<THREADS>& sc) {
  constexpr int WARPS = THREADS / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int len = nrows + nnzs;

  // Owner of row end ri = the thread whose IPT-item window holds its path diagonal
  // ri + (row_end - j0).  Threads learn their starting row as the first row end owned by any
  // thread >= them (suffix minimum).
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

  // Block-wide inclusive segmented scan of (has_row_end, tail value).
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

// One tile per CTA; A is staged with coalesced streaming loads (all IPT loads of a thread in
// flight before any use, then all IPT x gathers).
template <int THREADS, int IPT, int XMODE>
__global__ void __launch_bounds__(THREADS, 4) merge_spmv_kernel(
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
      if (k < nnzs) vv[i] *= ld_xm<XMODE>(x + cv[i], pl);
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

// Persistent, TMA-pipelined variant.  Each CTA walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...;
// one thread streams the next tiles' col_ind / data / row-end slices into a STAGES-deep ring of
// shared-memory buffers with 1-D bulk copies (cp.async.bulk, completion on an mbarrier, L2
// evict-first), so A arrives with no per-thread load instructions while the CTA gathers x and
// merges the current tile.  Products overwrite the staged values in place.
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
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      const uint32_t t = blockIdx.x + s * gridDim.x;
      if (t < tiles) issue(t, s);
    }
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

template <int THREADS, int IPT, int XMODE>
void launch_merge_direct(const Format& f, const double* x, double* y, cudaStream_t s) {
  merge_spmv_kernel<THREADS, IPT, XMODE><<<f.merge_tiles, THREADS, 0, s>>>(
      f.find("row_ptr")->as<uint32_t>(), f.find("col_ind")->as<uint32_t>(), f.find("data")->as<double>(),
      x, y, f.find("merge_tile_row")->as<uint32_t>(), f.find("merge_tile_nnz")->as<uint32_t>(),
      f.find("merge_carry_row")->as<uint32_t>(), f.find("merge_carry_val")->as<double>());
}

template <int THREADS, int IPT, int STAGES>
void launch_merge_tma(const Format& f, const double* x, double* y, cudaStream_t s) {
  using Cfg = MergeTmaCfg<THREADS, IPT, STAGES>;
  auto kern = merge_spmv_tma_kernel<THREADS, IPT, STAGES>;
  static int grid_per_sm = [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, Cfg::SMEM);
    return occ > 0 ? occ : 1;
  }();
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t grid = std::min<uint32_t>(f.merge_tiles, (uint32_t)(sms * grid_per_sm));
  kern<<<grid, THREADS, Cfg::SMEM, s>>>(
      f.find("row_ptr")->as<uint32_t>(), f.find("col_ind")->as<uint32_t>(), f.find("data")->as<double>(),
      x, y, f.find("merge_tile_row")->as<uint32_t>(), f.find("merge_tile_nnz")->as<uint32_t>(),
      f.find("merge_carry_row")->as<uint32_t>(), f.find("merge_carry_val")->as<double>(), f.merge_tiles);
}

}  // namespace

int spmv_seq_crs(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.m == 0) return kOk;
  timing_begin("seq_crs_kernel", s);
  seq_crs_kernel<<<(f.m + 127) / 128, 128, 0, s>>>(f.find("row_ptr")->as<uint32_t>(),
                                                   f.find("col_ind")->as<uint32_t>(),
                                                   f.find("data")->as<double>(), x, y, f.m);
  timing_end(s);
  note_launch();
  return check_launch("spmv_seq_crs");
}

int spmv_par_crs(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.m == 0) return kOk;
  const uint32_t* rp = f.find("row_ptr")->as<uint32_t>();
  const uint32_t* ci = f.find("col_ind")->as<uint32_t>();
  const double* d = f.find("data")->as<double>();
  const unsigned blocks = grid_for((uint64_t)f.m * f.par_group, 256, kNumSMs * 8);
  note_launch();
  switch (f.par_group) {
    case 2: par_crs_kernel<2><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    case 4: par_crs_kernel<4><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    case 8: par_crs_kernel<8><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    case 16: par_crs_kernel<16><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
    default: par_crs_kernel<32><<<blocks, 256, 0, s>>>(rp, ci, d, x, y, f.m); break;
  }
  return check_launch("spmv_par_crs");
}

// Tile shapes instantiated for the merge engine: (threads, items per thread, variant).
// variant 0 = one tile per CTA, direct loads; 1 = persistent TMA-pipelined.
bool merge_shape_supported(int threads, int ipt, int variant) {
#define SPMV_MERGE_SHAPE(T, I, V) if (threads == T && ipt == I && variant == V) return true;
#include "merge_shapes.inc"
#undef SPMV_MERGE_SHAPE
  return false;
}

int spmv_merge(const Format& f, const double* x, double* y, cudaStream_t s) {
  if (f.merge_tiles == 0) return kOk;
  const int threads = (int)f.merge_threads, ipt = (int)f.merge_ipt, variant = (int)f.merge_variant;
  bool launched = false;
  timing_begin(variant == 1 ? "merge_spmv_tma_kernel" : "merge_spmv_kernel", s);
#define SPMV_MERGE_SHAPE(T, I, V)                                    \
  if (!launched && threads == T && ipt == I && variant == V) {       \
    if (V == 0) launch_merge_direct<T, I, 0>(f, x, y, s);            \
    else if (V == 1) launch_merge_tma<T, I, 2>(f, x, y, s);          \
    else launch_merge_direct<T, I, (V >= 10 ? V - 10 : 0)>(f, x, y, s); \
    launched = true;                                                 \
  }
#include "merge_shapes.inc"
#undef SPMV_MERGE_SHAPE
  timing_end(s);
  if (!launched) {
    g_last_error = "merge tile shape not instantiated";
    return kInvalidArgument;
  }
  note_launch(2);
  merge_fixup_kernel<<<(f.merge_tiles + 255) / 256, 256, 0, s>>>(
      f.find("merge_carry_row")->as<uint32_t>(), f.find("merge_carry_val")->as<double>(), f.merge_tiles, y, f.m);
  return check_launch("spmv_merge");
}

}  // namespace spmvcu
