// kernels.cuh -- host launchers for the conversions and the multiplies.
#pragma once

#include <cstdint>
#include <functional>
#include <mutex>
#include <cuda_runtime.h>

#include "../../include/spmvlab_cuda.h"
#include "format.hpp"
#include "primitives.cuh"

namespace spmvcu {

// merge-CSR tile kernel (spmv_crs.cu): one warp tile of 32 * ipt merge items, ipt picked from
// {32, 16, 8} by matrix size at build time (256 threads per CTA).
constexpr int kMergeThreads = 256;
constexpr int kMergeIpt = 32;
// ParCRS: rows longer than kParLongIters * group width are summed by a whole CTA (a sub-warp group
// would walk them serially -- R-MAT s22 row 0 has ~10^5 nonzeros); those CTAs come first in the grid.
constexpr uint32_t kParLongIters = 32;
// Column panels of the merge engine: one panel per kPanelXBytes of x, at most kAutoMergePanels by
// default (SPMVLAB_MERGE_PANELS forces up to kMaxMergePanels); the B200 L2 is 126 MB, so x up to
// 96 MB runs unpanelled (R-MAT s22: 33.5 MB).  B200 sweep (us per multiply, K = 1/2/3/4/6/8):
// cfg3 1012/710/741/792/907/1025, cfg4 834/685/748/831/1016/1117, cfg5 6153/5412/5388/5447/5576/
// 5762 -- every panel pays its rows again, so beyond 2-3 panels the x locality no longer pays.
constexpr int kMaxMergePanels = 16;
constexpr int kAutoMergePanels = 3;
constexpr uint64_t kPanelXBytes = 96ull << 20;
bool merge_shape_supported(int threads, int ipt);
// Hot-x plan of the merge engine (build_hot_columns, convert_crs.cu): at most kHotMaxSlots x
// entries (96 KB of shared memory per SM, beside 16 KB of row maps: more shared memory starves the
// L1 the gathers need in flight) for the columns referenced at least kHotMinRefs times (sampled
// counts), kept when they cover at least kHotMinShare of the nonzeros; the persistent tile kernel
// then runs kHotTilesPerWarp tiles per resident warp (equal merge-path shares).
constexpr uint32_t kHotMaxSlots = 12288;
constexpr uint32_t kHotMinRefs = 32;
constexpr double kHotMinShare = 0.10;
constexpr uint32_t kHotTilesPerWarp = 4;
constexpr int kHotWarps = 32;  // warps of the persistent hot-x CTA (one per SM)
// (adopt: build the plan; always: the column-skew flag merge_x_noalloc)
int build_hot_columns(Format& f, Arena& ar, bool adopt);

// ---- conversions (COO -> format); each returns a Status
int build_crs(Format& f, const spmvlab_cuda_coo& a, Arena& ar);
int build_merge_plan(Format& f, Arena& ar);
int build_csb(Format& f, const spmvlab_cuda_coo& a, unsigned log2_beta, bool hilbert, uint64_t split_threshold, Arena& ar);
int build_mergeb(Format& f, const spmvlab_cuda_coo& a, unsigned log2_beta, bool hilbert, Arena& ar);
int build_bcoh(Format& f, const spmvlab_cuda_coo& a, unsigned log2_beta, unsigned p, Arena& ar);

// Extra destinations of every finished y row (the fused multi-GPU exchange): row r is also stored
// to p[i][off + r] for i < n -- peers' x buffers mapped through CUDA IPC, written over NVLink.
constexpr unsigned kMaxRowDest = 8;
struct RowDest {
  double* p[kMaxRowDest];
  unsigned n;
  uint64_t off;
};
// SCATTER = false compiles to the plain store (the destination list is then never touched, so the
// kernels keep their register / stack budget); kernels take the list as __grid_constant__.
// LAST = false: the value is a column panel's partial sum that the next panel reads back, so it
// is stored with the default L2 policy; the final y is written once and leaves with evict-first
// (keeps the L2 for x: cfg3 / cfg4, x ~ L2 size: -2..3 %).
// (evict-first for the intermediate panels too measured the same at cfg3-5: 704 / 662 / 5468 us)
template <bool SCATTER, bool LAST = true>
__device__ __forceinline__ void put_row(double* y, const RowDest& d, uint32_t r, double v) {
  if constexpr (LAST) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(y + r), "d"(v), "l"(pol) : "memory");
  } else {
    y[r] = v;
  }
  if constexpr (SCATTER)
    for (unsigned i = 0; i < d.n; ++i) d.p[i][d.off + r] = v;
}

// ---- multiplies (stream-ordered; y fully overwritten)
int spmv_seq_crs(const Format& f, const double* x, double* y, cudaStream_t s);
int spmv_par_crs(const Format& f, const double* x, double* y, cudaStream_t s);
int spmv_merge(const Format& f, const double* x, double* y, cudaStream_t s, const RowDest* dest = nullptr);
int spmv_blocked(const Format& f, const double* x, double* y, cudaStream_t s);

// ---- iterated multiply (iterate.cu): x <- A x, `iters` times, with optional norms / rescaling
using SpmvFn = std::function<int(const double* x, double* y, cudaStream_t s)>;
// merge_engine: the multiply is the merge engine on this (CRS) format, so a hot-x plan may run the
// loop's norms inside the multiply (spmv_merge_norms)
int iterate(const Format& f, const SpmvFn& multiply, double* x, double* work, uint32_t iters, int flags,
            double* norms, cudaStream_t s, bool merge_engine = false);

// Device state of the loop (iterate.cu; the fused merge epilogue in spmv_crs.cu updates it too).
constexpr unsigned kRedBlocks = 8 * kNumSMs;
struct IterScratch {
  double partial[2 * kRedBlocks];
  double pair[2];    // (residual, mass) of the current iteration when the caller keeps no norms
  double scale;      // s_k: x_k = scale * stored vector
  unsigned ticket;   // CTAs finished in the current reduction
  unsigned iter;     // iteration index (selects norms + 2 * iter)
  double cpart[kNumSMs];      // per-CTA mass of the fused merge kernel
  double pscale;              // fused loop: factor on the next multiply's products (drift correction)
};
// One rescaled iteration without norms, y = A u with the mass fused into the merge engine's hot-x
// plan (tile kernel: products summed per CTA; carry fix-up: its last block sums them in a fixed
// order and updates the scale as iter_pass_kernel does).  kInvalidArgument without a hot-x plan.
bool merge_norms_supported(const Format& f);
int spmv_merge_norms(const Format& f, const double* u, double* y, cudaStream_t s, IterScratch* sc);

// ---- primitives
int merge_path_search(const uint32_t* a, uint64_t a_len, const uint32_t* b, uint64_t b_len, const uint64_t* diags,
                      uint64_t count, uint64_t* out_i, cudaStream_t s);
int curve_keys(int kind, const uint32_t* rows, const uint32_t* cols, uint64_t count, unsigned level,
               uint64_t* keys, cudaStream_t s);
int validate_coo(const spmvlab_cuda_coo& a, Arena& ar);
int row_prefix(const spmvlab_cuda_coo& a, uint32_t* prefix, Arena& ar);
int cache_read(const char* path, spmvlab_cuda_coo* a, cudaStream_t s);
int cache_info(const char* path, uint32_t* m, uint32_t* n, uint64_t* nnz);
int cache_write(const char* path, const spmvlab_cuda_coo& a, cudaStream_t s);
int mm_read_host(const char* path, spmvlab_cuda_host_coo* out, spmvlab_cuda_mm_header* header);
int mm_read_device(const char* path, spmvlab_cuda_coo* a, spmvlab_cuda_mm_header* header, cudaStream_t s);
int load_matrix(const char* path, spmvlab_cuda_coo* a, cudaStream_t s);
int crs_to_icrs(const Format& f, spmvlab_cuda_bicrs* out, cudaStream_t s);
int triplet_to_bicrs(const spmvlab_cuda_coo& a, const uint32_t* order, spmvlab_cuda_bicrs* out, cudaStream_t s);
int bicrs_decode_all(const spmvlab_cuda_bicrs& b, uint32_t* rows, uint32_t* cols, uint64_t* stats, cudaStream_t s);
int bicrs_spmv(const spmvlab_cuda_bicrs& b, const double* x, double* y, uint64_t* stats, cudaStream_t s);
int format_to_triplet(const Format& f, uint32_t* rows, uint32_t* cols, double* vals, cudaStream_t s);
int csb_work_items(const Format& f, uint64_t split_threshold, spmvlab_cuda_csb_item* items, uint64_t capacity,
                   uint64_t* count, cudaStream_t s);

// ---- instrumentation: launch counter and dominant-kernel event brackets (capi.cu)
void note_launch(unsigned n = 1);
void timing_begin(const char* kernel, cudaStream_t s);  // no-op unless enabled
void timing_end(cudaStream_t s);
bool timing_enable(bool on);  // returns the previous state (graph capture suspends the brackets)

inline unsigned grid_for(uint64_t n, unsigned threads, unsigned max_blocks = kNumSMs * 16) {
  uint64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (unsigned)(b < max_blocks ? b : max_blocks);
}

}  // namespace spmvcu
