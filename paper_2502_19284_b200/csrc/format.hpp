// format.hpp -- the device-resident format object behind the C ABI (include/spmvlab_cuda.h).
//
// A format is a list of named device arrays.  The first `nstorage` arrays are exactly the arrays
// of the reference's storage_report() for that format (inc/storage.hpp:62-123), with identical
// element widths and lengths, so storage_report() byte counts match the reference.  BCOH bands are
// concatenated end to end; per-band slices are delimited by the auxiliary off_* tables.
// Everything a multiply needs beyond the storage arrays (merge-path tile coordinates, carry slots,
// block work queues) is built with the format, so the timed multiply allocates nothing.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

struct DevArray {
  std::string name;
  void* ptr = nullptr;
  uint64_t bytes = 0;   // logical bytes (reported)
  uint32_t esz = 0;
  template <typename T>
  T* as() const { return static_cast<T*>(ptr); }
  uint64_t count() const { return esz ? bytes / esz : 0; }
};

struct spmvlab_cuda_format {
  int alg = 0;
  uint32_t m = 0, n = 0;
  uint64_t nnz = 0;
  uint32_t log2_beta = 0, block_rows = 0, block_cols = 0;
  uint32_t element_level = 0, block_level = 0, bands = 0;
  int nstorage = 0;
  std::vector<DevArray> arrays;

  // ---- merge-path plan (CRS formats), spmv_parallel.hpp:82-86 at tile granularity
  uint32_t merge_tiles = 0;
  uint32_t merge_threads = 256, merge_ipt = 32;  // warp tile = 32 * ipt merge items
  // column panels (merge engine, x larger than the L2): panel k = columns [k*W, (k+1)*W), its
  // tiles at merge_tile_row/nnz[panel_tile_off[k] + k ...], carries at [panel_tile_off[k] ...].
  // Panel 0 walks all m rows (it stores y); a panel k >= 1 with entries in at most half of the
  // rows is doubly compressed: panel_nrows[k] rows (ids at merge_panel_rows[panel_rows_off[k] ...])
  // whose row pointer starts at merge_panel_row_ptr[panel_rp_off[k]]; the others keep a full
  // pointer there (panel_rows_off[k] = ~0).
  uint32_t merge_panels = 1, merge_panel_width = 0;
  std::vector<uint32_t> panel_tile_off{0, 0};
  std::vector<uint32_t> panel_nrows{0}, panel_rp_off{0}, panel_rows_off{0};
  uint64_t merge_panel_row_visits = 0;  // rows with entries, summed over panels >= 1
  std::vector<uint32_t> merge_panel_cuts;  // panel k = columns [cuts[k], cuts[k+1])
  // hot-x plan (one panel only): merge_hot x entries copied to shared memory per SM; their column
  // indices in the plan copy "merge_hot_col" carry 0x80000000 | slot, "merge_hot_cols" lists them
  uint32_t merge_hot = 0;
  bool merge_persist = false;    // persistent 8-wide tile kernel (always with a hot-x plan)
  bool merge_x_noalloc = false;  // no column skew: the tile kernels gather x without L1 allocation
  double merge_hot_share = 0.0;  // share of the nonzeros whose x comes from the copy

  // ---- ParCRS launch shape
  uint32_t par_group = 32;
  uint32_t par_long = 0;  // rows with > par_lim nonzeros ("par_long_rows", one CTA each)
  uint32_t par_lim = 0xFFFFFFFFu;

  // ---- blocked plan (CSB / MergeB / BCOH): work items = (element range, y window)
  uint32_t work_items = 0;
  bool needs_zero_y = false;
  // column panels of the chunk schedule (x larger than the L2): chunks run panel by panel
  // ("chunk_order" / the window items), so one panel's x window stays L2-resident
  uint32_t blk_panels = 1;
  // deterministic build (blocked formats): whole-block-row window items, the bucketed window kernel
  bool deterministic = false;

  // ---- per-stream multiply scratch (merge carries), so one immutable format can serve
  // concurrent multiplies on different streams / host threads (inc/engine.hpp ownership rules).
  struct Scratch {
    uint32_t* carry_row = nullptr;
    double* carry_val = nullptr;
  };
  mutable std::mutex scratch_mu;
  mutable std::map<cudaStream_t, Scratch> scratch;
  const Scratch* stream_scratch(cudaStream_t s) const;  // nullptr on allocation failure

  ~spmvlab_cuda_format();
  DevArray* find(const std::string& name);
  const DevArray* find(const std::string& name) const;
  // Allocates a named device array (16-byte padded); returns nullptr on failure.
  void* add(const std::string& name, uint64_t count, uint32_t esz, cudaStream_t s);
  void set_count(const std::string& name, uint64_t count);
  void drop(const std::string& name);  // frees and forgets an array (no-op if absent)
};

namespace spmvcu {
using Format = spmvlab_cuda_format;
}
