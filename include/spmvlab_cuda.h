/*
 * spmvlab_cuda.h -- C ABI of the B200-native (sm_100a) SpMV hot path.
 *
 * This is the drop-in boundary for the reference library's algorithm interface
 * (/root/reference/proj/include/spmvlab/engine.hpp).  Each entry point names the reference
 * function it replaces.  Plain pointers and sizes only; all matrix / vector pointers are DEVICE
 * pointers unless the name says _host.  `stream` is a cudaStream_t passed as void* (NULL = the
 * legacy default stream).  Calls are stream-ordered; the C++ wrapper in
 * include/spmvlab_cuda/engine.hpp synchronises to give the reference's synchronous semantics.
 *
 * Return codes: 0 = ok; 1 + spmvlab::ErrorKind ordinal (inc/types.hpp:47-62), i.e.
 *   1 DimensionMismatch, 2 InvalidArgument, 3 CorruptFormat, 4 Overflow, 9 IndexOutOfRange,
 *   10 DuplicateEntry; >= 100 CUDA / allocation faults.  spmvlab_cuda_last_error() describes the
 *   last failure on the calling thread.
 *
 * Algorithm ordinals follow inc/engine.hpp:30-42:
 *   0 crs, 1 parcrs, 2 merge, 3 csb, 4 csbh, 5 bcoh, 6 bcohc, 7 bcohch, 8 bcohchp, 9 mergeb,
 *   10 mergebh.
 */
#ifndef SPMVLAB_CUDA_H
#define SPMVLAB_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPMVLAB_CUDA_ABI_VERSION 3

/* Opaque, device-resident, immutable format (a BuiltFormat, inc/engine.hpp:82). */
typedef struct spmvlab_cuda_format spmvlab_cuda_format;

/* TripletMatrix view (inc/triplet.hpp:30-38), device pointers, u32 indices, f64 values. */
typedef struct {
  uint32_t m;
  uint32_t n;
  uint64_t nnz;
  const uint32_t* row_ind;
  const uint32_t* col_ind;
  const double* data;
} spmvlab_cuda_coo;

/* EngineOptions (inc/engine.hpp:75-79). */
typedef struct {
  uint64_t l2_bytes;        /* default 512 KiB (inc/block_size.hpp:39) */
  uint64_t split_threshold; /* 0 = 2*beta (inc/spmv_parallel.hpp:205-207) */
  uint32_t build_threads;   /* accepted for interface parity; the GPU build ignores it */
  uint32_t deterministic;   /* build option, blocked formats (3-10): bitwise-reproducible y -- every
                               block row owned by one CTA that adds into its rows in a fixed order
                               (the reference's exclusive rows, inc/spmv_parallel.hpp:311-350);
                               slower than the default atomics.  The CRS engines always are. */
} spmvlab_cuda_options;

/* StorageArray (inc/storage.hpp:32-36). */
typedef struct {
  char name[32];
  uint64_t bytes;
} spmvlab_cuda_storage_array;

typedef struct {
  int alg;
  uint32_t m, n;
  uint64_t nnz;
  uint32_t log2_beta, block_rows, block_cols;
  uint32_t element_level, block_level, bands;
  uint32_t merge_tiles, work_items;
  uint32_t merge_ipt, merge_panels; /* merge-CSR warp tile = 32 * merge_ipt items; column panels */
  uint64_t merge_panel_row_visits;  /* rows with entries, summed over panels >= 1 (each re-reads y) */
  uint32_t merge_hot_slots;         /* merge-CSR hot-x plan: x entries kept in shared memory (0: none) */
  double merge_hot_share;           /* share of the nonzeros whose x is read from that copy */
} spmvlab_cuda_format_info;

int spmvlab_cuda_abi_version(void);
const char* spmvlab_cuda_last_error(void);

/* Returns the free blocks the library keeps in the device's stream-ordered pool (conversion scratch
 * is kept between builds) to the driver, e.g. before another allocator needs the memory.  No
 * reference counterpart (the reference's scratch is std::vector). */
int spmvlab_cuda_release_pool(void);

/* build_format(Algorithm, const TripletMatrix&, threads, EngineOptions)  -- inc/engine.hpp:96-122.
 * `threads` is the BCOH band count p (inc/engine.hpp:108-115), ignored by the other formats. */
int spmvlab_cuda_build_format(int alg, const spmvlab_cuda_coo* a, unsigned threads,
                              const spmvlab_cuda_options* opt, spmvlab_cuda_format** out,
                              void* stream);

/* The per-format builders with an explicit block size beta = 2^log2_beta:
 * build_csb(a, beta, ZMorton|Hilbert) (inc/csb.hpp:51-57) for algorithms 3/4,
 * build_mergeb(a, beta, hilbert_inside) (inc/mergeb.hpp:50-56) for 9/10,
 * build_bcoh(a, beta, p = threads, variant) (inc/bcoh.hpp:194-205) for 5-8.
 * InvalidArgument: a CRS algorithm, beta outside [2, 2^16] ([2, 2^15] for BCOH), p < 1. */
int spmvlab_cuda_build_format_beta(int alg, const spmvlab_cuda_coo* a, unsigned log2_beta, unsigned threads,
                                   spmvlab_cuda_format** out, void* stream);

/* run_spmv(Algorithm, const BuiltFormat&, const DenseVector& x, DenseVector& y, p, opt)
 * -- inc/engine.hpp:126-148.  y (length m) is fully overwritten.  p must be >= 1 and, for BCOH,
 * equal to the band count (inc/spmv_parallel.hpp:339-341). */
int spmvlab_cuda_run_spmv(int alg, const spmvlab_cuda_format* f, const double* x, uint64_t x_len,
                          double* y, uint64_t y_len, unsigned p, const spmvlab_cuda_options* opt,
                          void* stream);

/* Same multiply with HOST x / y (pinned or pageable): H2D x, multiply, D2H y on `stream`, using
 * caller-provided device staging buffers x_dev (n doubles) and y_dev (m doubles). */
int spmvlab_cuda_run_spmv_host(int alg, const spmvlab_cuda_format* f, const double* x_host,
                               uint64_t x_len, double* y_host, uint64_t y_len, unsigned p,
                               const spmvlab_cuda_options* opt, double* x_dev, double* y_dev,
                               void* stream);

/* Iterated multiply x_{k+1} = A x_k (square A), `iters` times: the cfg5 application loop around
 * run_spmv (BASELINE configs[4], "x <- A x for 100 iterations"; the reference has no loop of its
 * own, its caller repeats inc/engine.hpp:126-148).  x (device, n) holds x_0 on entry and x_iters on
 * return; work is a device buffer of n doubles.  With SPMVLAB_ITER_NORMALIZE each iterate is
 * rescaled to unit L1 mass.  If `norms` (device, 2 * iters doubles) is non-NULL, iteration k writes
 * norms[2k] = ||A x_k - x_k||_1 (the residual; = ||x_{k+1} - x_k||_1 without rescaling) and
 * norms[2k+1] = sum_i (A x_k)_i, the mass before any rescale (its drop from the previous mass is the
 * leakage through empty columns), both by deterministic fixed-order reductions.  One pass per
 * iteration after the multiply computes them and (rescaling) writes A x_k back; the rescale itself
 * is deferred to a scalar, x_{k+1} = (stored A x_k) / mass_k, and applied once at the end.  SPMVLAB_ITER_GRAPH captures one iteration pair (x -> work -> x) as a
 * CUDA graph and replays it iters / 2 times (requires a non-default stream). */
#define SPMVLAB_ITER_NORMALIZE 1
#define SPMVLAB_ITER_GRAPH 2
int spmvlab_cuda_iterate(int alg, const spmvlab_cuda_format* f, double* x, double* work, uint32_t iters,
                         unsigned p, int flags, double* norms, void* stream);

/* --- fused multi-GPU exchange (SURVEY.md §8e stretch: the y slices written straight into the
 * peers' x over NVLink instead of a separate all-gather) ------------------------------------- */

/* Exchange buffers: plain device allocations that can be mapped into the other ranks' processes
 * through CUDA IPC.  alloc fills a 64-byte IPC handle; open maps a peer's handle (peer access
 * enabled lazily); close unmaps (opened != 0) or frees. */
int spmvlab_cuda_exchange_alloc(uint64_t bytes, void** dev_ptr, unsigned char ipc_handle[64]);
int spmvlab_cuda_exchange_open(const unsigned char ipc_handle[64], void** dev_ptr);
int spmvlab_cuda_exchange_close(void* dev_ptr, int opened);

/* Merge-CSR multiply (algorithm 2) of a row shard that also stores every finished row r of y into
 * dest[i][row_offset + r] for i < ndest (<= 8; device pointers valid in this process, e.g. the
 * peers' next-x buffers opened above, each dest_len doubles long): the all-gather of the y slices
 * fused into the multiply -- each warp tile copies its finished rows to the peers as one
 * contiguous run when it ends, the carry fix-up the rows it completes.  y (length m) is written as
 * by run_spmv.  InvalidArgument if row_offset + m > dest_len.  Synchronise the ranks before
 * reading the destinations. */
int spmvlab_cuda_run_spmv_scatter(const spmvlab_cuda_format* f, const double* x, uint64_t x_len, double* y,
                                  uint64_t y_len, double* const* dest, unsigned ndest, uint64_t dest_len,
                                  uint64_t row_offset, void* stream);

/* storage_report(const BuiltFormat&) -- inc/engine.hpp:158-160 / inc/storage.hpp:62-123. */
int spmvlab_cuda_storage_report(const spmvlab_cuda_format* f, spmvlab_cuda_storage_array* rows,
                                size_t capacity, size_t* count);

int spmvlab_cuda_get_format_info(const spmvlab_cuda_format* f, spmvlab_cuda_format_info* info);

/* Device pointer + byte count of one named array (storage arrays use the reference's names;
 * BCOH also exposes band_* and off_* tables).  For parity downloads. */
int spmvlab_cuda_format_array(const spmvlab_cuda_format* f, const char* name, const void** dev_ptr,
                              uint64_t* bytes);

/* Synchronous copy of one named array into host memory (capacity in bytes; *bytes = its size). */
int spmvlab_cuda_download_array(const spmvlab_cuda_format* f, const char* name, void* host_dst,
                                uint64_t capacity, uint64_t* bytes);

void spmvlab_cuda_free_format(spmvlab_cuda_format* f);

/* validate(const TripletMatrix&) -- inc/triplet.hpp:42-59 (range + duplicate check on device). */
int spmvlab_cuda_validate(const spmvlab_cuda_coo* a, void* stream);

/* row_counts + row_prefix (inc/triplet.hpp:75-87): prefix (device, m + 1 entries) = exclusive
 * prefix sums of the entries per row.  IndexOutOfRange for a row >= m.  Synchronises `stream`. */
int spmvlab_cuda_row_prefix(const spmvlab_cuda_coo* a, uint32_t* prefix, void* stream);

/* --- SPMVLAB1 binary triplet cache (inc/cache_io.hpp:31-91, inc/io.hpp:29-40) ----------------- */

/* cache_read: tag "SPMVLAB1", m, n, nnz as u64 LE, then nnz u64 row indices, nnz u64 column
 * indices and nnz u64 value bit patterns.  The file is read in large chunks into pinned staging
 * buffers while earlier chunks are copied to the device and narrowed there (indices are cast to
 * the 32-bit index type as the reference does), then the triplet is validated on the device
 * (inc/triplet.hpp:42-59).  If a->row_ind / col_ind / data are non-NULL they are caller-owned
 * device buffers of capacity a->nnz entries (size them with spmvlab_cuda_cache_info); otherwise
 * the library allocates them and they must be released with spmvlab_cuda_free_coo().  Errors:
 * BadMagic, Truncated, Overflow, IndexOutOfRange, DuplicateEntry, IoError, InvalidArgument (buffer
 * too small). */
int spmvlab_cuda_cache_read(const char* path, spmvlab_cuda_coo* a, void* stream);

/* Header of a cache file: m, n, nnz (checks the tag and the dimension limits). */
int spmvlab_cuda_cache_info(const char* path, uint32_t* m, uint32_t* n, uint64_t* nnz);

/* cache_write (inc/cache_io.hpp:58-66) of a device triplet; byte-identical to the reference's. */
int spmvlab_cuda_cache_write(const char* path, const spmvlab_cuda_coo* a, void* stream);

/* Releases the arrays of a triplet returned by spmvlab_cuda_cache_read. */
void spmvlab_cuda_free_coo(spmvlab_cuda_coo* a);

/* --- Matrix Market coordinate text (inc/matrix_market.hpp:94-190) ------------------------------ */

/* MatrixHeader (inc/matrix_market.hpp:35-41): field 0 real, 1 integer, 2 pattern; symmetry
 * 0 general, 1 symmetric; declared_nnz = the size line's entry count (before mirroring). */
typedef struct {
  int field;
  int symmetry;
  uint32_t m, n;
  uint64_t declared_nnz;
} spmvlab_cuda_mm_header;

/* A triplet in HOST memory (malloc'd by the library; release with spmvlab_cuda_free_host_coo). */
typedef struct {
  uint32_t m;
  uint32_t n;
  uint64_t nnz;
  uint32_t* row_ind;
  uint32_t* col_ind;
  double* data;
} spmvlab_cuda_host_coo;

/* read_matrix_market (inc/matrix_market.hpp:94-190): banner checks, 1-based -> 0-based, symmetric
 * off-diagonals mirrored right after their entry, pattern -> 1.0, then validate() -- into device
 * buffers (caller-owned with capacity a->nnz, or library-allocated when a's pointers are NULL:
 * release with spmvlab_cuda_free_coo).  header may be NULL.  Errors: BadHeader, UnsupportedFormat,
 * UnsupportedField, UnsupportedSymmetry, Truncated, ParseError, Overflow, IndexOutOfRange,
 * DuplicateEntry, IoError. */
int spmvlab_cuda_read_matrix_market(const char* path, spmvlab_cuda_coo* a, spmvlab_cuda_mm_header* header,
                                    void* stream);

/* The same parse + validate entirely on the host (no CUDA calls). */
int spmvlab_cuda_read_matrix_market_host(const char* path, spmvlab_cuda_host_coo* out,
                                         spmvlab_cuda_mm_header* header);
void spmvlab_cuda_free_host_coo(spmvlab_cuda_host_coo* a);

/* load_matrix (inc/io.hpp:29-40): SPMVLAB1 cache if the file starts with the magic, else Matrix
 * Market text; device buffers as in spmvlab_cuda_cache_read. */
int spmvlab_cuda_load_matrix(const char* path, spmvlab_cuda_coo* a, void* stream);

/* --- standalone ICRS / BICRS (inc/bicrs.hpp) --------------------------------------------------- */

/* IncrementalRowStorage (bicrs.hpp:33-45) in device memory.  kind 0 = ICRS (u32 increments and
 * row jumps, index_t), kind 1 = BICRS (i64, signed_index_t).  col_inc has nnz + 1 entries. */
typedef struct {
  uint32_t m, n;
  uint64_t nnz;
  int kind;
  void* col_inc;
  void* row_jump;
  uint64_t n_row_jump;
  double* data;
} spmvlab_cuda_bicrs;

/* crs_to_icrs (bicrs.hpp:120-150) from a CRS-family format (algorithms 0-2); library-allocated
 * arrays, release with spmvlab_cuda_free_bicrs.  Bit-identical to the reference. */
int spmvlab_cuda_crs_to_icrs(const spmvlab_cuda_format* crs, spmvlab_cuda_bicrs* out, void* stream);

/* triplet_to_bicrs (bicrs.hpp:154-200) with the elements in `order` (device, a permutation of
 * [0, nnz); otherwise InvalidArgument). */
int spmvlab_cuda_triplet_to_bicrs(const spmvlab_cuda_coo* a, const uint32_t* order, spmvlab_cuda_bicrs* out,
                                  void* stream);

/* spmv_bicrs_seq (bicrs.hpp:98-109): y (length m) fully overwritten; stats_host (2 entries, may be
 * NULL) = ReplayStats {overflow_events, row_jumps_consumed}.  DimensionMismatch, CorruptFormat. */
int spmvlab_cuda_bicrs_spmv(const spmvlab_cuda_bicrs* a, const double* x, uint64_t x_len, double* y,
                            uint64_t y_len, uint64_t* stats_host, void* stream);

/* bicrs_to_triplet (bicrs.hpp:111-118): row and column of every element (device, nnz each); the
 * values are a->data.  CorruptFormat. */
int spmvlab_cuda_bicrs_to_triplet(const spmvlab_cuda_bicrs* a, uint32_t* rows, uint32_t* cols, void* stream);

void spmvlab_cuda_free_bicrs(spmvlab_cuda_bicrs* a);

/* --- format -> triplet ------------------------------------------------------------------------ */

/* crs_to_triplet (crs.hpp:94-105), csb_to_triplet (csb.hpp:103-120), mergeb_to_triplet
 * (mergeb.hpp:110-127), bcoh_to_triplet (bcoh.hpp:379-392) for any built format: the row, column
 * and value (vals may be NULL) of every element in the reference's output order (storage order;
 * BCOH band by band), into device arrays of nnz entries.  Stream-ordered. */
int spmvlab_cuda_format_to_triplet(const spmvlab_cuda_format* f, uint32_t* rows, uint32_t* cols, double* vals,
                                   void* stream);

/* --- CSB work items (inc/spmv_parallel.hpp:167-264) ------------------------------------------ */

/* CsbWorkItem (spmv_parallel.hpp:167-174): cells [cell_begin, cell_end) of block_row clipped to
 * elements [elem_begin, elem_end); temp_slot -1 = the item owns its block row. */
typedef struct {
  uint32_t block_row, cell_begin, cell_end;
  int32_t temp_slot;
  uint64_t elem_begin, elem_end;
} spmvlab_cuda_csb_item;

/* The work-item list spmv_csb builds (spmv_parallel.hpp:202-264: per block row one item, or
 * greedy cell chunks plus the quadrant leaves of split_block_range :178-193 for cells above the
 * threshold), built on the device and bit-identical to the reference's, in the reference's order.
 * Algorithms 3 (csb) and 4 (csbh) only (else InvalidArgument).  split_threshold 0 = 2 * beta.
 * *count receives the list length; items (device, may be NULL to only count) must hold
 * `capacity` >= *count entries, else InvalidArgument.  Synchronises `stream`. */
int spmvlab_cuda_csb_work_items(const spmvlab_cuda_format* f, uint64_t split_threshold,
                                spmvlab_cuda_csb_item* items, uint64_t capacity, uint64_t* count,
                                void* stream);

/* --- primitives, exposed for parity tests ---------------------------------------------------- */

/* select_block_size -- inc/block_size.hpp:47-61 (value_size 8). Host computation. */
unsigned spmvlab_cuda_select_block_size(uint64_t n, unsigned index_bits_cap, uint64_t l2_bytes);

/* partition_rows_by_nnz -- inc/block_size.hpp:73-102.  Host arrays. */
int spmvlab_cuda_partition_rows_by_nnz(const uint32_t* prefix_host, uint32_t m, unsigned p,
                                       unsigned log2_beta, uint32_t* bounds_host);

/* diagonal_search over A = a[0..a_len) and B = b[0..b_len) (b == NULL: B[j] = j, the CRS case)
 * (inc/spmv_parallel.hpp:47-69), for `count` diagonals at once on the device:
 * out_i[k] = i of diags[k] (j = diag - i). */
int spmvlab_cuda_merge_path_search(const uint32_t* a, uint64_t a_len, const uint32_t* b,
                                   uint64_t b_len, const uint64_t* diags, uint64_t count,
                                   uint64_t* out_i, void* stream);

/* Curve keys on device: kind 0 = Z-Morton, 1 = Hilbert (inc/curves.hpp:107-143). */
int spmvlab_cuda_curve_keys(int kind, const uint32_t* rows, const uint32_t* cols, uint64_t count,
                            unsigned level, uint64_t* keys, void* stream);

/* Radix sort of (key, value) pairs by key bits [begin_bit, end_bit), in place, stable. */
int spmvlab_cuda_sort_pairs(uint64_t* keys, uint32_t* values, uint64_t count, int begin_bit,
                            int end_bit, void* stream);

/* Exclusive scan: out[0..n] (out[n] = total). */
int spmvlab_cuda_exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, void* stream);

/* --- instrumentation (benchmark harness only) -------------------------------------------------- */

/* Number of CUDA kernels this library has launched since load. */
uint64_t spmvlab_cuda_launch_count(void);

/* While enabled, the dominant kernel of every multiply is bracketed by CUDA events recorded on
 * the stream it is launched on.  spmvlab_cuda_kernel_time() waits for those events and returns
 * the summed kernel duration (ms), the launch count and the kernel's name, then resets. */
void spmvlab_cuda_kernel_timing(int enable);
int spmvlab_cuda_kernel_time(double* total_ms, uint64_t* launches, char* name, size_t name_cap);

#ifdef __cplusplus
}
#endif
#endif /* SPMVLAB_CUDA_H */
