// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference headers (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile directly against /root/reference/proj/include (nothing is copied)
// into oracle/_ref/libspmvref.so.  It lets the tests pin the C restatement (spmv_oracle.c)
// against the reference itself, lets tests/golden/make_golden.py record golden vectors, and is
// bench.py --impl reference's CPU arm (the reference's own engines, multithreaded).
//
// Formats are exported with the same named-array layout as orc_format (spmv_oracle.h): the
// storage_report arrays first (inc/storage.hpp:62-123), BCOH bands concatenated with off_* tables.
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "spmv_oracle.h"
#include <fstream>

#include "spmvlab/bench.hpp"
#include "spmvlab/engine.hpp"
#include "spmvlab/io.hpp"

using namespace spmvlab;

namespace {

thread_local std::string g_err;

int code_of(const Error& e) { return static_cast<int>(e.kind()) + 1; }

template <typename T>
void put(orc_format* f, const char* name, const std::vector<T>& v) {
  orc_array* a = &f->arrays[f->narrays++];
  std::strncpy(a->name, name, sizeof(a->name) - 1);
  a->elem_size = sizeof(T);
  a->bytes = v.size() * sizeof(T);
  a->data = std::malloc(a->bytes ? a->bytes : 1);
  if (a->bytes) std::memcpy(a->data, v.data(), a->bytes);
}

struct Handle {
  Algorithm alg;
  BuiltFormat fmt;
};

TripletMatrix make_triplet(uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows,
                           const uint32_t* cols, const double* vals) {
  TripletMatrix a;
  a.m = m;
  a.n = n;
  a.row_ind.assign(rows, rows + nnz);
  a.col_ind.assign(cols, cols + nnz);
  a.data.assign(vals, vals + nnz);
  return a;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_build(int alg, uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows,
              const uint32_t* cols, const double* vals, unsigned threads, uint64_t l2_bytes,
              unsigned build_threads, void** out) {
  try {
    auto a = make_triplet(m, n, nnz, rows, cols, vals);
    EngineOptions opt{l2_bytes, 0, build_threads};
    auto h = std::make_unique<Handle>(
        Handle{static_cast<Algorithm>(alg), build_format(static_cast<Algorithm>(alg), a, threads, opt)});
    *out = h.release();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

// The reference's per-format builders with an explicit block size (csb.hpp:51, mergeb.hpp:50,
// bcoh.hpp:194); threads = band count p for BCOH.
int ref_build_beta(int alg, uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows, const uint32_t* cols,
                   const double* vals, unsigned log2_beta, unsigned threads, void** out) {
  try {
    auto a = make_triplet(m, n, nnz, rows, cols, vals);
    const BlockSize bs = make_block_size(log2_beta);
    const auto A = static_cast<Algorithm>(alg);
    BuiltFormat f;
    switch (A) {
      case Algorithm::Csb: f = build_csb(a, bs, CurveKind::ZMorton, 1); break;
      case Algorithm::Csbh: f = build_csb(a, bs, CurveKind::Hilbert, 1); break;
      case Algorithm::MergeB: f = build_mergeb(a, bs, false, 1); break;
      case Algorithm::MergeBH: f = build_mergeb(a, bs, true, 1); break;
      case Algorithm::Bcoh: f = build_bcoh(a, bs, threads, bcoh_variant, 1); break;
      case Algorithm::Bcohc: f = build_bcoh(a, bs, threads, bcohc_variant, 1); break;
      case Algorithm::Bcohch: f = build_bcoh(a, bs, threads, bcohch_variant, 1); break;
      case Algorithm::Bcohchp: f = build_bcoh(a, bs, threads, bcohchp_variant, 1); break;
      default: g_err = "no block size for CRS"; return 2;
    }
    *out = new Handle{A, std::move(f)};
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

void ref_free(void* h) { delete static_cast<Handle*>(h); }

int ref_run(void* hv, int alg, const double* x, uint64_t x_len, double* y, uint64_t y_len,
            unsigned p, uint64_t split_threshold) {
  try {
    auto* h = static_cast<Handle*>(hv);
    DenseVector xv(x, x + x_len), yv(y_len, 0.0);
    EngineOptions opt{default_l2_bytes, split_threshold, 1};
    run_spmv(static_cast<Algorithm>(alg), h->fmt, xv, yv, p, opt);
    std::memcpy(y, yv.data(), y_len * sizeof(double));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

// Times `reps` multiplies after `warmup` (min and total seconds), on resident std::vectors, i.e.
// exactly the reference's min_time_of protocol (inc/bench.hpp:98-110).
int ref_time_spmv(void* hv, int alg, const double* x, uint64_t x_len, uint64_t y_len, unsigned p,
                  unsigned reps, unsigned warmup, double* min_s, double* total_s) {
  try {
    auto* h = static_cast<Handle*>(hv);
    DenseVector xv(x, x + x_len), yv(y_len, 0.0);
    EngineOptions opt{};
    for (unsigned w = 0; w < warmup; ++w) run_spmv(static_cast<Algorithm>(alg), h->fmt, xv, yv, p, opt);
    double best = 1e300, tot = 0;
    for (unsigned r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      run_spmv(static_cast<Algorithm>(alg), h->fmt, xv, yv, p, opt);
      auto t1 = std::chrono::steady_clock::now();
      const double s = std::chrono::duration<double>(t1 - t0).count();
      best = s < best ? s : best;
      tot += s;
    }
    *min_s = best;
    *total_s = tot;
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// Exports the built format as an orc_format (named arrays).
int ref_export(void* hv, orc_format** out) {
  auto* h = static_cast<Handle*>(hv);
  auto* f = static_cast<orc_format*>(std::calloc(1, sizeof(orc_format)));
  f->alg = static_cast<int>(h->alg);
  if (auto* c = std::get_if<CrsMatrix>(&h->fmt)) {
    f->m = c->m; f->n = c->n; f->nnz = c->nnz();
    put(f, "row_ptr", c->row_ptr); put(f, "col_ind", c->col_ind); put(f, "data", c->data);
    f->nstorage = 3;
  } else if (auto* c = std::get_if<CsbMatrix>(&h->fmt)) {
    f->m = c->m; f->n = c->n; f->nnz = c->nnz();
    f->log2_beta = c->beta.log2_beta; f->block_rows = c->block_rows; f->block_cols = c->block_cols;
    put(f, "blk_ptr", c->blk_ptr); put(f, "packed", c->packed); put(f, "data", c->data);
    f->nstorage = 3;
  } else if (auto* c = std::get_if<MergeBlockMatrix>(&h->fmt)) {
    f->m = c->m; f->n = c->n; f->nnz = c->nnz();
    f->log2_beta = c->beta.log2_beta; f->block_rows = c->block_rows; f->block_cols = c->block_cols;
    put(f, "blk_row_ptr", c->blk_row_ptr); put(f, "blk_col_ind", c->blk_col_ind);
    put(f, "blk_data_ptr", c->blk_data_ptr); put(f, "packed", c->packed); put(f, "data", c->data);
    f->nstorage = 5;
  } else {
    const auto& bm = std::get<BcohMatrix>(h->fmt);
    f->m = bm.m; f->n = bm.n; f->nnz = bm.nnz();
    f->log2_beta = bm.beta.log2_beta; f->block_rows = bm.block_rows; f->block_cols = bm.block_cols;
    f->element_level = bm.element_level; f->block_level = bm.block_level;
    f->bands = static_cast<uint32_t>(bm.bands.size());
    std::vector<uint32_t> block_nnz, blk_ptr, packed, bfr, brc, bfbr, bbrc;
    std::vector<int16_t> rjb, cjb;
    std::vector<uint16_t> col_inc, row_jump;
    std::vector<double> data;
    std::vector<uint64_t> oe, ob, orjb, obp, orj;
    for (const auto& b : bm.bands) {
      oe.push_back(data.size()); ob.push_back(block_nnz.size()); orjb.push_back(rjb.size());
      obp.push_back(blk_ptr.size()); orj.push_back(row_jump.size());
      block_nnz.insert(block_nnz.end(), b.block_nnz.begin(), b.block_nnz.end());
      rjb.insert(rjb.end(), b.row_jump_block.begin(), b.row_jump_block.end());
      cjb.insert(cjb.end(), b.col_jump_block.begin(), b.col_jump_block.end());
      blk_ptr.insert(blk_ptr.end(), b.blk_ptr.begin(), b.blk_ptr.end());
      col_inc.insert(col_inc.end(), b.col_inc.begin(), b.col_inc.end());
      row_jump.insert(row_jump.end(), b.row_jump.begin(), b.row_jump.end());
      packed.insert(packed.end(), b.packed.begin(), b.packed.end());
      data.insert(data.end(), b.data.begin(), b.data.end());
      bfr.push_back(b.first_row); brc.push_back(b.row_count);
      bfbr.push_back(b.first_block_row); bbrc.push_back(b.block_row_count);
    }
    oe.push_back(data.size()); ob.push_back(block_nnz.size()); orjb.push_back(rjb.size());
    obp.push_back(blk_ptr.size()); orj.push_back(row_jump.size());
    put(f, "block_nnz", block_nnz); put(f, "row_jump_block", rjb); put(f, "col_jump_block", cjb);
    put(f, "blk_ptr", blk_ptr); put(f, "col_inc", col_inc); put(f, "row_jump", row_jump);
    put(f, "packed", packed); put(f, "data", data);
    f->nstorage = 8;
    put(f, "band_first_row", bfr); put(f, "band_row_count", brc);
    put(f, "band_first_block_row", bfbr); put(f, "band_block_row_count", bbrc);
    put(f, "off_elem", oe); put(f, "off_block", ob); put(f, "off_row_jump_block", orjb);
    put(f, "off_blk_ptr", obp); put(f, "off_row_jump", orj);
  }
  // storage_report totals are checked against these arrays by the tests.
  *out = f;
  return 0;
}

void ref_free_export(orc_format* f) {
  if (!f) return;
  for (int i = 0; i < f->narrays; ++i) std::free(f->arrays[i].data);
  std::free(f);
}

uint64_t ref_storage_total(void* hv) {
  return storage_report(static_cast<Handle*>(hv)->fmt).total();
}

// --- SPMVLAB1 cache (inc/cache_io.hpp:58-91) --------------------------------------------------
int ref_cache_write(const char* path, uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows,
                    const uint32_t* cols, const double* vals) {
  try {
    auto a = make_triplet(m, n, nnz, rows, cols, vals);
    save_cache(a, path);
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// Reads a cache; on success *nnz_out and the malloc'ed arrays are returned (free with ref_free_buf).
int ref_cache_read(const char* path, uint32_t* m, uint32_t* n, uint64_t* nnz_out, uint32_t** rows,
                   uint32_t** cols, double** vals) {
  try {
    std::ifstream in(path, std::ios::binary);
    require(in.is_open(), ErrorKind::IoError, std::string("cannot open ") + path);
    TripletMatrix a = cache_read(in);
    *m = a.m;
    *n = a.n;
    *nnz_out = a.data.size();
    *rows = static_cast<uint32_t*>(std::malloc(4 * (a.data.size() + 1)));
    *cols = static_cast<uint32_t*>(std::malloc(4 * (a.data.size() + 1)));
    *vals = static_cast<double*>(std::malloc(8 * (a.data.size() + 1)));
    std::memcpy(*rows, a.row_ind.data(), 4 * a.data.size());
    std::memcpy(*cols, a.col_ind.data(), 4 * a.data.size());
    std::memcpy(*vals, a.data.data(), 8 * a.data.size());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  }
}

void ref_free_buf(void* p) { std::free(p); }

// --- primitives (for golden vectors) ---------------------------------------------------------
unsigned ref_select_block_size(uint64_t n, unsigned cap, uint64_t l2) {
  return select_block_size(n, cap, l2).log2_beta;
}
uint64_t ref_morton(uint32_t r, uint32_t c, unsigned level) { return morton_encode(r, c, level).value; }
uint64_t ref_hilbert(uint32_t r, uint32_t c, unsigned level) { return hilbert_encode(r, c, level).value; }
void ref_diagonal_search(const uint32_t* a, uint64_t a_len, const uint32_t* b, uint64_t b_len,
                         uint64_t diag, uint64_t* i, uint64_t* j) {
  auto pt = diagonal_search(std::span<const index_t>(a, a_len), std::span<const index_t>(b, b_len), diag);
  *i = pt.i;
  *j = pt.j;
}
int ref_partition_rows_by_nnz(const uint32_t* prefix, uint32_t m, unsigned p, unsigned lb,
                              uint32_t* bounds) {
  try {
    auto v = partition_rows_by_nnz(std::span<const index_t>(prefix, m + 1), p, make_block_size(lb));
    std::memcpy(bounds, v.data(), v.size() * sizeof(uint32_t));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  }
}
void ref_verification_input(uint32_t n, uint64_t seed, double* x) {
  auto v = verification_input(n, seed);
  std::memcpy(x, v.data(), n * sizeof(double));
}
unsigned ref_hardware_threads() { return hardware_threads(); }

// The reference's *_to_triplet of a built format (crs.hpp:94, csb.hpp:103, mergeb.hpp:110,
// bcoh.hpp:379): nnz coordinates and values in its output order.
int ref_to_triplet(void* hv, uint32_t* rows, uint32_t* cols, double* vals) {
  try {
    auto* h = static_cast<Handle*>(hv);
    TripletMatrix t;
    if (auto* c = std::get_if<CrsMatrix>(&h->fmt)) t = crs_to_triplet(*c);
    else if (auto* c = std::get_if<CsbMatrix>(&h->fmt)) t = csb_to_triplet(*c);
    else if (auto* c = std::get_if<MergeBlockMatrix>(&h->fmt)) t = mergeb_to_triplet(*c);
    else t = bcoh_to_triplet(std::get<BcohMatrix>(h->fmt));
    std::memcpy(rows, t.row_ind.data(), t.row_ind.size() * sizeof(uint32_t));
    std::memcpy(cols, t.col_ind.data(), t.col_ind.size() * sizeof(uint32_t));
    std::memcpy(vals, t.data.data(), t.data.size() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// The reference's own quadrant leaves (detail::split_block_range, spmv_parallel.hpp:178-193) of
// every cell holding more than `threshold` elements of a built CSB format, cells ascending:
// out[3k..3k+2] = (cell, first element, end element).  Returns the leaf count (-1: not CSB;
// -2: capacity too small).
int64_t ref_csb_leaves(void* hv, uint64_t threshold, uint64_t* out, uint64_t capacity) {
  auto* h = static_cast<Handle*>(hv);
  const auto* a = std::get_if<CsbMatrix>(&h->fmt);
  if (!a) return -1;
  uint64_t k = 0;
  const uint64_t cells = static_cast<uint64_t>(a->block_rows) * a->block_cols;
  std::vector<std::pair<std::size_t, std::size_t>> leaves;
  for (uint64_t cell = 0; cell < cells; ++cell) {
    if (a->blk_ptr[cell + 1] - a->blk_ptr[cell] <= threshold) continue;
    leaves.clear();
    detail::split_block_range(*a, a->blk_ptr[cell], a->blk_ptr[cell + 1], a->beta.beta, {},
                              threshold, leaves);
    for (const auto& [lo, hi] : leaves) {
      if (k >= capacity) return -2;
      out[3 * k] = cell;
      out[3 * k + 1] = lo;
      out[3 * k + 2] = hi;
      ++k;
    }
  }
  return static_cast<int64_t>(k);
}

// The reference's own measurement protocol (inc/bench.hpp:239-329), unmodified: kind 0 =
// bench_spmv (build per (algorithm, threads), verify against spmv_triplet, min of spmv_reps
// multiplies; speedup over the sequential CRS baseline), kind 1 = bench_convert (min of
// convert_reps conversions; ratio to the fastest ParCRS multiply).  One record per (alg, p).
struct ref_bench_record {
  int alg;
  unsigned threads;
  double min_time, speedup, convert_time, convert_ratio, density;
  char status[128];
};

int64_t ref_bench(int kind, uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows, const uint32_t* cols,
                  const double* vals, const int* algs, unsigned nalgs, const unsigned* threads, unsigned nthreads,
                  unsigned spmv_reps, unsigned convert_reps, unsigned warmup, ref_bench_record* out,
                  uint64_t capacity) {
  try {
    auto a = make_triplet(m, n, nnz, rows, cols, vals);
    BenchConfig cfg;
    cfg.algorithms.clear();
    for (unsigned i = 0; i < nalgs; ++i) cfg.algorithms.push_back(static_cast<Algorithm>(algs[i]));
    cfg.threads.assign(threads, threads + nthreads);
    cfg.spmv_reps = spmv_reps;
    cfg.convert_reps = convert_reps;
    cfg.warmup = warmup;
    const auto recs = kind == 0 ? bench_spmv(a, "m", cfg) : bench_convert(a, "m", cfg);
    uint64_t k = 0;
    for (const auto& r : recs) {
      if (k >= capacity) return -2;
      ref_bench_record& o = out[k++];
      o.alg = static_cast<int>(r.algorithm);
      o.threads = r.threads;
      o.min_time = r.min_time;
      o.speedup = r.speedup;
      o.convert_time = r.convert_time ? *r.convert_time : -1.0;
      o.convert_ratio = r.convert_ratio ? *r.convert_ratio : -1.0;
      o.density = r.density;
      std::memset(o.status, 0, sizeof(o.status));
      std::strncpy(o.status, r.status.c_str(), sizeof(o.status) - 1);
    }
    return static_cast<int64_t>(k);
  } catch (const Error& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
