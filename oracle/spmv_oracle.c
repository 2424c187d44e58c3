/*
 * spmv_oracle.c -- CPU restatement of the spmvlab SpMV hot path.  TEST INFRASTRUCTURE ONLY:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use
 * it, as the checker.  The product path (paper_2502_19284_b200/, libspmvlab_cuda.so) never
 * links or calls it.
 *
 * Citations are relative to /root/reference/proj/include/spmvlab/.  Every sort below is
 * restated as a sort over explicit lexicographic keys (k1, k2, k3, index); the reference sorts a
 * permutation with a comparator over the same tuple, and because the tuples are unique (no
 * duplicate coordinates, triplet.hpp:42-59) both produce the identical order.  Kernels replay the
 * reference loops in the same order, so y is bitwise equal to the reference's for every engine.
 *
 * Parity: pinned against tests/golden/ (made from the reference itself, oracle/_ref) and, where
 * oracle/_ref is built, against the reference on seeded random matrices.
 */
#include "spmv_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAX_DIMENSION (UINT64_C(1) << 31) /* types.hpp:45 */

static unsigned bit_width64(uint64_t v) {
  unsigned w = 0;
  while (v) { ++w; v >>= 1; }
  return w;
}

/* ---------------------------------------------------------------- block size (block_size.hpp) */

/* select_block_size, block_size.hpp:47-61 (value_size = sizeof(double)). */
unsigned orc_select_block_size(uint64_t n, unsigned cap, uint64_t l2_bytes) {
  const unsigned ceil_log2_n = n <= 1 ? 0 : bit_width64(n - 1);
  unsigned lb = 3 + (ceil_log2_n + 1) / 2;
  for (;;) {
    if (lb <= 1) break;
    const uint64_t beta = UINT64_C(1) << lb;
    const int fits = lb <= cap && 2 * beta * 8 <= l2_bytes / 2;
    if (fits) break;
    --lb;
  }
  return lb;
}

static int is_bcoh(int alg) {
  return alg == ORC_BCOH || alg == ORC_BCOHC || alg == ORC_BCOHCH || alg == ORC_BCOHCHP;
}

/* engine_block_size, engine.hpp:84-91: cap 15 for BCOH (bcoh.hpp:59), 16 otherwise (csb.hpp:47). */
unsigned orc_engine_log2_beta(int alg, uint32_t n, uint64_t l2_bytes) {
  return orc_select_block_size(n < 1 ? 1 : n, is_bcoh(alg) ? 15 : 16, l2_bytes);
}

static uint32_t blocks_covering(uint32_t extent, unsigned lb) { /* block_size.hpp:64-66 */
  return (uint32_t)((extent + (UINT32_C(1) << lb) - 1) >> lb);
}

/* partition_rows_by_nnz, block_size.hpp:73-102. */
int orc_partition_rows_by_nnz(const uint32_t* prefix, uint32_t m, unsigned p, unsigned lb,
                              uint32_t* bounds) {
  if (p < 1) return ORC_INVALID_ARGUMENT;
  const uint64_t nnz = prefix[m];
  const uint32_t beta = UINT32_C(1) << lb;
  const uint32_t block_rows = blocks_covering(m, lb);
  for (unsigned k = 0; k <= p; ++k) bounds[k] = m;
  bounds[0] = 0;
  uint32_t prev_cut = 0;
  for (unsigned k = 1; k < p; ++k) {
    const uint64_t target = nnz * k;
    /* lower_bound: first r with prefix[r] * p >= target */
    uint64_t lo = 0, hi = (uint64_t)m + 1;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if ((uint64_t)prefix[mid] * p < target) lo = mid + 1; else hi = mid;
    }
    const uint32_t greedy_row = (uint32_t)lo;
    uint32_t cut = (uint32_t)((greedy_row + beta / 2) >> lb);
    const uint32_t hic = block_rows >= p ? block_rows - (p - k) : block_rows;
    uint32_t loc = prev_cut + 1 < hic ? prev_cut + 1 : hic;
    if (cut < loc) cut = loc;
    if (cut > hic) cut = hic;
    const uint32_t b = cut << lb;
    bounds[k] = b < m ? b : m;
    prev_cut = cut;
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------- curves (curves.hpp) */

/* HilbertOrientation::position / child / cell, curves.hpp:60-103; state bit0 = swapped,
 * bit1 = flipped. */
static unsigned hil_position(unsigned st, unsigned rbit, unsigned cbit) {
  unsigned x = cbit, y = rbit;
  if (st & 2u) { x ^= 1u; y ^= 1u; }
  if (st & 1u) { unsigned t = x; x = y; y = t; }
  return (3u * x) ^ y;
}
static unsigned hil_child(unsigned st, unsigned pos) {
  if (pos == 0) return st ^ 1u;
  if (pos == 3) return st ^ 3u;
  return st;
}
static void hil_cell(unsigned st, unsigned pos, unsigned* rbit, unsigned* cbit) {
  static const unsigned rx[4] = {0u, 0u, 1u, 1u};
  static const unsigned ry[4] = {0u, 1u, 1u, 0u};
  unsigned x = rx[pos], y = ry[pos];
  if (st & 2u) { x ^= 1u; y ^= 1u; }
  if (st & 1u) { unsigned t = x; x = y; y = t; }
  *rbit = y;
  *cbit = x;
}

/* morton_encode, curves.hpp:107-117 */
uint64_t orc_morton_encode(uint32_t row, uint32_t col, unsigned level) {
  uint64_t v = 0;
  for (unsigned b = level; b-- > 0;)
    v = (v << 2) | ((uint64_t)((row >> b) & 1u) << 1) | ((col >> b) & 1u);
  return v;
}
/* morton_decode, curves.hpp:119-130 */
void orc_morton_decode(uint64_t d, unsigned level, uint32_t* row, uint32_t* col) {
  uint32_t r = 0, c = 0;
  for (unsigned b = 0; b < level; ++b) {
    c |= (uint32_t)((d >> (2 * b)) & 1u) << b;
    r |= (uint32_t)((d >> (2 * b + 1)) & 1u) << b;
  }
  *row = r;
  *col = c;
}
/* hilbert_encode, curves.hpp:133-143 */
uint64_t orc_hilbert_encode(uint32_t row, uint32_t col, unsigned level) {
  unsigned st = 0;
  uint64_t v = 0;
  for (unsigned b = level; b-- > 0;) {
    const unsigned pos = hil_position(st, (row >> b) & 1u, (col >> b) & 1u);
    v = (v << 2) | pos;
    st = hil_child(st, pos);
  }
  return v;
}
/* hilbert_decode, curves.hpp:145-161 */
void orc_hilbert_decode(uint64_t d, unsigned level, uint32_t* row, uint32_t* col) {
  unsigned st = 0;
  uint32_t r = 0, c = 0;
  for (unsigned b = level; b-- > 0;) {
    const unsigned pos = (unsigned)((d >> (2 * b)) & 3u);
    unsigned rb, cb;
    hil_cell(st, pos, &rb, &cb);
    r |= rb << b;
    c |= cb << b;
    st = hil_child(st, pos);
  }
  *row = r;
  *col = c;
}
/* covering_level, curves.hpp:164-171 */
unsigned orc_covering_level(uint32_t rows, uint32_t cols) {
  uint32_t e = rows > cols ? rows : cols;
  if (e < 1) e = 1;
  return bit_width64((uint64_t)e - 1);
}

/* ---------------------------------------------------------------- merge path (spmv_parallel.hpp) */

/* diagonal_search, spmv_parallel.hpp:47-69.  List A is a[0..a_len); list B is b[0..b_len) or,
 * with b_natural, B[j] = j. */
int orc_diagonal_search(const uint32_t* a, uint64_t a_len, uint64_t b_len, uint64_t diag,
                        int b_natural, const uint32_t* b, uint64_t* i_out, uint64_t* j_out) {
  if (diag > a_len + b_len) return ORC_INVALID_ARGUMENT;
  uint64_t lo = diag > b_len ? diag - b_len : 0;
  uint64_t hi = diag < a_len ? diag : a_len;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;
    int pred;
    const uint64_t j = diag - mid;
    if (j >= b_len) pred = 1;
    else {
      const uint64_t bj = b_natural ? j : b[j];
      pred = !(bj < a[mid - 1]);
    }
    if (pred) lo = mid; else hi = mid - 1;
  }
  *i_out = lo;
  *j_out = diag - lo;
  return ORC_OK;
}

/* ---------------------------------------------------------------- triplet (triplet.hpp) */

/* row_prefix, triplet.hpp:82-87 */
void orc_row_prefix(uint32_t m, uint64_t nnz, const uint32_t* rows, uint32_t* prefix) {
  memset(prefix, 0, sizeof(uint32_t) * ((size_t)m + 1));
  for (uint64_t k = 0; k < nnz; ++k) ++prefix[(size_t)rows[k] + 1];
  for (uint64_t i = 1; i <= m; ++i) prefix[i] += prefix[i - 1];
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* validate, triplet.hpp:42-59 */
int orc_validate(uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows, const uint32_t* cols) {
  if (m > MAX_DIMENSION || n > MAX_DIMENSION) return ORC_OVERFLOW;
  for (uint64_t i = 0; i < nnz; ++i)
    if (rows[i] >= m || cols[i] >= n) return ORC_INDEX_OUT_OF_RANGE;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (nnz ? nnz : 1));
  if (!keys) return ORC_NO_MEMORY;
  for (uint64_t i = 0; i < nnz; ++i) keys[i] = ((uint64_t)rows[i] << 32) | cols[i];
  qsort(keys, nnz, sizeof(uint64_t), cmp_u64);
  int rc = ORC_OK;
  for (uint64_t i = 1; i < nnz; ++i)
    if (keys[i] == keys[i - 1]) { rc = ORC_DUPLICATE_ENTRY; break; }
  free(keys);
  return rc;
}

/* spmv_triplet, triplet.hpp:63-72 */
void orc_spmv_triplet(uint32_t m, uint64_t nnz, const uint32_t* rows, const uint32_t* cols,
                      const double* vals, const double* x, double* y) {
  for (uint32_t i = 0; i < m; ++i) y[i] = 0.0;
  for (uint64_t k = 0; k < nnz; ++k) y[rows[k]] += vals[k] * x[cols[k]];
}

void orc_abs_spmv(uint32_t m, uint64_t nnz, const uint32_t* rows, const uint32_t* cols,
                  const double* vals, const double* x, double* y) {
  for (uint32_t i = 0; i < m; ++i) y[i] = 0.0;
  for (uint64_t k = 0; k < nnz; ++k) {
    const double a = vals[k] < 0 ? -vals[k] : vals[k];
    const double b = x[cols[k]] < 0 ? -x[cols[k]] : x[cols[k]];
    y[rows[k]] += a * b;
  }
}

/* verification_input, bench.hpp:153-161 */
void orc_verification_input(uint32_t n, uint64_t seed, double* x) {
  uint64_t state = seed * UINT64_C(0x9E3779B97F4A7C15) + 1;
  for (uint32_t i = 0; i < n; ++i) {
    state = state * UINT64_C(6364136223846793005) + UINT64_C(1442695040888963407);
    x[i] = 0.5 + (double)(state >> 11) * 0x1.0p-53;
  }
}

/* ---------------------------------------------------------------- SPMVLAB1 cache (cache_io.hpp) */

static int get_u64_le(FILE* f, uint64_t* v) { /* cache_io.hpp:47-54 */
  unsigned char b[8];
  if (fread(b, 1, 8, f) != 8) return ORC_TRUNCATED;
  uint64_t x = 0;
  for (int i = 0; i < 8; ++i) x |= (uint64_t)b[i] << (8 * i);
  *v = x;
  return ORC_OK;
}

static void put_u64_le(FILE* f, uint64_t v) { /* cache_io.hpp:41-45 */
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
  fwrite(b, 1, 8, f);
}

void orc_free(void* p) { free(p); }

/* cache_read, cache_io.hpp:69-91: magic, m, n, nnz, then the three streams; validate(). */
int orc_cache_read(const char* path, uint32_t* m, uint32_t* n, uint64_t* nnz, uint32_t** rows,
                   uint32_t** cols, double** vals) {
  static const char magic[8] = {'S', 'P', 'M', 'V', 'L', 'A', 'B', '1'};
  *rows = NULL;
  *cols = NULL;
  *vals = NULL;
  FILE* f = fopen(path, "rb");
  if (!f) return ORC_IO_ERROR;
  char head[8];
  if (fread(head, 1, 8, f) != 8 || memcmp(head, magic, 8) != 0) { fclose(f); return ORC_BAD_MAGIC; }
  uint64_t mm, nn, cnt;
  if (get_u64_le(f, &mm) || get_u64_le(f, &nn) || get_u64_le(f, &cnt)) { fclose(f); return ORC_TRUNCATED; }
  if (mm > MAX_DIMENSION || nn > MAX_DIMENSION) { fclose(f); return ORC_OVERFLOW; }
  uint32_t* r = (uint32_t*)malloc(4 * (cnt ? cnt : 1));
  uint32_t* c = (uint32_t*)malloc(4 * (cnt ? cnt : 1));
  double* v = (double*)malloc(8 * (cnt ? cnt : 1));
  int rc = ORC_OK;
  uint64_t x;
  for (uint64_t k = 0; k < cnt && !rc; ++k) { rc = get_u64_le(f, &x); r[k] = (uint32_t)x; }
  for (uint64_t k = 0; k < cnt && !rc; ++k) { rc = get_u64_le(f, &x); c[k] = (uint32_t)x; }
  for (uint64_t k = 0; k < cnt && !rc; ++k) { rc = get_u64_le(f, &x); memcpy(&v[k], &x, 8); }
  fclose(f);
  if (!rc) rc = orc_validate((uint32_t)mm, (uint32_t)nn, cnt, r, c);
  if (rc) { free(r); free(c); free(v); return rc; }
  *m = (uint32_t)mm;
  *n = (uint32_t)nn;
  *nnz = cnt;
  *rows = r;
  *cols = c;
  *vals = v;
  return ORC_OK;
}

/* cache_write, cache_io.hpp:58-66 */
int orc_cache_write(const char* path, uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows,
                    const uint32_t* cols, const double* vals) {
  FILE* f = fopen(path, "wb");
  if (!f) return ORC_IO_ERROR;
  fwrite("SPMVLAB1", 1, 8, f);
  put_u64_le(f, m);
  put_u64_le(f, n);
  put_u64_le(f, nnz);
  for (uint64_t k = 0; k < nnz; ++k) put_u64_le(f, rows[k]);
  for (uint64_t k = 0; k < nnz; ++k) put_u64_le(f, cols[k]);
  for (uint64_t k = 0; k < nnz; ++k) {
    uint64_t b;
    memcpy(&b, &vals[k], 8);
    put_u64_le(f, b);
  }
  const int bad = ferror(f);
  fclose(f);
  return bad ? ORC_IO_ERROR : ORC_OK;
}

/* ---------------------------------------------------------------- key sort helper */

typedef struct {
  uint64_t k1, k2, k3;
  uint32_t idx;
} sort_item;

static int cmp_item(const void* a, const void* b) {
  const sort_item* x = (const sort_item*)a;
  const sort_item* y = (const sort_item*)b;
  if (x->k1 != y->k1) return x->k1 < y->k1 ? -1 : 1;
  if (x->k2 != y->k2) return x->k2 < y->k2 ? -1 : 1;
  if (x->k3 != y->k3) return x->k3 < y->k3 ? -1 : 1;
  return 0;
}

/* ---------------------------------------------------------------- format bookkeeping */

static orc_format* new_format(int alg, uint32_t m, uint32_t n, uint32_t nnz) {
  orc_format* f = (orc_format*)calloc(1, sizeof(orc_format));
  if (!f) return NULL;
  f->alg = alg;
  f->m = m;
  f->n = n;
  f->nnz = nnz;
  return f;
}

static void* add_array(orc_format* f, const char* name, uint64_t count, uint32_t esz) {
  orc_array* a = &f->arrays[f->narrays++];
  strncpy(a->name, name, sizeof(a->name) - 1);
  a->elem_size = esz;
  a->bytes = count * esz;
  a->data = calloc(count ? count : 1, esz);
  return a->data;
}

static void shrink_array(orc_format* f, const char* name, uint64_t count) {
  for (int i = 0; i < f->narrays; ++i)
    if (!strcmp(f->arrays[i].name, name)) f->arrays[i].bytes = count * f->arrays[i].elem_size;
}

void orc_free_format(orc_format* f) {
  if (!f) return;
  for (int i = 0; i < f->narrays; ++i) free(f->arrays[i].data);
  free(f);
}

const orc_array* orc_find_array(const orc_format* f, const char* name) {
  for (int i = 0; i < f->narrays; ++i)
    if (!strcmp(f->arrays[i].name, name)) return &f->arrays[i];
  return NULL;
}

#define ARR(f, name, type) ((type*)orc_find_array((f), (name))->data)
#define ARRN(f, name) (orc_find_array((f), (name))->bytes / orc_find_array((f), (name))->elem_size)

/* ---------------------------------------------------------------- CRS (crs.hpp) */

/* triplet_to_crs, crs.hpp:67-91: sort by (row, col); row_ptr = counts + partial_sum; gather. */
static int build_crs(int alg, uint32_t m, uint32_t n, uint32_t nnz, const uint32_t* rows,
                     const uint32_t* cols, const double* vals, orc_format** out) {
  orc_format* f = new_format(alg, m, n, nnz);
  sort_item* it = (sort_item*)malloc(sizeof(sort_item) * (nnz ? nnz : 1));
  for (uint32_t k = 0; k < nnz; ++k) {
    it[k].k1 = rows[k]; it[k].k2 = cols[k]; it[k].k3 = 0; it[k].idx = k;
  }
  qsort(it, nnz, sizeof(sort_item), cmp_item);
  uint32_t* row_ptr = (uint32_t*)add_array(f, "row_ptr", (uint64_t)m + 1, 4);
  uint32_t* col_ind = (uint32_t*)add_array(f, "col_ind", nnz, 4);
  double* data = (double*)add_array(f, "data", nnz, 8);
  f->nstorage = 3;
  for (uint32_t k = 0; k < nnz; ++k) ++row_ptr[(size_t)rows[k] + 1];
  for (uint64_t i = 1; i <= m; ++i) row_ptr[i] += row_ptr[i - 1];
  for (uint32_t k = 0; k < nnz; ++k) {
    col_ind[k] = cols[it[k].idx];
    data[k] = vals[it[k].idx];
  }
  free(it);
  *out = f;
  return ORC_OK;
}

/* ---------------------------------------------------------------- CSB (csb.hpp) */

static uint64_t curve_rank(int hilbert, uint32_t r, uint32_t c, unsigned level) {
  return hilbert ? orc_hilbert_encode(r, c, level) : orc_morton_encode(r, c, level);
}

/* build_csb, csb.hpp:51-100: sort by (br, bc, curve rank in block); blk_ptr over the dense
 * block_rows x block_cols cell grid; packed = in_row << 16 | in_col (packed_index.hpp:29-34). */
static int build_csb(int alg, uint32_t m, uint32_t n, uint32_t nnz, const uint32_t* rows,
                     const uint32_t* cols, const double* vals, unsigned lb, orc_format** out) {
  if ((uint64_t)m > MAX_DIMENSION || (uint64_t)n > MAX_DIMENSION) return ORC_OVERFLOW;
  if (lb < 1 || lb > 16) return ORC_INVALID_ARGUMENT;
  const int hilbert = alg == ORC_CSBH;
  orc_format* f = new_format(alg, m, n, nnz);
  f->log2_beta = lb;
  f->block_rows = blocks_covering(m, lb);
  f->block_cols = blocks_covering(n, lb);
  const uint32_t mask = (UINT32_C(1) << lb) - 1;
  sort_item* it = (sort_item*)malloc(sizeof(sort_item) * (nnz ? nnz : 1));
  for (uint32_t k = 0; k < nnz; ++k) {
    it[k].k1 = rows[k] >> lb;
    it[k].k2 = cols[k] >> lb;
    it[k].k3 = curve_rank(hilbert, rows[k] & mask, cols[k] & mask, lb);
    it[k].idx = k;
  }
  qsort(it, nnz, sizeof(sort_item), cmp_item);
  const uint64_t cells = (uint64_t)f->block_rows * f->block_cols;
  uint32_t* blk_ptr = (uint32_t*)add_array(f, "blk_ptr", cells + 1, 4);
  uint32_t* packed = (uint32_t*)add_array(f, "packed", nnz, 4);
  double* data = (double*)add_array(f, "data", nnz, 8);
  f->nstorage = 3;
  for (uint32_t k = 0; k < nnz; ++k)
    ++blk_ptr[(uint64_t)(rows[k] >> lb) * f->block_cols + (cols[k] >> lb) + 1];
  for (uint64_t c = 1; c <= cells; ++c) blk_ptr[c] += blk_ptr[c - 1];
  for (uint32_t k = 0; k < nnz; ++k) {
    const uint32_t id = it[k].idx;
    packed[k] = ((rows[id] & mask) << 16) | (cols[id] & mask);
    data[k] = vals[id];
  }
  free(it);
  *out = f;
  return ORC_OK;
}

/* ---------------------------------------------------------------- MergeB (mergeb.hpp) */

/* build_mergeb, mergeb.hpp:50-108: sort by (br, bc, in_row, in_col) or (br, bc, Hilbert rank);
 * block runs become a CRS over nonempty blocks. */
static int build_mergeb(int alg, uint32_t m, uint32_t n, uint32_t nnz, const uint32_t* rows,
                        const uint32_t* cols, const double* vals, unsigned lb, orc_format** out) {
  if ((uint64_t)m > MAX_DIMENSION || (uint64_t)n > MAX_DIMENSION) return ORC_OVERFLOW;
  if (lb < 1 || lb > 16) return ORC_INVALID_ARGUMENT;
  const int hilbert = alg == ORC_MERGEBH;
  orc_format* f = new_format(alg, m, n, nnz);
  f->log2_beta = lb;
  f->block_rows = blocks_covering(m, lb);
  f->block_cols = blocks_covering(n, lb);
  const uint32_t mask = (UINT32_C(1) << lb) - 1;
  sort_item* it = (sort_item*)malloc(sizeof(sort_item) * (nnz ? nnz : 1));
  for (uint32_t k = 0; k < nnz; ++k) {
    it[k].k1 = ((uint64_t)(rows[k] >> lb) << 32) | (cols[k] >> lb);
    it[k].k2 = hilbert ? orc_hilbert_encode(rows[k] & mask, cols[k] & mask, lb)
                       : (((uint64_t)(rows[k] & mask) << 32) | (cols[k] & mask));
    it[k].k3 = 0;
    it[k].idx = k;
  }
  qsort(it, nnz, sizeof(sort_item), cmp_item);
  uint32_t* blk_row_ptr = (uint32_t*)add_array(f, "blk_row_ptr", (uint64_t)f->block_rows + 1, 4);
  uint32_t* blk_col_ind = (uint32_t*)add_array(f, "blk_col_ind", nnz, 4);
  uint32_t* blk_data_ptr = (uint32_t*)add_array(f, "blk_data_ptr", (uint64_t)nnz + 1, 4);
  uint32_t* packed = (uint32_t*)add_array(f, "packed", nnz, 4);
  double* data = (double*)add_array(f, "data", nnz, 8);
  f->nstorage = 5;
  uint32_t nblk = 0;
  for (uint32_t k = 0; k < nnz; ++k) {
    const uint32_t id = it[k].idx;
    const uint32_t br = rows[id] >> lb, bc = cols[id] >> lb;
    if (k == 0 || br != (rows[it[k - 1].idx] >> lb) || bc != (cols[it[k - 1].idx] >> lb)) {
      ++blk_row_ptr[br + 1];
      blk_col_ind[nblk] = bc;
      blk_data_ptr[nblk] = k;
      ++nblk;
    }
    packed[k] = ((rows[id] & mask) << 16) | (cols[id] & mask);
    data[k] = vals[id];
  }
  blk_data_ptr[nblk] = nnz;
  for (uint64_t i = 1; i <= f->block_rows; ++i) blk_row_ptr[i] += blk_row_ptr[i - 1];
  shrink_array(f, "blk_col_ind", nblk);
  shrink_array(f, "blk_data_ptr", (uint64_t)nblk + 1);
  free(it);
  *out = f;
  return ORC_OK;
}

/* ---------------------------------------------------------------- BCOH (bcoh.hpp) */

typedef struct { uint32_t row, col, count; } block_ref;

/* Hilbert rect walk, curves.hpp:225-254 (recursive, pruned). */
typedef struct {
  uint32_t row0, row1, col0, col1;
  void (*fn)(void*, uint32_t, uint32_t);
  void* ctx;
} walk_ctx;

static void walk_rec(const walk_ctx* w, uint64_t rb, uint64_t cb, uint64_t dim, unsigned st) {
  if (rb >= w->row1 || cb >= w->col1 || rb + dim <= w->row0 || cb + dim <= w->col0) return;
  if (dim == 1) { w->fn(w->ctx, (uint32_t)rb, (uint32_t)cb); return; }
  const uint64_t half = dim >> 1;
  for (unsigned pos = 0; pos < 4; ++pos) {
    unsigned r, c;
    hil_cell(st, pos, &r, &c);
    walk_rec(w, rb + r * half, cb + c * half, half, hil_child(st, pos));
  }
}

static void hilbert_rect_walk(unsigned level, uint32_t row0, uint32_t row1, uint32_t col0,
                              uint32_t col1, void (*fn)(void*, uint32_t, uint32_t), void* ctx) {
  if (row0 >= row1 || col0 >= col1) return;
  walk_ctx w = {row0, row1, col0, col1, fn, ctx};
  walk_rec(&w, 0, 0, UINT64_C(1) << level, 0);
}

typedef struct {
  const block_ref* blocks;
  uint32_t nblocks, t, cum;
  uint32_t* blk_ptr;
  uint64_t pos;
} ptr_fill_ctx;

static void ptr_fill(void* vctx, uint32_t br, uint32_t bc) {
  ptr_fill_ctx* c = (ptr_fill_ctx*)vctx;
  if (c->t < c->nblocks && c->blocks[c->t].row == br && c->blocks[c->t].col == bc) {
    c->cum += c->blocks[c->t].count;
    ++c->t;
  }
  c->blk_ptr[c->pos++] = c->cum;
}

static uint32_t band_of(const uint32_t* bounds, unsigned p, uint32_t row) {
  /* upper_bound(bounds, row) - 1, bcoh.hpp:224-227 */
  unsigned lo = 0, hi = p + 1;
  while (lo < hi) {
    unsigned mid = (lo + hi) / 2;
    if (bounds[mid] <= row) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

/* build_bcoh, bcoh.hpp:194-376.  Variant: BCOH = (ICRS, row-wise, BICRS), BCOHC = (packed,
 * row-wise, BICRS), BCOHCH = (packed, Hilbert, BICRS), BCOHCHP = (packed, Hilbert, HilbertPtr)
 * (bcoh.hpp:45-56). */
static int build_bcoh(int alg, uint32_t m, uint32_t n, uint32_t nnz, const uint32_t* rows,
                      const uint32_t* cols, const double* vals, unsigned lb, unsigned p,
                      orc_format** out) {
  if ((uint64_t)m > MAX_DIMENSION || (uint64_t)n > MAX_DIMENSION) return ORC_OVERFLOW;
  if (lb < 1 || lb > 15) return ORC_INVALID_ARGUMENT;
  if (p < 1) return ORC_INVALID_ARGUMENT;
  const int icrs = alg == ORC_BCOH;
  const int hilbert_elements = alg == ORC_BCOHCH || alg == ORC_BCOHCHP;
  const int ptr_level = alg == ORC_BCOHCHP;
  const uint32_t beta = UINT32_C(1) << lb;
  const uint32_t mask = beta - 1;

  const unsigned cov = orc_covering_level(m, n);
  if (cov > 31) return ORC_OVERFLOW;
  const uint32_t block_rows = blocks_covering(m, lb);
  const uint32_t block_cols = blocks_covering(n, lb);
  const unsigned element_level = cov > lb ? cov : lb;
  const unsigned block_level = element_level - lb;

  uint32_t* prefix = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)m + 1));
  orc_row_prefix(m, nnz, rows, prefix);
  uint32_t* bounds = (uint32_t*)malloc(sizeof(uint32_t) * (p + 1));
  orc_partition_rows_by_nnz(prefix, m, p, lb, bounds);
  free(prefix);
  if (block_cols >= (UINT32_C(1) << 15)) { free(bounds); return ORC_OVERFLOW; }

  /* per-band geometry, bcoh.hpp:262-273 */
  uint32_t* first_block_row = (uint32_t*)malloc(sizeof(uint32_t) * p);
  uint32_t* block_row_count = (uint32_t*)malloc(sizeof(uint32_t) * p);
  for (unsigned b = 0; b < p; ++b) {
    const uint32_t row_count = bounds[b + 1] - bounds[b];
    first_block_row[b] = bounds[b] >> lb;
    block_row_count[b] = row_count == 0 ? 0 : blocks_covering(bounds[b + 1], lb) - first_block_row[b];
    if (block_row_count[b] >= (UINT32_C(1) << 15)) {
      free(bounds); free(first_block_row); free(block_row_count);
      return ORC_OVERFLOW;
    }
  }

  /* sort, bcoh.hpp:235-252 */
  sort_item* it = (sort_item*)malloc(sizeof(sort_item) * (nnz ? nnz : 1));
  for (uint32_t k = 0; k < nnz; ++k) {
    it[k].k1 = band_of(bounds, p, rows[k]);
    if (hilbert_elements) {
      it[k].k2 = orc_hilbert_encode(rows[k], cols[k], element_level);
      it[k].k3 = 0;
    } else {
      it[k].k2 = orc_hilbert_encode(rows[k] >> lb, cols[k] >> lb, block_level);
      it[k].k3 = ((uint64_t)(rows[k] & mask) << 32) | (cols[k] & mask);
    }
    it[k].idx = k;
  }
  qsort(it, nnz, sizeof(sort_item), cmp_item);

  orc_format* f = new_format(alg, m, n, nnz);
  f->log2_beta = lb;
  f->block_rows = block_rows;
  f->block_cols = block_cols;
  f->element_level = element_level;
  f->block_level = block_level;
  f->bands = p;

  /* capacities: blocks <= nnz, row jumps <= nnz, cells <= sum over bands */
  uint64_t total_cells = 0;
  for (unsigned b = 0; b < p; ++b) total_cells += (uint64_t)block_row_count[b] * block_cols + 1;
  uint32_t* block_nnz = (uint32_t*)add_array(f, "block_nnz", ptr_level ? 0 : nnz, 4);
  int16_t* row_jump_block = (int16_t*)add_array(f, "row_jump_block", ptr_level ? 0 : nnz, 2);
  int16_t* col_jump_block = (int16_t*)add_array(f, "col_jump_block", ptr_level ? 0 : nnz, 2);
  uint32_t* blk_ptr = (uint32_t*)add_array(f, "blk_ptr", ptr_level ? total_cells : 0, 4);
  uint16_t* col_inc = (uint16_t*)add_array(f, "col_inc", icrs ? nnz : 0, 2);
  uint16_t* row_jump = (uint16_t*)add_array(f, "row_jump", icrs ? nnz : 0, 2);
  uint32_t* packed = (uint32_t*)add_array(f, "packed", icrs ? 0 : nnz, 4);
  double* data = (double*)add_array(f, "data", nnz, 8);
  f->nstorage = 8;
  uint32_t* band_first_row = (uint32_t*)add_array(f, "band_first_row", p, 4);
  uint32_t* band_row_count = (uint32_t*)add_array(f, "band_row_count", p, 4);
  uint32_t* band_first_block_row = (uint32_t*)add_array(f, "band_first_block_row", p, 4);
  uint32_t* band_block_row_count = (uint32_t*)add_array(f, "band_block_row_count", p, 4);
  uint64_t* off_elem = (uint64_t*)add_array(f, "off_elem", p + 1, 8);
  uint64_t* off_block = (uint64_t*)add_array(f, "off_block", p + 1, 8);
  uint64_t* off_row_jump_block = (uint64_t*)add_array(f, "off_row_jump_block", p + 1, 8);
  uint64_t* off_blk_ptr = (uint64_t*)add_array(f, "off_blk_ptr", p + 1, 8);
  uint64_t* off_row_jump = (uint64_t*)add_array(f, "off_row_jump", p + 1, 8);

  /* band_begin, bcoh.hpp:254-260 */
  uint64_t* band_begin = (uint64_t*)malloc(sizeof(uint64_t) * (p + 1));
  for (unsigned b = 0; b <= p; ++b) band_begin[b] = nnz;
  band_begin[0] = 0;
  {
    uint64_t b = 0;
    for (uint32_t k = 0; k < nnz; ++k) {
      const uint64_t band = it[k].k1;
      while (b < band) band_begin[++b] = k;
    }
  }

  block_ref* blocks = (block_ref*)malloc(sizeof(block_ref) * (nnz ? nnz : 1));
  uint64_t n_blk = 0, n_rjb = 0, n_ptr = 0, n_rj = 0;
  for (unsigned b = 0; b < p; ++b) {
    band_first_row[b] = bounds[b];
    band_row_count[b] = bounds[b + 1] - bounds[b];
    band_first_block_row[b] = first_block_row[b];
    band_block_row_count[b] = block_row_count[b];
    off_elem[b] = band_begin[b];
    off_block[b] = n_blk;
    off_row_jump_block[b] = n_rjb;
    off_blk_ptr[b] = n_ptr;
    off_row_jump[b] = n_rj;

    /* populate_band, bcoh.hpp:275-366 */
    const uint64_t lo = band_begin[b], hi = band_begin[b + 1];
    uint32_t nb = 0;
    uint32_t prev_in_row = 0, prev_in_col = 0;
    for (uint64_t k = lo; k < hi; ++k) {
      const uint32_t id = it[k].idx;
      const uint32_t row = rows[id], col = cols[id];
      const uint32_t br = row >> lb, bc = col >> lb;
      const uint32_t in_row = row & mask, in_col = col & mask;
      const int new_block = nb == 0 || blocks[nb - 1].row != br || blocks[nb - 1].col != bc;
      if (new_block) { blocks[nb].row = br; blocks[nb].col = bc; blocks[nb].count = 0; ++nb; }
      ++blocks[nb - 1].count;
      if (!icrs) {
        packed[k] = (in_row << 16) | in_col;
      } else {
        if (new_block) {
          col_inc[k] = (uint16_t)in_col;
          row_jump[n_rj++] = (uint16_t)in_row;
        } else if (in_row == prev_in_row) {
          col_inc[k] = (uint16_t)(in_col - prev_in_col);
        } else {
          col_inc[k] = (uint16_t)(in_col - prev_in_col + beta);
          row_jump[n_rj++] = (uint16_t)(in_row - prev_in_row);
        }
        prev_in_row = in_row;
        prev_in_col = in_col;
      }
      data[k] = vals[id];
    }
    if (!ptr_level) {
      uint32_t prev_br = 0, prev_bc = 0;
      for (uint32_t t = 0; t < nb; ++t) {
        block_nnz[n_blk] = blocks[t].count;
        if (t == 0) {
          col_jump_block[n_blk] = (int16_t)blocks[t].col;
          row_jump_block[n_rjb++] = (int16_t)(uint16_t)(blocks[t].row - first_block_row[b]);
        } else if (blocks[t].row == prev_br) {
          col_jump_block[n_blk] = (int16_t)(uint16_t)((int64_t)blocks[t].col - prev_bc);
        } else {
          col_jump_block[n_blk] =
              (int16_t)(uint16_t)((int64_t)blocks[t].col - prev_bc + block_cols);
          row_jump_block[n_rjb++] = (int16_t)(uint16_t)((int64_t)blocks[t].row - prev_br);
        }
        prev_br = blocks[t].row;
        prev_bc = blocks[t].col;
        ++n_blk;
      }
    } else {
      ptr_fill_ctx c = {blocks, nb, 0, 0, blk_ptr + n_ptr, 1};
      blk_ptr[n_ptr] = 0;
      hilbert_rect_walk(block_level, first_block_row[b], first_block_row[b] + block_row_count[b],
                        0, block_cols, ptr_fill, &c);
      if (c.t != nb) { /* bcoh.hpp:363-364 */
        free(blocks); free(band_begin); free(it); free(bounds);
        free(first_block_row); free(block_row_count); orc_free_format(f);
        return ORC_CORRUPT_FORMAT;
      }
      n_ptr += c.pos;
    }
  }
  off_elem[p] = nnz;
  off_block[p] = n_blk;
  off_row_jump_block[p] = n_rjb;
  off_blk_ptr[p] = n_ptr;
  off_row_jump[p] = n_rj;
  shrink_array(f, "block_nnz", n_blk);
  shrink_array(f, "col_jump_block", n_blk);
  shrink_array(f, "row_jump_block", n_rjb);
  shrink_array(f, "blk_ptr", n_ptr);
  shrink_array(f, "row_jump", n_rj);
  free(blocks); free(band_begin); free(it); free(bounds);
  free(first_block_row); free(block_row_count);
  *out = f;
  return ORC_OK;
}

/* build_format, engine.hpp:96-122 */
int orc_build_format(int alg, uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows,
                     const uint32_t* cols, const double* vals, unsigned threads,
                     uint64_t l2_bytes, orc_format** out) {
  *out = NULL;
  if (alg < 0 || alg > ORC_MERGEBH) return ORC_INVALID_ARGUMENT;
  if (nnz > UINT32_MAX) return ORC_OVERFLOW;
  const unsigned lb = orc_engine_log2_beta(alg, n, l2_bytes);
  switch (alg) {
    case ORC_SEQ_CRS: case ORC_PAR_CRS: case ORC_MERGE:
      return build_crs(alg, m, n, (uint32_t)nnz, rows, cols, vals, out);
    case ORC_CSB: case ORC_CSBH:
      return build_csb(alg, m, n, (uint32_t)nnz, rows, cols, vals, lb, out);
    case ORC_MERGEB: case ORC_MERGEBH:
      return build_mergeb(alg, m, n, (uint32_t)nnz, rows, cols, vals, lb, out);
    default:
      return build_bcoh(alg, m, n, (uint32_t)nnz, rows, cols, vals, lb, threads, out);
  }
}

/* build_csb / build_mergeb / build_bcoh with an explicit block size (csb.hpp:51-57,
 * mergeb.hpp:50-56, bcoh.hpp:194-205): beta in [2, 2^16] ([2, 2^15] for BCOH), p >= 1. */
int orc_build_format_beta(int alg, uint32_t m, uint32_t n, uint64_t nnz, const uint32_t* rows,
                          const uint32_t* cols, const double* vals, unsigned log2_beta, unsigned threads,
                          orc_format** out) {
  *out = NULL;
  if (alg <= ORC_MERGE || alg > ORC_MERGEBH) return ORC_INVALID_ARGUMENT;
  if (nnz > UINT32_MAX) return ORC_OVERFLOW;
  const unsigned cap = is_bcoh(alg) ? 15u : 16u;
  if (log2_beta < 1 || log2_beta > cap) return ORC_INVALID_ARGUMENT;
  switch (alg) {
    case ORC_CSB: case ORC_CSBH:
      return build_csb(alg, m, n, (uint32_t)nnz, rows, cols, vals, log2_beta, out);
    case ORC_MERGEB: case ORC_MERGEBH:
      return build_mergeb(alg, m, n, (uint32_t)nnz, rows, cols, vals, log2_beta, out);
    default:
      if (threads < 1) return ORC_INVALID_ARGUMENT;
      return build_bcoh(alg, m, n, (uint32_t)nnz, rows, cols, vals, log2_beta, threads, out);
  }
}

/* ---------------------------------------------------------------- kernels */

/* spmv_crs_seq, crs.hpp:43-57 (ParCRS is bitwise equal, spmv_parallel.hpp:106-125) */
static void spmv_crs(const orc_format* f, const double* x, double* y) {
  const uint32_t* rp = ARR(f, "row_ptr", uint32_t);
  const uint32_t* ci = ARR(f, "col_ind", uint32_t);
  const double* d = ARR(f, "data", double);
  for (uint32_t i = 0; i < f->m; ++i) {
    double sum = 0.0;
    for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) sum += d[k] * x[ci[k]];
    y[i] = sum;
  }
}

/* spmv_merge, spmv_parallel.hpp:130-160: p merge-path bands, carry-outs fixed up sequentially. */
static void spmv_merge(const orc_format* f, const double* x, double* y, unsigned p) {
  const uint32_t* rp = ARR(f, "row_ptr", uint32_t);
  const uint32_t* ci = ARR(f, "col_ind", uint32_t);
  const double* d = ARR(f, "data", double);
  const uint64_t m = f->m, nnz = f->nnz, total = m + nnz;
  if (total == 0) return;
  uint32_t* carry_row = (uint32_t*)malloc(sizeof(uint32_t) * p);
  double* carry_val = (double*)malloc(sizeof(double) * p);
  for (unsigned w = 0; w < p; ++w) {
    uint64_t i, j, ie, je;
    orc_diagonal_search(rp + 1, m, nnz, total * w / p, 1, NULL, &i, &j);
    orc_diagonal_search(rp + 1, m, nnz, total * (w + 1) / p, 1, NULL, &ie, &je);
    double temp = 0.0;
    for (; i < ie; ++i) {
      for (; j < rp[i + 1]; ++j) temp += d[j] * x[ci[j]];
      y[i] = temp;
      temp = 0.0;
    }
    for (; j < je; ++j) temp += d[j] * x[ci[j]];
    carry_row[w] = (uint32_t)ie;
    carry_val[w] = temp;
  }
  for (unsigned w = 0; w < p; ++w)
    if (carry_row[w] < m) y[carry_row[w]] += carry_val[w];
  free(carry_row);
  free(carry_val);
}

/* quadrant_boundaries, curves.hpp:185-211 (partition_point over curve positions). */
static unsigned quad_position(int hilbert, unsigned st, uint32_t pk, uint32_t half) {
  const unsigned rbit = ((pk >> 16) & half) ? 1u : 0u;
  const unsigned cbit = ((pk & 0xFFFFu) & half) ? 1u : 0u;
  return hilbert ? hil_position(st, rbit, cbit) : ((rbit << 1) | cbit);
}

typedef struct { uint64_t lo, hi; } range64;

/* split_block_range, spmv_parallel.hpp:178-193 */
static void split_block_range(const uint32_t* packed, int hilbert, uint64_t begin, uint64_t end,
                              uint32_t dim, unsigned st, uint64_t threshold, range64* leaves,
                              uint64_t* nleaves) {
  if (end - begin <= threshold || dim == 1) {
    if (end > begin) { leaves[*nleaves].lo = begin; leaves[*nleaves].hi = end; ++*nleaves; }
    return;
  }
  const uint32_t half = dim >> 1;
  uint64_t cut[5];
  cut[0] = 0;
  cut[4] = end - begin;
  for (unsigned q = 1; q <= 3; ++q) {
    uint64_t lo = 0, hi = end - begin;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (quad_position(hilbert, st, packed[begin + mid], half) < q) lo = mid + 1; else hi = mid;
    }
    cut[q] = lo;
  }
  for (unsigned pos = 0; pos < 4; ++pos)
    split_block_range(packed, hilbert, begin + cut[pos], begin + cut[pos + 1], dim >> 1,
                      hilbert ? hil_child(st, pos) : st, threshold, leaves, nleaves);
}

/* The work-item list of spmv_csb, spmv_parallel.hpp:209-264.  Returns the number of items; items
 * must hold nnz + block_rows * (block_cols + 1) entries (an upper bound). */
static uint64_t csb_items(const orc_format* f, uint64_t threshold, orc_csb_item* items) {
  const uint32_t* blk_ptr = ARR(f, "blk_ptr", uint32_t);
  const uint32_t* packed = ARR(f, "packed", uint32_t);
  const uint32_t beta = UINT32_C(1) << f->log2_beta;
  const int hilbert = f->alg == ORC_CSBH;
  const uint32_t bcs = f->block_cols;
  uint64_t nitems = 0;
  int32_t slot = 0;
  range64* leaves = (range64*)malloc(sizeof(range64) * ((uint64_t)f->nnz + 1));

  for (uint32_t br = 0; br < f->block_rows; ++br) {
    const uint64_t row_cell = (uint64_t)br * bcs;
    const uint64_t rb = blk_ptr[row_cell], re = blk_ptr[row_cell + bcs];
    if (re == rb) continue;
    if (re - rb <= threshold) {
      orc_csb_item t = {br, 0, bcs, -1, rb, re};
      items[nitems++] = t;
      continue;
    }
    uint32_t chunk_first = 0;
    uint64_t chunk_count = 0;
#define FLUSH_CHUNK(cell_end)                                                          \
  do {                                                                                 \
    if (chunk_count != 0) {                                                            \
      orc_csb_item t = {br, chunk_first, (cell_end), slot++,                           \
                        blk_ptr[row_cell + chunk_first], blk_ptr[row_cell + (cell_end)]}; \
      items[nitems++] = t;                                                             \
      chunk_count = 0;                                                                 \
    }                                                                                  \
  } while (0)
    for (uint32_t c = 0; c < bcs; ++c) {
      const uint64_t cell_nnz = blk_ptr[row_cell + c + 1] - blk_ptr[row_cell + c];
      if (cell_nnz > threshold) {
        FLUSH_CHUNK(c);
        uint64_t nl = 0;
        split_block_range(packed, hilbert, blk_ptr[row_cell + c], blk_ptr[row_cell + c + 1], beta,
                          0, threshold, leaves, &nl);
        for (uint64_t l = 0; l < nl; ++l) {
          orc_csb_item t = {br, c, c + 1, slot++, leaves[l].lo, leaves[l].hi};
          items[nitems++] = t;
        }
        chunk_first = c + 1;
        continue;
      }
      if (chunk_count == 0) chunk_first = c;
      if (chunk_count + cell_nnz > threshold) {
        FLUSH_CHUNK(c);
        chunk_first = c;
      }
      chunk_count += cell_nnz;
    }
    FLUSH_CHUNK(bcs);
#undef FLUSH_CHUNK
  }
  free(leaves);
  return nitems;
}

int orc_csb_work_items(const orc_format* f, uint64_t split_threshold, orc_csb_item* items,
                       uint64_t capacity, uint64_t* count) {
  if (f->alg != ORC_CSB && f->alg != ORC_CSBH) return ORC_INVALID_ARGUMENT;
  const uint64_t threshold = split_threshold == 0 ? 2 * ((uint64_t)1 << f->log2_beta) : split_threshold;
  const uint64_t cap = (uint64_t)f->nnz + (uint64_t)f->block_rows * (f->block_cols + 1) + 16;
  orc_csb_item* all = (orc_csb_item*)malloc(sizeof(orc_csb_item) * cap);
  if (!all) return ORC_NO_MEMORY;
  const uint64_t n = csb_items(f, threshold, all);
  *count = n;
  int rc = ORC_OK;
  if (items) {
    if (capacity < n) rc = ORC_INVALID_ARGUMENT;
    else memcpy(items, all, sizeof(orc_csb_item) * n);
  }
  free(all);
  return rc;
}

/* spmv_csb, spmv_parallel.hpp:202-331: work items, temp slots, pairwise slot reduction.  The
 * result is independent of p (deterministic reduction order), so it is replayed sequentially. */
static void spmv_csb(const orc_format* f, const double* x, double* y, uint64_t split_threshold) {
  const uint32_t* blk_ptr = ARR(f, "blk_ptr", uint32_t);
  const uint32_t* packed = ARR(f, "packed", uint32_t);
  const double* d = ARR(f, "data", double);
  const unsigned lb = f->log2_beta;
  const uint32_t beta = UINT32_C(1) << lb;
  const uint64_t threshold = split_threshold == 0 ? 2 * (uint64_t)beta : split_threshold;
  const uint32_t bcs = f->block_cols;

  uint64_t cap = (uint64_t)f->nnz + (uint64_t)f->block_rows * (bcs + 1) + 16;
  orc_csb_item* items = (orc_csb_item*)malloc(sizeof(orc_csb_item) * cap);
  const uint64_t nitems = csb_items(f, threshold, items);
  /* split rows: consecutive items with slots, in block-row order */
  typedef struct { uint32_t block_row; uint64_t slot_begin, slot_count; } split_row;
  split_row* srows = (split_row*)malloc(sizeof(split_row) * (f->block_rows + 1));
  uint64_t nsrows = 0, total_slots = 0;
  for (uint64_t t = 0; t < nitems; ++t) {
    if (items[t].temp_slot < 0) continue;
    if (nsrows == 0 || srows[nsrows - 1].block_row != items[t].block_row) {
      srows[nsrows].block_row = items[t].block_row;
      srows[nsrows].slot_begin = (uint64_t)items[t].temp_slot;
      srows[nsrows].slot_count = 0;
      ++nsrows;
    }
    ++srows[nsrows - 1].slot_count;
    ++total_slots;
  }

  double** temps = (double**)calloc(total_slots ? total_slots : 1, sizeof(double*));
  for (uint64_t r = 0; r < nsrows; ++r) {
    const uint64_t rem = f->m - ((uint64_t)srows[r].block_row << lb);
    const uint64_t height = beta < rem ? beta : rem;
    for (uint64_t s = 0; s < srows[r].slot_count; ++s)
      temps[srows[r].slot_begin + s] = (double*)calloc(height ? height : 1, sizeof(double));
  }
  for (uint32_t i = 0; i < f->m; ++i) y[i] = 0.0;
  for (uint64_t t = 0; t < nitems; ++t) {
    const orc_csb_item* it = &items[t];
    double* target = it->temp_slot < 0 ? y + ((uint64_t)it->block_row << lb) : temps[it->temp_slot];
    const uint64_t row_cell = (uint64_t)it->block_row * bcs;
    for (uint32_t c = it->cell_begin; c < it->cell_end; ++c) {
      uint64_t lo = blk_ptr[row_cell + c], hi = blk_ptr[row_cell + c + 1];
      if (lo < it->elem_begin) lo = it->elem_begin;
      if (hi > it->elem_end) hi = it->elem_end;
      const uint64_t col_base = (uint64_t)c << lb;
      for (uint64_t k = lo; k < hi; ++k)
        target[packed[k] >> 16] += d[k] * x[col_base + (packed[k] & 0xFFFFu)];
    }
  }
  for (uint64_t r = 0; r < nsrows; ++r) {
    const split_row* row = &srows[r];
    const uint64_t rem = f->m - ((uint64_t)row->block_row << lb);
    const uint64_t height = beta < rem ? beta : rem;
    for (uint64_t stride = 1; stride < row->slot_count; stride *= 2)
      for (uint64_t s = 0; s + stride < row->slot_count; s += 2 * stride) {
        double* dst = temps[row->slot_begin + s];
        const double* src = temps[row->slot_begin + s + stride];
        for (uint64_t q = 0; q < height; ++q) dst[q] += src[q];
      }
    double* outp = y + ((uint64_t)row->block_row << lb);
    const double* tot = temps[row->slot_begin];
    for (uint64_t q = 0; q < height; ++q) outp[q] += tot[q];
  }
  for (uint64_t s = 0; s < total_slots; ++s) free(temps[s]);
  free(temps);
  free(items);
  free(srows);
}

/* bcoh_for_each_block / bcoh_for_each_element replay (bcoh.hpp:115-187) and spmv_bcoh
 * (spmv_parallel.hpp:336-350). */
typedef struct {
  const orc_format* f;
  unsigned band;
  const double* x;
  double* y;
  uint64_t cell;
  uint64_t rj;
  int err;
  uint32_t* rows; /* decode mode (bcoh_to_triplet): coordinates at storage positions, no multiply */
  uint32_t* cols;
} bcoh_ctx;

/* one element of the band replay: y += a * x, or record its coordinates */
static void bcoh_visit(bcoh_ctx* c, uint64_t e0, uint64_t k, uint64_t row, uint64_t col, const double* d) {
  if (c->rows) {
    c->rows[e0 + k] = (uint32_t)row;
    c->cols[e0 + k] = (uint32_t)col;
  } else {
    c->y[row] += d[k] * c->x[col];
  }
}

static void bcoh_block(bcoh_ctx* c, uint32_t br, uint32_t bc, uint64_t begin, uint64_t count) {
  const orc_format* f = c->f;
  const unsigned lb = f->log2_beta;
  const uint32_t beta = UINT32_C(1) << lb;
  const uint64_t e0 = ARR(f, "off_elem", uint64_t)[c->band];
  const double* d = ARR(f, "data", double) + e0;
  const uint64_t row_base = (uint64_t)br << lb, col_base = (uint64_t)bc << lb;
  if (f->alg != ORC_BCOH) {
    const uint32_t* pk = ARR(f, "packed", uint32_t) + e0;
    for (uint64_t k = begin; k < begin + count; ++k)
      bcoh_visit(c, e0, k, row_base + (pk[k] >> 16), col_base + (pk[k] & 0xFFFFu), d);
  } else {
    const uint16_t* ci = ARR(f, "col_inc", uint16_t) + e0;
    const uint16_t* rj = ARR(f, "row_jump", uint16_t) + ARR(f, "off_row_jump", uint64_t)[c->band];
    uint32_t in_col = ci[begin];
    uint32_t in_row = rj[c->rj++];
    bcoh_visit(c, e0, begin, row_base + in_row, col_base + in_col, d);
    for (uint64_t k = begin + 1; k < begin + count; ++k) {
      in_col += ci[k];
      if (in_col >= beta) { in_col -= beta; in_row += rj[c->rj++]; }
      bcoh_visit(c, e0, k, row_base + in_row, col_base + in_col, d);
    }
  }
}

static void bcoh_walk_fn(void* vctx, uint32_t br, uint32_t bc) {
  bcoh_ctx* c = (bcoh_ctx*)vctx;
  const uint32_t* bp = ARR(c->f, "blk_ptr", uint32_t) + ARR(c->f, "off_blk_ptr", uint64_t)[c->band];
  const uint64_t begin = bp[c->cell], end = bp[c->cell + 1];
  ++c->cell;
  if (end > begin) bcoh_block(c, br, bc, begin, end - begin);
}

/* Replays every band; y == NULL: decode mode into rows / cols (bcoh_to_triplet, bcoh.hpp:379-392). */
static int bcoh_replay(const orc_format* f, const double* x, double* y, unsigned p, uint32_t* rows,
                       uint32_t* cols) {
  if (p != f->bands) return ORC_INVALID_ARGUMENT; /* spmv_parallel.hpp:339-341 */
  for (unsigned b = 0; b < p; ++b) {
    const uint32_t first_row = ARR(f, "band_first_row", uint32_t)[b];
    const uint32_t row_count = ARR(f, "band_row_count", uint32_t)[b];
    const uint32_t fbr = ARR(f, "band_first_block_row", uint32_t)[b];
    const uint32_t nbr = ARR(f, "band_block_row_count", uint32_t)[b];
    if (y)
      for (uint32_t i = first_row; i < first_row + row_count; ++i) y[i] = 0.0;
    bcoh_ctx c = {f, b, x, y, 0, 0, 0, y ? NULL : rows, y ? NULL : cols};
    if (f->alg != ORC_BCOHCHP) {
      const uint64_t b0 = ARR(f, "off_block", uint64_t)[b], b1 = ARR(f, "off_block", uint64_t)[b + 1];
      const uint32_t* bn = ARR(f, "block_nnz", uint32_t) + b0;
      const int16_t* cj = ARR(f, "col_jump_block", int16_t) + b0;
      const int16_t* rjb = ARR(f, "row_jump_block", int16_t) + ARR(f, "off_row_jump_block", uint64_t)[b];
      uint32_t col = 0;
      int32_t local_row = 0;
      uint64_t rj = 0, begin = 0;
      for (uint64_t t = 0; t < b1 - b0; ++t) {
        if (t == 0) {
          col = (uint32_t)(int32_t)cj[0];
          local_row = rjb[0];
          rj = 1;
        } else {
          const uint16_t raw = (uint16_t)((uint16_t)col + (uint16_t)cj[t]);
          if (raw >= f->block_cols) { col = raw - f->block_cols; local_row += rjb[rj++]; }
          else col = raw;
        }
        bcoh_block(&c, fbr + (uint32_t)local_row, col, begin, bn[t]);
        begin += bn[t];
      }
    } else {
      hilbert_rect_walk(f->block_level, fbr, fbr + nbr, 0, f->block_cols, bcoh_walk_fn, &c);
    }
  }
  return ORC_OK;
}

static int spmv_bcoh(const orc_format* f, const double* x, double* y, unsigned p) {
  return bcoh_replay(f, x, y, p, NULL, NULL);
}

/* crs_to_triplet (crs.hpp:94-105), csb_to_triplet (csb.hpp:103-120), mergeb_to_triplet
 * (mergeb.hpp:110-127), bcoh_to_triplet (bcoh.hpp:379-392): coordinates in storage order. */
int orc_format_to_triplet(const orc_format* f, uint32_t* rows, uint32_t* cols, double* vals) {
  const unsigned lb = f->log2_beta;
  if (vals && f->nnz) memcpy(vals, ARR(f, "data", double), sizeof(double) * f->nnz);
  if (f->alg <= ORC_MERGE) {
    const uint32_t* rp = ARR(f, "row_ptr", uint32_t);
    if (f->nnz) memcpy(cols, ARR(f, "col_ind", uint32_t), sizeof(uint32_t) * f->nnz);
    for (uint32_t i = 0; i < f->m; ++i)
      for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) rows[k] = i;
  } else if (f->alg == ORC_CSB || f->alg == ORC_CSBH) {
    const uint32_t* bp = ARR(f, "blk_ptr", uint32_t);
    const uint32_t* pk = ARR(f, "packed", uint32_t);
    for (uint32_t br = 0; br < f->block_rows; ++br)
      for (uint32_t bc = 0; bc < f->block_cols; ++bc) {
        const uint64_t cell = (uint64_t)br * f->block_cols + bc;
        for (uint32_t k = bp[cell]; k < bp[cell + 1]; ++k) {
          rows[k] = (br << lb) + (pk[k] >> 16);
          cols[k] = (bc << lb) + (pk[k] & 0xFFFFu);
        }
      }
  } else if (f->alg == ORC_MERGEB || f->alg == ORC_MERGEBH) {
    const uint32_t* brp = ARR(f, "blk_row_ptr", uint32_t);
    const uint32_t* bci = ARR(f, "blk_col_ind", uint32_t);
    const uint32_t* bdp = ARR(f, "blk_data_ptr", uint32_t);
    const uint32_t* pk = ARR(f, "packed", uint32_t);
    for (uint32_t br = 0; br < f->block_rows; ++br)
      for (uint32_t t = brp[br]; t < brp[br + 1]; ++t)
        for (uint32_t k = bdp[t]; k < bdp[t + 1]; ++k) {
          rows[k] = (br << lb) + (pk[k] >> 16);
          cols[k] = (bci[t] << lb) + (pk[k] & 0xFFFFu);
        }
  } else {
    return bcoh_replay(f, NULL, NULL, f->bands, rows, cols);
  }
  return ORC_OK;
}

/* spmv_mergeb, spmv_parallel.hpp:355-402 */
static void spmv_mergeb(const orc_format* f, const double* x, double* y, unsigned p) {
  const uint32_t* brp = ARR(f, "blk_row_ptr", uint32_t);
  const uint32_t* bci = ARR(f, "blk_col_ind", uint32_t);
  const uint32_t* bdp = ARR(f, "blk_data_ptr", uint32_t);
  const uint32_t* pk = ARR(f, "packed", uint32_t);
  const double* d = ARR(f, "data", double);
  const uint64_t blocks = ARRN(f, "blk_col_ind");
  const uint64_t total = (uint64_t)f->block_rows + blocks;
  if (total == 0) return;
  const unsigned lb = f->log2_beta;
  const uint32_t beta = UINT32_C(1) << lb;
  uint32_t* carry_row = (uint32_t*)malloc(sizeof(uint32_t) * p);
  double** carry_slice = (double**)calloc(p, sizeof(double*));
  for (unsigned w = 0; w < p; ++w) {
    uint64_t i, t, ie, te;
    orc_diagonal_search(brp + 1, f->block_rows, blocks, total * w / p, 1, NULL, &i, &t);
    orc_diagonal_search(brp + 1, f->block_rows, blocks, total * (w + 1) / p, 1, NULL, &ie, &te);
    double* slice = (double*)calloc(beta, sizeof(double));
    for (; i < ie; ++i) {
      for (; t < brp[i + 1]; ++t) {
        const uint64_t col_base = (uint64_t)bci[t] << lb;
        for (uint32_t k = bdp[t]; k < bdp[t + 1]; ++k)
          slice[pk[k] >> 16] += d[k] * x[col_base + (pk[k] & 0xFFFFu)];
      }
      const uint64_t row_base = i << lb;
      const uint64_t rem = f->m - row_base;
      const uint64_t height = beta < rem ? beta : rem;
      for (uint64_t q = 0; q < height; ++q) { y[row_base + q] = slice[q]; slice[q] = 0.0; }
    }
    for (; t < te; ++t) {
      const uint64_t col_base = (uint64_t)bci[t] << lb;
      for (uint32_t k = bdp[t]; k < bdp[t + 1]; ++k)
        slice[pk[k] >> 16] += d[k] * x[col_base + (pk[k] & 0xFFFFu)];
    }
    carry_row[w] = (uint32_t)ie;
    carry_slice[w] = slice;
  }
  for (unsigned w = 0; w < p; ++w) {
    if (carry_row[w] < f->block_rows) {
      const uint64_t row_base = (uint64_t)carry_row[w] << lb;
      const uint64_t rem = f->m - row_base;
      const uint64_t height = beta < rem ? beta : rem;
      for (uint64_t q = 0; q < height; ++q) y[row_base + q] += carry_slice[w][q];
    }
    free(carry_slice[w]);
  }
  free(carry_row);
  free(carry_slice);
}

/* run_spmv, engine.hpp:126-148, with check_spmv_args (spmv_parallel.hpp:90-99). */
int orc_run_spmv(int alg, const orc_format* f, const double* x, uint64_t x_len, double* y,
                 uint64_t y_len, unsigned p, uint64_t split_threshold) {
  if (x_len != f->n || y_len != f->m) return ORC_DIMENSION_MISMATCH;
  if (alg != ORC_SEQ_CRS && p < 1) return ORC_INVALID_ARGUMENT;
  switch (alg) {
    case ORC_SEQ_CRS: case ORC_PAR_CRS:
      if (f->alg > ORC_MERGE) return ORC_INVALID_ARGUMENT;
      spmv_crs(f, x, y);
      return ORC_OK;
    case ORC_MERGE:
      if (f->alg > ORC_MERGE) return ORC_INVALID_ARGUMENT;
      spmv_merge(f, x, y, p);
      return ORC_OK;
    case ORC_CSB: case ORC_CSBH:
      if (f->alg != ORC_CSB && f->alg != ORC_CSBH) return ORC_INVALID_ARGUMENT;
      spmv_csb(f, x, y, split_threshold);
      return ORC_OK;
    case ORC_MERGEB: case ORC_MERGEBH:
      if (f->alg != ORC_MERGEB && f->alg != ORC_MERGEBH) return ORC_INVALID_ARGUMENT;
      spmv_mergeb(f, x, y, p);
      return ORC_OK;
    default:
      if (!is_bcoh(f->alg)) return ORC_INVALID_ARGUMENT;
      return spmv_bcoh(f, x, y, p);
  }
}
