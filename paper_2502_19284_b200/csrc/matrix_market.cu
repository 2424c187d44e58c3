// matrix_market.cu -- Matrix Market coordinate ingest and the format
// sniffing loader.
//
// Restates read_matrix_market (inc/matrix_market.hpp:94-190) -- the same banner rules, error kinds
// and entry order (1-based -> 0-based, symmetric off-diagonals mirrored right after their entry,
// pattern -> 1.0, integer values widened) -- as a single pass over the file bytes instead of
// istream line reads, then validate() (inc/triplet.hpp:42-59): on the host for the host variant,
// on the device (radix-sorted duplicate check) for the device variant.  load_matrix
// (inc/io.hpp:29-40) sniffs the SPMVLAB1 magic and dispatches to the cache or the text reader.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {

extern thread_local std::string g_last_error;

namespace {

constexpr uint64_t kMaxDimension = uint64_t(1) << 31;  // inc/types.hpp:45

int mm_fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// istream >> token whitespace (C locale isspace)
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

struct Lines {
  const char* p;
  const char* end;
  bool more() const { return p < end; }
  // std::getline: the text up to the next '\n' (the last line may lack one); false at EOF
  bool getline(std::string& line) {
    if (p >= end) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    const char* e = nl ? nl : end;
    line.assign(p, e);
    p = nl ? nl + 1 : end;
    return true;
  }
  // detail::next_content_line (matrix_market.hpp:50-59)
  bool next_content(std::string& line) {
    while (getline(line)) {
      if (!line.empty() && line.back() == '\r') line.pop_back();
      const size_t first = line.find_first_not_of(" \t");
      if (first == std::string::npos) continue;
      if (line[first] == '%') continue;
      return true;
    }
    return false;
  }
};

void split_fields(const std::string& line, std::vector<std::string>& out) {
  out.clear();
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_ws(line[i])) ++i;
    size_t j = i;
    while (j < line.size() && !is_ws(line[j])) ++j;
    if (j > i) out.emplace_back(line, i, j - i);
    i = j;
  }
}

bool parse_u64(const std::string& t, uint64_t& v) {
  auto [ptr, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
  return ec == std::errc{} && ptr == t.data() + t.size();
}

bool parse_value(const std::string& t, double& v) {
  char* e = nullptr;
  v = std::strtod(t.c_str(), &e);
  return !t.empty() && e == t.c_str() + t.size();
}

}  // namespace

struct MmResult {
  uint32_t m = 0, n = 0;
  int field = 0, symmetry = 0;
  uint64_t declared = 0;
  std::vector<uint32_t> rows, cols;
  std::vector<double> vals;
};

static int read_file(const char* path, std::string& buf) {
  FILE* f = fopen(path, "rb");
  if (!f) return mm_fail(kIoError, std::string("cannot open ") + path);
  std::fseek(f, 0, SEEK_END);
  const long size = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  buf.resize(size > 0 ? (size_t)size : 0);
  const size_t got = buf.empty() ? 0 : fread(&buf[0], 1, buf.size(), f);
  fclose(f);
  if (got != buf.size()) return mm_fail(kIoError, std::string("read failed: ") + path);
  return kOk;
}

// read_matrix_market minus the final validate(): parse errors only.
static int mm_parse(const std::string& text, MmResult& r) {
  Lines in{text.data(), text.data() + text.size()};
  std::string line;
  std::vector<std::string> f;
  if (!in.getline(line)) return mm_fail(kBadHeader, "empty input");
  if (!line.empty() && line.back() == '\r') line.pop_back();
  for (char& c : line)
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
  split_fields(line, f);
  if (f.size() != 5 || f[0] != "%%matrixmarket")
    return mm_fail(kBadHeader, "first line must be a %%MatrixMarket banner");
  if (f[1] != "matrix") return mm_fail(kBadHeader, "unsupported object '" + f[1] + "'");
  if (f[2] == "array") return mm_fail(kUnsupportedFormat, "dense 'array' bodies are not supported");
  if (f[2] != "coordinate") return mm_fail(kBadHeader, "unknown format '" + f[2] + "'");
  if (f[3] == "real") r.field = 0;
  else if (f[3] == "integer") r.field = 1;
  else if (f[3] == "pattern") r.field = 2;
  else return mm_fail(kUnsupportedField, "unsupported field '" + f[3] + "'");
  if (f[4] == "general") r.symmetry = 0;
  else if (f[4] == "symmetric") r.symmetry = 1;
  else return mm_fail(kUnsupportedSymmetry, "unsupported symmetry '" + f[4] + "'");

  size_t line_no = 1;
  if (!in.next_content(line)) return mm_fail(kTruncated, "missing size line");
  ++line_no;
  split_fields(line, f);
  if (f.size() != 3) return mm_fail(kParseError, "size line must read 'rows cols entries'");
  uint64_t m = 0, n = 0, declared = 0;
  for (int k = 0; k < 3; ++k) {
    uint64_t& v = k == 0 ? m : (k == 1 ? n : declared);
    if (!parse_u64(f[k], v))
      return mm_fail(kParseError, "line " + std::to_string(line_no) + ": expected an integer, got '" + f[k] + "'");
  }
  if (m > kMaxDimension || n > kMaxDimension)
    return mm_fail(kOverflow, "matrix dimension exceeds the supported index width");
  r.m = (uint32_t)m;
  r.n = (uint32_t)n;
  r.declared = declared;
  const size_t expected = r.field == 2 ? 2u : 3u;
  const size_t reserve = (size_t)std::min<uint64_t>(declared, text.size() / 4 + 1) * (r.symmetry ? 2 : 1);
  r.rows.reserve(reserve);
  r.cols.reserve(reserve);
  r.vals.reserve(reserve);
  for (uint64_t k = 0; k < declared; ++k) {
    if (!in.next_content(line))
      return mm_fail(kTruncated, "entry " + std::to_string(k + 1) + " of " + std::to_string(declared) + " missing");
    ++line_no;
    split_fields(line, f);
    if (f.size() != expected)
      return mm_fail(kParseError, "line " + std::to_string(line_no) + ": expected " + std::to_string(expected) +
                                      " fields");
    uint64_t i = 0, j = 0;
    if (!parse_u64(f[0], i))
      return mm_fail(kParseError, "line " + std::to_string(line_no) + ": expected an integer, got '" + f[0] + "'");
    if (!parse_u64(f[1], j))
      return mm_fail(kParseError, "line " + std::to_string(line_no) + ": expected an integer, got '" + f[1] + "'");
    if (!(i >= 1 && i <= m && j >= 1 && j <= n))
      return mm_fail(kIndexOutOfRange, "line " + std::to_string(line_no) + ": entry (" + std::to_string(i) + ", " +
                                           std::to_string(j) + ") outside " + std::to_string(m) + "x" +
                                           std::to_string(n));
    double value = 1.0;
    if (r.field != 2 && !parse_value(f[2], value))
      return mm_fail(kParseError, "line " + std::to_string(line_no) + ": expected a number, got '" + f[2] + "'");
    r.rows.push_back((uint32_t)(i - 1));
    r.cols.push_back((uint32_t)(j - 1));
    r.vals.push_back(value);
    if (r.symmetry == 1 && i != j) {
      r.rows.push_back((uint32_t)(j - 1));
      r.cols.push_back((uint32_t)(i - 1));
      r.vals.push_back(value);
    }
  }
  if (in.next_content(line))
    return mm_fail(kParseError, "more entries than the " + std::to_string(declared) + " declared");
  if (r.vals.size() > 0xFFFFFFFFull) return mm_fail(kOverflow, "nnz exceeds the 32-bit index type");
  return kOk;
}

// validate() on the host (inc/triplet.hpp:42-59); ranges were checked while parsing
static int host_duplicates(const MmResult& r) {
  std::vector<uint64_t> keys(r.vals.size());
  for (size_t i = 0; i < keys.size(); ++i) keys[i] = ((uint64_t)r.rows[i] << 32) | r.cols[i];
  std::sort(keys.begin(), keys.end());
  if (std::adjacent_find(keys.begin(), keys.end()) != keys.end())
    return mm_fail(kDuplicateEntry, "duplicate (row, col) coordinate");
  return kOk;
}

static void fill_header(const MmResult& r, spmvlab_cuda_mm_header* h) {
  if (!h) return;
  h->field = r.field;
  h->symmetry = r.symmetry;
  h->m = r.m;
  h->n = r.n;
  h->declared_nnz = r.declared;
}

int mm_read_host(const char* path, spmvlab_cuda_host_coo* out, spmvlab_cuda_mm_header* header) {
  std::string text;
  if (int rc = read_file(path, text)) return rc;
  MmResult r;
  if (int rc = mm_parse(text, r)) return rc;
  if (int rc = host_duplicates(r)) return rc;
  const size_t nnz = r.vals.size();
  std::memset(out, 0, sizeof(*out));
  out->row_ind = static_cast<uint32_t*>(std::malloc(nnz ? nnz * 4 : 1));
  out->col_ind = static_cast<uint32_t*>(std::malloc(nnz ? nnz * 4 : 1));
  out->data = static_cast<double*>(std::malloc(nnz ? nnz * 8 : 1));
  if (!out->row_ind || !out->col_ind || !out->data) {
    std::free(out->row_ind);
    std::free(out->col_ind);
    std::free(out->data);
    std::memset(out, 0, sizeof(*out));
    return mm_fail(kNoMemory, "host allocation failed");
  }
  std::memcpy(out->row_ind, r.rows.data(), nnz * 4);
  std::memcpy(out->col_ind, r.cols.data(), nnz * 4);
  std::memcpy(out->data, r.vals.data(), nnz * 8);
  out->m = r.m;
  out->n = r.n;
  out->nnz = nnz;
  fill_header(r, header);
  return kOk;
}

int mm_read_device(const char* path, spmvlab_cuda_coo* a, spmvlab_cuda_mm_header* header, cudaStream_t s) {
  const bool caller_buffers = a->row_ind && a->col_ind && a->data;
  const uint64_t capacity = a->nnz;
  std::string text;
  if (int rc = read_file(path, text)) return rc;
  MmResult r;
  if (int rc = mm_parse(text, r)) return rc;
  text.clear();
  text.shrink_to_fit();
  const uint64_t nnz = r.vals.size();
  uint32_t *rows = nullptr, *cols = nullptr;
  double* vals = nullptr;
  if (caller_buffers) {
    if (capacity < nnz) return mm_fail(kInvalidArgument, "caller buffers smaller than the matrix's nnz");
    rows = const_cast<uint32_t*>(a->row_ind);
    cols = const_cast<uint32_t*>(a->col_ind);
    vals = const_cast<double*>(a->data);
  } else if (cudaMalloc(&rows, (nnz ? nnz : 1) * 4) != cudaSuccess ||
             cudaMalloc(&cols, (nnz ? nnz : 1) * 4) != cudaSuccess ||
             cudaMalloc(&vals, (nnz ? nnz : 1) * 8) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(rows);
    cudaFree(cols);
    return mm_fail(kNoMemory, "device allocation failed");
  }
  if (nnz) {
    cudaMemcpyAsync(rows, r.rows.data(), nnz * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(cols, r.cols.data(), nnz * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(vals, r.vals.data(), nnz * 8, cudaMemcpyHostToDevice, s);
  }
  spmvlab_cuda_coo d{r.m, r.n, nnz, rows, cols, vals};
  Arena ar(s);
  int rc = validate_coo(d, ar);  // read_matrix_market ends with validate(out) (matrix_market.hpp:187)
  ar.release();
  cudaStreamSynchronize(s);
  if (rc == kDuplicateEntry) g_last_error = "duplicate (row, col) coordinate";
  if (rc == kOk) rc = check_launch("read_matrix_market");
  if (rc != kOk) {
    if (!caller_buffers) {
      cudaFree(rows);
      cudaFree(cols);
      cudaFree(vals);
    }
    return rc;
  }
  *a = d;
  fill_header(r, header);
  return kOk;
}

int load_matrix(const char* path, spmvlab_cuda_coo* a, cudaStream_t s) {
  FILE* f = fopen(path, "rb");
  if (!f) return mm_fail(kIoError, std::string("cannot open ") + path);
  char head[8];
  const size_t got = fread(head, 1, 8, f);
  fclose(f);
  static const char magic[8] = {'S', 'P', 'M', 'V', 'L', 'A', 'B', '1'};
  if (got == 8 && std::memcmp(head, magic, 8) == 0) return cache_read(path, a, s);
  return mm_read_device(path, a, nullptr, s);
}

}  // namespace spmvcu
