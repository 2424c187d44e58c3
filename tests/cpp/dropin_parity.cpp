// dropin_parity.cpp -- exercises the C++ drop-in header (include/spmvlab_cuda/engine.hpp) exactly
// the way the reference's callers use include/spmvlab/engine.hpp (build_format / run_spmv /
// storage_report on host vectors), and checks every engine against the C oracle
// (oracle/spmv_oracle.c, test infrastructure linked only into this test binary).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "spmv_oracle.h"
#include "spmvlab_cuda/engine.hpp"

namespace sc = spmvlab::cuda;

// Same members as spmvlab::TripletMatrix (inc/triplet.hpp:30-38).
struct TripletMatrix {
  std::uint32_t m = 0, n = 0;
  std::vector<std::uint32_t> row_ind, col_ind;
  std::vector<double> data;
};

static int failures = 0, checks = 0;
#define EXPECT(cond, ...)                   \
  do {                                      \
    ++checks;                               \
    if (!(cond)) {                          \
      ++failures;                           \
      std::printf("FAIL: " __VA_ARGS__);    \
      std::printf("\n");                    \
    }                                       \
  } while (0)

static TripletMatrix random_matrix(std::uint32_t m, std::uint32_t n, double density, std::uint64_t seed,
                                   std::uint32_t dense_row = 0) {
  std::mt19937_64 rng(seed);
  std::set<std::pair<std::uint32_t, std::uint32_t>> coords;
  const auto target = static_cast<std::size_t>(density * m * n);
  while (coords.size() < target) coords.emplace(rng() % m, rng() % n);
  for (std::uint32_t k = 0; k < dense_row && k < n; ++k) coords.emplace(0, k);
  TripletMatrix a;
  a.m = m;
  a.n = n;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> v(coords.begin(), coords.end());
  std::shuffle(v.begin(), v.end(), rng);
  for (auto [r, c] : v) {
    a.row_ind.push_back(r);
    a.col_ind.push_back(c);
    a.data.push_back(std::uniform_real_distribution<double>(-1.0, 1.0)(rng));
  }
  return a;
}

static void check_matrix(const TripletMatrix& a, const std::string& tag, std::uint64_t l2) {
  std::vector<double> x(a.n);
  orc_verification_input(a.n, 5, x.data());
  std::vector<double> bound(a.m);
  orc_abs_spmv(a.m, a.data.size(), a.row_ind.data(), a.col_ind.data(), a.data.data(), x.data(), bound.data());
  for (sc::Algorithm alg : sc::all_algorithms) {
    for (unsigned p : {1u, 4u}) {
      sc::EngineOptions opt;
      opt.l2_bytes = l2;
      sc::BuiltFormat f = sc::build_format(alg, a, p, opt);
      orc_format* ref = nullptr;
      const int rc = orc_build_format(static_cast<int>(alg), a.m, a.n, a.data.size(), a.row_ind.data(),
                                      a.col_ind.data(), a.data.data(), p, l2, &ref);
      EXPECT(rc == 0, "%s oracle build failed", tag.c_str());
      const sc::StorageBreakdown rep = sc::storage_report(f);
      EXPECT(static_cast<int>(rep.arrays.size()) == ref->nstorage, "%s %s storage count", tag.c_str(),
             sc::algorithm_name(alg));
      for (int i = 0; i < ref->nstorage && i < static_cast<int>(rep.arrays.size()); ++i) {
        const orc_array& ra = ref->arrays[i];
        EXPECT(rep.arrays[i].name == ra.name && rep.arrays[i].bytes == ra.bytes, "%s %s array %s bytes",
               tag.c_str(), sc::algorithm_name(alg), ra.name);
        const std::vector<unsigned char> got = f.download<unsigned char>(ra.name);
        EXPECT(got.size() == ra.bytes && (ra.bytes == 0 || std::memcmp(got.data(), ra.data, ra.bytes) == 0),
               "%s %s array %s differs", tag.c_str(), sc::algorithm_name(alg), ra.name);
      }
      {  // *_to_triplet: storage-order coordinates and values bitwise the oracle's
        const TripletMatrix t = sc::to_triplet<TripletMatrix>(f);
        const std::size_t nnz = a.data.size();
        std::vector<std::uint32_t> rr(nnz), rc(nnz);
        std::vector<double> rv(nnz);
        orc_format_to_triplet(ref, rr.data(), rc.data(), rv.data());
        EXPECT(t.row_ind == rr && t.col_ind == rc && t.data == rv, "%s %s to_triplet differs", tag.c_str(),
               sc::algorithm_name(alg));
      }
      if (alg == sc::Algorithm::Csb || alg == sc::Algorithm::Csbh) {
        for (std::size_t thr : {std::size_t{0}, std::size_t{1}, std::size_t{9}}) {
          const std::vector<spmvlab_cuda_csb_item> got = sc::csb_work_items(f, thr);
          std::uint64_t cnt = 0;
          orc_csb_work_items(ref, thr, nullptr, 0, &cnt);
          std::vector<orc_csb_item> want(cnt);
          orc_csb_work_items(ref, thr, want.data(), cnt, &cnt);
          EXPECT(got.size() == want.size() &&
                     (want.empty() || std::memcmp(got.data(), want.data(), sizeof(orc_csb_item) * cnt) == 0),
                 "%s %s csb_work_items(%zu) differs", tag.c_str(), sc::algorithm_name(alg), thr);
        }
      }
      const std::vector<double> y = sc::run_spmv(alg, f, x, p, opt);
      std::vector<double> yr(a.m);
      orc_run_spmv(static_cast<int>(alg), ref, x.data(), x.size(), yr.data(), yr.size(), p, 0);
      for (std::uint32_t i = 0; i < a.m; ++i)
        EXPECT(std::fabs(y[i] - yr[i]) <= 1e-12 * bound[i], "%s %s y[%u] %.17g vs %.17g", tag.c_str(),
               sc::algorithm_name(alg), i, y[i], yr[i]);
      orc_free_format(ref);
    }
  }
}

int main() {
  // E4 (tests/oracles.hpp:37-44): y = [3, 3, 0, 9] for every engine.
  TripletMatrix e4;
  e4.m = e4.n = 4;
  e4.row_ind = {0, 0, 1, 3, 3};
  e4.col_ind = {0, 2, 1, 0, 3};
  e4.data = {1, 2, 3, 4, 5};
  for (sc::Algorithm alg : sc::all_algorithms) {
    sc::BuiltFormat f = sc::build_format(alg, e4, 2);
    const std::vector<double> y = sc::run_spmv(alg, f, std::vector<double>(4, 1.0), 2);
    EXPECT(y == (std::vector<double>{3, 3, 0, 9}), "e4 %s", sc::algorithm_name(alg));
  }
  // build_format_beta: the per-format builders at explicit block sizes, every array bitwise the oracle's
  {
    const TripletMatrix a = random_matrix(200, 150, 0.04, 21, 150);
    for (sc::Algorithm alg : sc::all_algorithms) {
      if (static_cast<int>(alg) <= 2) continue;
      for (unsigned lb : {1u, 3u, 6u}) {
        const unsigned p = 3;
        sc::BuiltFormat f = sc::build_format_beta(alg, a, lb, p);
        orc_format* ref = nullptr;
        const int rc = orc_build_format_beta(static_cast<int>(alg), a.m, a.n, a.data.size(), a.row_ind.data(),
                                             a.col_ind.data(), a.data.data(), lb, p, &ref);
        EXPECT(rc == 0, "oracle build_beta failed");
        for (int i = 0; rc == 0 && i < ref->nstorage; ++i) {
          const orc_array& ra = ref->arrays[i];
          const std::vector<unsigned char> got = f.download<unsigned char>(ra.name);
          EXPECT(got.size() == ra.bytes && (ra.bytes == 0 || std::memcmp(got.data(), ra.data, ra.bytes) == 0),
                 "build_format_beta %s lb %u array %s differs", sc::algorithm_name(alg), lb, ra.name);
        }
        orc_free_format(ref);
      }
    }
    bool thrown = false;
    try {
      sc::build_format_beta(sc::Algorithm::Bcoh, a, 16, 2);
    } catch (const sc::Error& e) {
      thrown = e.kind() == sc::ErrorKind::InvalidArgument;
    }
    EXPECT(thrown, "BCOH beta 2^16 not rejected");
  }
  check_matrix(random_matrix(300, 250, 0.03, 11, 250), "rand300", 4096);
  check_matrix(random_matrix(1000, 1200, 0.01, 12), "rand1000", 512 * 1024);
  check_matrix(random_matrix(77, 5, 0.3, 13), "tall", 64);
  // iterate_device: 10 SeqCrs iterations are bitwise the oracle's repeated sequential CRS multiply
  {
    TripletMatrix a = random_matrix(400, 400, 0.02, 14, 400);
    for (double& v : a.data) v = std::fabs(v);
    sc::BuiltFormat f = sc::build_format(sc::Algorithm::SeqCrs, a, 1);
    orc_format* ref = nullptr;
    orc_build_format(0, a.m, a.n, a.data.size(), a.row_ind.data(), a.col_ind.data(), a.data.data(), 1, 512 * 1024,
                     &ref);
    std::vector<double> x(a.n), y(a.n);
    orc_verification_input(a.n, 9, x.data());
    double *xd = nullptr, *wd = nullptr;
    cudaMalloc(&xd, 8 * a.n);
    cudaMalloc(&wd, 8 * a.n);
    cudaMemcpy(xd, x.data(), 8 * a.n, cudaMemcpyHostToDevice);
    sc::iterate_device(sc::Algorithm::SeqCrs, f, xd, wd, 10, 1);
    std::vector<double> got(a.n);
    cudaMemcpy(got.data(), xd, 8 * a.n, cudaMemcpyDeviceToHost);
    for (int k = 0; k < 10; ++k) {
      orc_run_spmv(0, ref, x.data(), x.size(), y.data(), y.size(), 1, 0);
      std::swap(x, y);
    }
    EXPECT(got == x, "iterate_device SeqCrs x_10 differs from the oracle loop");
    cudaFree(xd);
    cudaFree(wd);
    orc_free_format(ref);
  }
  // errors: DimensionMismatch (spmv_parallel.hpp:90-99), band mismatch (:339-341)
  {
    sc::BuiltFormat f = sc::build_format(sc::Algorithm::Merge, e4, 1);
    std::vector<double> x(3, 1.0), y(4);
    bool thrown = false;
    try {
      sc::run_spmv(sc::Algorithm::Merge, f, x, y, 1);
    } catch (const sc::Error& e) {
      thrown = e.kind() == sc::ErrorKind::DimensionMismatch;
    }
    EXPECT(thrown, "DimensionMismatch not raised");
    sc::BuiltFormat b = sc::build_format(sc::Algorithm::Bcohch, e4, 2);
    thrown = false;
    try {
      std::vector<double> x4(4, 1.0);
      sc::run_spmv(sc::Algorithm::Bcohch, b, x4, y, 3);
    } catch (const sc::Error& e) {
      thrown = e.kind() == sc::ErrorKind::InvalidArgument;
    }
    EXPECT(thrown, "band mismatch not raised");
  }
  std::printf("%s: %d checks, %d failures\n", failures ? "FAIL" : "PASS", checks, failures);
  return failures ? 1 : 0;
}
