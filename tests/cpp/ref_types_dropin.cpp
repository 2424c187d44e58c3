// ref_types_dropin.cpp -- the C++ drop-in (include/spmvlab_cuda/engine.hpp) driven with the
// reference's OWN types, helpers and acceptance criterion.  Compiled against the unmodified
// reference headers (/root/reference/proj/include, and proj/tests/oracles.hpp for the corpus
// generator random_matrix) by tests/cpp/Makefile where that tree exists; the binary travels to the
// GPU box and tests/test_gpu_dropin.py runs it.
//
// What it checks, per matrix of a randomized corpus (spmvlab::TripletMatrix from random_matrix,
// shuffled entry order, empty leading rows, an almost-dense row, shapes below one block):
//   * the oracle-equivalence criterion of /root/reference/proj/tests/acceptance.cpp:113-153 --
//     every engine at p in {1, 2, 4, 8}, BCOH rebuilt per p (its band count), y within
//     spmvlab::verify_rel_tolerance of spmvlab::spmv_triplet by spmvlab::relative_error, with
//     x = spmvlab::verification_input(n, idx + 1) -- through spmvlab::cuda::build_format /
//     run_spmv on the reference's TripletMatrix and DenseVector;
//   * storage_report(): the same array names and byte counts as spmvlab::storage_report of the
//     reference's own build_format;
//   * the CRS arrays bit for bit against the reference's triplet_to_crs, and SeqCrs y bit for bit
//     against the reference's spmv_crs_seq.
#include <algorithm>
#include <cstdio>
#include <random>
#include <string>
#include <variant>
#include <vector>

#include "oracles.hpp"          // reference test helper: RandomMatrixSpec, random_matrix
#include "spmvlab/bench.hpp"    // verification_input, relative_error, verify_rel_tolerance
#include "spmvlab/engine.hpp"   // the reference engines (CPU)
#include "spmvlab_cuda/engine.hpp"

namespace eng = spmvlab::cuda;  // the drop-in: swap this alias for `spmvlab` to run the CPU engines

static int failures = 0;
static long checks = 0;
static void expect(bool ok, const std::string& what) {
  ++checks;
  if (!ok && ++failures <= 20) std::printf("FAIL: %s\n", what.c_str());
}

static std::vector<spmvlab::TripletMatrix> corpus() {
  std::vector<spmvlab::TripletMatrix> out;
  std::mt19937_64 rng(424242);
  for (int t = 0; t < 60; ++t) {
    spmvlab::testing::RandomMatrixSpec spec;
    const int shape = t % 6;
    spec.m = shape == 0 ? 3 + rng() % 12 : (shape < 4 ? 1 + rng() % 300 : 200 + rng() % 1500);
    spec.n = shape == 0 ? 3 + rng() % 12 : (shape < 4 ? 1 + rng() % 300 : 200 + rng() % 1500);
    spec.density = shape == 0 ? 0.25 : 0.0005 + 0.004 * (t % 7);
    spec.leading_empty_rows = t % 4 == 1;
    if (t % 9 == 5) spec.dense_row_nnz = spec.n - spec.n / 10;
    out.push_back(spmvlab::testing::random_matrix(spec, rng()));
  }
  return out;
}

int main() {
  const auto mats = corpus();
  const std::vector<unsigned> worker_counts{1, 2, 4, 8};
  long runs = 0;
  for (std::size_t idx = 0; idx < mats.size(); ++idx) {
    const spmvlab::TripletMatrix& a = mats[idx];
    const spmvlab::DenseVector x = spmvlab::verification_input(a.n, idx + 1);
    const spmvlab::DenseVector expected = spmvlab::spmv_triplet(a, x);
    const std::string tag = "matrix " + std::to_string(idx) + " (" + std::to_string(a.m) + "x" +
                            std::to_string(a.n) + ", nnz " + std::to_string(a.data.size()) + ")";
    const eng::EngineOptions opt;
    // formats shared across p (the acceptance criterion builds these once)
    for (eng::Algorithm alg : {eng::Algorithm::SeqCrs, eng::Algorithm::ParCrs, eng::Algorithm::Merge,
                               eng::Algorithm::Csb, eng::Algorithm::Csbh, eng::Algorithm::MergeB,
                               eng::Algorithm::MergeBH}) {
      const eng::BuiltFormat f = eng::build_format(alg, a, 1, opt);
      const auto ref_alg = static_cast<spmvlab::Algorithm>(static_cast<int>(alg));
      const spmvlab::BuiltFormat rf = spmvlab::build_format(ref_alg, a, 1);
      const auto gs = eng::storage_report(f);
      const auto rs = spmvlab::storage_report(rf);
      expect(gs.arrays.size() == rs.arrays.size(), tag + " storage_report arrays " + eng::algorithm_name(alg));
      for (std::size_t i = 0; i < std::min(gs.arrays.size(), rs.arrays.size()); ++i)
        expect(gs.arrays[i].name == rs.arrays[i].name && gs.arrays[i].bytes == rs.arrays[i].bytes,
               tag + " storage_report " + eng::algorithm_name(alg) + " " + rs.arrays[i].name);
      if (alg == eng::Algorithm::SeqCrs) {
        const auto& crs = std::get<spmvlab::CrsMatrix>(rf);
        expect(f.download<std::uint32_t>("row_ptr") == crs.row_ptr, tag + " CRS row_ptr");
        expect(f.download<std::uint32_t>("col_ind") == crs.col_ind, tag + " CRS col_ind");
        expect(f.download<double>("data") == crs.data, tag + " CRS data");
        spmvlab::DenseVector y_ref(a.m, 0.0);
        spmvlab::spmv_crs_seq(crs, x, y_ref);
        expect(eng::run_spmv(alg, f, x, 1, opt) == y_ref, tag + " SeqCrs bitwise");
      }
      for (unsigned p : worker_counts) {
        const spmvlab::DenseVector y = eng::run_spmv(alg, f, x, p, opt);
        for (std::size_t i = 0; i < a.m; ++i)
          expect(spmvlab::relative_error(y[i], expected[i]) <= spmvlab::verify_rel_tolerance,
                 std::string("engine ") + eng::algorithm_name(alg) + " mismatch at p=" + std::to_string(p) + ", " +
                     tag + ", element " + std::to_string(i));
        ++runs;
      }
    }
    for (unsigned p : worker_counts) {
      for (eng::Algorithm alg :
           {eng::Algorithm::Bcoh, eng::Algorithm::Bcohc, eng::Algorithm::Bcohch, eng::Algorithm::Bcohchp}) {
        const eng::BuiltFormat f = eng::build_format(alg, a, p, opt);
        const spmvlab::BuiltFormat rf = spmvlab::build_format(static_cast<spmvlab::Algorithm>(static_cast<int>(alg)), a, p);
        expect(eng::storage_report(f).total() == spmvlab::storage_report(rf).total(),
               tag + " storage_report total " + eng::algorithm_name(alg) + " p=" + std::to_string(p));
        const spmvlab::DenseVector y = eng::run_spmv(alg, f, x, p, opt);
        for (std::size_t i = 0; i < a.m; ++i)
          expect(spmvlab::relative_error(y[i], expected[i]) <= spmvlab::verify_rel_tolerance,
                 std::string("engine ") + eng::algorithm_name(alg) + " mismatch at p=" + std::to_string(p) + ", " +
                     tag + ", element " + std::to_string(i));
        // the band-count check (spmv_parallel.hpp:339-341): p must equal the format's bands
        if (p > 1) {
          bool threw = false;
          try {
            (void)eng::run_spmv(alg, f, x, p - 1, opt);
          } catch (const eng::Error& e) {
            threw = e.kind() == eng::ErrorKind::InvalidArgument;
          }
          expect(threw, tag + " BCOH band mismatch must raise InvalidArgument");
        }
        ++runs;
      }
    }
  }
  std::printf("%zu matrices, %ld engine runs (11 engines x p in {1,2,4,8}), %ld checks, %d failures\n", mats.size(),
              runs, checks, failures);
  return failures ? 1 : 0;
}
