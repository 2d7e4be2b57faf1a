// Adapter containers and the decomposed forward (include/lorakv/lora.hpp) against the CPU oracle;
// mirrors proj/tests/test_lora.cpp and the matmul pins of proj/tests/test_matrix.cpp:43-68.
#include <cmath>

#include "check.hpp"
#include "lorakv/lora.hpp"
#include "oracle_glue.hpp"

using namespace lorakv;

namespace {
template <class T>
LoraAdapter<T> make_adapter(idx d_in, idx d_out, idx r, double alpha, std::uint64_t seed_a, std::uint64_t seed_b) {
  return LoraAdapter<T>(Matrix<T>::gaussian(d_in, r, Rng(seed_a), 1.0 / std::sqrt(double(d_in))),
                        Matrix<T>::gaussian(r, d_out, Rng(seed_b), 0.02), r, alpha);
}
}  // namespace

TEST_CASE("device matmul reproduces the reference's triple loop bit for bit") {
  const Matrix<double> a = Matrix<double>::gaussian(13, 29, Rng(1), 1.0), b = Matrix<double>::gaussian(29, 7, Rng(2), 1.0);
  CHECK(max_abs_diff(matmul(a, b), oracle::matmul(a, b)) == 0.0);
  const Matrix<float> af = Matrix<float>::gaussian(33, 65, Rng(3), 1.0), bf = Matrix<float>::gaussian(65, 17, Rng(4), 1.0);
  CHECK(max_abs_diff(matmul(af, bf), oracle::matmul(af, bf)) == 0.0);
  CHECK_THROWS_WITH_AS(matmul(Matrix<double>(2, 3), Matrix<double>(4, 5)), "2x3", std::runtime_error);
}

TEST_CASE("adapter invariants") {
  CHECK_THROWS_AS(LoraAdapter<double>(Matrix<double>(8, 0), Matrix<double>(0, 8), 0, 16.0), std::runtime_error);
  CHECK_THROWS_AS(LoraAdapter<double>(Matrix<double>(8, 2), Matrix<double>(3, 8), 2, 16.0), std::runtime_error);
  CHECK_THROWS_AS(LoraAdapter<double>(Matrix<double>(2, 4), Matrix<double>(4, 8), 4, 16.0), std::runtime_error);
  CHECK_THROWS_AS(LoraAdapter<double>(Matrix<double>(8, 2), Matrix<double>(2, 8), 2, 0.0), std::runtime_error);
  const LoraAdapter<double> ok = make_adapter<double>(8, 6, 2, 16.0, 5, 6);
  CHECK(ok.d_in() == 8); CHECK(ok.d_out() == 6); CHECK(ok.lora_scale() == 8.0);
}

TEST_CASE("shared-A equality is enforced") {
  const Matrix<double> w = Matrix<double>::gaussian(8, 6, Rng(7), 1.0);
  std::vector<LoraAdapter<double>> same{make_adapter<double>(8, 6, 2, 16.0, 8, 9), make_adapter<double>(8, 6, 2, 16.0, 8, 10)};
  CHECK_NOTHROW(MultiLoraSet<double>(w, same, true));
  std::vector<LoraAdapter<double>> differ{make_adapter<double>(8, 6, 2, 16.0, 8, 9), make_adapter<double>(8, 6, 2, 16.0, 11, 10)};
  CHECK_THROWS_WITH_AS(MultiLoraSet<double>(w, differ, true), "down-projections differ", std::runtime_error);
  CHECK_NOTHROW(MultiLoraSet<double>(w, differ, false));
  const MultiLoraSet<double> set(w, same, true);
  CHECK_THROWS_WITH_AS(set.adapter(2), "out of range", std::runtime_error);
}

TEST_CASE("decomposed forward equals the merged weight; y_lr is unscaled and agent-independent under shared A") {
  const idx d_in = 24, d_out = 16, r = 4;
  const Matrix<double> w = Matrix<double>::gaussian(d_in, d_out, Rng(12), 1.0 / std::sqrt(double(d_in)));
  std::vector<LoraAdapter<double>> ads{make_adapter<double>(d_in, d_out, r, 16.0, 13, 14), make_adapter<double>(d_in, d_out, r, 16.0, 13, 15)};
  const MultiLoraSet<double> set(w, ads, true);
  const Matrix<double> x = Matrix<double>::gaussian(9, d_in, Rng(16), 1.0);
  const ForwardParts<double> p0 = forward_decomposed(set, 0, x), p1 = forward_decomposed(set, 1, x);
  CHECK(max_abs_diff(p0.y_lr, p1.y_lr) == 0.0);
  CHECK(max_abs_diff(p0.y_lr, oracle::matmul(x, ads[0].a)) == 0.0);
  // merged weight W0 + s * A B, composed on the CPU checker
  Matrix<double> merged = oracle::matmul(ads[1].a, ads[1].b);
  for (std::size_t i = 0; i < merged.data.size(); ++i) merged.data[i] = w.data[i] + 4.0 * merged.data[i];
  CHECK_LE(max_rel_error(p1.y_full, oracle::matmul(x, merged)), 1e-12);
  CHECK_THROWS_AS(forward_decomposed(set, 0, Matrix<double>(3, d_in + 1)), std::runtime_error);
}

TEST_CASE("expand_lr matches the oracle bit for bit; doubling alpha doubles it exactly") {
  const LoraAdapter<double> ad = make_adapter<double>(12, 10, 3, 16.0, 17, 18);
  const Matrix<double> y = Matrix<double>::gaussian(7, 3, Rng(19), 1.0);
  Matrix<double> want(7, 10);
  oracle::ok(orc_expand_lr_f64(oracle::sp(y.view()), oracle::sp(ad.b.view()), 3, 16.0, want.data.data()));
  const Matrix<double> got = expand_lr(y, ad);
  CHECK(max_abs_diff(got, want) == 0.0);
  const LoraAdapter<double> twice(ad.a, ad.b, 3, 32.0);
  const Matrix<double> got2 = expand_lr(y, twice);
  for (std::size_t i = 0; i < got.data.size(); ++i) CHECK(got2.data[i] == 2.0 * got.data[i]);
  CHECK_THROWS_WITH_AS(expand_lr(Matrix<double>(7, 4), ad), "rank mismatch", std::runtime_error);
}
