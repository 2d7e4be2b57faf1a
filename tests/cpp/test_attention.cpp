// Parity suite of the attention operators behind include/lorakv/attention.hpp, on the GPU, against
// the CPU oracle.  Mirrors what proj/tests/test_attention.cpp pins: closed-form
// cases, kernel-vs-oracle sweeps at 1e-10 (f64) / 1e-4 (f32), exact masking, softmax statistics,
// MAC counters, error paths and the GQA head mapping.
#include <cmath>
#include <vector>

#include "check.hpp"
#include "lorakv/attention.hpp"
#include "lorakv/fuzz.hpp"
#include "oracle_glue.hpp"

using namespace lorakv;

namespace {

template <class T>
struct Case {
  Matrix<T> q, k, v, v_lr, b_up;
  T scale = T(0.5);
  idx offset = 0;
  AttentionInputs<T> inputs() const {
    return AttentionInputs<T>{q.view(), k.view(), v.view(), v_lr.view(), b_up.view(), scale, offset};
  }
};

// same generator keys as the reference's random_case (test_attention.cpp:32-43)
template <class T>
Case<T> random_case(idx L, idx L_c, idx d, idx r, idx offset, std::uint64_t seed) {
  Rng rng(seed);
  Case<T> c;
  c.q = Matrix<T>::gaussian(L_c, d, rng.child(1), 1.0);
  c.k = Matrix<T>::gaussian(L, d, rng.child(2), 1.0);
  c.v = Matrix<T>::gaussian(L, d, rng.child(3), 1.0);
  c.v_lr = Matrix<T>::gaussian(L, r, rng.child(4), 1.0);
  c.b_up = Matrix<T>::gaussian(r, d, rng.child(5), 1.0);
  c.offset = offset;
  return c;
}

}  // namespace

TEST_CASE("single cached token returns v_base + scale * v_lr * B") {
  const Case<double> c = random_case<double>(1, 1, 8, 3, 0, 31);
  const Matrix<double> out = flash_lora_attention(c.inputs(), BlockConfig{});
  for (idx p = 0; p < 8; ++p) {
    double want = c.v(0, p);
    for (idx t = 0; t < 3; ++t) want += 0.5 * c.v_lr(0, t) * c.b_up(t, p);
    CHECK(std::abs(out(0, p) - want) <= 1e-12);
  }
}

TEST_CASE("device naive and flash kernels equal the oracle on random cases") {
  for (std::uint64_t seed : {40, 41, 42, 140, 141}) {
    const Case<double> c = random_case<double>(37, 11, 16, 4, 26, seed);
    const Matrix<double> want = oracle::naive(c.inputs());
    CHECK_LE(max_rel_error(naive_attention(c.inputs()), want), 1e-12);
    CHECK_LE(max_rel_error(flash_lora_attention(c.inputs(), BlockConfig{8, 8}), want), 1e-10);
    CHECK_LE(max_rel_error(expand_first_attention(c.inputs(), BlockConfig{3, 64}), want), 1e-10);
    const Case<float> f = random_case<float>(37, 11, 16, 4, 26, seed);
    const Matrix<float> wantf = oracle::naive(f.inputs());
    CHECK_LE(max_rel_error(flash_lora_attention(f.inputs(), BlockConfig{}), wantf), 1e-4);
    CHECK_LE(max_rel_error(expand_first_attention(f.inputs(), BlockConfig{}), wantf), 1e-4);
  }
}

TEST_CASE("zero queries give uniform weights over the visible prefix") {
  Case<double> c = random_case<double>(9, 9, 4, 2, 0, 47);
  for (double& x : c.q.data) x = 0.0;
  const Matrix<double> out = flash_lora_attention(c.inputs(), BlockConfig{4, 2});
  for (idx i = 0; i < 9; ++i)
    for (idx p = 0; p < 4; ++p) {
      double mean = 0.0;
      for (idx j = 0; j <= i; ++j) {
        double val = c.v(j, p);
        for (idx t = 0; t < 2; ++t) val += 0.5 * c.v_lr(j, t) * c.b_up(t, p);
        mean += val;
      }
      CHECK(std::abs(out(i, p) - mean / double(i + 1)) <= 1e-12);
    }
}

TEST_CASE("first row with offset 0 sees only token 0") {
  const Case<double> c = random_case<double>(12, 5, 8, 2, 0, 53);
  const Matrix<double> out = flash_lora_attention(c.inputs(), BlockConfig{2, 3});
  for (idx p = 0; p < 8; ++p) {
    double want = c.v(0, p);
    for (idx t = 0; t < 2; ++t) want += 0.5 * c.v_lr(0, t) * c.b_up(t, p);
    CHECK(std::abs(out(0, p) - want) <= 1e-12);
  }
}

TEST_CASE("kernel fuzz: 40 base cases x 16 tilings, f64 <= 1e-10 and f32 <= 1e-4") {
  const KernelFuzzResult d = run_kernel_fuzz<double>(40, 7001, 48);
  CHECK(d.comparisons == 640);
  CHECK_LE(d.max_rel(), 1e-10);
  const KernelFuzzResult f = run_kernel_fuzz<float>(40, 7002, 48);
  CHECK(f.comparisons == 640);
  CHECK_LE(f.max_rel(), 1e-4);
}

TEST_CASE("masked keys contribute exactly zero, even with 1e6 magnitudes") {
  // queries at positions 3..6 of a 20-token cache: keys 7..19 are invisible to every row
  Case<double> c = random_case<double>(20, 4, 8, 3, 3, 61);
  Case<double> cut = c;
  cut.k = Matrix<double>(7, 8); cut.v = Matrix<double>(7, 8); cut.v_lr = Matrix<double>(7, 3);
  for (idx j = 0; j < 7; ++j) {
    for (idx p = 0; p < 8; ++p) { cut.k(j, p) = c.k(j, p); cut.v(j, p) = c.v(j, p); }
    for (idx t = 0; t < 3; ++t) cut.v_lr(j, t) = c.v_lr(j, t);
  }
  for (idx j = 7; j < 20; ++j) {
    for (idx p = 0; p < 8; ++p) { c.k(j, p) = 1e6; c.v(j, p) = -1e6; }
    for (idx t = 0; t < 3; ++t) c.v_lr(j, t) = 1e6;
  }
  const Matrix<double> full = flash_lora_attention(c.inputs(), BlockConfig{2, 4});
  const Matrix<double> truncated = flash_lora_attention(cut.inputs(), BlockConfig{2, 4});
  CHECK(max_abs_diff(full, truncated) == 0.0);
}

TEST_CASE("online softmax statistics match the oracle") {
  const Case<double> c = random_case<double>(33, 9, 16, 2, 20, 83);
  OnlineSoftmaxStats<double> got, want;
  flash_lora_attention(c.inputs(), BlockConfig{4, 8}, nullptr, &got);
  oracle::flash(c.inputs(), BlockConfig{64, 64}, nullptr, &want);
  REQUIRE(got.row_max.size() == 9);
  for (std::size_t i = 0; i < 9; ++i) {
    CHECK(std::abs(got.row_max[i] - want.row_max[i]) <= 1e-12 * std::max(1.0, std::abs(want.row_max[i])));
    CHECK(std::abs(got.row_denom[i] - want.row_denom[i]) <= 1e-10 * want.row_denom[i]);
  }
}

TEST_CASE("closed-form MAC counts") {
  const LrMacCounts c = lr_mac_counts(4096, 1, 8, 128);
  CHECK(c.reorder == 33792u);
  CHECK(c.no_reorder == 4718592u);
}

TEST_CASE("AttnMacs equal the oracle's instrumented counters for random shapes and tilings") {
  Rng rng(97);
  for (int trial = 0; trial < 24; ++trial) {
    const idx L = 1 + idx(rng.next_u64() % 40), L_c = 1 + idx(rng.next_u64() % std::uint64_t(L));
    const idx d = idx(4) << (rng.next_u64() % 3), r = idx(rng.next_u64() % 5);
    const Case<double> c = random_case<double>(L, L_c, d, r, L - L_c, 1000 + trial);
    const BlockConfig cfg{1 + idx(rng.next_u64() % 9), 1 + idx(rng.next_u64() % 9)};
    AttnMacs got, want, got_e, want_e;
    flash_lora_attention(c.inputs(), cfg, &got);
    oracle::flash(c.inputs(), cfg, &want);
    expand_first_attention(c.inputs(), cfg, &got_e);
    oracle::expand_first(c.inputs(), cfg, &want_e);
    CHECK(got.qk == want.qk); CHECK(got.pv == want.pv); CHECK(got.lr == want.lr);
    CHECK(got.lr == lr_mac_counts(L, L_c, r, d).reorder);
    CHECK(got_e.qk == want_e.qk); CHECK(got_e.pv == want_e.pv); CHECK(got_e.lr == want_e.lr);
  }
}

TEST_CASE("rank 0 is plain attention and costs no low-rank MACs") {
  const Case<double> c = random_case<double>(25, 6, 8, 0, 19, 113);
  AttnMacs macs;
  const Matrix<double> out = flash_lora_attention(c.inputs(), BlockConfig{}, &macs);
  CHECK(macs.lr == 0u);
  CHECK_LE(max_rel_error(out, oracle::naive(c.inputs())), 1e-12);
}

TEST_CASE("bad block sizes, offsets and shapes throw std::runtime_error") {
  const Case<double> c = random_case<double>(10, 4, 8, 2, 6, 127);
  CHECK_THROWS_AS(flash_lora_attention(c.inputs(), BlockConfig{0, 8}), std::runtime_error);
  CHECK_THROWS_AS(expand_first_attention(c.inputs(), BlockConfig{8, 0}), std::runtime_error);
  Case<double> bad = c;
  bad.offset = 7;
  CHECK_THROWS_WITH_AS(flash_lora_attention(bad.inputs(), BlockConfig{}), "exceeds L", std::runtime_error);
  bad = c;
  bad.v_lr = Matrix<double>(9, 2);
  CHECK_THROWS_WITH_AS(flash_lora_attention(bad.inputs(), BlockConfig{}), "v_lr rows", std::runtime_error);
  bad = c;
  bad.v = Matrix<double>(10, 7);
  CHECK_THROWS_WITH_AS(naive_attention(bad.inputs()), "10x7", std::runtime_error);
}

TEST_CASE("gqa_attention: head mapping, shared V_lr, per-kv-head slices of B") {
  const idx L = 29, L_c = 5, d = 8, r = 3, n_q = 6, n_kv = 2;
  Rng rng(149);
  const Matrix<double> q = Matrix<double>::gaussian(L_c, n_q * d, rng.child(1), 1.0);
  const Matrix<double> k = Matrix<double>::gaussian(L, n_kv * d, rng.child(2), 1.0);
  const Matrix<double> v = Matrix<double>::gaussian(L, n_kv * d, rng.child(3), 1.0);
  const Matrix<double> v_lr = Matrix<double>::gaussian(L, r, rng.child(4), 1.0);
  const Matrix<double> b = Matrix<double>::gaussian(r, n_kv * d, rng.child(5), 1.0);
  AttnMacs macs;
  const Matrix<double> got = gqa_attention(q.view(), k.view(), v.view(), v_lr.view(), b.view(), 0.5, L - L_c, n_q, n_kv,
                                           BlockConfig{}, &macs);
  CHECK_LE(max_rel_error(got, oracle::gqa(q.view(), k.view(), v.view(), v_lr.view(), b.view(), 0.5, L - L_c, n_q, n_kv)), 1e-10);
  CHECK(macs.qk == std::uint64_t(n_q * L_c * L * d));
  // every q head equals the per-head operator on its column slices
  const idx group = n_q / n_kv;
  for (idx h = 0; h < n_q; ++h) {
    const idx kv = h / group;
    AttentionInputs<double> in{q.view().col_range(h * d, (h + 1) * d), k.view().col_range(kv * d, (kv + 1) * d),
                               v.view().col_range(kv * d, (kv + 1) * d), v_lr.view(),
                               b.view().col_range(kv * d, (kv + 1) * d), 0.5, L - L_c};
    const Matrix<double> head = flash_lora_attention(in, BlockConfig{});
    for (idx i = 0; i < L_c; ++i)
      for (idx p = 0; p < d; ++p) CHECK(std::abs(head(i, p) - got(i, h * d + p)) <= 1e-12);
  }
  CHECK_THROWS_WITH_AS(gqa_attention(q.view(), k.view(), v.view(), v_lr.view(), b.view(), 0.5, L - L_c, idx(6), idx(4), BlockConfig{}),
                       "not divisible", std::runtime_error);
}
