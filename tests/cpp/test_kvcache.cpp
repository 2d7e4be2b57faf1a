// The scheme-aware cache store behind include/lorakv/kvcache.hpp (paged HBM pool + host bookkeeping).
// Mirrors proj/tests/test_kvcache.cpp: planner intervals, first-writer-wins, the gap / forbidden
// errors, exact byte identities, monotone seen_upto -- all integer results bit-exact -- plus the page
// table, which the reference does not have (first-touch order, checked against the oracle's page model).
#include <cstdint>
#include <vector>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>

#include "check.hpp"
#include "lorakv/kvcache.hpp"
#include "oracle_glue.hpp"

using namespace lorakv;

namespace {

Matrix<float> fill_rows(idx rows, idx cols, float tag) {   // small integers: exact in fp32 and bf16-free
  Matrix<float> m(rows, cols);
  for (idx i = 0; i < rows; ++i)
    for (idx j = 0; j < cols; ++j) m(i, j) = tag + float(i * cols + j);
  return m;
}

bool same(Span2D<const float> a, const Matrix<float>& b) {
  if (a.rows != b.rows || a.cols != b.cols) return false;
  for (idx i = 0; i < a.rows; ++i)
    for (idx j = 0; j < a.cols; ++j)
      if (a(i, j) != b(i, j)) return false;
  return true;
}

CacheScheme scheme(SchemeKind k) { return CacheScheme{k, {}}; }

}  // namespace

TEST_CASE("plan_core: cold start plans the fresh range under every scheme") {
  for (SchemeKind k : {SchemeKind::NonShared, SchemeKind::FullShared, SchemeKind::BaseShared, SchemeKind::BaseLRShared}) {
    const PrefillPlan p = plan_core(scheme(k), 0, 0, 128);
    CHECK(p.hidden_pass == (Interval{0, 128}));
    CHECK(p.kv_project == (Interval{0, 128}));
    CHECK(p.lr_project == (Interval{0, 128}));
  }
  CHECK_THROWS_AS(plan_core(scheme(SchemeKind::FullShared), 10, 11, 1), std::runtime_error);
  CHECK_THROWS_AS(plan_core(scheme(SchemeKind::FullShared), 10, 0, -1), std::runtime_error);
}

TEST_CASE("plan_core: an agent switch after 1000 tokens") {
  // the agent last saw 200 tokens, the trajectory holds 1000 and 16 new tokens arrive
  const Interval fresh{1000, 1016}, unseen{200, 1016};
  PrefillPlan p = plan_core(scheme(SchemeKind::NonShared), 1000, 200, 16);
  CHECK(p.hidden_pass == unseen); CHECK(p.kv_project == unseen); CHECK(p.lr_project == unseen);
  p = plan_core(scheme(SchemeKind::FullShared), 1000, 200, 16);
  CHECK(p.hidden_pass == fresh); CHECK(p.kv_project == fresh); CHECK(p.lr_project == fresh);
  p = plan_core(scheme(SchemeKind::BaseShared), 1000, 200, 16);
  CHECK(p.hidden_pass == unseen); CHECK(p.kv_project == fresh); CHECK(p.lr_project == unseen);
  p = plan_core(scheme(SchemeKind::BaseLRShared), 1000, 200, 16);
  CHECK(p.hidden_pass == fresh); CHECK(p.kv_project == fresh); CHECK(p.lr_project == fresh);
  // the oracle's restatement of plan_core agrees on every field
  for (int k = 0; k < 4; ++k) {
    std::int64_t want[9];
    oracle::ok(orc_plan_core(k, 0, 1000, 200, 16, want));
    const PrefillPlan g = plan_core(scheme(static_cast<SchemeKind>(k)), 1000, 200, 16);
    CHECK(g.hidden_pass.begin == want[0]); CHECK(g.hidden_pass.end == want[1]);
    CHECK(g.kv_project.begin == want[2]); CHECK(g.lr_project.begin == want[4]);
  }
}

TEST_CASE("first writer wins; a gap is an error") {
  KvStore<float> st(scheme(SchemeKind::BaseLRShared), StoreDims{2, 8, 16, 4, 3}, DeviceOptions{2, 256});
  const Matrix<float> k0 = fill_rows(10, 8, 0.f), k1 = fill_rows(10, 8, 500.f);
  st.append_tokens(std::vector<std::int32_t>(10, 7));
  st.append_key(0, 0, 0, k0.view());
  st.append_key(0, 1, 0, k1.view());                 // second writer: content unchanged
  CHECK(same(st.key_view(0, 2), k0));
  const Matrix<float> tail = fill_rows(6, 8, 900.f);  // rows 8..13: only 10..13 are new
  st.append_key(0, 1, 8, tail.view());
  const Span2D<const float> kv = st.key_view(0, 0);
  REQUIRE(kv.rows == 14);
  CHECK(kv(9, 0) == k0(9, 0));
  CHECK(kv(10, 0) == tail(2, 0));
  CHECK_THROWS_WITH_AS(st.append_key(0, 0, 20, k0.view()), "gap", std::runtime_error);
  CHECK_THROWS_WITH_AS(st.append_value(1, 0, 1, k0.view()), "gap at row 0", std::runtime_error);
  CHECK_THROWS_AS(st.append_key(2, 0, 0, k0.view()), std::runtime_error);     // layer out of range
  CHECK_NOTHROW(st.key_view(0, 3));   // shared caches ignore the agent index (kvcache.hpp:307-311)
}

TEST_CASE("FullShared: a second writer adds no bytes; NonShared keeps disjoint caches") {
  KvStore<float> fs(scheme(SchemeKind::FullShared), StoreDims{1, 8, 16, 0, 2}, DeviceOptions{1, 128});
  const Matrix<float> rows = fill_rows(5, 8, 1.f);
  fs.append_key(0, 0, 0, rows.view()); fs.append_value(0, 0, 0, rows.view());
  const CacheBytes before = fs.bytes();
  fs.append_key(0, 1, 0, rows.view()); fs.append_value(0, 1, 0, rows.view());
  CHECK(fs.bytes().total() == before.total());
  CHECK(before.key == 5u * 8u * sizeof(float));
  CHECK(fs.lr_view(0, 0).rows == 5); CHECK(fs.lr_view(0, 0).cols == 0);
  CHECK_THROWS_WITH_AS(fs.append_lr(0, 0, 0, Matrix<float>(5, 0).view()), "has no LR cache", std::runtime_error);

  KvStore<float> ns(scheme(SchemeKind::NonShared), StoreDims{1, 8, 16, 0, 2}, DeviceOptions{1, 128});
  const Matrix<float> other = fill_rows(3, 8, 100.f);
  ns.append_key(0, 0, 0, rows.view()); ns.append_key(0, 1, 0, other.view());
  CHECK(same(ns.key_view(0, 0), rows)); CHECK(same(ns.key_view(0, 1), other));
  CHECK(ns.bytes().key == (5u + 3u) * 8u * sizeof(float));
  CHECK_THROWS_WITH_AS(ns.key_view(0, 2), "unknown agent", std::runtime_error);
}

TEST_CASE("overwrites are forbidden; schemes without a hidden cache say so") {
  KvStore<float> st(scheme(SchemeKind::BaseShared), StoreDims{1, 8, 16, 2, 2}, DeviceOptions{1, 64});
  const Matrix<float> rows = fill_rows(2, 8, 0.f);
  CHECK_THROWS_WITH_AS(st.recompute_overwrite(0, 0, rows.view(), rows.view()), "forbidden", std::runtime_error);
  CHECK_THROWS_WITH_AS(st.append_hidden(0, rows.view()), "no hidden-state cache", std::runtime_error);
  // SelectiveRecompute (kvcache.hpp:229-246, 289-305): needs a recompute set; keeps one hidden-state cache; only its recompute
  // layers may overwrite rows that exist (the rest stays first-writer-wins)
  CHECK_THROWS_WITH_AS(KvStore<float>(CacheScheme{SchemeKind::SelectiveRecompute, {}}, StoreDims{1, 8, 16, 2, 2}), "non-empty recompute set",
                       std::runtime_error);
  KvStore<float> sel(CacheScheme{SchemeKind::SelectiveRecompute, {1}}, StoreDims{2, 8, 16, 0, 2}, DeviceOptions{1, 64});
  const Matrix<float> hid = fill_rows(2, 16, 50.f), other = fill_rows(2, 8, 7.f);
  for (idx l = 0; l < 2; ++l) { sel.append_key(l, 0, 0, rows.view()); sel.append_value(l, 0, 0, rows.view()); }
  sel.append_hidden(0, hid.view());
  CHECK(sel.hidden_size() == 2);
  CHECK(same(sel.hidden_rows(0, 2), hid));
  CHECK(sel.bytes().hidden == 2u * 16u * sizeof(float));
  CHECK_THROWS_WITH_AS(sel.recompute_overwrite(0, 0, other.view(), other.view()), "forbidden", std::runtime_error);
  sel.recompute_overwrite(1, 0, other.view(), other.view());
  CHECK(same(sel.key_view(1, 0), other)); CHECK(same(sel.value_view(1, 1), other)); CHECK(same(sel.key_view(0, 0), rows));
  CHECK_THROWS_WITH_AS(sel.recompute_overwrite(1, 1, other.view(), other.view()), "not materialized", std::runtime_error);
  // KvStore<double>: fp64 pages keep every bit; a copy is a second pool with equal contents
  KvStore<double> dbl(scheme(SchemeKind::BaseLRShared), StoreDims{1, 8, 16, 2, 2}, DeviceOptions{1, 64});
  Matrix<double> fine(3, 8);
  for (std::size_t i = 0; i < fine.data.size(); ++i) fine.data[i] = 1.0 / 3.0 + 1e-13 * double(i);
  dbl.append_tokens({1, 2, 3}); dbl.append_key(0, 0, 0, fine.view()); dbl.mark_seen(1);
  const auto kv = dbl.key_view(0, 0);
  CHECK(kv.rows == 3);
  for (idx i = 0; i < 3; ++i) for (idx j = 0; j < 8; ++j) CHECK(kv(i, j) == fine(i, j));
  CHECK(dbl.bytes().key == 3u * 8u * sizeof(double));
  const KvStore<double> twin = dbl;
  CHECK(twin == dbl); CHECK(twin.seen(1) == 3); CHECK(twin.seen(0) == 0);
  CHECK_THROWS_WITH_AS(CacheScheme::parse("Shared"), "unknown cache scheme", std::runtime_error);
  CHECK(CacheScheme::parse("BaseLRShared").kind == SchemeKind::BaseLRShared);
}

TEST_CASE("byte ratios are the exact rationals 1/N + r/d_out, 1/N + r/(N d_out) and 1/N") {
  for (idx r : {4, 8, 16, 32})
    for (idx d_out : {256, 1024}) {
      const idx N = 3, L = 40, layers = 2;
      auto fill = [&](SchemeKind k) {
        KvStore<float> st(scheme(k), StoreDims{layers, d_out, 64, r, N}, DeviceOptions{d_out / 64, 64});
        const Matrix<float> kv = fill_rows(L, d_out, 0.f), lr = fill_rows(L, r, 0.f);
        for (idx a = 0; a < N; ++a)
          for (idx l = 0; l < layers; ++l) {
            st.append_key(l, a, 0, kv.view()); st.append_value(l, a, 0, kv.view());
            if (k == SchemeKind::BaseShared || k == SchemeKind::BaseLRShared) st.append_lr(l, a, 0, lr.view());
          }
        CHECK(st.bytes().total() == st.allocated_elements() * sizeof(float));
        return st.bytes();
      };
      const CacheBytes ns = fill(SchemeKind::NonShared), bs = fill(SchemeKind::BaseShared), bl = fill(SchemeKind::BaseLRShared);
      const std::uint64_t n = N, d = std::uint64_t(d_out), rr = std::uint64_t(r);
      CHECK(bs.key * n == ns.key); CHECK(bl.key * n == ns.key);
      CHECK((bs.value + bs.lr) * n * d == ns.value * (d + n * rr));     // 1/N + r/d_out
      CHECK((bl.value + bl.lr) * n * d == ns.value * (d + rr));         // 1/N + r/(N d_out)
    }
}

TEST_CASE("seen_upto is monotone; plan_step reads the store") {
  KvStore<float> st(scheme(SchemeKind::BaseShared), StoreDims{1, 8, 16, 2, 2}, DeviceOptions{1, 64});
  st.append_tokens(std::vector<std::int32_t>(12, 1));
  st.mark_seen(0);
  CHECK(st.seen(0) == 12); CHECK(st.seen(1) == 0);
  st.append_tokens(std::vector<std::int32_t>(3, 2));
  CHECK(st.length() == 15); CHECK(st.tokens().size() == 15u);
  const PrefillPlan p = plan_step(st, 1, 4);
  CHECK(p.hidden_pass == (Interval{0, 19})); CHECK(p.kv_project == (Interval{15, 19})); CHECK(p.lr_project == (Interval{0, 19}));
  st.mark_seen(1);
  CHECK(st.seen(1) == 15);
  CHECK_THROWS_AS(st.seen(2), std::runtime_error);
}

TEST_CASE("pages are handed out in first-touch order (logical row -> row / P, row % P)") {
  const idx P = 16;
  KvStore<float> st(scheme(SchemeKind::NonShared), StoreDims{1, 8, 16, 0, 2}, DeviceOptions{1, 256, false, P});
  const Matrix<float> a = fill_rows(20, 8, 0.f), b = fill_rows(40, 8, 0.f);
  st.append_key(0, 1, 0, a.view());       // agent 1 touches logical pages 0,1 first -> physical 0,1
  st.append_key(0, 0, 0, b.view());       // agent 0: logical 0,1,2 -> physical 2,3,4
  st.append_key(0, 1, 20, a.view());      // agent 1 grows to 40 rows: logical 2 -> physical 5
  std::int64_t page, slot;
  orc_page_of(39, P, &page, &slot);
  CHECK(page == 2); CHECK(slot == 7);
  CHECK(st.page_table(LORAKV_KEY, 1) == (std::vector<std::int32_t>{0, 1, 5}));
  CHECK(st.page_table(LORAKV_KEY, 0) == (std::vector<std::int32_t>{2, 3, 4}));
  CHECK(same(st.key_view(0, 0), b));
}

// test_kvcache.cpp:279-305 of the reference: a snapshot round-trips bit-exactly and re-dumps identically
TEST_CASE("snapshot round-trips bit-exactly and re-dumps identically (paged store)") {
  for (SchemeKind kind : {SchemeKind::NonShared, SchemeKind::FullShared, SchemeKind::BaseShared, SchemeKind::BaseLRShared}) {
    for (int bf16 = 0; bf16 < 2; ++bf16) {
      const idx L = 9, n_layers = 2, d_kv = 16, rank = 2, n_agents = 3;
      KvStore<float> store(CacheScheme{kind, {}}, StoreDims{n_layers, d_kv, 16, rank, n_agents}, DeviceOptions{2, 32, bf16 != 0, 8});
      store.append_tokens(std::vector<std::int32_t>(static_cast<std::size_t>(L), 7));
      auto rows = [](idx n, idx cols, double base) {
        Matrix<float> m(n, cols);
        for (idx i = 0; i < n; ++i) for (idx j = 0; j < cols; ++j) m(i, j) = float(std::fmod(base + double(i * cols + j), 200.0) - 100.0);
        return m;
      };
      for (idx l = 0; l < n_layers; ++l) {
        for (idx a = 0; a < (kind == SchemeKind::NonShared ? n_agents : 1); ++a) {
          store.append_key(l, a, 0, rows(L, d_kv, 10.0 * double(l) + double(a)).view());
          store.append_value(l, a, 0, rows(L, d_kv, 50.0 + 10.0 * double(l) + double(a)).view());
        }
        if (kind == SchemeKind::BaseShared) for (idx a = 0; a < n_agents; ++a) store.append_lr(l, a, 0, rows(L - a, rank, 3.0 * double(a)).view());
        if (kind == SchemeKind::BaseLRShared) store.append_lr(l, 0, 0, rows(L, rank, 5.0).view());
      }
      store.mark_seen(1);
      const std::string path = "/tmp/lorakv_b200_snapshot_test.bin", path2 = path + ".again";
      store.save_snapshot(path);
      KvStore<float> loaded = KvStore<float>::load_snapshot(path, DeviceOptions{2, 64, bf16 != 0, 16});
      CHECK(loaded.length() == store.length());
      CHECK(loaded.tokens() == store.tokens());
      CHECK(loaded.seen(1) == L); CHECK(loaded.seen(0) == 0);
      CHECK(loaded.bytes().total() == store.bytes().total());
      for (idx l = 0; l < n_layers; ++l) {
        const Span2D<const float> a = store.key_view(l, 0), b = loaded.key_view(l, 0);
        REQUIRE(a.rows == b.rows); REQUIRE(a.cols == b.cols);
        for (idx i = 0; i < a.rows; ++i) for (idx j = 0; j < a.cols; ++j) REQUIRE(a(i, j) == b(i, j));
      }
      loaded.save_snapshot(path2);
      std::ifstream f1(path, std::ios::binary), f2(path2, std::ios::binary);
      const std::string b1((std::istreambuf_iterator<char>(f1)), std::istreambuf_iterator<char>());
      const std::string b2((std::istreambuf_iterator<char>(f2)), std::istreambuf_iterator<char>());
      CHECK(b1 == b2);
      CHECK(b1.size() > 8);
      std::remove(path.c_str()); std::remove(path2.c_str());
    }
  }
}
