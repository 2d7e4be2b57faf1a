// The device-resident fast paths (include/lorakv/device.hpp) against what they stand for: one
// gqa_attention call per (agent, layer) over the store's views, as engine.hpp:429-443 composes it.
// fp32 pages: max_rel_error <= 1e-4; bf16 pages (inputs rounded to bf16 once, the oracle consumes the
// rounded values): <= 2e-2 -- BASELINE.json north_star tolerances.
#include <cmath>
#include <vector>

#include "check.hpp"
#include "lorakv/device.hpp"
#include "oracle_glue.hpp"

using namespace lorakv;

namespace {

struct Layer {
  Matrix<float> k, v, x, a;
  std::vector<Matrix<float>> q, b;
};

void run_config(bool bf16, double tol, idx L, idx n_q, idx n_kv, idx d, idx r, idx agents, idx layers, idx d_model) {
  auto rnd = [&](Matrix<float> m) { return bf16 ? oracle::round_bf16(m) : m; };
  KvStore<float> store(CacheScheme{SchemeKind::BaseLRShared, {}}, StoreDims{layers, n_kv * d, d_model, r, agents},
                       DeviceOptions{n_kv, L, bf16});
  AdapterTable tables(store, n_q);
  store.append_tokens(std::vector<std::int32_t>(static_cast<std::size_t>(L), 1));
  std::vector<Layer> model;
  const Rng root(4242);
  for (idx l = 0; l < layers; ++l) {
    const Rng rng = root.child(std::uint64_t(l));
    Layer ly;
    ly.k = rnd(Matrix<float>::gaussian(L, n_kv * d, rng.child(2), 1.0 / std::sqrt(double(d))));
    ly.v = rnd(Matrix<float>::gaussian(L, n_kv * d, rng.child(3), 1.0));
    ly.x = rnd(Matrix<float>::gaussian(L, d_model, rng.child(6), 1.0));
    ly.a = rnd(Matrix<float>::gaussian(d_model, r, rng.child(7), 1.0 / std::sqrt(double(d_model))));
    std::vector<LoraAdapter<float>> ads;
    for (idx a = 0; a < agents; ++a) {
      ly.q.push_back(rnd(Matrix<float>::gaussian(1, n_q * d, rng.child(100 + std::uint64_t(a)), 1.0 / std::sqrt(double(d)))));
      ly.b.push_back(rnd(Matrix<float>::gaussian(r, n_kv * d, rng.child(200 + std::uint64_t(a)), 0.02 / std::sqrt(double(r)))));
      ads.emplace_back(ly.a, ly.b.back(), r, 16.0);
    }
    const MultiLoraSet<float> set(Matrix<float>(d_model, n_kv * d), ads, /*shared_a=*/true);
    tables.set_layer(l, set);
    store.append_key(l, 0, 0, ly.k.view());
    store.append_value(l, 0, 0, ly.v.view());
    CHECK(append_lr_project(store, tables, l, 0, 0, ly.x.view()) == L);   // V_lr = X A once for all agents
    CHECK(append_lr_project(store, tables, l, 1, 0, ly.x.view()) == 0);   // the next agent finds it there
    model.push_back(std::move(ly));
  }
  std::vector<std::int32_t> batch;
  for (idx a = 0; a < agents; ++a) batch.push_back(std::int32_t(a));
  Matrix<float> q(layers * agents, n_q * d);
  for (idx l = 0; l < layers; ++l)
    for (idx a = 0; a < agents; ++a)
      for (idx c = 0; c < n_q * d; ++c) q(l * agents + a, c) = model[l].q[a](0, c);
  const Matrix<float> out = decode_batched(store, &tables, 0, layers, batch, n_q, q);
  for (idx l = 0; l < layers; ++l) {
    const Layer& ly = model[l];
    // the oracle attends over what the store holds: its own views (bit-exact K/V, device-projected V_lr)
    const Matrix<float> v_lr_want = oracle::matmul(ly.x, ly.a);
    const Span2D<const float> lr = store.lr_view(l, 0);
    REQUIRE(lr.rows == L);
    Matrix<float> lr_got(L, r);
    for (idx i = 0; i < L; ++i) for (idx c = 0; c < r; ++c) lr_got(i, c) = lr(i, c);
    CHECK_LE(max_rel_error(lr_got, v_lr_want), bf16 ? 1e-2 : 1e-5);
    for (idx a = 0; a < agents; ++a) {
      const Matrix<float> want = oracle::gqa<float>(ly.q[a].view(), ly.k.view(), ly.v.view(), v_lr_want.view(), ly.b[a].view(),
                                                    float(16.0 / double(r)), L - 1, n_q, n_kv);
      Matrix<float> got(1, n_q * d);
      for (idx c = 0; c < n_q * d; ++c) got(0, c) = out(l * agents + a, c);
      CHECK_LE(max_rel_error(got, want), tol);
    }
  }
  // the same step ending in the peer-memory output gather: with one rank the gathered rows ARE the decode's rows
  {
    OutputGather gather(0, 1, layers * agents * n_q * d);
    CHECK(gather.handle().size() == std::size_t(LORAKV_GATHER_HANDLE_BYTES));
    for (int rep = 0; rep < 3; ++rep) {      // both buffers of the pair
      const Matrix<float> full = decode_batched_gather(store, &tables, gather, 0, layers, batch, n_q, q);
      REQUIRE(full.rows == out.rows); REQUIRE(full.cols == out.cols);
      CHECK(full.data == out.data);
    }
    CHECK(gather.steps() == 3);
  }
  // prefill block of agent 1 on layer 0 at the tail of the cache
  const idx L_c = std::min<idx>(L, 9);
  const Matrix<float> qp = rnd(Matrix<float>::gaussian(L_c, n_q * d, Rng(99), 1.0 / std::sqrt(double(d))));
  const Matrix<float> got = prefill(store, &tables, 0, 1, n_q, qp, L - L_c);
  const Matrix<float> v_lr0 = oracle::matmul(model[0].x, model[0].a);
  const Matrix<float> want = oracle::gqa<float>(qp.view(), model[0].k.view(), model[0].v.view(), v_lr0.view(), model[0].b[1].view(),
                                                float(16.0 / double(r)), L - L_c, n_q, n_kv);
  CHECK_LE(max_rel_error(got, want), tol);
}

}  // namespace

TEST_CASE("tiny config (BASELINE configs[0]): 4q/2kv heads, d=64, r=8, 2 agents, 512 tokens, fp32 pages") {
  run_config(false, 1e-4, 512, 4, 2, 64, 8, 2, 1, 256);
}

TEST_CASE("tiny config on bf16 pages") { run_config(true, 2e-2, 512, 4, 2, 64, 8, 2, 1, 256); }

TEST_CASE("Llama-shaped heads (32q/8kv, d=128, r=16, 3 agents), two layers, bf16 pages, ragged length") {
  run_config(true, 2e-2, 1000, 32, 8, 128, 16, 3, 2, 512);
}

// engine.hpp:376-403 through the drop-in header: project, rotate, append in one device pass, read back through the
// store's views and compare with matmul + apply_rope of the checker
TEST_CASE("append_kv_project == append_key(rope(x Wk)), append_value(x Wv) on bf16 and fp32 pages") {
  for (int bf16 = 0; bf16 < 2; ++bf16) {
    const idx L = 150, d_model = 128, n_kv = 2, d = 128;
    auto rnd = [&](Matrix<float> m) { return bf16 ? oracle::round_bf16(m) : m; };
    KvStore<float> store(CacheScheme{SchemeKind::FullShared, {}}, StoreDims{1, n_kv * d, d_model, 0, 1}, DeviceOptions{n_kv, L, bf16 != 0});
    ProjectionTable weights(store);
    const Matrix<float> x = rnd(Matrix<float>::gaussian(L, d_model, Rng(5), 1.0));
    const Matrix<float> wk = rnd(Matrix<float>::gaussian(d_model, n_kv * d, Rng(6), 1.0 / std::sqrt(double(d_model))));
    const Matrix<float> wv = rnd(Matrix<float>::gaussian(d_model, n_kv * d, Rng(7), 1.0 / std::sqrt(double(d_model))));
    weights.set_layer(0, wk, wv);
    store.append_tokens(std::vector<std::int32_t>(static_cast<std::size_t>(L), 1));
    CHECK(append_kv_project(store, weights, 0, 0, 0, x.view().row_range(0, 60)) == 60);
    CHECK(append_kv_project(store, weights, 0, 0, 60, x.view().row_range(60, L)) == L - 60);
    CHECK(append_kv_project(store, weights, 0, 0, 0, x.view()) == 0);
    Matrix<float> k_want = oracle::matmul(x, wk);
    oracle::ok(orc_apply_rope_f32(k_want.data.data(), L, n_kv * d, n_kv, d, 0));
    const Matrix<float> v_want = oracle::matmul(x, wv);
    const Span2D<const float> kv = store.key_view(0, 0), vv = store.value_view(0, 0);
    REQUIRE(kv.rows == L); REQUIRE(vv.rows == L);
    Matrix<float> k_got(L, n_kv * d), v_got(L, n_kv * d);
    for (idx i = 0; i < L; ++i) for (idx c = 0; c < n_kv * d; ++c) { k_got(i, c) = kv(i, c); v_got(i, c) = vv(i, c); }
    CHECK_LE(max_rel_error(k_got, k_want), bf16 ? 4e-3 : 1e-6);
    CHECK_LE(max_rel_error(v_got, v_want), bf16 ? 4e-3 : 0.0);
    bool threw = false;
    try { append_kv_project(store, weights, 0, 0, L + 5, x.view()); } catch (const std::runtime_error& e) {
      threw = std::string(e.what()).find("gap") != std::string::npos;     // kvcache.hpp:401-403
    }
    CHECK(threw);
  }
}

TEST_CASE("project_query == rope(x Wq + s (x A_q) B_q[agent]) through the drop-in header") {
  const idx L = 70, d_model = 128, n_q = 4, n_kv = 2, d = 128, r = 8, agents = 2;
  KvStore<float> store(CacheScheme{SchemeKind::FullShared, {}}, StoreDims{1, n_kv * d, d_model, 0, agents}, DeviceOptions{n_kv, L, true});
  ProjectionTable weights(store);
  auto rnd = [](Matrix<float> m) { return oracle::round_bf16(m); };
  const Matrix<float> x = rnd(Matrix<float>::gaussian(L, d_model, Rng(15), 1.0));
  const Matrix<float> wq = rnd(Matrix<float>::gaussian(d_model, n_q * d, Rng(16), 1.0 / std::sqrt(double(d_model))));
  const Matrix<float> a = rnd(Matrix<float>::gaussian(d_model, r, Rng(17), 1.0 / std::sqrt(double(d_model))));
  std::vector<LoraAdapter<float>> ads;
  for (idx i = 0; i < agents; ++i)
    ads.emplace_back(a, rnd(Matrix<float>::gaussian(r, n_q * d, Rng(18 + std::uint64_t(i)), 0.02 / std::sqrt(double(r)))), r, 16.0);
  const MultiLoraSet<float> set(wq, ads, /*shared_a=*/true);
  weights.set_query_layer(0, n_q, wq, &set);
  const Matrix<float> got = project_query(weights, 0, 1, 9, x.view(), n_q * d);
  Matrix<float> want = oracle::matmul(x, wq);
  const Matrix<float> upm = oracle::matmul(oracle::matmul(x, a), ads[1].b);
  for (std::size_t i = 0; i < want.data.size(); ++i) want.data[i] += float(16.0 / double(r)) * upm.data[i];
  oracle::ok(orc_apply_rope_f32(want.data.data(), L, n_q * d, n_q, d, 9));
  CHECK_LE(max_rel_error(got, want), 1e-4);
}
