// The trace replay (include/lorakv/replay.hpp) against the reference path composed from the CPU checker: for every
// step() call of a short multi-agent trace -- plan (kvcache.hpp:112-142), k = rope(x Wk), v = x Wv (+ the value
// adapter under the full-values schemes), V_lr = x A_v, first-writer-wins appends, q = rope(x Wq + s (x A_q) B_q),
// gqa_attention over the store's views (engine.hpp:362-443) -- the last layer's attention output must match.
// fp32 pages: 1e-4; bf16 pages (tcgen05 projection, prefill and decode kernels): 2e-2.  Cache bytes are exact.
#include <cmath>
#include <vector>

#include "check.hpp"
#include "lorakv/replay.hpp"
#include "oracle_glue.hpp"

using namespace lorakv;

namespace {

struct RefStore {
  orc_store* s = nullptr;
  RefStore(int scheme, idx n_layers, idx d_kv, idx d_model, idx rank, idx n_agents) {
    s = orc_store_create(scheme, n_layers, d_kv, d_model, rank, n_agents, 4);
    REQUIRE(s != nullptr);
  }
  ~RefStore() { orc_store_destroy(s); }
  Span2D<const float> view(int which, idx layer, idx agent) const {
    const void* data = nullptr; int64_t rows = 0, cols = 0;
    oracle::ok(orc_store_view(s, which, layer, agent, &data, &rows, &cols));
    return Span2D<const float>{static_cast<const float*>(data), rows, cols, cols};
  }
};

Matrix<float> rows_of(const Matrix<float>& m, idx b, idx e) {
  Matrix<float> out(e - b, m.cols);
  for (idx i = b; i < e; ++i) for (idx j = 0; j < m.cols; ++j) out(i - b, j) = m(i, j);
  return out;
}

void run(SchemeKind kind, bool bf16, idx d_head, double tol) {
  const idx n_layers = 2, n_q = 4, n_kv = 2, d_model = 64, rank = 4, n_agents = 3;
  const idx dq = n_q * d_head, dkv = n_kv * d_head;
  const std::vector<TraceStep> trace{{0, 20, 3}, {1, 5, 2}, {0, 7, 2}, {2, 9, 1}, {1, 3, 2}, {2, 0, 2}};
  const idx total = trace_total_len(trace);
  auto rnd = [&](Matrix<float> m) { return bf16 ? oracle::round_bf16(m) : m; };
  const Rng root(77);
  const Matrix<float> xall = rnd(Matrix<float>::gaussian(total, d_model, root.child(1), 1.0));
  std::vector<SublayerWeights> layers;
  for (idx l = 0; l < n_layers; ++l) {
    const Rng r = root.child(100 + std::uint64_t(l));
    SublayerWeights w;
    const double ws = 1.0 / std::sqrt(double(d_model));
    w.wq = rnd(Matrix<float>::gaussian(d_model, dq, r.child(0), ws));
    w.wk = rnd(Matrix<float>::gaussian(d_model, dkv, r.child(1), ws));
    w.wv = rnd(Matrix<float>::gaussian(d_model, dkv, r.child(2), ws));
    w.a_q = rnd(Matrix<float>::gaussian(d_model, rank, r.child(10), ws));
    w.a_v = rnd(Matrix<float>::gaussian(d_model, rank, r.child(11), ws));
    for (idx a = 0; a < n_agents; ++a) {
      w.b_q.push_back(rnd(Matrix<float>::gaussian(rank, dq, r.child(0x200 + std::uint64_t(a)), 0.02 / std::sqrt(double(rank)))));
      w.b_v.push_back(rnd(Matrix<float>::gaussian(rank, dkv, r.child(0x300 + std::uint64_t(a)), 0.02 / std::sqrt(double(rank)))));
    }
    layers.push_back(std::move(w));
  }
  const CacheScheme scheme{kind, {}};
  std::vector<Matrix<float>> got;
  DeviceOptions opt; opt.bf16 = bf16; opt.page_tokens = 16;
  const ReplayReport rep = replay_trace(layers, n_q, n_kv, d_head, d_model, rank, n_agents, scheme, trace,
                                        [&](idx p, float* row) { for (idx j = 0; j < d_model; ++j) row[j] = xall(p, j); }, opt, true, &got);
  CHECK(rep.total_seq_len == total);
  CHECK(rep.steps.size() == trace.size());

  // ---- the reference path, step by step ----
  const bool full_values = kind == SchemeKind::NonShared || kind == SchemeKind::FullShared;
  const bool lr_cached = !full_values;
  RefStore ref(static_cast<int>(kind), n_layers, dkv, d_model, rank, n_agents);
  const float s = float(16.0 / double(rank));
  std::size_t call = 0;
  auto step = [&](idx agent, idx n_new) {
    int64_t seen = 0;
    oracle::ok(orc_store_seen(ref.s, agent, &seen));
    const PrefillPlan plan = plan_core(scheme, orc_store_length(ref.s), seen, n_new);
    oracle::ok(orc_store_append_tokens(ref.s, n_new));
    if (plan.hidden_pass.empty()) { oracle::ok(orc_store_mark_seen(ref.s, agent)); return; }
    const idx p0 = plan.hidden_pass.begin, p1 = plan.hidden_pass.end;
    const Matrix<float> x = rows_of(xall, p0, p1);
    Matrix<float> attn;
    for (idx l = 0; l < n_layers; ++l) {
      const SublayerWeights& w = layers[std::size_t(l)];
      const Interval kv = plan.kv_project;
      if (!kv.empty()) {
        const Matrix<float> xkv = rows_of(xall, kv.begin, kv.end);
        Matrix<float> k = oracle::matmul(xkv, w.wk);
        oracle::ok(orc_apply_rope_f32(k.data.data(), k.rows, k.cols, n_kv, d_head, kv.begin));
        Matrix<float> v = oracle::matmul(xkv, w.wv);
        if (full_values) {
          const Matrix<float> upm = oracle::matmul(oracle::matmul(xkv, w.a_v), w.b_v[std::size_t(agent)]);
          for (std::size_t i = 0; i < v.data.size(); ++i) v.data[i] += s * upm.data[i];
        }
        oracle::ok(orc_store_append(ref.s, 0, l, agent, kv.begin, k.data.data(), k.rows, k.cols));
        oracle::ok(orc_store_append(ref.s, 1, l, agent, kv.begin, v.data.data(), v.rows, v.cols));
      }
      if (lr_cached && !plan.lr_project.empty()) {
        const Matrix<float> lr = oracle::matmul(rows_of(xall, plan.lr_project.begin, plan.lr_project.end), w.a_v);
        oracle::ok(orc_store_append(ref.s, 2, l, agent, plan.lr_project.begin, lr.data.data(), lr.rows, lr.cols));
      }
      Matrix<float> q = oracle::matmul(x, w.wq);
      const Matrix<float> qup = oracle::matmul(oracle::matmul(x, w.a_q), w.b_q[std::size_t(agent)]);
      for (std::size_t i = 0; i < q.data.size(); ++i) q.data[i] += s * qup.data[i];
      oracle::ok(orc_apply_rope_f32(q.data.data(), q.rows, q.cols, n_q, d_head, p0));
      const Span2D<const float> kview = ref.view(0, l, agent), vview = ref.view(1, l, agent);
      Span2D<const float> lrview{nullptr, kview.rows, 0, 0}, bview{nullptr, 0, dkv, dkv};
      float scale = 1.f;
      if (lr_cached) { lrview = ref.view(2, l, agent); bview = w.b_v[std::size_t(agent)].view(); scale = s; }
      attn = oracle::gqa<float>(q.view(), kview, vview, lrview, bview, scale, p0, n_q, n_kv);
    }
    oracle::ok(orc_store_mark_seen(ref.s, agent));
    REQUIRE(call < got.size());
    REQUIRE(got[call].rows == attn.rows);
    CHECK_LE(max_rel_error(got[call], attn), tol);
    ++call;
  };
  for (const TraceStep& ts : trace) {
    step(ts.agent, ts.prefill_len);
    for (idx g = 0; g < ts.gen_len; ++g) step(ts.agent, 1);
  }
  CHECK(call == got.size());
  uint64_t b[4];
  orc_store_bytes(ref.s, b);
  const std::uint64_t esz = bf16 ? 2 : 4;                 // CacheBytes counts elements x sizeof(T); the checker stores float
  CHECK(rep.bytes.key * 4 == b[0] * esz);
  CHECK(rep.bytes.value * 4 == b[1] * esz);
  CHECK(rep.bytes.lr * 4 == b[2] * esz);
}

}  // namespace

TEST_CASE("trace replay == the reference path, fp32 pages, every scheme on the path") {
  for (SchemeKind k : {SchemeKind::NonShared, SchemeKind::FullShared, SchemeKind::BaseShared, SchemeKind::BaseLRShared}) run(k, false, 32, 1e-4);
}

TEST_CASE("trace replay == the reference path, bf16 pages and the tcgen05 kernels (d_head 128), every scheme on the path") {
  for (SchemeKind k : {SchemeKind::NonShared, SchemeKind::FullShared, SchemeKind::BaseShared, SchemeKind::BaseLRShared}) run(k, true, 128, 2e-2);
}

TEST_CASE("generate_trace: 17 steps, 912 + 4 l_ctx tokens (trace.cpp:11-25)") {
  const std::vector<TraceStep> t = generate_trace(100);
  CHECK(t.size() == 17);
  CHECK(trace_total_len(t) == 912 + 400);
  CHECK(t[0].agent == kPlanAgent); CHECK(t[0].prefill_len == 512); CHECK(t[0].gen_len == 32);
  CHECK(t[3].prefill_len == 100); CHECK(t[5].agent == kActionAgent);
  CHECK(t[15].agent == kReflectAgent); CHECK(t[15].prefill_len == 32); CHECK(t[16].gen_len == 8);
  CHECK(synth_token(42, 3, 17, 1000) == std::int32_t(Rng::mix(Rng::mix(42, 0x70c5u), Rng::mix(3, 17)) % 1000));
}
