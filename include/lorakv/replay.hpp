// replay.hpp -- the multi-agent trace of the reference's cost study, driven through the B200 cache path
// (SURVEY 8(f) row 4).
//
// The reference replays a fixed 17-step plan / action / reflect schedule through step() and reports MAC-count
// proxies for TTFT and throughput per cache scheme (proj/include/lorakv/trace.hpp:84-155, schedule
// proj/src/trace.cpp:11-25; the paper's Tables 3 / 4).  Here the same schedule runs through the part of step()
// this library implements -- per layer: plan (kvcache.hpp:112-142), K / V projection + RoPE + append
// (engine.hpp:376-403), V_lr = X A append (:411-419), query projection (:362-373, :422) and Flash-LoRA-Attention
// over the store (:429-443) -- and reports DEVICE TIME instead of MAC proxies.  The MLP, the output projection and
// the embeddings are not part of this path, so the hidden state of a trajectory position comes from the caller
// (`RowSource`); every scheme replays the same rows, which keeps the comparison between schemes like-for-like.
#pragma once

#include <functional>
#include <string>
#include <vector>

#include "lorakv/device.hpp"
#include "lorakv/rng.hpp"

namespace lorakv {

struct TraceStep {
  idx agent = 0;
  idx prefill_len = 0;   // context appended to the trajectory by this step
  idx gen_len = 0;       // tokens generated afterwards, one decode step each
};

inline constexpr idx kPlanAgent = 0, kActionAgent = 1, kReflectAgent = 2;

// plan(512 + 32), plan(8 + 8), action(8 + 8), four retrieval cycles {plan(l_ctx + 32), plan(8 + 8), action(8 + 8)},
// reflect(32 + 32), reflect(8 + 8): 17 steps, 912 + 4 l_ctx tokens
inline std::vector<TraceStep> generate_trace(idx l_ctx) {
  if (l_ctx < 0) fail("generate_trace: l_ctx must be >= 0");
  const TraceStep shortp{kPlanAgent, 8, 8}, shorta{kActionAgent, 8, 8};
  std::vector<TraceStep> t{{kPlanAgent, 512, 32}, shortp, shorta};
  for (int cycle = 0; cycle < 4; ++cycle) t.insert(t.end(), {TraceStep{kPlanAgent, l_ctx, 32}, shortp, shorta});
  t.insert(t.end(), {TraceStep{kReflectAgent, 32, 32}, TraceStep{kReflectAgent, 8, 8}});
  return t;
}

inline idx trace_total_len(const std::vector<TraceStep>& trace) {
  idx n = 0;
  for (const TraceStep& s : trace) n += s.prefill_len + s.gen_len;
  return n;
}

// token id of (seed, step, position), independent of the scheme (trace.hpp:41-47)
inline std::int32_t synth_token(std::uint64_t seed, idx step_index, idx position, idx vocab) {
  const std::uint64_t h = Rng::mix(Rng::mix(seed, 0x70c5u), Rng::mix(std::uint64_t(step_index), std::uint64_t(position)));
  return std::int32_t(h % std::uint64_t(vocab));
}

// attention-sublayer weights of one layer (engine.hpp LayerWeights without wo / MLP); the adapters follow the
// shared-A rule (lora.hpp:69-73): one down-projection per side, one up-projection per agent
struct SublayerWeights {
  Matrix<float> wq, wk, wv;            // d_model x n_q*d, d_model x n_kv*d (twice)
  Matrix<float> a_q, a_v;              // d_model x rank
  std::vector<Matrix<float>> b_q, b_v; // per agent: rank x n_q*d, rank x n_kv*d
  double alpha = 16.0;
};

struct ReplayStepLog {
  idx step_index = 0, agent = 0, len_before = 0, len_after = 0;
  Interval hidden_pass, kv_project, lr_project;   // of the prefill part of the step
  double prefill_ms = 0.0, decode_ms = 0.0;       // device time
};

struct ReplayReport {
  std::string scheme;
  idx total_seq_len = 0;
  CacheBytes bytes;
  double ttft_ms = 0.0, total_ms = 0.0;           // sum of the prefill parts / of everything
  std::vector<ReplayStepLog> steps;
};

using RowSource = std::function<void(idx position, float* row)>;   // hidden state (d_model floats) of a position

namespace detail {
class DeviceBuffer {
 public:
  explicit DeviceBuffer(std::int64_t bytes) { b200::check(lorakv_dev_alloc(b200::Runtime::ctx(), bytes, &p_)); }
  ~DeviceBuffer() { lorakv_dev_free(b200::Runtime::ctx(), p_); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  float* f() const { return static_cast<float*>(p_); }

 private:
  void* p_ = nullptr;
};
class Timer {
 public:
  Timer() {
    b200::check(lorakv_event_create(b200::Runtime::ctx(), &a_));
    b200::check(lorakv_event_create(b200::Runtime::ctx(), &b_));
  }
  ~Timer() { lorakv_event_destroy(a_); lorakv_event_destroy(b_); }
  void start() { b200::check(lorakv_event_record(b200::Runtime::ctx(), a_)); }
  double stop_ms() {
    float ms = 0.f;
    b200::check(lorakv_event_record(b200::Runtime::ctx(), b_));
    b200::check(lorakv_event_elapsed_ms(a_, b_, &ms));
    return ms;
  }

 private:
  lorakv_event *a_ = nullptr, *b_ = nullptr;
};
}  // namespace detail

// `outputs`, when given, receives the attention output of the LAST layer of every step() call in order
// (prefill part first, then one row per generated token) -- what the parity test compares.
inline ReplayReport replay_trace(const std::vector<SublayerWeights>& layers, idx n_q_heads, idx n_kv_heads, idx d_head, idx d_model,
                                 idx rank, idx n_agents, const CacheScheme& scheme, const std::vector<TraceStep>& trace,
                                 const RowSource& x_of, DeviceOptions opt, bool rope = true,
                                 std::vector<Matrix<float>>* outputs = nullptr, std::uint64_t seed = 42, idx vocab = 1000) {
  const idx n_layers = static_cast<idx>(layers.size());
  if (n_layers < 1) fail("replay_trace: no layers");
  const bool full_values = scheme.kind == SchemeKind::NonShared || scheme.kind == SchemeKind::FullShared;
  const bool lr_cached = scheme.kind == SchemeKind::BaseShared || scheme.kind == SchemeKind::BaseLRShared;
  if (!full_values && !lr_cached) fail("replay_trace: scheme " + scheme.name() + " is outside the B200 hot path");
  const bool has_lora = rank > 0;
  const idx total = trace_total_len(trace), dq = n_q_heads * d_head, dkv = n_kv_heads * d_head;
  opt.n_kv_heads = n_kv_heads;
  if (opt.max_tokens < total) opt.max_tokens = total;
  KvStore<float> store(scheme, StoreDims{n_layers, dkv, d_model, lr_cached ? rank : 0, n_agents}, opt);
  ProjectionTable weights(store);
  AdapterTable tables(store, n_q_heads, has_lora ? rank : 1);
  for (idx l = 0; l < n_layers; ++l) {
    const SublayerWeights& w = layers[static_cast<std::size_t>(l)];
    weights.set_layer(l, w.wk, w.wv);
    b200::check(lorakv_proj_set_q(weights.handle(), l, n_q_heads, w.wq.data.data()));
    if (has_lora)
      for (idx a = 0; a < n_agents; ++a) {
        b200::check(lorakv_proj_set_q_lora(weights.handle(), l, a, n_agents, rank, w.a_q.data.data(),
                                           w.b_q[static_cast<std::size_t>(a)].data.data(), w.alpha));
        tables.set(l, a, LoraAdapter<float>(w.a_v, w.b_v[static_cast<std::size_t>(a)], rank, w.alpha), a == 0);
      }
  }
  lorakv_ctx* ctx = b200::Runtime::ctx();
  detail::DeviceBuffer xbuf(total * d_model * std::int64_t(sizeof(float))), qbuf(total * dq * std::int64_t(sizeof(float))),
      obuf(total * dq * std::int64_t(sizeof(float)));
  std::vector<float> xhost;
  detail::Timer timer;

  ReplayReport report;
  report.scheme = scheme.name();
  // one call of step() (engine.hpp:279-443) restricted to the attention sublayer
  auto step = [&](idx si, idx agent, idx n_new, ReplayStepLog* log) {
    const PrefillPlan plan = plan_step(store, agent, n_new);
    std::vector<std::int32_t> ids;
    for (idx i = 0; i < n_new; ++i) ids.push_back(synth_token(seed, si, store.length() + i, vocab));
    store.append_tokens(ids);
    if (log) { log->hidden_pass = plan.hidden_pass; log->kv_project = plan.kv_project; log->lr_project = plan.lr_project; }
    if (plan.hidden_pass.empty()) { store.mark_seen(agent); return 0.0; }
    const idx p0 = plan.hidden_pass.begin, p1 = plan.hidden_pass.end, n = p1 - p0;
    xhost.resize(static_cast<std::size_t>(n * d_model));
    for (idx p = p0; p < p1; ++p) x_of(p, xhost.data() + (p - p0) * d_model);
    b200::check(lorakv_copy_h2d(ctx, xbuf.f(), xhost.data(), n * d_model * std::int64_t(sizeof(float))));
    timer.start();
    for (idx l = 0; l < n_layers; ++l) {
      const Interval kv = plan.kv_project_at(l, scheme);
      // A decode step (a handful of fresh rows, every cache of the layer ending where they begin) is ONE library call:
      // lorakv_step_layer chains the projections, the appends, the attention and its epilogue as four dependent
      // launches.  Anything else (prefills, agent switches that re-project a longer range) takes the calls below.
      const Interval lr_iv = (lr_cached && has_lora) ? plan.lr_project_at(l, scheme) : plan.hidden_pass;
      if (n <= 8 && kv.begin == p0 && kv.end == p1 && lr_iv.begin == p0 && lr_iv.end == p1 && (has_lora || !lr_cached)) {
        b200::check(lorakv_step_layer(store.handle(), weights.handle(), has_lora ? tables.handle() : nullptr, l, agent, p0, xbuf.f(), n,
                                      d_model, rope ? 1 : 0, n_q_heads, qbuf.f(), obuf.f(), LORAKV_DEVICE));
        continue;
      }
      if (!kv.empty()) {
        const float* xkv = xbuf.f() + (kv.begin - p0) * d_model;
        if (full_values && has_lora)
          b200::check(lorakv_pool_append_kv_project_full(store.handle(), weights.handle(), tables.handle(), l, agent, kv.begin, xkv,
                                                         kv.size(), d_model, LORAKV_DEVICE, rope ? 1 : 0, nullptr));
        else
          b200::check(lorakv_pool_append_kv_project(store.handle(), weights.handle(), l, agent, kv.begin, xkv, kv.size(), d_model,
                                                    LORAKV_DEVICE, rope ? 1 : 0, nullptr));
      }
      if (lr_cached && has_lora) {
        const Interval lr = plan.lr_project_at(l, scheme);
        if (!lr.empty())
          b200::check(lorakv_pool_append_lr_project(store.handle(), tables.handle(), l, agent, lr.begin,
                                                    xbuf.f() + (lr.begin - p0) * d_model, lr.size(), d_model, LORAKV_DEVICE, nullptr));
      }
      b200::check(lorakv_proj_query(weights.handle(), l, has_lora ? agent : -1, p0, xbuf.f(), n, d_model, rope ? 1 : 0, qbuf.f(),
                                    LORAKV_DEVICE));
      b200::check(lorakv_fla_prefill(store.handle(), lr_cached && has_lora ? tables.handle() : nullptr, l, agent, n_q_heads, qbuf.f(), n,
                                     p0, obuf.f(), LORAKV_DEVICE));
    }
    const double ms = timer.stop_ms();
    if (outputs) {
      Matrix<float> o(n, dq);
      b200::check(lorakv_copy_d2h(ctx, o.data.data(), obuf.f(), n * dq * std::int64_t(sizeof(float))));
      b200::check(lorakv_ctx_synchronize(ctx));
      outputs->push_back(std::move(o));
    }
    store.mark_seen(agent);
    return ms;
  };

  for (std::size_t si = 0; si < trace.size(); ++si) {
    const TraceStep& ts = trace[si];
    if (ts.agent < 0 || ts.agent >= n_agents) fail("run_trace: trace agent " + std::to_string(ts.agent) + " outside the model's " + std::to_string(n_agents) + " agents");
    if (ts.prefill_len < 0 || ts.gen_len < 0) fail("run_trace: negative step length");
    ReplayStepLog log;
    log.step_index = idx(si); log.agent = ts.agent; log.len_before = store.length();
    log.prefill_ms = step(idx(si), ts.agent, ts.prefill_len, &log);
    for (idx g = 0; g < ts.gen_len; ++g) log.decode_ms += step(idx(si), ts.agent, 1, nullptr);
    log.len_after = store.length();
    report.ttft_ms += log.prefill_ms;
    report.total_ms += log.prefill_ms + log.decode_ms;
    report.steps.push_back(log);
  }
  report.total_seq_len = store.length();
  report.bytes = store.bytes();
  return report;
}

}  // namespace lorakv
