// lorakv/device.hpp -- device-resident fast paths over the paged cache.  NOT part of the reference's
// header set: the reference attends over host views (engine.hpp:429-443 hands key_view / value_view /
// lr_view to gqa_attention); here the cache already lives in HBM, so the engine-level call becomes
//
//   decode_batched(store, tables, layer_begin, layer_end, agents, n_q_heads, q)
//       == for every layer, for every batch entry: gqa_attention(q_row, key_view, value_view, lr_view,
//          B[agent], alpha/rank, query_offset = L-1, n_q, n_kv)            (attention.hpp:332-363)
//   prefill(store, tables, layer, agent, n_q_heads, q, query_offset)
//       == gqa_attention(q, key_view, value_view, lr_view, B[agent], alpha/rank, query_offset, ...)
//   append_lr_project(store, tables, layer, agent, row_begin, x)
//       == store.append_lr(layer, agent, row_begin, matmul(x, A))           (engine.hpp:414-418)
//   append_kv_project(store, weights, layer, agent, row_begin, x, rope)
//       == k = matmul(x, Wk); if (rope) apply_rope(k, n_kv_heads, d_head, row_begin); v = matmul(x, Wv);
//          store.append_key(layer, agent, row_begin, k); store.append_value(layer, agent, row_begin, v)
//                                                                           (engine.hpp:376-403, :225-243)
//
// AdapterTable keeps the shared down-projection A per layer and B / alpha per (layer, agent) in HBM
// (lora.hpp:13-87; shared-A multi-LoRA, lora.hpp:69-73).
#pragma once

#include <vector>

#include "lorakv/kvcache.hpp"
#include "lorakv/lora.hpp"

namespace lorakv {

class AdapterTable {
 public:
  // rank = 0 takes the store's; the "full values" schemes keep no LR cache (store rank 0) but still merge a rank-r
  // value adapter into the rows they store (engine.hpp:385-393), so their tables name the rank explicitly
  AdapterTable(const KvStore<float>& store, idx n_q_heads, idx rank = 0)
      : n_q_heads_(n_q_heads), n_kv_heads_(store.device_options().n_kv_heads),
        per_agent_a_(store.scheme().kind == SchemeKind::BaseShared) {
    StoreDims d = store.dims();
    if (rank > 0) d.rank = rank;
    const DeviceOptions& o = store.device_options();
    b200::check(lorakv_adapters_create(b200::Runtime::ctx(), d.n_layers, d.n_agents, d.d_model, d.rank, o.n_kv_heads,
                                       d.d_kv / o.n_kv_heads, o.kv_head_begin, o.n_kv_local,
                                       o.bf16 ? LORAKV_BF16 : LORAKV_F32, &h_));
  }
  ~AdapterTable() { lorakv_adapters_destroy(h_); }
  AdapterTable(const AdapterTable&) = delete;
  AdapterTable& operator=(const AdapterTable&) = delete;

  // one adapter of one layer; under shared-A every agent's `a` is the same matrix and is uploaded once
  // (BaseShared keeps one LR cache per agent because the down-projections differ: there every agent's A is kept)
  void set(idx layer, idx agent, const LoraAdapter<float>& adapter, bool upload_a = true) {
    if (per_agent_a_) b200::check(lorakv_adapters_set_a_agent(h_, layer, agent, adapter.a.data.data()));
    else if (upload_a) b200::check(lorakv_adapters_set_a(h_, layer, adapter.a.data.data()));
    b200::check(lorakv_adapters_set_b(h_, layer, agent, adapter.b.data.data(), adapter.alpha));
  }
  // A MultiLoraSet without shared_a may carry a different down-projection per agent (legal for NonShared / FullShared,
  // engine.hpp:375-379 reads adapter(agent).a): every agent's A is then kept on the device, not only agent 0's.
  void set_layer(idx layer, const MultiLoraSet<float>& set) {
    for (idx a = 0; a < set.num_agents(); ++a) {
      const LoraAdapter<float>& ad = set.adapter(a);
      if (per_agent_a_ || !set.shared_a) {
        b200::check(lorakv_adapters_set_a_agent(h_, layer, a, ad.a.data.data()));
        if (a == 0 && !per_agent_a_) b200::check(lorakv_adapters_set_a(h_, layer, ad.a.data.data()));
        b200::check(lorakv_adapters_set_b(h_, layer, a, ad.b.data.data(), ad.alpha));
      } else {
        this->set(layer, a, ad, a == 0);
      }
    }
  }
  lorakv_adapters* handle() const { return h_; }
  idx n_q_heads() const { return n_q_heads_; }

 private:
  lorakv_adapters* h_ = nullptr;
  idx n_q_heads_, n_kv_heads_;
  bool per_agent_a_;
};

// q: [(layer_end - layer_begin) * agents.size()] rows x (n_q_local * d_head); same-shaped result
inline Matrix<float> decode_batched(KvStore<float>& store, const AdapterTable* tables, idx layer_begin, idx layer_end,
                                    const std::vector<std::int32_t>& agents, idx n_q_heads, const Matrix<float>& q) {
  const idx n_batch = static_cast<idx>(agents.size());
  if (q.rows != (layer_end - layer_begin) * n_batch)
    fail("decode_batched: q has " + std::to_string(q.rows) + " rows, expected layers x batch = " +
         std::to_string((layer_end - layer_begin) * n_batch));
  Matrix<float> out(q.rows, q.cols);
  b200::check(lorakv_fla_decode_batched(store.handle(), tables ? tables->handle() : nullptr, layer_begin, layer_end,
                                        agents.data(), n_batch, n_q_heads, q.data.data(), out.data.data(), LORAKV_HOST));
  return out;
}

// End-of-step output gather of a kv-head-sharded decode over peer memory (lorakv_gather_*, csrc/peer_gather.cu):
// every rank's decode epilogue stores its column slice of the output rows straight into all ranks' buffers.
//   OutputGather g(rank, world, layers * batch * n_q_heads * d_head);
//   exchange g.handle() with the other ranks (MPI_Allgather, a file, ...), g.connect(all handles in rank order);
//   each step: Matrix<float> full = decode_batched_gather(store, tables, g, ...);   // rows x (n_q_heads * d_head)
//   tear-down: g.disconnect(); barrier; destructor.
class OutputGather {
 public:
  OutputGather(int rank, int world, idx full_elems) { b200::check(lorakv_gather_create(b200::Runtime::ctx(), rank, world, full_elems, &h_)); }
  ~OutputGather() { lorakv_gather_destroy(h_); }
  OutputGather(const OutputGather&) = delete;
  OutputGather& operator=(const OutputGather&) = delete;
  std::vector<unsigned char> handle() const {
    std::vector<unsigned char> h(LORAKV_GATHER_HANDLE_BYTES);
    b200::check(lorakv_gather_export(h_, h.data()));
    return h;
  }
  void connect(const std::vector<unsigned char>& handles_in_rank_order) { b200::check(lorakv_gather_connect(h_, handles_in_rank_order.data())); }
  void disconnect() { b200::check(lorakv_gather_disconnect(h_)); }
  idx steps() const { std::int64_t n = 0; b200::check(lorakv_gather_steps(h_, &n)); return n; }
  lorakv_gather* raw() const { return h_; }

 private:
  lorakv_gather* h_ = nullptr;
};

// q: this rank's heads, [(layer_end - layer_begin) * agents.size()] rows x (n_q_local * d_head);
// result: the gathered rows of ALL heads, same row count x (n_q_heads * d_head)
inline Matrix<float> decode_batched_gather(KvStore<float>& store, const AdapterTable* tables, OutputGather& gather, idx layer_begin,
                                           idx layer_end, const std::vector<std::int32_t>& agents, idx n_q_heads, const Matrix<float>& q) {
  const idx n_batch = static_cast<idx>(agents.size());
  if (q.rows != (layer_end - layer_begin) * n_batch)
    fail("decode_batched: q has " + std::to_string(q.rows) + " rows, expected layers x batch = " +
         std::to_string((layer_end - layer_begin) * n_batch));
  const DeviceOptions& o = store.device_options();
  Matrix<float> out(q.rows, n_q_heads * (store.dims().d_kv / o.n_kv_heads));
  b200::check(lorakv_fla_decode_batched_gather(store.handle(), tables ? tables->handle() : nullptr, gather.raw(), layer_begin, layer_end,
                                               agents.data(), n_batch, n_q_heads, q.data.data(), LORAKV_HOST, out.data.data(), nullptr));
  return out;
}

inline Matrix<float> prefill(KvStore<float>& store, const AdapterTable* tables, idx layer, idx agent, idx n_q_heads,
                             const Matrix<float>& q, idx query_offset) {
  Matrix<float> out(q.rows, q.cols);
  b200::check(lorakv_fla_prefill(store.handle(), tables ? tables->handle() : nullptr, layer, agent, n_q_heads,
                                 q.data.data(), q.rows, query_offset, out.data.data(), LORAKV_HOST));
  return out;
}

// V_lr rows = x * A computed on the device once for all agents, written straight into the LR pages;
// returns the rows actually appended (first writer wins)
inline idx append_lr_project(KvStore<float>& store, const AdapterTable& tables, idx layer, idx agent, idx row_begin,
                             Span2D<const float> x) {
  std::int64_t added = 0;
  b200::check(lorakv_pool_append_lr_project(store.handle(), tables.handle(), layer, agent, row_begin, x.data, x.rows,
                                            x.stride, LORAKV_HOST, &added));
  return added;
}

// Wk / Wv of every layer (engine.hpp LayerWeights::wk, wv), restricted to the store's kv-head shard
class ProjectionTable {
 public:
  explicit ProjectionTable(const KvStore<float>& store) {
    const StoreDims& d = store.dims();
    const DeviceOptions& o = store.device_options();
    b200::check(lorakv_proj_create(b200::Runtime::ctx(), d.n_layers, d.d_model, o.n_kv_heads, d.d_kv / o.n_kv_heads,
                                   o.kv_head_begin, o.n_kv_local, o.bf16 ? LORAKV_BF16 : LORAKV_F32, &h_));
  }
  ~ProjectionTable() { lorakv_proj_destroy(h_); }
  ProjectionTable(const ProjectionTable&) = delete;
  ProjectionTable& operator=(const ProjectionTable&) = delete;
  // wk, wv: d_model x d_kv, row-major (Matrix<float> storage)
  void set_layer(idx layer, const Matrix<float>& wk, const Matrix<float>& wv) {
    if (wk.rows != wv.rows || wk.cols != wv.cols)
      fail("ProjectionTable: wk is " + shape_str(wk.rows, wk.cols) + " but wv is " + shape_str(wv.rows, wv.cols));
    b200::check(lorakv_proj_set_kv(h_, layer, wk.data.data(), wv.data.data()));
  }
  // query side (engine.hpp LayerWeights::wq, q_lora): wq d_model x d_model; shared-A adapters of every agent
  void set_query_layer(idx layer, idx n_q_heads, const Matrix<float>& wq, const MultiLoraSet<float>* q_lora = nullptr) {
    b200::check(lorakv_proj_set_q(h_, layer, n_q_heads, wq.data.data()));
    n_q_cols_ = wq.cols;
    if (q_lora)
      for (idx a = 0; a < q_lora->num_agents(); ++a) {
        const LoraAdapter<float>& ad = q_lora->adapter(a);
        b200::check(lorakv_proj_set_q_lora(h_, layer, a, q_lora->num_agents(), ad.rank, ad.a.data.data(), ad.b.data.data(), ad.alpha));
      }
  }
  lorakv_proj* handle() const { return h_; }
  idx n_q_cols() const { return n_q_cols_; }

 private:
  lorakv_proj* h_ = nullptr;
  idx n_q_cols_ = 0;
};

// q = rope(x Wq + (alpha/rank) (x A_q) B_q[agent]) for rows at positions [pos_begin, pos_begin + x.rows)
// (engine.hpp:362-373, :422); agent < 0 skips the adapter.  n_q_local_cols = columns of the store's q-head shard.
inline Matrix<float> project_query(const ProjectionTable& weights, idx layer, idx agent, idx pos_begin, Span2D<const float> x,
                                   idx n_q_local_cols, bool rope = true) {
  Matrix<float> q(x.rows, n_q_local_cols);
  b200::check(lorakv_proj_query(weights.handle(), layer, agent, pos_begin, x.data, x.rows, x.stride, rope ? 1 : 0, q.data.data(),
                                LORAKV_HOST));
  return q;
}

// K / V_base projection of new context rows, rotation of the keys and the append, in one device pass;
// returns the rows actually appended (first writer wins)
inline idx append_kv_project(KvStore<float>& store, const ProjectionTable& weights, idx layer, idx agent, idx row_begin,
                             Span2D<const float> x, bool rope = true) {
  std::int64_t added = 0;
  b200::check(lorakv_pool_append_kv_project(store.handle(), weights.handle(), layer, agent, row_begin, x.data, x.rows,
                                            x.stride, LORAKV_HOST, rope ? 1 : 0, &added));
  return added;
}

}  // namespace lorakv
