// ref_shim.cpp -- extern "C" window onto the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  This file contains no algorithm: it includes the reference's
// own headers where they lie (/root/reference/proj/include, passed with -I by oracle/Makefile)
// and forwards to them, so that tests can (a) pin oracle/lorakv_oracle.c bit-for-bit and
// (b) time the reference's real CPU path (bench.py --impl reference, cpu_baseline.kind
// "reference").  The built library lands in oracle/_ref/ (git-ignored, shipped to the GPU box).
// Symbols mirror lorakv_oracle.h with the prefix ref_ instead of orc_.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lorakv/attention.hpp"
#include "lorakv/engine.hpp"
#include "lorakv/fuzz.hpp"
#include "lorakv/kvcache.hpp"
#include "lorakv/lora.hpp"
#include "lorakv/matrix.hpp"
#include "lorakv/rng.hpp"

#include "lorakv_oracle.h"  // span structs + status codes only

using namespace lorakv;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_ERR;
  }
}

template <class T, class S>
Span2D<const T> sp(S s) { return Span2D<const T>{s.data, s.rows, s.cols, s.stride}; }

template <class T, class S>
AttentionInputs<T> inputs(S q, S k, S v, S vlr, S b, T scale, idx off) {
  AttentionInputs<T> in;
  in.q = sp<T>(q); in.k = sp<T>(k); in.v_base = sp<T>(v); in.v_lr = sp<T>(vlr); in.b_up = sp<T>(b);
  in.lr_scale = scale; in.query_offset = off;
  return in;
}

template <class T>
void put(const Matrix<T>& m, T* out) { std::memcpy(out, m.data.data(), m.data.size() * sizeof(T)); }

void macs_out(const AttnMacs& m, orc_attn_macs* o) {
  if (o) { o->qk += m.qk; o->pv += m.pv; o->lr += m.lr; }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_rng_mix(uint64_t a, uint64_t b) { return Rng::mix(a, b); }
uint64_t ref_rng_child_seed(uint64_t seed, uint64_t key) { return Rng(seed).child(key).seed(); }
void ref_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  Rng g(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = g.next_u64();
}
void ref_fill_gaussian_f32(uint64_t seed, int64_t n, double scale, float* out) {
  put(Matrix<float>::gaussian(1, n, Rng(seed), scale), out);
}
void ref_fill_gaussian_f64(uint64_t seed, int64_t n, double scale, double* out) {
  put(Matrix<double>::gaussian(1, n, Rng(seed), scale), out);
}

void ref_lr_mac_counts(int64_t L, int64_t Lc, int64_t r, int64_t d, uint64_t* no_reorder,
                       uint64_t* reorder) {
  const LrMacCounts c = lr_mac_counts(L, Lc, r, d);
  *no_reorder = c.no_reorder; *reorder = c.reorder;
}

#define REF_ATTENTION(SUF, T, S)                                                                   \
  int ref_naive_attention_##SUF(S q, S k, S v, S vlr, S b, T scale, int64_t off, T* out) {         \
    return guarded([&] { put(naive_attention(inputs<T>(q, k, v, vlr, b, scale, off)), out); });    \
  }                                                                                                \
  int ref_flash_lora_attention_##SUF(S q, S k, S v, S vlr, S b, T scale, int64_t off, int64_t br,  \
                                     int64_t bc, T* out, orc_attn_macs* macs, T* row_max,          \
                                     T* row_denom) {                                               \
    return guarded([&] {                                                                           \
      AttnMacs m;                                                                                  \
      OnlineSoftmaxStats<T> st;                                                                    \
      put(flash_lora_attention(inputs<T>(q, k, v, vlr, b, scale, off), BlockConfig{br, bc}, &m,    \
                               &st), out);                                                         \
      macs_out(m, macs);                                                                           \
      if (row_max) std::memcpy(row_max, st.row_max.data(), st.row_max.size() * sizeof(T));         \
      if (row_denom) std::memcpy(row_denom, st.row_denom.data(), st.row_denom.size() * sizeof(T)); \
    });                                                                                            \
  }                                                                                                \
  int ref_expand_first_attention_##SUF(S q, S k, S v, S vlr, S b, T scale, int64_t off,            \
                                       int64_t br, int64_t bc, T* out, orc_attn_macs* macs) {      \
    return guarded([&] {                                                                           \
      AttnMacs m;                                                                                  \
      put(expand_first_attention(inputs<T>(q, k, v, vlr, b, scale, off), BlockConfig{br, bc}, &m), \
          out);                                                                                    \
      macs_out(m, macs);                                                                           \
    });                                                                                            \
  }                                                                                                \
  int ref_gqa_attention_##SUF(S q, S k, S v, S vlr, S b, T scale, int64_t off, int64_t n_q,        \
                              int64_t n_kv, int64_t br, int64_t bc, T* out, orc_attn_macs* macs) { \
    return guarded([&] {                                                                           \
      AttnMacs m;                                                                                  \
      put(gqa_attention<T>(sp<T>(q), sp<T>(k), sp<T>(v), sp<T>(vlr), sp<T>(b), scale, off, n_q,    \
                           n_kv, BlockConfig{br, bc}, &m), out);                                   \
      macs_out(m, macs);                                                                           \
    });                                                                                            \
  }                                                                                                \
  int ref_matmul_##SUF(S a, S b, T* out) {                                                         \
    return guarded([&] { put(matmul(sp<T>(a), sp<T>(b)), out); });                                 \
  }                                                                                                \
  double ref_max_rel_error_##SUF(const T* a, const T* b, int64_t n) {                              \
    Matrix<T> ma(1, n), mb(1, n);                                                                  \
    std::memcpy(ma.data.data(), a, n * sizeof(T));                                                 \
    std::memcpy(mb.data.data(), b, n * sizeof(T));                                                 \
    return max_rel_error(ma, mb);                                                                  \
  }                                                                                                \
  double ref_max_abs_diff_##SUF(const T* a, const T* b, int64_t n) {                               \
    Matrix<T> ma(1, n), mb(1, n);                                                                  \
    std::memcpy(ma.data.data(), a, n * sizeof(T));                                                 \
    std::memcpy(mb.data.data(), b, n * sizeof(T));                                                 \
    return max_abs_diff(ma, mb);                                                                   \
  }                                                                                                \
  int ref_expand_lr_##SUF(S y, S b, int64_t rank, double alpha, T* out) {                          \
    return guarded([&] {                                                                           \
      Matrix<T> ym(y.rows, y.cols), bm(b.rows, b.cols);                                            \
      for (idx i = 0; i < y.rows; ++i)                                                             \
        for (idx j = 0; j < y.cols; ++j) ym(i, j) = y.data[i * y.stride + j];                      \
      for (idx i = 0; i < b.rows; ++i)                                                             \
        for (idx j = 0; j < b.cols; ++j) bm(i, j) = b.data[i * b.stride + j];                      \
      /* a is irrelevant to expand_lr; give it a valid shape */                                    \
      LoraAdapter<T> ad(Matrix<T>(std::max<idx>(rank, b.cols), rank), bm, rank, alpha);            \
      put(expand_lr(ym, ad), out);                                                                 \
    });                                                                                            \
  }

REF_ATTENTION(f32, float, orc_span_f32)
REF_ATTENTION(f64, double, orc_span_f64)

// The reference's head loop spread over host threads: each q head is an independent, pure
// call of flash_lora_attention (SPEC.md:229-230 permits this), exactly what gqa_attention
// does serially at attention.hpp:347-361.
int ref_gqa_attention_f32_mt(orc_span_f32 q, orc_span_f32 k, orc_span_f32 v, orc_span_f32 vlr,
                             orc_span_f32 b, float scale, int64_t off, int64_t n_q, int64_t n_kv,
                             int64_t br, int64_t bc, float* out, int threads) {
  return guarded([&] {
    if (n_q < 1 || n_kv < 1 || n_q % n_kv != 0) fail("gqa_attention: head counts not divisible");
    if (threads < 1) threads = 1;
    const idx d_head = q.cols / n_q, group = n_q / n_kv;
    std::vector<std::string> errs(static_cast<std::size_t>(threads));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        try {
          for (idx h = t; h < n_q; h += threads) {
            const idx kvh = h / group;
            AttentionInputs<float> in;
            in.q = sp<float>(q).col_range(h * d_head, (h + 1) * d_head);
            in.k = sp<float>(k).col_range(kvh * d_head, (kvh + 1) * d_head);
            in.v_base = sp<float>(v).col_range(kvh * d_head, (kvh + 1) * d_head);
            in.v_lr = sp<float>(vlr);
            in.b_up = vlr.cols > 0 ? sp<float>(b).col_range(kvh * d_head, (kvh + 1) * d_head)
                                   : Span2D<const float>{nullptr, 0, d_head, 0};
            in.lr_scale = scale;
            in.query_offset = off;
            const Matrix<float> ho = flash_lora_attention(in, BlockConfig{br, bc});
            for (idx i = 0; i < ho.rows; ++i)
              for (idx j = 0; j < d_head; ++j) out[i * q.cols + h * d_head + j] = ho(i, j);
          }
        } catch (const std::exception& e) {
          errs[static_cast<std::size_t>(t)] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) fail(e);
  });
}

// run_kernel_fuzz, fuzz.hpp:25-72
int ref_kernel_fuzz_f32(int64_t cases, uint64_t seed, int64_t max_len, int64_t* comparisons,
                        double* max_rel_flash, double* max_rel_expand) {
  return guarded([&] {
    const KernelFuzzResult r = run_kernel_fuzz<float>(cases, seed, max_len);
    *comparisons = r.comparisons; *max_rel_flash = r.max_rel_flash; *max_rel_expand = r.max_rel_expand;
  });
}
int ref_kernel_fuzz_f64(int64_t cases, uint64_t seed, int64_t max_len, int64_t* comparisons,
                        double* max_rel_flash, double* max_rel_expand) {
  return guarded([&] {
    const KernelFuzzResult r = run_kernel_fuzz<double>(cases, seed, max_len);
    *comparisons = r.comparisons; *max_rel_flash = r.max_rel_flash; *max_rel_expand = r.max_rel_expand;
  });
}

int ref_plan_core(int scheme, int64_t first_recompute, int64_t length, int64_t seen,
                  int64_t new_tokens, int64_t out[9]) {
  return guarded([&] {
    CacheScheme cs{static_cast<SchemeKind>(scheme), {}};
    if (cs.kind == SchemeKind::SelectiveRecompute) cs.recompute_layers = {first_recompute};
    const PrefillPlan p = plan_core(cs, length, seen, new_tokens);
    out[0] = p.hidden_pass.begin; out[1] = p.hidden_pass.end;
    out[2] = p.kv_project.begin; out[3] = p.kv_project.end;
    out[4] = p.lr_project.begin; out[5] = p.lr_project.end;
    out[6] = p.kv_recompute.begin; out[7] = p.kv_recompute.end;
    out[8] = p.skip_layers_below;
  });
}

// KvStore<T> behind an opaque handle; elem_size picks float or double.
struct ref_store {
  int elem;
  KvStore<float>* f;
  KvStore<double>* d;
};

ref_store* ref_store_create(int scheme, int64_t n_layers, int64_t d_kv, int64_t d_model,
                            int64_t rank, int64_t n_agents, int elem_size) {
  ref_store* s = nullptr;
  const int rc = guarded([&] {
    CacheScheme cs{static_cast<SchemeKind>(scheme), {}};
    StoreDims dims{n_layers, d_kv, d_model, rank, n_agents};
    s = new ref_store{elem_size, nullptr, nullptr};
    if (elem_size == 4) s->f = new KvStore<float>(cs, dims);
    else s->d = new KvStore<double>(cs, dims);
  });
  if (rc != ORC_OK) { delete s; return nullptr; }
  return s;
}
void ref_store_destroy(ref_store* s) {
  if (!s) return;
  delete s->f; delete s->d; delete s;
}
#define ON_STORE(expr_f, expr_d) (s->elem == 4 ? (expr_f) : (expr_d))
int ref_store_append_tokens(ref_store* s, int64_t n) {
  return guarded([&] {
    std::vector<std::int32_t> ids(static_cast<std::size_t>(n), 1);
    if (s->elem == 4) s->f->append_tokens(ids); else s->d->append_tokens(ids);
  });
}
int64_t ref_store_length(const ref_store* s) { return ON_STORE(s->f->length(), s->d->length()); }
int ref_store_seen(const ref_store* s, int64_t agent, int64_t* out) {
  return guarded([&] { *out = ON_STORE(s->f->seen(agent), s->d->seen(agent)); });
}
int ref_store_mark_seen(ref_store* s, int64_t agent) {
  return guarded([&] { if (s->elem == 4) s->f->mark_seen(agent); else s->d->mark_seen(agent); });
}
int ref_store_append(ref_store* s, int which, int64_t layer, int64_t agent, int64_t row_begin,
                     const void* rows, int64_t n, int64_t stride) {
  return guarded([&] {
    auto go = [&](auto* st, auto* typed) {
      using T = std::remove_cv_t<std::remove_pointer_t<decltype(typed)>>;
      const idx cols = which == 2 ? st->dims().rank : st->dims().d_kv;
      Span2D<const T> v{typed, n, cols, stride};
      if (which == 0) st->append_key(layer, agent, row_begin, v);
      else if (which == 1) st->append_value(layer, agent, row_begin, v);
      else st->append_lr(layer, agent, row_begin, v);
    };
    if (s->elem == 4) go(s->f, static_cast<const float*>(rows));
    else go(s->d, static_cast<const double*>(rows));
  });
}
int ref_store_view(const ref_store* s, int which, int64_t layer, int64_t agent, const void** data,
                   int64_t* rows, int64_t* cols) {
  return guarded([&] {
    auto go = [&](auto* st) {
      auto v = which == 0 ? st->key_view(layer, agent)
               : which == 1 ? st->value_view(layer, agent) : st->lr_view(layer, agent);
      *data = v.data; *rows = v.rows; *cols = v.cols;
    };
    if (s->elem == 4) go(s->f); else go(s->d);
  });
}
void ref_store_bytes(const ref_store* s, uint64_t out[4]) {
  const CacheBytes b = ON_STORE(s->f->bytes(), s->d->bytes());
  out[0] = b.key; out[1] = b.value; out[2] = b.lr; out[3] = b.hidden;
}
uint64_t ref_store_allocated_elements(const ref_store* s) {
  return ON_STORE(s->f->allocated_elements(), s->d->allocated_elements());
}


// KvStore::save_snapshot / load_snapshot (kvcache.hpp:438-546): the reference's own writer and reader
int ref_store_save_snapshot(const ref_store* s, const char* path) {
  return guarded([&] { if (s->elem == 4) s->f->save_snapshot(path); else s->d->save_snapshot(path); });
}
ref_store* ref_store_load_snapshot(const char* path, int elem_size) {
  ref_store* s = nullptr;
  const int rc = guarded([&] {
    s = new ref_store{elem_size, nullptr, nullptr};
    if (elem_size == 4) s->f = new KvStore<float>(KvStore<float>::load_snapshot(path));
    else s->d = new KvStore<double>(KvStore<double>::load_snapshot(path));
  });
  if (rc != ORC_OK) { delete s; return nullptr; }
  return s;
}

// detail::apply_rope (engine.hpp:225-243) on a strided row-major matrix, in place
#define REF_ROPE(SUF, T)                                                                                  \
  int ref_apply_rope_##SUF(T* m, int64_t rows, int64_t stride, int64_t n_heads, int64_t d_head,           \
                           int64_t pos_begin) {                                                           \
    return guarded([&] {                                                                                  \
      Matrix<T> tmp(rows, n_heads * d_head);                                                              \
      for (int64_t i = 0; i < rows; ++i)                                                                  \
        for (int64_t j = 0; j < n_heads * d_head; ++j) tmp(i, j) = m[i * stride + j];                     \
      detail::apply_rope(tmp, n_heads, d_head, pos_begin);                                                \
      for (int64_t i = 0; i < rows; ++i)                                                                  \
        for (int64_t j = 0; j < n_heads * d_head; ++j) m[i * stride + j] = tmp(i, j);                     \
    });                                                                                                   \
  }
REF_ROPE(f32, float)
REF_ROPE(f64, double)

}  // extern "C"
