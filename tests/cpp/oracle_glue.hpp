// oracle_glue.hpp -- the CPU checker (oracle/liblorakv_oracle.so, a restatement of the reference pinned
// to it by tests/test_oracle_*.py) behind lorakv-typed helpers.  TEST CODE ONLY: the product headers
// in include/lorakv never see the oracle.
#pragma once

#include <type_traits>

#include "lorakv/attention.hpp"
#include "lorakv/lora.hpp"
extern "C" {
#include "lorakv_oracle.h"
}

namespace oracle {

using lorakv::idx;
using lorakv::Matrix;
using lorakv::Span2D;

inline void ok(int rc) { if (rc != ORC_OK) throw std::runtime_error(std::string("oracle: ") + orc_last_error()); }
inline orc_span_f32 sp(Span2D<const float> s) { return orc_span_f32{s.data, s.rows, s.cols, s.stride}; }
inline orc_span_f64 sp(Span2D<const double> s) { return orc_span_f64{s.data, s.rows, s.cols, s.stride}; }

template <class T>
Matrix<T> naive(const lorakv::AttentionInputs<T>& in) {
  Matrix<T> out(in.q.rows, in.q.cols);
  if constexpr (std::is_same_v<T, float>)
    ok(orc_naive_attention_f32(sp(in.q), sp(in.k), sp(in.v_base), sp(in.v_lr), sp(in.b_up), in.lr_scale, in.query_offset, out.data.data()));
  else
    ok(orc_naive_attention_f64(sp(in.q), sp(in.k), sp(in.v_base), sp(in.v_lr), sp(in.b_up), in.lr_scale, in.query_offset, out.data.data()));
  return out;
}

template <class T>
Matrix<T> flash(const lorakv::AttentionInputs<T>& in, lorakv::BlockConfig cfg, lorakv::AttnMacs* macs = nullptr,
                lorakv::OnlineSoftmaxStats<T>* stats = nullptr) {
  Matrix<T> out(in.q.rows, in.q.cols);
  orc_attn_macs m{0, 0, 0};
  T* rm = nullptr; T* rd = nullptr;
  if (stats) {
    stats->row_max.assign((size_t)in.q.rows, T(0)); stats->row_denom.assign((size_t)in.q.rows, T(0));
    rm = stats->row_max.data(); rd = stats->row_denom.data();
  }
  if constexpr (std::is_same_v<T, float>)
    ok(orc_flash_lora_attention_f32(sp(in.q), sp(in.k), sp(in.v_base), sp(in.v_lr), sp(in.b_up), in.lr_scale, in.query_offset, cfg.b_r, cfg.b_c, out.data.data(), &m, rm, rd));
  else
    ok(orc_flash_lora_attention_f64(sp(in.q), sp(in.k), sp(in.v_base), sp(in.v_lr), sp(in.b_up), in.lr_scale, in.query_offset, cfg.b_r, cfg.b_c, out.data.data(), &m, rm, rd));
  if (macs) { macs->qk += m.qk; macs->pv += m.pv; macs->lr += m.lr; }
  return out;
}

template <class T>
Matrix<T> expand_first(const lorakv::AttentionInputs<T>& in, lorakv::BlockConfig cfg, lorakv::AttnMacs* macs = nullptr) {
  Matrix<T> out(in.q.rows, in.q.cols);
  orc_attn_macs m{0, 0, 0};
  if constexpr (std::is_same_v<T, float>)
    ok(orc_expand_first_attention_f32(sp(in.q), sp(in.k), sp(in.v_base), sp(in.v_lr), sp(in.b_up), in.lr_scale, in.query_offset, cfg.b_r, cfg.b_c, out.data.data(), &m));
  else
    ok(orc_expand_first_attention_f64(sp(in.q), sp(in.k), sp(in.v_base), sp(in.v_lr), sp(in.b_up), in.lr_scale, in.query_offset, cfg.b_r, cfg.b_c, out.data.data(), &m));
  if (macs) { macs->qk += m.qk; macs->pv += m.pv; macs->lr += m.lr; }
  return out;
}

template <class T>
Matrix<T> gqa(Span2D<const T> q, Span2D<const T> k, Span2D<const T> v, Span2D<const T> v_lr, Span2D<const T> b, T s,
              idx off, idx n_q, idx n_kv, lorakv::AttnMacs* macs = nullptr) {
  Matrix<T> out(q.rows, q.cols);
  orc_attn_macs m{0, 0, 0};
  if constexpr (std::is_same_v<T, float>)
    ok(orc_gqa_attention_f32(sp(q), sp(k), sp(v), sp(v_lr), sp(b), s, off, n_q, n_kv, 64, 64, out.data.data(), &m));
  else
    ok(orc_gqa_attention_f64(sp(q), sp(k), sp(v), sp(v_lr), sp(b), s, off, n_q, n_kv, 64, 64, out.data.data(), &m));
  if (macs) { macs->qk += m.qk; macs->pv += m.pv; macs->lr += m.lr; }
  return out;
}

template <class T>
Matrix<T> matmul(const Matrix<T>& a, const Matrix<T>& b) {
  Matrix<T> out(a.rows, b.cols);
  if constexpr (std::is_same_v<T, float>) ok(orc_matmul_f32(sp(a.view()), sp(b.view()), out.data.data()));
  else ok(orc_matmul_f64(sp(a.view()), sp(b.view()), out.data.data()));
  return out;
}

inline Matrix<float> round_bf16(const Matrix<float>& a) {
  Matrix<float> out(a.rows, a.cols);
  orc_round_bf16_array(a.data.data(), out.data.data(), (int64_t)a.data.size());
  return out;
}

}  // namespace oracle
