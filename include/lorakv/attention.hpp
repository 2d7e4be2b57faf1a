// lorakv/attention.hpp -- the attention operators of the reference (proj/include/lorakv/attention.hpp)
// with the same signatures, executed on the B200 through the C ABI (include/lorakv_b200.h).
//
//   flash_lora_attention   -> lorakv_fla_forward_*           (attention.hpp:210-268)
//   expand_first_attention -> lorakv_expand_first_forward_*  (attention.hpp:274-326)
//   naive_attention        -> lorakv_naive_forward_*         (attention.hpp:81-112)
//   gqa_attention          -> lorakv_gqa_forward_*           (attention.hpp:332-363), all q heads in one launch
//
// Argument meaning, validation order, error text and the optional AttnMacs / OnlineSoftmaxStats
// outputs follow the reference.  BlockConfig is validated but does not steer the device kernels:
// the result is independent of tiling up to rounding (SPEC, attention.hpp:18-21), and the dense MAC
// counters are tiling-independent closed forms, filled from lorakv_attn_macs.
// These header-level operators take HOST views and therefore copy operands per call; the
// device-resident fast paths over the paged cache are in lorakv/device.hpp.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "lorakv/matrix.hpp"

namespace lorakv {

struct BlockConfig {
  idx b_r = 64;   // query rows per block
  idx b_c = 64;   // keys per tile
};

// Dense MAC counters (masked entries included, so they equal the closed-form cost model for any tiling)
struct AttnMacs {
  std::uint64_t qk = 0;   // Q K^T
  std::uint64_t pv = 0;   // P V_base
  std::uint64_t lr = 0;   // P V_lr + (P V_lr) B  -- or V_lr B + P (V_lr B) for expand-first
};

struct LrMacCounts {
  std::uint64_t no_reorder = 0;   // L r d + L_c L d
  std::uint64_t reorder = 0;      // L_c L r + L_c r d
};

inline LrMacCounts lr_mac_counts(idx total_len, idx cur_len, idx rank, idx d_head) {
  LrMacCounts c;
  lorakv_lr_mac_counts(total_len, cur_len, rank, d_head, &c.no_reorder, &c.reorder);
  return c;
}

// Operands of one head.  Query row i sits at sequence position query_offset + i and sees key j iff
// j <= query_offset + i.  A zero-column v_lr means plain attention over v_base.
template <class T>
struct AttentionInputs {
  Span2D<const T> q;        // L_c x d
  Span2D<const T> k;        // L x d
  Span2D<const T> v_base;   // L x d
  Span2D<const T> v_lr;     // L x r
  Span2D<const T> b_up;     // r x d
  T lr_scale = T(1);
  idx query_offset = 0;
};

template <class T>
inline void validate_attention_inputs(const AttentionInputs<T>& in) {
  const idx L = in.k.rows, d = in.q.cols, r = in.v_lr.cols;
  if (in.k.cols != d) fail("attention: q/k head dim mismatch");
  if (in.v_base.rows != L || in.v_base.cols != d)
    fail("attention: v_base shape " + shape_str(in.v_base.rows, in.v_base.cols) + " does not match k " + shape_str(L, d));
  if (r != 0 && in.v_lr.rows != L)
    fail("attention: v_lr rows " + std::to_string(in.v_lr.rows) + " != sequence length " + std::to_string(L));
  if (in.b_up.rows != r || (r > 0 && in.b_up.cols != d))
    fail("attention: b_up shape " + shape_str(in.b_up.rows, in.b_up.cols) + " does not match rank " + std::to_string(r));
  if (in.query_offset < 0 || in.query_offset + in.q.rows > L)
    fail("attention: query_offset " + std::to_string(in.query_offset) + " with L_c " + std::to_string(in.q.rows) +
         " exceeds L " + std::to_string(L));
}

// final online-softmax state per query row
template <class T>
struct OnlineSoftmaxStats {
  std::vector<T> row_max;
  std::vector<T> row_denom;
};

namespace detail {

inline void add_macs(AttnMacs* macs, idx L_c, idx L, idx d, idx r, bool expand_first) {
  if (!macs) return;
  std::uint64_t m[3];
  lorakv_attn_macs(L_c, L, d, r, expand_first ? 1 : 0, m);
  macs->qk += m[0];
  macs->pv += m[1];
  macs->lr += m[2];
}

}  // namespace detail

// Materialising algorithm (full score matrix, row softmax, expanded values), kept as an independent
// device implementation so kernel-vs-oracle sweeps (lorakv/fuzz.hpp) still compare two algorithms.
template <class T>
inline Matrix<T> naive_attention(const AttentionInputs<T>& in) {
  static_assert(b200::is_supported<T>, "lorakv operators exist for float and double");
  validate_attention_inputs(in);
  Matrix<T> out(in.q.rows, in.q.cols);
  lorakv_ctx* ctx = b200::Runtime::ctx();
  const idx L_c = in.q.rows, L = in.k.rows, d = in.q.cols, r = in.v_lr.cols;
  if constexpr (std::is_same_v<T, float>)
    b200::check(lorakv_naive_forward_f32(ctx, in.q.data, in.q.stride, in.k.data, in.k.stride, in.v_base.data, in.v_base.stride,
                                         in.v_lr.data, in.v_lr.stride, in.b_up.data, in.b_up.stride, in.lr_scale, L_c, L, d,
                                         r, in.query_offset, out.data.data()));
  else
    b200::check(lorakv_naive_forward_f64(ctx, in.q.data, in.q.stride, in.k.data, in.k.stride, in.v_base.data, in.v_base.stride,
                                         in.v_lr.data, in.v_lr.stride, in.b_up.data, in.b_up.stride, in.lr_scale, L_c, L, d,
                                         r, in.query_offset, out.data.data()));
  return out;
}

// Flash-LoRA-Attention: online softmax over key tiles, P V_base in d columns and P V_lr in r columns,
// then o += (lr_scale * o_lr[p]) * b_up[p,:] and the division by the denominator.
template <class T>
inline Matrix<T> flash_lora_attention(const AttentionInputs<T>& in, const BlockConfig& cfg, AttnMacs* macs = nullptr,
                                      OnlineSoftmaxStats<T>* stats = nullptr) {
  static_assert(b200::is_supported<T>, "lorakv operators exist for float and double");
  validate_attention_inputs(in);
  if (cfg.b_r < 1 || cfg.b_c < 1) fail("flash_lora_attention: block sizes must be >= 1");
  const idx L_c = in.q.rows, L = in.k.rows, d = in.q.cols, r = in.v_lr.cols;
  Matrix<T> out(L_c, d);
  T* row_max = nullptr;
  T* row_denom = nullptr;
  if (stats) {
    stats->row_max.assign(static_cast<std::size_t>(L_c), T(0));
    stats->row_denom.assign(static_cast<std::size_t>(L_c), T(0));
    row_max = stats->row_max.data();
    row_denom = stats->row_denom.data();
  }
  lorakv_ctx* ctx = b200::Runtime::ctx();
  if constexpr (std::is_same_v<T, float>)
    b200::check(lorakv_fla_forward_f32(ctx, in.q.data, in.q.stride, in.k.data, in.k.stride, in.v_base.data, in.v_base.stride,
                                       in.v_lr.data, in.v_lr.stride, in.b_up.data, in.b_up.stride, in.lr_scale, L_c, L, d, r,
                                       in.query_offset, out.data.data(), row_max, row_denom));
  else
    b200::check(lorakv_fla_forward_f64(ctx, in.q.data, in.q.stride, in.k.data, in.k.stride, in.v_base.data, in.v_base.stride,
                                       in.v_lr.data, in.v_lr.stride, in.b_up.data, in.b_up.stride, in.lr_scale, L_c, L, d, r,
                                       in.query_offset, out.data.data(), row_max, row_denom));
  detail::add_macs(macs, L_c, L, d, r, false);
  return out;
}

// Baseline: materialise lr_scale * (V_lr B) over the whole sequence, then attend with a second d-wide
// accumulator.  Its lr counter follows the no-reorder cost form.
template <class T>
inline Matrix<T> expand_first_attention(const AttentionInputs<T>& in, const BlockConfig& cfg, AttnMacs* macs = nullptr) {
  static_assert(b200::is_supported<T>, "lorakv operators exist for float and double");
  validate_attention_inputs(in);
  if (cfg.b_r < 1 || cfg.b_c < 1) fail("expand_first_attention: block sizes must be >= 1");
  const idx L_c = in.q.rows, L = in.k.rows, d = in.q.cols, r = in.v_lr.cols;
  Matrix<T> out(L_c, d);
  lorakv_ctx* ctx = b200::Runtime::ctx();
  if constexpr (std::is_same_v<T, float>)
    b200::check(lorakv_expand_first_forward_f32(ctx, in.q.data, in.q.stride, in.k.data, in.k.stride, in.v_base.data,
                                                in.v_base.stride, in.v_lr.data, in.v_lr.stride, in.b_up.data, in.b_up.stride,
                                                in.lr_scale, L_c, L, d, r, in.query_offset, out.data.data()));
  else
    b200::check(lorakv_expand_first_forward_f64(ctx, in.q.data, in.q.stride, in.k.data, in.k.stride, in.v_base.data,
                                                in.v_base.stride, in.v_lr.data, in.v_lr.stride, in.b_up.data, in.b_up.stride,
                                                in.lr_scale, L_c, L, d, r, in.query_offset, out.data.data()));
  detail::add_macs(macs, L_c, L, d, r, true);
  return out;
}

// Grouped-query multi-head wrapper: q head h reads kv head h / (n_q / n_kv); one L x r value cache
// serves every head and kv head h' owns columns [h' d, (h'+1) d) of b_up.
template <class T>
inline Matrix<T> gqa_attention(Span2D<const T> q, Span2D<const T> k, Span2D<const T> v_base, Span2D<const T> v_lr,
                               Span2D<const T> b_up, T lr_scale, idx query_offset, idx n_q_heads, idx n_kv_heads,
                               const BlockConfig& cfg, AttnMacs* macs = nullptr) {
  static_assert(b200::is_supported<T>, "lorakv operators exist for float and double");
  if (n_q_heads < 1 || n_kv_heads < 1 || n_q_heads % n_kv_heads != 0)
    fail("gqa_attention: n_q_heads " + std::to_string(n_q_heads) + " not divisible by n_kv_heads " +
         std::to_string(n_kv_heads));
  if (q.cols % n_q_heads != 0) fail("gqa_attention: q width not divisible by head count");
  const idx d = q.cols / n_q_heads;
  if (k.cols != n_kv_heads * d || v_base.cols != n_kv_heads * d)
    fail("gqa_attention: k/v width does not match n_kv_heads * d_head");
  {   // the per-head checks of the reference, once (every head has the same shapes)
    AttentionInputs<T> head;
    head.q = q.col_range(0, d);
    head.k = k.col_range(0, d);
    head.v_base = v_base.col_range(0, d);
    head.v_lr = v_lr;
    head.b_up = v_lr.cols > 0 ? b_up.col_range(0, d) : Span2D<const T>{nullptr, 0, d, 0};
    head.query_offset = query_offset;
    validate_attention_inputs(head);
  }
  if (cfg.b_r < 1 || cfg.b_c < 1) fail("flash_lora_attention: block sizes must be >= 1");
  const idx L_c = q.rows, L = k.rows, r = v_lr.cols;
  Matrix<T> out(q.rows, q.cols);
  lorakv_ctx* ctx = b200::Runtime::ctx();
  if constexpr (std::is_same_v<T, float>)
    b200::check(lorakv_gqa_forward_f32(ctx, q.data, q.stride, k.data, k.stride, v_base.data, v_base.stride, v_lr.data,
                                       v_lr.stride, b_up.data, b_up.stride, lr_scale, L_c, L, n_q_heads, n_kv_heads, d, r,
                                       query_offset, out.data.data()));
  else
    b200::check(lorakv_gqa_forward_f64(ctx, q.data, q.stride, k.data, k.stride, v_base.data, v_base.stride, v_lr.data,
                                       v_lr.stride, b_up.data, b_up.stride, lr_scale, L_c, L, n_q_heads, n_kv_heads, d, r,
                                       query_offset, out.data.data()));
  for (idx h = 0; h < n_q_heads; ++h) detail::add_macs(macs, L_c, L, d, r, false);
  return out;
}

}  // namespace lorakv
