/*
 * lorakv_oracle.h -- CPU restatement of the reference's Flash-LoRA-Attention path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library, and there only as the checker / the CPU baseline.
 * The product path (paper_2602_01053_b200/csrc -> liblorakv_b200.so) never links,
 * loads or calls it.
 *
 * Parity status: PINNED.  Every function below follows a cited function of the
 * reference (file:line under /root/reference/proj) with the same operation order,
 * and tests/test_oracle_*.py check it (a) bit-for-bit against oracle/_ref (the
 * reference's own headers compiled by oracle/Makefile) when that library is
 * present and (b) against the committed fixtures in tests/golden/ that
 * oracle/gen_golden.py produced from the reference.
 *
 * The one function with no reference counterpart is orc_page_of() (the reference
 * has no pages); it is the trivial "row -> (row / P, row % P), pages
 * handed out in first-touch order" model the GPU page table must match.
 *
 * All matrices are row-major with an explicit row stride in elements
 * (reference: Span2D, include/lorakv/matrix.hpp:31-38).
 */
#ifndef LORAKV_ORACLE_H
#define LORAKV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* borrowed view, mirrors Span2D<const T> */
typedef struct { const float* data; int64_t rows, cols, stride; } orc_span_f32;
typedef struct { const double* data; int64_t rows, cols, stride; } orc_span_f64;

/* status codes; message of the last failure on this thread via orc_last_error() */
enum { ORC_OK = 0, ORC_ERR = 1 };
const char* orc_last_error(void);

/* ---- rng.hpp:10-53 ------------------------------------------------------ */
uint64_t orc_rng_mix(uint64_t a, uint64_t b);                 /* Rng::mix      :41 */
uint64_t orc_rng_child_seed(uint64_t seed, uint64_t key);     /* Rng::child    :39 */
/* n consecutive next_u64() draws of Rng(seed)                 rng.hpp:14-20 */
void orc_rng_u64(uint64_t seed, int64_t n, uint64_t* out);
/* Matrix<T>::gaussian(rows*cols, Rng(seed), scale)            matrix.hpp:83-87 */
void orc_fill_gaussian_f32(uint64_t seed, int64_t n, double scale, float* out);
void orc_fill_gaussian_f64(uint64_t seed, int64_t n, double scale, double* out);

/* ---- attention.hpp ------------------------------------------------------ */
typedef struct { uint64_t qk, pv, lr; } orc_attn_macs;            /* :22 */
void orc_lr_mac_counts(int64_t total_len, int64_t cur_len, int64_t rank, int64_t d_head,
                       uint64_t* no_reorder, uint64_t* reorder);  /* :35 */

/* naive_attention :81-112; out is L_c x d dense */
int orc_naive_attention_f32(orc_span_f32 q, orc_span_f32 k, orc_span_f32 v_base, orc_span_f32 v_lr,
                            orc_span_f32 b_up, float lr_scale, int64_t query_offset, float* out);
int orc_naive_attention_f64(orc_span_f64 q, orc_span_f64 k, orc_span_f64 v_base, orc_span_f64 v_lr,
                            orc_span_f64 b_up, double lr_scale, int64_t query_offset, double* out);

/* flash_lora_attention :210-268 (+ flash_tile_update :140-200).
 * macs / row_max / row_denom may be NULL. */
int orc_flash_lora_attention_f32(orc_span_f32 q, orc_span_f32 k, orc_span_f32 v_base,
                                 orc_span_f32 v_lr, orc_span_f32 b_up, float lr_scale,
                                 int64_t query_offset, int64_t b_r, int64_t b_c, float* out,
                                 orc_attn_macs* macs, float* row_max, float* row_denom);
int orc_flash_lora_attention_f64(orc_span_f64 q, orc_span_f64 k, orc_span_f64 v_base,
                                 orc_span_f64 v_lr, orc_span_f64 b_up, double lr_scale,
                                 int64_t query_offset, int64_t b_r, int64_t b_c, double* out,
                                 orc_attn_macs* macs, double* row_max, double* row_denom);

/* expand_first_attention :274-326 */
int orc_expand_first_attention_f32(orc_span_f32 q, orc_span_f32 k, orc_span_f32 v_base,
                                   orc_span_f32 v_lr, orc_span_f32 b_up, float lr_scale,
                                   int64_t query_offset, int64_t b_r, int64_t b_c, float* out,
                                   orc_attn_macs* macs);
int orc_expand_first_attention_f64(orc_span_f64 q, orc_span_f64 k, orc_span_f64 v_base,
                                   orc_span_f64 v_lr, orc_span_f64 b_up, double lr_scale,
                                   int64_t query_offset, int64_t b_r, int64_t b_c, double* out,
                                   orc_attn_macs* macs);

/* gqa_attention :332-363; out is L_c x (n_q*d_head) dense */
int orc_gqa_attention_f32(orc_span_f32 q, orc_span_f32 k, orc_span_f32 v_base, orc_span_f32 v_lr,
                          orc_span_f32 b_up, float lr_scale, int64_t query_offset,
                          int64_t n_q_heads, int64_t n_kv_heads, int64_t b_r, int64_t b_c,
                          float* out, orc_attn_macs* macs);
int orc_gqa_attention_f64(orc_span_f64 q, orc_span_f64 k, orc_span_f64 v_base, orc_span_f64 v_lr,
                          orc_span_f64 b_up, double lr_scale, int64_t query_offset,
                          int64_t n_q_heads, int64_t n_kv_heads, int64_t b_r, int64_t b_c,
                          double* out, orc_attn_macs* macs);

/* Same as orc_gqa_attention_f32 but the q heads are spread over `threads` host
 * threads (pure, independent calls: SPEC.md:229-230).  Used by the CPU baseline. */
int orc_gqa_attention_f32_mt(orc_span_f32 q, orc_span_f32 k, orc_span_f32 v_base,
                             orc_span_f32 v_lr, orc_span_f32 b_up, float lr_scale,
                             int64_t query_offset, int64_t n_q_heads, int64_t n_kv_heads,
                             int64_t b_r, int64_t b_c, float* out, int threads);

/* ---- matrix.hpp --------------------------------------------------------- */
/* matmul :114-122 (matmul_accumulate :101-111, i-p-j order); out rows(a) x cols(b) */
int orc_matmul_f32(orc_span_f32 a, orc_span_f32 b, float* out);
int orc_matmul_f64(orc_span_f64 a, orc_span_f64 b, double* out);
/* max_rel_error :202-214 and max_abs_diff :217-223 over n elements */
double orc_max_rel_error_f32(const float* a, const float* b, int64_t n);
double orc_max_rel_error_f64(const double* a, const double* b, int64_t n);
double orc_max_abs_diff_f32(const float* a, const float* b, int64_t n);
double orc_max_abs_diff_f64(const double* a, const double* b, int64_t n);

/* ---- lora.hpp ----------------------------------------------------------- */
/* expand_lr :39-47: out = scale * (y_lr * b), scale = (T)(alpha / rank) */
int orc_expand_lr_f32(orc_span_f32 y_lr, orc_span_f32 b, int64_t rank, double alpha, float* out);
int orc_expand_lr_f64(orc_span_f64 y_lr, orc_span_f64 b, int64_t rank, double alpha, double* out);

/* ---- kvcache.hpp -------------------------------------------------------- */
enum { ORC_NONSHARED = 0, ORC_FULLSHARED = 1, ORC_BASESHARED = 2, ORC_BASELRSHARED = 3,
       ORC_SELECTIVE = 4 };                                        /* SchemeKind :15-21 */
/* plan_core :112-142.  out[0..1]=hidden_pass, [2..3]=kv_project, [4..5]=lr_project,
 * [6..7]=kv_recompute, [8]=skip_layers_below (first_recompute passed by caller). */
int orc_plan_core(int scheme, int64_t first_recompute, int64_t length, int64_t seen,
                  int64_t new_tokens, int64_t out[9]);

/* append_fww :400-407 arithmetic on one buffer with `rows` rows:
 * returns ORC_ERR on a gap; otherwise *skip = rows of the source already present and
 * *appended = rows actually appended (0 when fully present). */
int orc_append_fww(int64_t rows, int64_t row_begin, int64_t n_src, int64_t* skip, int64_t* appended);

/* KvStore<T> :213-420 restated with double/float payloads kept in growable buffers.
 * elem_size selects sizeof(T) (4 or 8) for bytes(). */
typedef struct orc_store orc_store;
orc_store* orc_store_create(int scheme, int64_t n_layers, int64_t d_kv, int64_t d_model,
                            int64_t rank, int64_t n_agents, int elem_size);
void orc_store_destroy(orc_store*);
int  orc_store_append_tokens(orc_store*, int64_t n);                 /* :254-257 */
int64_t orc_store_length(const orc_store*);
int  orc_store_seen(const orc_store*, int64_t agent, int64_t* out);   /* :259 */
int  orc_store_mark_seen(orc_store*, int64_t agent);                 /* :260-264 */
/* which: 0 = key, 1 = value, 2 = lr.  rows is n x cols(which) with the given stride;
 * data is float when elem_size==4 else double. */
int  orc_store_append(orc_store*, int which, int64_t layer, int64_t agent, int64_t row_begin,
                      const void* rows, int64_t n, int64_t stride);  /* :268-288 */
/* view: rows/cols of the buffer the scheme resolves (layer, agent) to, pointer to data */
int  orc_store_view(const orc_store*, int which, int64_t layer, int64_t agent,
                    const void** data, int64_t* rows, int64_t* cols);/* :307-324 */
void orc_store_bytes(const orc_store*, uint64_t out[4]);             /* :330-344 key,value,lr,hidden */
uint64_t orc_store_allocated_elements(const orc_store*);             /* :346-358 */

/* Page model (no reference counterpart, see header comment): logical row -> page slot. */
void orc_page_of(int64_t row, int64_t page_tokens, int64_t* logical_page, int64_t* row_in_page);

/* bf16 helpers for the bf16 storage mode: round-to-nearest-even to bf16 and back. */
float orc_round_bf16(float x);
void  orc_round_bf16_array(const float* in, float* out, int64_t n);

/* engine.hpp:225-243 (detail::apply_rope), in place on a row-major matrix with the given row stride */
int orc_apply_rope_f32(float* m, int64_t rows, int64_t stride, int64_t n_heads, int64_t d_head, int64_t pos_begin);
int orc_apply_rope_f64(double* m, int64_t rows, int64_t stride, int64_t n_heads, int64_t d_head, int64_t pos_begin);

#ifdef __cplusplus
}
#endif
#endif
