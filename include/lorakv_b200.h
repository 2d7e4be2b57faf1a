/*
 * lorakv_b200.h -- C ABI of the B200-native Flash-LoRA-Attention path (liblorakv_b200.so).
 *
 * This is the drop-in boundary.  The reference (lorakv, arXiv 2602.01053) has no FFI layer: its
 * operator API is the C++ header surface in proj/include/lorakv/.  Every entry point below names
 * the reference symbol (file:line under /root/reference) it stands in for; the source-compatible
 * C++ headers in include/lorakv/ are thin wrappers over exactly these functions, and
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions
 *   - plain pointers and sizes only; opaque handles for device-resident state;
 *   - every function returns 0 on success, non-zero on failure; the message (same wording as the
 *     reference's std::runtime_error text where one exists, matrix.hpp:17-19) is returned by
 *     lorakv_last_error() for the calling thread;
 *   - matrices are row-major with an explicit row stride in ELEMENTS (Span2D, matrix.hpp:31-38);
 *   - there is no CPU fallback: without a CUDA device every compute entry point fails loudly.
 */
#ifndef LORAKV_B200_H
#define LORAKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LORAKV_ABI_VERSION 6   /* 2: projections (lorakv_proj_*), snapshot / resume; 3: output gather over peer memory;
                                  4: lorakv_step_layer, lorakv_snapshot_tokens, fp64 pools, SelectiveRecompute store;
                                  5: key-side low-rank term (lorakv_pool_dims.rank_k, lorakv_adapters_*_k, *_keylr_*);
                                  6: fp32 mode on tcgen05 (plane kernels), lorakv_ctx_set_prefill_split_keys */

typedef struct lorakv_ctx lorakv_ctx;           /* device + stream + scratch */
typedef struct lorakv_pool lorakv_pool;         /* paged cache of one trajectory (KvStore<T>) */
typedef struct lorakv_adapters lorakv_adapters; /* shared A per layer, B per (layer, agent) */

enum { LORAKV_OK = 0, LORAKV_ERR = 1 };

/* storage / arithmetic modes */
enum { LORAKV_F32 = 0, LORAKV_BF16 = 1,
       LORAKV_F64 = 2 };  /* fp64 pages: KvStore<double> of the reference API (exact rows, lorakv_pool_append_f64 / _read_f64);
                             storage only -- attention over such a store goes through the views and lorakv_gqa_forward_f64 */
/* where a caller buffer lives */
enum { LORAKV_HOST = 0, LORAKV_DEVICE = 1 };
/* SchemeKind, kvcache.hpp:15-21 (SelectiveRecompute is outside the hot path) */
enum { LORAKV_NONSHARED = 0, LORAKV_FULLSHARED = 1, LORAKV_BASESHARED = 2, LORAKV_BASELRSHARED = 3,
       LORAKV_SELECTIVE = 4 };
/* which cache (LORAKV_HIDDEN: the hidden-state cache of SelectiveRecompute, kvcache.hpp:245-246, 289-293; layer ignored) */
enum { LORAKV_KEY = 0, LORAKV_VALUE = 1, LORAKV_LR = 2, LORAKV_HIDDEN = 3,
       LORAKV_LK = 4 };   /* the key-side low-rank cache L_k = X A_k (extension; lorakv_pool_dims.rank_k > 0; layer-wide, no agent) */

int lorakv_abi_version(void);
const char* lorakv_last_error(void);

/* ---- context ------------------------------------------------------------------------------- */
/* stream: a cudaStream_t to launch on (borrowed), or NULL to create a private one. */
int lorakv_ctx_create(int device, void* stream, lorakv_ctx** out);
void lorakv_ctx_destroy(lorakv_ctx* ctx);
int lorakv_ctx_synchronize(lorakv_ctx* ctx);
void* lorakv_ctx_stream(lorakv_ctx* ctx);
int lorakv_ctx_sm_count(lorakv_ctx* ctx);
/* L2 capacity the decode path plans with (default: the device's).  The low-rank cache V_lr is shared by the kv heads
 * of a layer; the decode keeps it L2-resident (evict-last hint) when the launch's share fits, and otherwise walks the
 * layers in equal chunks inside the kernel so that one chunk's share does.  Tests shrink it to force the chunked path. */
int lorakv_ctx_set_l2_bytes(lorakv_ctx* ctx, int64_t bytes);
/* Keys per split of the fp32-mode tensor-core prefill (fla_prefill_split; default 4096, rounded up to 64).  A tensor-core
 * accumulate truncates, so a CTA accumulates over one split only and the splits of a row are combined with rounded fp32
 * adds: shorter splits = less truncation bias, more partials.  0 restores the default.  Tests shrink it to cover many
 * splits, empty splits and ragged row blocks at small sizes. */
int lorakv_ctx_set_prefill_split_keys(lorakv_ctx* ctx, int64_t keys);
/* number of kernels this library has launched on ctx since creation (bench.py's gpu_launches) */
int64_t lorakv_ctx_launch_count(lorakv_ctx* ctx);

/* device / pinned-host buffers for callers that do not link the CUDA runtime themselves */
int lorakv_dev_alloc(lorakv_ctx* ctx, int64_t bytes, void** out);
int lorakv_dev_free(lorakv_ctx* ctx, void* p);
int lorakv_host_alloc(lorakv_ctx* ctx, int64_t bytes, void** out); /* pinned */
int lorakv_host_free(lorakv_ctx* ctx, void* p);
int lorakv_copy_h2d(lorakv_ctx* ctx, void* dst_dev, const void* src_host, int64_t bytes); /* async on ctx stream */
int lorakv_copy_d2h(lorakv_ctx* ctx, void* dst_host, const void* src_dev, int64_t bytes); /* async on ctx stream */
/* writes `bytes` of a scratch buffer (> L2) so that the next kernel starts with a cold L2 */
int lorakv_flush_l2(lorakv_ctx* ctx);
/* CUDA events recorded on the ctx stream -- the stream every kernel of this library launches on --
 * so a caller can time the library on the device without linking the CUDA runtime.
 * lorakv_event_elapsed_ms waits for `stop` and returns the device time between the two records. */
typedef struct lorakv_event lorakv_event;
int lorakv_event_create(lorakv_ctx* ctx, lorakv_event** out);
int lorakv_event_record(lorakv_ctx* ctx, lorakv_event* ev);
int lorakv_event_elapsed_ms(lorakv_event* start, lorakv_event* stop, float* ms);
void lorakv_event_destroy(lorakv_event* ev);

/* ---- per-head operators over caller memory (HOST pointers) ----------------------------------
 * flash_lora_attention<T>, attention.hpp:210-268.  q: L_c x d, k/v_base: L x d, v_lr: L x r,
 * b_up: r x d, out: L_c x d dense.  row_max / row_denom (OnlineSoftmaxStats, :116-119) may be NULL.
 * Result is independent of any tiling, so BlockConfig only needs validating by the caller. */
int lorakv_fla_forward_f32(lorakv_ctx* ctx, const float* q, int64_t ldq, const float* k, int64_t ldk,
                           const float* v_base, int64_t ldv, const float* v_lr, int64_t ldlr,
                           const float* b_up, int64_t ldb, float lr_scale, int64_t L_c, int64_t L,
                           int64_t d, int64_t r, int64_t query_offset, float* out, float* row_max,
                           float* row_denom);
int lorakv_fla_forward_f64(lorakv_ctx* ctx, const double* q, int64_t ldq, const double* k, int64_t ldk,
                           const double* v_base, int64_t ldv, const double* v_lr, int64_t ldlr,
                           const double* b_up, int64_t ldb, double lr_scale, int64_t L_c, int64_t L,
                           int64_t d, int64_t r, int64_t query_offset, double* out, double* row_max,
                           double* row_denom);
/* expand_first_attention<T>, attention.hpp:274-326: materialises lr_scale*(V_lr*B) (L x d) on the
 * device, then attends with a second d-wide accumulator.  The baseline the paper compares with. */
int lorakv_expand_first_forward_f32(lorakv_ctx* ctx, const float* q, int64_t ldq, const float* k,
                                    int64_t ldk, const float* v_base, int64_t ldv, const float* v_lr,
                                    int64_t ldlr, const float* b_up, int64_t ldb, float lr_scale,
                                    int64_t L_c, int64_t L, int64_t d, int64_t r,
                                    int64_t query_offset, float* out);
int lorakv_expand_first_forward_f64(lorakv_ctx* ctx, const double* q, int64_t ldq, const double* k,
                                    int64_t ldk, const double* v_base, int64_t ldv,
                                    const double* v_lr, int64_t ldlr, const double* b_up, int64_t ldb,
                                    double lr_scale, int64_t L_c, int64_t L, int64_t d, int64_t r,
                                    int64_t query_offset, double* out);
/* naive_attention<T>, attention.hpp:81-112: full score matrix, row softmax, expanded values --
 * the materialising algorithm, kept as an independent device implementation for cross-checks. */
int lorakv_naive_forward_f32(lorakv_ctx* ctx, const float* q, int64_t ldq, const float* k, int64_t ldk,
                             const float* v_base, int64_t ldv, const float* v_lr, int64_t ldlr,
                             const float* b_up, int64_t ldb, float lr_scale, int64_t L_c, int64_t L,
                             int64_t d, int64_t r, int64_t query_offset, float* out);
int lorakv_naive_forward_f64(lorakv_ctx* ctx, const double* q, int64_t ldq, const double* k,
                             int64_t ldk, const double* v_base, int64_t ldv, const double* v_lr,
                             int64_t ldlr, const double* b_up, int64_t ldb, double lr_scale,
                             int64_t L_c, int64_t L, int64_t d, int64_t r, int64_t query_offset,
                             double* out);
/* gqa_attention<T>, attention.hpp:332-363: all q heads in one launch.  q: L_c x (n_q*d_head),
 * k/v_base: L x (n_kv*d_head), v_lr: L x r (shared by all heads), b_up: r x (n_kv*d_head). */
int lorakv_gqa_forward_f32(lorakv_ctx* ctx, const float* q, int64_t ldq, const float* k, int64_t ldk,
                           const float* v_base, int64_t ldv, const float* v_lr, int64_t ldlr,
                           const float* b_up, int64_t ldb, float lr_scale, int64_t L_c, int64_t L,
                           int64_t n_q_heads, int64_t n_kv_heads, int64_t d_head, int64_t r,
                           int64_t query_offset, float* out);
int lorakv_gqa_forward_f64(lorakv_ctx* ctx, const double* q, int64_t ldq, const double* k, int64_t ldk,
                           const double* v_base, int64_t ldv, const double* v_lr, int64_t ldlr,
                           const double* b_up, int64_t ldb, double lr_scale, int64_t L_c, int64_t L,
                           int64_t n_q_heads, int64_t n_kv_heads, int64_t d_head, int64_t r,
                           int64_t query_offset, double* out);

/* gqa_attention with a KEY-side low-rank term (the north star's "q K_base^T + (q B_k^T) L_k^T"): the effective keys are
 * K_base + k_scale * L_k B_k with l_k: L x r_k (shared by all heads, like v_lr) and b_k: r_k x (n_kv_heads*d_head); the
 * full-width adapter keys are never formed.  The reference has NO key adapter (engine.hpp:129-130, attention.hpp:47-56;
 * ruled out under RoPE): this is an extension, parity unpinned (the checker materialises K_eff and calls the
 * reference's attention); r_k = 0 is exactly lorakv_gqa_forward_*.  n_q_heads = n_kv_heads = 1 gives the per-head operator. */
int lorakv_gqa_forward_keylr_f32(lorakv_ctx* ctx, const float* q, int64_t ldq, const float* k, int64_t ldk,
                                 const float* v_base, int64_t ldv, const float* v_lr, int64_t ldlr, const float* b_up,
                                 int64_t ldb, float lr_scale, const float* l_k, int64_t ld_lk, const float* b_k,
                                 int64_t ld_bk, float k_scale, int64_t L_c, int64_t L, int64_t n_q_heads,
                                 int64_t n_kv_heads, int64_t d_head, int64_t r, int64_t r_k, int64_t query_offset,
                                 float* out);
int lorakv_gqa_forward_keylr_f64(lorakv_ctx* ctx, const double* q, int64_t ldq, const double* k, int64_t ldk,
                                 const double* v_base, int64_t ldv, const double* v_lr, int64_t ldlr,
                                 const double* b_up, int64_t ldb, double lr_scale, const double* l_k, int64_t ld_lk,
                                 const double* b_k, int64_t ld_bk, double k_scale, int64_t L_c, int64_t L,
                                 int64_t n_q_heads, int64_t n_kv_heads, int64_t d_head, int64_t r, int64_t r_k,
                                 int64_t query_offset, double* out);

/* matmul, matrix.hpp:101-135: out (M x N, dense) = a (M x K, stride lda) * b (K x N, stride ldb) over
 * HOST pointers.  Ascending-k accumulation with separately rounded multiply and add, i.e. the bits the
 * reference's triple loop produces under -ffp-contract=off.  Used by expand_lr / forward_decomposed
 * (lora.hpp:39-47,97-108). */
int lorakv_matmul_f32(lorakv_ctx* ctx, const float* a, int64_t lda, const float* b, int64_t ldb,
                      int64_t M, int64_t K, int64_t N, float* out);
int lorakv_matmul_f64(lorakv_ctx* ctx, const double* a, int64_t lda, const double* b, int64_t ldb,
                      int64_t M, int64_t K, int64_t N, double* out);

/* lr_mac_counts, attention.hpp:35-41, and the dense AttnMacs closed forms (:229-243):
 * macs[0]=qk, [1]=pv, [2]=lr (reordered).  Pure integer arithmetic on the host. */
void lorakv_lr_mac_counts(int64_t total_len, int64_t cur_len, int64_t rank, int64_t d_head,
                          uint64_t* no_reorder, uint64_t* reorder);
void lorakv_attn_macs(int64_t L_c, int64_t L, int64_t d, int64_t r, int expand_first,
                      uint64_t macs[3]);

/* ---- planning (pure integers) --------------------------------------------------------------
 * plan_core, kvcache.hpp:112-142.  out[0..1]=hidden_pass, [2..3]=kv_project, [4..5]=lr_project,
 * [6..7]=kv_recompute, [8]=skip_layers_below. */
int lorakv_plan_core(int scheme, int64_t first_recompute, int64_t length, int64_t seen,
                     int64_t new_tokens, int64_t out[9]);

/* ---- paged cache pool: KvStore<T>, kvcache.hpp:213-420 ---------------------------------------- */
typedef struct {
  int32_t scheme;        /* LORAKV_NONSHARED .. LORAKV_BASELRSHARED */
  int32_t dtype;         /* LORAKV_F32 or LORAKV_BF16 storage in HBM */
  int64_t n_layers;
  int64_t n_kv_heads;    /* kv heads of the whole model */
  int64_t d_head;
  int64_t d_model;
  int64_t rank;          /* 0 = no low-rank cache */
  int64_t n_agents;
  int64_t page_tokens;   /* tokens per page; 0 = default (64) */
  int64_t max_tokens;    /* capacity of the trajectory, rounded up to whole pages */
  int64_t kv_head_begin; /* this pool stores kv heads [kv_head_begin, kv_head_begin + n_kv_local) */
  int64_t n_kv_local;    /* 0 = all heads (single GPU) */
  int64_t rank_k;        /* key-side low-rank cache L_k (extension, lorakv_gqa_forward_keylr_*); 0 = none, the reference */
} lorakv_pool_dims;

int lorakv_pool_create(lorakv_ctx* ctx, const lorakv_pool_dims* dims, lorakv_pool** out);
void lorakv_pool_destroy(lorakv_pool* pool);
int lorakv_pool_dims_get(const lorakv_pool* pool, lorakv_pool_dims* out);

int lorakv_pool_append_tokens(lorakv_pool* pool, int64_t n);            /* :254-257 */
int64_t lorakv_pool_length(const lorakv_pool* pool);                    /* :251 */
int lorakv_pool_seen(const lorakv_pool* pool, int64_t agent, int64_t* out); /* :259 */
int lorakv_pool_mark_seen(lorakv_pool* pool, int64_t agent);            /* :260-264 */
int lorakv_pool_plan_step(const lorakv_pool* pool, int64_t agent, int64_t new_tokens,
                          int64_t out[9]);                              /* plan_step :423-425 */

/* append_key / append_value / append_lr, :268-288, with first-writer-wins (:400-407) resolved on
 * the host before any launch.  rows: n_rows x cols(which) float32, row stride ld, in HOST or
 * DEVICE memory; cols = n_kv_heads*d_head for key/value (the FULL width -- the pool keeps its own
 * head slice) and rank for lr.  *appended (may be NULL) receives the rows actually written. */
int lorakv_pool_append(lorakv_pool* pool, int which, int64_t layer, int64_t agent,
                       int64_t row_begin, const float* rows, int64_t n_rows, int64_t ld,
                       int mem_kind, int64_t* appended);
/* The append path of engine.hpp:414-418: V_lr rows = X * A (unscaled) computed on the device and
 * written straight into the LR pages.  x: n_rows x d_model float32. */
int lorakv_pool_append_lr_project(lorakv_pool* pool, const lorakv_adapters* adapters, int64_t layer,
                                  int64_t agent, int64_t row_begin, const float* x, int64_t n_rows,
                                  int64_t ld, int mem_kind, int64_t* appended);
/* ---- the projection that feeds the cache ------------------------------------
 * Replaces, for the rows of the plan's kv range (proj/include/lorakv/engine.hpp:376-403):
 *     k_rows = x_norm * Wk;  if (rope) apply_rope(k_rows, n_kv_heads, d_head, row_begin);   (:380-383, :225-243)
 *     v_rows = x_norm * Wv;                                                                  (:384)
 *     store.append_key(layer, agent, row_begin, k_rows); store.append_value(..., v_rows);    (:402-403)
 * lorakv_proj holds Wk, Wv (d_model x n_kv_heads*d_head, row-major float32, HOST) per layer; the shard
 * arguments and dtype must equal the pool's.  bf16 pools with d_head 128 run ONE tcgen05 kernel that
 * projects, rotates and writes bf16 pages; other pools use the reference's summation order in fp32. */
typedef struct lorakv_proj lorakv_proj;
int lorakv_proj_create(lorakv_ctx* ctx, int64_t n_layers, int64_t d_model, int64_t n_kv_heads,
                       int64_t d_head, int64_t kv_head_begin, int64_t n_kv_local, int dtype,
                       lorakv_proj** out);
void lorakv_proj_destroy(lorakv_proj* proj);
int lorakv_proj_set_kv(lorakv_proj* proj, int64_t layer, const float* wk, const float* wv);
/* The query side of the same step (engine.hpp:362-373, :422):
 *     q = x_norm * Wq;  q += (alpha/rank) * ((x_norm * A_q) * B_q[agent]);  if (rope) apply_rope(q, n_q_heads, d_head, pos_begin)
 * wq: d_model x n_q_heads*d_head, a_q: d_model x rank (shared by all agents, lora.hpp:69-73), b_q: rank x
 * n_q_heads*d_head, all row-major float32 HOST.  lorakv_proj_query writes n_rows x (n_q_local*d_head) float32 rows
 * (the shard's q heads) into q_out, HOST or DEVICE like x; agent < 0 skips the adapter. */
int lorakv_proj_set_q(lorakv_proj* proj, int64_t layer, int64_t n_q_heads, const float* wq);
int lorakv_proj_set_q_lora(lorakv_proj* proj, int64_t layer, int64_t agent, int64_t n_agents, int64_t rank,
                           const float* a_q, const float* b_q, double alpha);
int lorakv_proj_query(lorakv_proj* proj, int64_t layer, int64_t agent, int64_t pos_begin, const float* x,
                      int64_t n_rows, int64_t ld, int rope, float* q_out, int mem_kind);
/* x: n_rows x d_model float32 (x_norm rows of logical rows [row_begin, row_begin+n_rows)), HOST or
 * DEVICE.  First-writer-wins as in lorakv_pool_append; *appended = rows newly written. */
int lorakv_pool_append_kv_project(lorakv_pool* pool, const lorakv_proj* proj, int64_t layer,
                                  int64_t agent, int64_t row_begin, const float* x, int64_t n_rows,
                                  int64_t ld, int mem_kind, int rope, int64_t* appended);
/* ---- snapshot / resume --------------------------------------------------------
 * KvStore::save_snapshot / load_snapshot (kvcache.hpp:438-546): the reference's "lorakv-cache-snapshot" v1
 * container, written from / read into the paged pool; dtype "f32" (bf16 pools de-paginate exactly).  A pool
 * holding the same state as a reference KvStore<float> writes the reference's file byte for byte.  The token
 * ids of the trajectory are the caller's (the pool keeps only their count); load returns them in tokens_out
 * (up to tokens_cap) and their number in *n_tokens (both may be NULL).  n_kv_heads / page_tokens / max_tokens /
 * dtype are the device options a snapshot does not carry. */
int lorakv_pool_save_snapshot(const lorakv_pool* pool, const char* path, const int32_t* tokens, int64_t n_tokens);
int lorakv_pool_load_snapshot(lorakv_ctx* ctx, const char* path, int dtype, int64_t n_kv_heads,
                              int64_t page_tokens, int64_t max_tokens, lorakv_pool** out,
                              int32_t* tokens_out, int64_t tokens_cap, int64_t* n_tokens);
/* The token ids a snapshot file holds, from its header alone: writes min(cap, n) ids, *n_tokens = n (both may be NULL). */
int lorakv_snapshot_tokens(const char* path, int32_t* tokens_out, int64_t cap, int64_t* n_tokens);
/* The "full values" variant of engine.hpp:385-393 (NonShared, FullShared): the stored value rows are
 * v_base + (alpha/rank) * ((x * A_v) * B_v[agent]) with A_v, B_v, alpha from the adapter table. */
int lorakv_pool_append_kv_project_full(lorakv_pool* pool, const lorakv_proj* proj,
                                       const lorakv_adapters* adapters, int64_t layer, int64_t agent,
                                       int64_t row_begin, const float* x, int64_t n_rows, int64_t ld,
                                       int mem_kind, int rope, int64_t* appended);
/* The same two calls for fp64 pools (dtype LORAKV_F64): rows / out are float64. */
int lorakv_pool_append_f64(lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t row_begin, const double* rows,
                           int64_t n_rows, int64_t ld, int mem_kind, int64_t* appended);
int lorakv_pool_read_f64(const lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t row_begin, int64_t n_rows,
                         double* out);
/* SelectiveRecompute (kvcache.hpp:53-58): the sorted, unique layers whose cached K / V rows a returning agent recomputes */
int lorakv_pool_set_recompute_layers(lorakv_pool* pool, const int64_t* layers, int64_t n);
int lorakv_pool_get_recompute_layers(const lorakv_pool* pool, int64_t* out, int64_t cap, int64_t* n);   /* writes min(cap, n) */
/* recompute_overwrite, kvcache.hpp:298-305 / GrowMat::overwrite :184-193: replace already materialised rows
 * [row_begin, row_begin + n_rows) of the key or value cache of a recompute layer (anything else is the reference's
 * "overwrite ... forbidden" error).  rows: float32 (lorakv_pool_overwrite) or float64 (_f64, fp64 pools). */
int lorakv_pool_overwrite(lorakv_pool* pool, int which, int64_t layer, int64_t row_begin, const float* rows, int64_t n_rows,
                          int64_t ld, int mem_kind);
int lorakv_pool_overwrite_f64(lorakv_pool* pool, int which, int64_t layer, int64_t row_begin, const double* rows, int64_t n_rows,
                              int64_t ld, int mem_kind);
/* rows currently materialised in the buffer (layer, agent) resolves to (GrowMat::rows) */
int lorakv_pool_rows(const lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t* rows);
/* key_view / value_view / lr_view, :307-324: de-paginate rows [row_begin, row_begin+n_rows) into a
 * dense float32 HOST matrix (n_rows x cols, cols = n_kv_local*d_head or rank). */
int lorakv_pool_read(const lorakv_pool* pool, int which, int64_t layer, int64_t agent,
                     int64_t row_begin, int64_t n_rows, float* out);
/* CacheBytes / bytes(), :144-150,330-344: {key, value, lr, hidden} = logical elements*sizeof(T);
 * allocated_elements(), :346-358. */
int lorakv_pool_bytes(const lorakv_pool* pool, uint64_t out[4]);
uint64_t lorakv_pool_allocated_elements(const lorakv_pool* pool);
/* bytes of HBM actually reserved for pages (capacity, not occupancy) */
uint64_t lorakv_pool_reserved_bytes(const lorakv_pool* pool);
/* logical page -> physical page of the page set that (which, agent) resolves to.  Pages are handed
 * out in first-touch order.  Writes min(cap, n_pages) entries, *n_pages = pages in use. */
int lorakv_pool_page_table(const lorakv_pool* pool, int which, int64_t agent, int32_t* out,
                           int64_t cap, int64_t* n_pages);

/* ---- adapter tables: LoraAdapter / MultiLoraSet, lora.hpp:13-87 -------------------------------- */
int lorakv_adapters_create(lorakv_ctx* ctx, int64_t n_layers, int64_t n_agents, int64_t d_model,
                           int64_t rank, int64_t n_kv_heads, int64_t d_head, int64_t kv_head_begin,
                           int64_t n_kv_local, int dtype, lorakv_adapters** out);
void lorakv_adapters_destroy(lorakv_adapters* ad);
/* shared down-projection A (d_model x rank, HOST float32, dense) of one layer: shared-A multi-LoRA,
 * lora.hpp:69-73 -- one A for every agent, so X*A is computed once */
int lorakv_adapters_set_a(lorakv_adapters* ad, int64_t layer, const float* a);
/* per-agent down-projection (d_model x rank, HOST float32, dense): the BaseShared scheme, whose adapters do NOT
 * share A and which therefore keeps one LR cache per agent (kvcache.hpp:127-130, 238-243).  When set, the X*A
 * append of that agent uses it instead of the shared A. */
int lorakv_adapters_set_a_agent(lorakv_adapters* ad, int64_t layer, int64_t agent, const float* a);
/* per-agent up-projection B (rank x n_kv_heads*d_head, HOST float32, dense, FULL width) and alpha;
 * the effective scale alpha/rank travels with B (lora.hpp:9-11,34) */
int lorakv_adapters_set_b(lorakv_adapters* ad, int64_t layer, int64_t agent, const float* b,
                          double alpha);

/* Key-side adapter tables (extension; see lorakv_gqa_forward_keylr_*): shared down-projection A_k (d_model x rank_k) per
 * layer, per-agent up-projection B_k (rank_k x n_kv_heads*d_head, FULL width) with alpha_k; scale alpha_k / rank_k.  A pool
 * with rank_k > 0 attends with S = (q K_base^T + (k_scale q B_k[agent]^T) L_k^T) / sqrt(d). */
int lorakv_adapters_enable_key(lorakv_adapters* ad, int64_t rank_k);
int lorakv_adapters_set_a_k(lorakv_adapters* ad, int64_t layer, const float* a_k);
int lorakv_adapters_set_b_k(lorakv_adapters* ad, int64_t layer, int64_t agent, const float* b_k, double alpha_k);
/* L_k rows = X * A_k computed on the device and written into the L_k pages (the key-side twin of lorakv_pool_append_lr_project) */
int lorakv_pool_append_lk_project(lorakv_pool* pool, const lorakv_adapters* adapters, int64_t layer, int64_t row_begin,
                                  const float* x, int64_t n_rows, int64_t ld, int mem_kind, int64_t* appended);

/* ---- device-resident fast paths --------------------------------------------------------------
 * Batched decode = one gqa_attention call (attention.hpp:332) per (layer, batch entry), every
 * entry attending to the whole shared cache (query_offset = L-1, engine.hpp:440-443), fused into
 * one launch over layers [layer_begin, layer_end).
 *   agent_ids: n_batch HOST int32 (which B table each query row group uses)
 *   q:   [layer_end-layer_begin][n_batch][n_q_local*d_head] float32
 *   out: same shape, float32                (n_q_local = n_kv_local * n_q_heads/n_kv_heads)
 * q/out live in HOST or DEVICE memory as mem_kind says (HOST: copies ride the ctx stream). */
int lorakv_fla_decode_batched(lorakv_pool* pool, const lorakv_adapters* adapters,
                              int64_t layer_begin, int64_t layer_end, const int32_t* agent_ids,
                              int64_t n_batch, int64_t n_q_heads, const float* q, float* out,
                              int mem_kind);
/* ---- end-of-step output gather of a kv-head-sharded decode, over peer memory --------------------
 * gqa_attention returns L_c x (n_q*d) rows (attention.hpp:346,359-360); q head h reads only kv head h/g
 * (:348-354), so a rank holding kv heads [kv_head_begin, +n_kv_local) (lorakv_pool_dims) owns a column slice of
 * every row and putting the slices side by side is the only exchange of a step.  A lorakv_gather
 * owns one device allocation per rank -- two full outputs (alternating by step) and a flag page -- mapped into
 * every other rank through CUDA IPC.  The decode epilogue stores its finished rows into ALL ranks' buffers
 * directly (NVLink / NVSwitch peer stores), a one-block kernel then publishes the step number to the peers
 * and waits for theirs; no collective library call, no local slab.
 *   create : full_elems = (layer_end-layer_begin) * n_batch * n_q_heads * d_head floats of one step's output
 *   export : writes this rank's LORAKV_GATHER_HANDLE_BYTES-byte handle; the caller all-gathers the handles of
 *            ranks 0..world-1 by whatever means it has (torch.distributed, MPI, a file) ...
 *   connect: ... and passes them back in rank order (world * LORAKV_GATHER_HANDLE_BYTES bytes)
 * world == 1 needs no export / connect.  Ranks must issue the same sequence of gather steps. */
typedef struct lorakv_gather lorakv_gather;
#define LORAKV_GATHER_HANDLE_BYTES 64
int lorakv_gather_create(lorakv_ctx* ctx, int rank, int world, int64_t full_elems, lorakv_gather** out);
/* Tear-down order across ranks: every rank disconnects (unmaps its peers), the caller runs a barrier, then every
 * rank destroys -- an exported allocation must outlive the mappings of it (CUDA IPC rule). */
int lorakv_gather_disconnect(lorakv_gather* g);
void lorakv_gather_destroy(lorakv_gather* g);
int lorakv_gather_export(lorakv_gather* g, unsigned char* handle);
int lorakv_gather_connect(lorakv_gather* g, const unsigned char* handles);
/* how long a rank waits for its peers before the step fails instead of hanging (default 20 s) */
int lorakv_gather_set_timeout_ms(lorakv_gather* g, int64_t ms);
int lorakv_gather_steps(const lorakv_gather* g, int64_t* steps);
/* Overlapped handshake (off by default).  On: the handshake kernel of a step runs on a side stream behind that step's
 * epilogue, so the ctx stream goes straight on with the next step's attention kernel; the library makes the ctx stream
 * wait for it only before the NEXT step's epilogue stores into the peers' buffers (the reuse guard of the buffer pair).
 * The gathered rows of a step are then complete on the ctx stream only after lorakv_gather_wait(g): call it before
 * enqueueing a reader of the pointer lorakv_fla_decode_batched_gather returned (the out_host path does it itself). */
int lorakv_gather_set_overlap(lorakv_gather* g, int enabled);
int lorakv_gather_wait(lorakv_gather* g);
/* synchronises the ctx stream and fails if a handshake enqueued so far timed out */
int lorakv_gather_check(lorakv_gather* g);
/* lorakv_fla_decode_batched on this rank's shard, ending in the gather.
 *   q: [layers][n_batch][n_q_local*d_head] float32 (this rank's heads), HOST or DEVICE per q_mem_kind
 *   out_host: NULL, or [layers][n_batch][n_q_heads*d_head] float32 HOST: the gathered rows (synchronises)
 *   out_dev : NULL, or receives the DEVICE pointer of the gathered rows of this step; valid until the step after
 *             next is issued; reads must be ordered on the ctx stream */
int lorakv_fla_decode_batched_gather(lorakv_pool* pool, const lorakv_adapters* adapters, lorakv_gather* g,
                                     int64_t layer_begin, int64_t layer_end, const int32_t* agent_ids,
                                     int64_t n_batch, int64_t n_q_heads, const float* q, int q_mem_kind,
                                     float* out_host, float** out_dev);

/* Prefill / append-step attention of one agent on one layer: q rows cover positions
 * [query_offset, query_offset+L_c) of the cached trajectory (causal rule attention.hpp:44-46).
 *   q/out: L_c x (n_q_local*d_head) float32, dense. */
int lorakv_fla_prefill(lorakv_pool* pool, const lorakv_adapters* adapters, int64_t layer,
                       int64_t agent, int64_t n_q_heads, const float* q, int64_t L_c,
                       int64_t query_offset, float* out, int mem_kind);

/* One decode layer-step of step() restricted to the attention sublayer (proj/include/lorakv/engine.hpp:331-443): for the rows
 * x (n_rows x d_model float32, logical rows [row_begin, row_begin + n_rows) of the trajectory, the positions of the new
 * tokens)
 *     q = rope(x Wq + (alpha/rank) (x A_q) B_q[agent])                                         (:352-373, :422-427)
 *     append_key(rope(x Wk)); append_value(x Wv [+ (alpha/rank) (x A_v) B_v[agent] under NonShared / FullShared])  (:376-403)
 *     append_lr(x A_v)                             (BaseShared / BaseLRShared, :411-419)
 *     out = gqa_attention(q, key_view, value_view, lr_view, B_v[agent], alpha/rank, query_offset = row_begin)    (:429-443)
 * i.e. lorakv_pool_append_kv_project[_full] + lorakv_pool_append_lr_project + lorakv_proj_query + lorakv_fla_prefill.  The q
 * adapter of (layer, agent) is applied when one was uploaded (lorakv_proj_set_q_lora).  adapters: the value-side tables
 * (required by the schemes with an LR cache; NonShared / FullShared merge them into the stored rows when given, NULL = none).
 * With DEVICE operands, a bf16 pool, d_head 128 and <= 8 fresh rows -- a decode step -- the whole call is four chained
 * kernel launches with no host synchronisation and no copy (all projections in two launches, attention, merge epilogue).
 *   q_scratch: NULL, or n_rows x (n_q_local*d_head) float32 in the same memory kind as x: receives the projected queries
 *   out      : n_rows x (n_q_local*d_head) float32 */
int lorakv_step_layer(lorakv_pool* pool, const lorakv_proj* proj, const lorakv_adapters* adapters, int64_t layer, int64_t agent,
                      int64_t row_begin, const float* x, int64_t n_rows, int64_t ld, int rope, int64_t n_q_heads,
                      float* q_scratch, float* out, int mem_kind);

/* Device time of the dominant kernel alone.  With profiling on, every fast-path call brackets its
 * main attention kernel (not the merge epilogue, not the staging copies) with two events on the ctx
 * stream; lorakv_ctx_last_kernel_ms waits for the second and returns the time between them. */
int lorakv_ctx_set_profiling(lorakv_ctx* ctx, int enabled);
int lorakv_ctx_last_kernel_ms(lorakv_ctx* ctx, float* ms);
/* Mean of that time over the fast-path calls made since profiling was switched on (or since the previous call of
 * this function; up to 256 calls), without a synchronisation between the calls: the kernel timed inside an
 * uninterrupted run of steps.  *n_calls (optional) = how many calls were averaged. */
int lorakv_ctx_mean_kernel_ms(lorakv_ctx* ctx, float* ms, int* n_calls);

/* One-tile tcgen05 self-test (diagnostics): D (128 x N) = A (128 x K) * B on the tensor cores with the
 * shared-memory operand layouts the prefill kernel uses; B is N x K row-major (b_mn_major = 0, the
 * K-page convention) or K x N row-major (b_mn_major = 1, the V / V_lr page convention).  HOST pointers,
 * operands rounded to bf16, fp32 accumulation in TMEM.  rescale != 0 additionally scales the
 * accumulator by alpha through tcgen05.ld/st and accumulates a second pass: D = (alpha + 1) * A B.
 * a_in_tmem != 0 feeds A from tensor memory (packed bf16 pairs written with tcgen05.st), the way the
 * prefill kernel feeds Q and P.  K = 64 or 128; with a_in_tmem and b_mn_major = 0 also K = 16 / 32: B rows of
 * 32 / 64 bytes (SWIZZLE_32B / 64B), the convention of a tile of the key-side low-rank cache L_k. */
int lorakv_selftest_umma(lorakv_ctx* ctx, const float* a, const float* b, int N, int K, int b_mn_major,
                         float alpha, int rescale, int a_in_tmem, float* d);

/* selects the kernel family for the fast paths: 0 = auto (tcgen05/TMA where the shape allows),
 * 1 = force the CUDA-core kernels, 2 = auto but keep decode on the mma.sync streaming kernel even for
 * many query rows, the fp32-mode prefill on the mma.sync TF32 kernel and the fp32 projections on the reference's
 * summation order (bit-identical K / V / q rows) instead of the tcgen05 plane kernels (A/B comparisons).
 * Returns the previous value. */
int lorakv_set_kernel_policy(lorakv_ctx* ctx, int policy);
/* name of the kernel family the last fast-path call on this ctx dispatched to */
const char* lorakv_last_kernel(lorakv_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
