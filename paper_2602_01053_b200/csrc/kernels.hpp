// kernels.hpp -- host-callable launchers implemented in the .cu files of this directory.
#pragma once

#include <cstdint>

#include "lorakv_b200.h"

struct lorakv_ctx;
struct lorakv_pool;
struct lorakv_adapters;

namespace lk {

// Key-side low-rank term of the north star: K_eff = K_base + k_scale * L_k B_k with L_k = X A_k (L x r_k, one per layer like
// V_lr) and B_k (r_k x n_kv d, per agent).  The kernels never form K_eff: q . K_eff[j] = q . K_base[j] + (k_scale q B_k^T) . L_k[j].
// The reference has no key adapter (engine.hpp:129-130; the paper rules it out under RoPE), so this is an
// extension whose parity is UNPINNED: the checker materialises K_eff and calls the reference's attention.  r_k = 0 is the reference.
template <class T>
struct KeyLowRank {
  const T* l_k; int64_t ld_lk;     // L x r_k
  const T* b_k; int64_t ld_bk;     // r_k x (n_kv * d)
  T k_scale;                       // alpha_k / r_k
  int64_t r_k;
};

// fla_generic.cu ------------------------------------------------------------------------------
template <class T>
int generic_forward(lorakv_ctx* ctx, const char* op, int mode, const T* q, int64_t ldq, const T* k,
                    int64_t ldk, const T* v, int64_t ldv, const T* vlr, int64_t ldlr, const T* b,
                    int64_t ldb, T lr_scale, int64_t Lc, int64_t L, int n_q, int n_kv, int64_t d,
                    int64_t r, int64_t off, T* out, T* row_max, T* row_denom, const KeyLowRank<T>* key = nullptr);
template <class T>
int naive_forward(lorakv_ctx* ctx, const T* q, int64_t ldq, const T* k, int64_t ldk, const T* v,
                  int64_t ldv, const T* vlr, int64_t ldlr, const T* b, int64_t ldb, T lr_scale,
                  int64_t Lc, int64_t L, int64_t d, int64_t r, int64_t off, T* out);

// linalg_kernels.cu ---------------------------------------------------------------------------
template <class T>
int matmul_forward(lorakv_ctx* ctx, const T* a, int64_t lda, const T* b, int64_t ldb, int64_t M, int64_t K,
                   int64_t N, T* out);

// cache_kernels.cu ----------------------------------------------------------------------------
// Copy `n_rows` float32 rows (device, row stride ld, already offset to the pool's first column)
// into pages, starting at logical row `row0` of the page set `set`.
int launch_append_scatter(lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                          const float* src_dev, int64_t n_rows, int64_t ld);
int launch_append_scatter(lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                          const double* src_dev, int64_t n_rows, int64_t ld);          // fp64 pools
// V_lr rows = X * A for one layer, written into the LR pages of `set` from logical row `row0`.
// (which = LORAKV_LK writes L_k = X * A_k into the key-side low-rank pages instead)
int launch_lr_project(lorakv_pool* pool, const float* a_dev, int64_t d_model, int64_t rank, int64_t layer, int64_t set,
                      int64_t row0, const float* x_dev, int64_t n_rows, int64_t ld, int which = LORAKV_LR);
// De-paginate rows [row0, row0+n_rows) into a dense float32 device matrix.
int launch_gather_rows(const lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                       int64_t n_rows, float* dst_dev);
int launch_gather_rows(const lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                       int64_t n_rows, double* dst_dev);                                // fp64 pools

// Where a finished output row goes when the step ends in the output gather of a kv-head-sharded run
// (peer_gather.cu): the epilogue stores its slice of the FULL row [n_q_total * d] straight into every rank's
// peer-mapped buffer over NVLink instead of a local slab that a collective would move afterwards.
constexpr int kMaxPeers = 8;
struct PeerOut {
  float* dst[kMaxPeers];   // [layers][n_batch][n_q_total * d] on every rank (own rank included)
  int n = 0;               // 0: plain local store
  int64_t n_q_total = 0;   // q heads of the full output row
  int64_t q_head_begin = 0;  // first q head this shard owns
  void* wait_event = nullptr;  // cudaEvent_t the launch stream waits for before the kernel that stores into the peers (or null)
};

// fla_paged_simt.cu ---------------------------------------------------------------------------
struct PagedAttnCall {
  lorakv_pool* pool;
  const lorakv_adapters* adapters;  // may be null when rank == 0
  int64_t layer_begin, layer_end;
  int64_t kv_set, lr_set;           // page sets to read (0 for the shared schemes)
  const int32_t* agent_ids_dev;     // [n_batch] which B table / scale each batch entry uses
  int64_t n_batch;                  // decode: batch entries; prefill: 1
  int64_t rows_per_entry;           // decode: 1; prefill: L_c
  int64_t query_offset;             // position of row 0 of every entry
  int64_t agent_host;               // agent of batch entry 0 (host copy; prefill has exactly one entry)
  int64_t n_q_local;                // q heads held by this pool
  int64_t L;                        // cached rows visible to the kernel (min over K, V, LR buffers)
  const float* q_dev;               // [layers][n_batch][rows_per_entry][n_q_local*d]
  float* out_dev;                   // same shape
  const PeerOut* peers = nullptr;   // decode only: store finished rows into the peers' gather buffers as well
  // BaseShared batch (kvcache.hpp:127-130, 238-243: shared K / V_base, one V_lr cache PER AGENT): batch entry i reads the
  // low-rank page set agent_ids[i] instead of lr_set, so that K / V_base are still streamed once for the whole batch
  bool per_entry_lr = false;
  // key-side low-rank term (KeyLowRank above; pool->rk_pad > 0): qk = k_scale * (q B_k[agent]^T) per query row and q head,
  // [layers][n_batch][rows_per_entry][n_q_local][rk_pad] float32 (zero-padded), written by launch_qk_project before the
  // attention kernel; the kernels add qk . L_k[j] to q . K_base[j]
  const float* qk_dev = nullptr;
};
int launch_qk_project(const PagedAttnCall& call, float* qk_out);
bool decode_tma_per_entry_lr_supported(const PagedAttnCall& call);
int launch_paged_simt(const PagedAttnCall& call);

// V_lr is per layer, not per head (attention.hpp:353): a decode launch reads every low-rank tile once per kv head, at
// different times of the launch.  While the low-rank cache of the whole launch fits in L2 beside the K / V stream, the
// decode kernels load its tiles with an evict-last hint (K / V keep evict-first) and DRAM serves them once instead of
// n_kv times (cfg 2: 4.56 -> 4.34 GB per step = the algorithmic bytes).  Larger ones (cfg 4: 268 MB) are cut into layer
// chunks INSIDE the kernel (fla_decode_tma: n_chunks); separate launches per chunk were measured first and do not pay
// (six launch pairs cost more than the saved traffic: 1.60 vs 1.57 ms per cfg-4 step).
// Budgets are fractions of the device's L2 (lorakv_ctx::l2_bytes, 126 MB on B200; lorakv_ctx_set_l2_bytes overrides it):
// a whole launch may keep 0.6 of it for V_lr, one in-kernel layer chunk 0.28 (two chunks can be live at once).
bool lr_fits_l2(const PagedAttnCall& c, int64_t lr_bytes_per_layer);
int64_t lr_chunk_budget(const PagedAttnCall& c);

// fla_decode_tma.cu (TMA bulk-copy rings + tensor-core MMA; bf16 pages, decode) -------------------
bool decode_tma_supported(const PagedAttnCall& call);
int launch_decode_tma(const PagedAttnCall& call);
// split merge + up-projection epilogue over the partial layout both decode kernels write
int launch_decode_merge(lorakv_ctx* ctx, const float* part, int d, int rp, int r, int mw, int group, int n_kv_local, int n_batch,
                        int rows_total, int row_blocks, int64_t T, int64_t G, int64_t layer_begin, int64_t n_q_local, int max_seg,
                        const int32_t* agent_ids_dev, const lorakv_adapters* adapters, float* out_dev, int64_t n_layers,
                        const PeerOut* peers = nullptr, int agent_fixed = -1, int64_t units_per_chunk = 0, int64_t n_workers = 0);

// fla_decode_f32.cu (the same streaming decode over fp32 pages: 3 x TF32 mma.sync, fp32 accuracy) ----------
bool decode_f32_supported(const PagedAttnCall& call);
int launch_decode_f32(const PagedAttnCall& call);
bool prefill_f32_supported(const PagedAttnCall& call);     // prefill blocks of one agent on one layer
int launch_prefill_f32(const PagedAttnCall& call);
// fp32 pages, blocks of >= 128 query rows per kv head: tcgen05 over bf16 planes of the fp32 rows (fla_prefill_split.cu)
bool prefill_split_supported(const PagedAttnCall& call);
int launch_prefill_split(const PagedAttnCall& call);

// fla_prefill_umma.cu (tcgen05 / TMEM / TMA; bf16 pages, prefill blocks) ---------------------------------
bool prefill_umma_supported(const PagedAttnCall& call);
int launch_prefill_umma(const PagedAttnCall& call);
bool decode_umma_supported(const PagedAttnCall& call);     // decode with 33..128 query rows per kv head
int launch_decode_umma(const PagedAttnCall& call);

// kv_project_umma.cu (K / V_base projection + RoPE + append in one pass; tcgen05 for bf16 pools) -----------
bool kv_project_fused_shape(int dtype, int64_t d_head, int64_t d_model);
int64_t kv_project_packed_elems(int64_t d_model, int64_t n_kv_local, int64_t d_head);
int launch_pack_w(lorakv_ctx* ctx, const float* w_dev, int64_t ldw, int64_t col0, int64_t n_cols, int64_t d_model, int64_t nb0, void* packed);
int launch_kv_project(lorakv_pool* pool, const void* w_packed, const float* wk_dev, const float* wv_dev, int64_t layer, int64_t set,
                      int64_t row0, int64_t k_from, int64_t v_from, const float* x_dev, int64_t n_rows, int64_t ld, bool rope,
                      const float* down_dev, const float* av_dev, const float* bv_dev, int64_t rank, float v_scale);

int launch_q_project(lorakv_ctx* ctx, bool fused, const void* wq_packed, const float* wq_dev, int64_t ldw, int64_t col0,
                     int64_t d_model, int64_t n_cols, int64_t d_head, const float* down_dev, const float* aq_dev, const float* bq_dev,
                     int64_t ldb, int64_t rank, float q_scale, int64_t pos0, const float* x_dev, int64_t n_rows, int64_t ld, bool rope,
                     float* q_dev, const void* bq_extra);
int launch_pack_lora_b(lorakv_ctx* ctx, const float* b_dev, int64_t ldb, int64_t col0, int64_t n_cols, int64_t rank, void* packed);
// cache_kernels.cu: x * A as dense float32 rows (tensor cores)
int launch_xa_dense(lorakv_ctx* ctx, const float* a_dev, int64_t d_model, int64_t rank, const float* x_dev, int64_t n_rows, int64_t ld,
                    float* out_dev);

// rows_project.cu: the same projections for <= 8 rows (a decode step) as weight-streaming GEMVs over all SMs
bool rows_project_supported(int64_t n_rows, int64_t d_model, int64_t rank);
int launch_rows_xa(lorakv_ctx* ctx, const float* a_dev, int64_t d_model, int64_t rank, const float* x_dev, int64_t n_rows, int64_t ld,
                   float* down_dev);
int launch_rows_kv_project(lorakv_pool* pool, const void* w_packed, int64_t layer, int64_t set, int64_t row0, int64_t k_from,
                           int64_t v_from, const float* x_dev, int64_t n_rows, int64_t ld, bool rope, const float* down_dev,
                           const float* bv_dev, int64_t rank, float v_scale);
int launch_rows_q_project(lorakv_ctx* ctx, const void* wq_packed, int64_t d_model, int64_t n_cols, int64_t d_head, const float* down_dev,
                          const float* bq_dev, int64_t ldb, int64_t rank, float q_scale, int64_t pos0, const float* x_dev, int64_t n_rows,
                          int64_t ld, bool rope, float* q_dev);
int launch_rows_lr_project(lorakv_pool* pool, const float* a_dev, int64_t d_model, int64_t rank, int64_t layer, int64_t set, int64_t row0,
                           const float* x_dev, int64_t n_rows, int64_t ld);

// step_layer.cu: all projections of one decode layer-step (<= 8 rows) in two launches: q (+ q-LoRA, RoPE) into float32
// rows, K (RoPE) / V (+ merged value adapter) into their pages, V_lr = x A_v into its LR page
struct StepLayerCall {
  int64_t layer, kv_set, lr_set, row0, n_rows;
  const float* x_dev; int64_t ld;
  const void* wq_packed; const void* wkv_packed;   // this layer's packed bf16 weights
  int64_t dq;                                      // q columns of this shard
  const float* a_q; const float* b_q; int64_t ldb_q, r_q; float s_q;   // q adapter (a_q null: none); b_q already at the shard's first column
  const float* a_v; const float* b_v; int64_t r_v; float s_v;          // value adapter: A for V_lr / the merge, B (shard-local width) for the merge
  bool merge_v;                                    // full-values schemes: v += s_v (x A_v) B_v
  bool append_lr;                                  // schemes with an LR cache: V_lr row = x A_v
  bool rope;
  float* q_dev;                                    // [n_rows][dq] float32
};
bool step_layer_supported(int64_t n_rows, int64_t d_model, int64_t d_head, int64_t r_q, int64_t r_v);
int launch_step_layer(lorakv_pool* pool, const StepLayerCall& call);

// peer_gather.cu: local slab [layers][n_batch][n_q_local * d] -> every peer's full buffer (paths without the merge epilogue)
int launch_peer_scatter(lorakv_ctx* ctx, const float* slab_dev, int64_t rows, int64_t n_q_local, int64_t d, const PeerOut& peers);

// umma_selftest.cu ------------------------------------------------------------------------------------
int umma_selftest(lorakv_ctx* ctx, const float* a, const float* b, int N, int K, int b_mn_major, float alpha, int rescale,
                  int a_in_tmem, float* d);

}  // namespace lk
