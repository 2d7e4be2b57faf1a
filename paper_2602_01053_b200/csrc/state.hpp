// state.hpp -- host-side state behind the C ABI (include/lorakv_b200.h).
//
// lorakv_ctx      : device, stream, scratch buffers, launch counter
// lorakv_pool     : paged HBM cache of one trajectory + the integer bookkeeping of the reference's
//                   KvStore<T> (proj/include/lorakv/kvcache.hpp:213-420), kept on the host
// lorakv_adapters : shared A per layer, per-agent B tables (proj/include/lorakv/lora.hpp:13-87)
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "lorakv_b200.h"

namespace lk {

// ---- errors: status code + thread-local message (the reference throws, matrix.hpp:17-19) ----
std::string& err_slot();
int fail(const char* fmt, ...);

#define LK_CUDA(expr)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return lk::fail("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, __LINE__, \
                      cudaGetErrorString(e_));                                             \
  } while (0)

#define LK_TRY(expr)            \
  do {                          \
    int rc_ = (expr);           \
    if (rc_ != LORAKV_OK) return rc_; \
  } while (0)

struct Scratch {            // grow-only device buffer
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace lk

namespace lk {
// Agent-id lists of the batched calls, staged once: a small ring of {pinned host, device} buffers keyed by content.  A call
// whose list equals a staged one reuses the device copy (a decode loop passes the same batch every layer and step: no
// copy at all); a new list takes the next slot, and the slot's event makes sure the pinned buffer is not rewritten while
// an earlier host-to-device copy of it is still pending.
struct IdSlot {
  int32_t* host = nullptr;
  int32_t* dev = nullptr;
  size_t cap = 0;                 // entries
  std::vector<int32_t> ids;       // what the device buffer holds (or will, in stream order)
  cudaEvent_t copied = nullptr;
};
}  // namespace lk

struct lorakv_pool;

struct lorakv_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  int sm_count = 0;
  int64_t l2_bytes = 0;               // device L2 size (cudaDevAttrL2CacheSize); sizes the V_lr residency decisions of the decode
  int64_t launches = 0;
  int policy = 0;
  int split_keys = 0;                 // keys per split of the fp32-mode tcgen05 prefill; 0 = the kernel's default
  bool pdl = true;                    // chain the decode kernels with programmatic dependent launches (LORAKV_NO_PDL=1 disables)
  bool speculate = true;              // prefetch certainly-complete cache rows before the dependent-launch wait (LORAKV_NO_SPECULATION=1)
  const char* last_kernel = "none";
  lk::Scratch in, out, work, flush;   // staging for host operands / results / partials / L2 flush
  lk::Scratch proj;                   // q-LoRA down-projection rows of the query projection; partial sums of a fused layer-step
  lk::Scratch planes;                 // bf16 planes of the visible fp32 cache rows of one layer (fla_prefill_split.cu)
  lk::Scratch qk;                     // queries seen through the key adapter (launch_qk_project)
  lk::Scratch qrows;                  // query rows of a fused layer-step when the caller passes no scratch
  static constexpr int kIdSlots = 8;
  lk::IdSlot id_slots[kIdSlots];
  int id_next = 0;
  void* pinned = nullptr;             // small pinned staging buffer
  size_t pinned_bytes = 0;
  bool profiling = false;             // bracket the dominant kernel of fast-path calls with events
  cudaEvent_t prof_ev[2] = {nullptr, nullptr};
  bool prof_valid = false;
  // back-to-back profiling: one event pair per fast-path call since profiling was switched on (up to kProfPairs), so
  // that the kernel can be timed inside an uninterrupted run of steps (lorakv_ctx_mean_kernel_ms)
  static constexpr int kProfPairs = 256;
  std::vector<cudaEvent_t> prof_ring;    // 2 * kProfPairs events, created with the first profiled call
  int prof_count = 0;
};

namespace lk {
// Kernel launch on the ctx stream, optionally as a programmatic dependent launch (umma.cuh: pdl_wait): the kernels of a
// decode layer-step chain this way so that each one's launch latency and prologue hide under its predecessor's tail.
template <class... KArgs, class... Args>
inline cudaError_t launch_kernel(lorakv_ctx* ctx, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr; cfg.numAttrs = (pdl && ctx->pdl) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, KArgs(std::forward<Args>(args))...);
}
// record the start (which = 0) / end (which = 1) of the dominant kernel when profiling is on
inline void prof_mark(lorakv_ctx* ctx, int which) {
  if (!ctx->profiling) return;
  cudaEventRecord(ctx->prof_ev[which], ctx->stream);
  if (ctx->prof_count < lorakv_ctx::kProfPairs && !ctx->prof_ring.empty())
    cudaEventRecord(ctx->prof_ring[(size_t)(2 * ctx->prof_count + which)], ctx->stream);
  if (which == 1) { ctx->prof_valid = true; if (ctx->prof_count < lorakv_ctx::kProfPairs) ++ctx->prof_count; }
}
}  // namespace lk

namespace lk {

int scratch_reserve(lorakv_ctx* ctx, Scratch& s, size_t bytes);
int pinned_reserve(lorakv_ctx* ctx, size_t bytes);
// device copy of an agent-id list (see IdSlot); valid for every kernel enqueued on the ctx stream after this call
int stage_agent_ids(lorakv_ctx* ctx, const int32_t* ids, int64_t n, const int32_t** dev);
// page-write tracking of a pool (see lorakv_pool::write_event)
int note_pages_written(lorakv_pool* pool, int64_t row0);
int64_t stable_rows(lorakv_pool* pool, int64_t L);        // rows [0, result) are complete on the device right now

// One page space: page ids handed out in first-touch order to the logical pages of its sets.
struct PageSpace {
  int64_t n_sets = 0, max_pages = 0;          // logical pages per set
  int32_t next_free = 0;
  std::vector<std::vector<int32_t>> table;    // [set][logical page] -> physical page
  int32_t* dev_table = nullptr;               // [n_sets][max_pages], mirrors `table`
  int64_t total_pages() const { return n_sets * max_pages; }
  // True when logical page i of `set` is physical page i for every i < n_pages (one trajectory appended in order: the
  // common case).  The decode kernel then skips the page-table load that its first bulk copy would otherwise wait for.
  // Tables are append-only, so the verified prefix is remembered.
  std::vector<int64_t> ident_upto;            // [set] pages verified so far; -1 once a mismatch was found
  bool identity(int64_t set, int64_t n_pages) {
    if (ident_upto.size() != table.size()) ident_upto.assign(table.size(), 0);
    int64_t& c = ident_upto[(size_t)set];
    const auto& tab = table[(size_t)set];
    while (c >= 0 && c < n_pages && c < (int64_t)tab.size()) c = tab[(size_t)c] == c ? c + 1 : -1;
    return c >= n_pages;
  }
};

}  // namespace lk

struct lorakv_pool {
  lorakv_ctx* ctx = nullptr;
  lorakv_pool_dims dims{};
  int64_t P = 64;            // page_tokens
  int64_t r_pad = 0;         // LR row width in HBM (rank zero-padded to 8/16/32/64/k*64; 0 when rank == 0)
  int64_t elem = 4;          // bytes per stored element
  int64_t n_kv_local = 0;
  int64_t length = 0;        // KvStore::length_
  std::vector<int64_t> seen; // KvStore::seen_
  // row counts of every logical buffer (GrowMat::rows): [set][layer]
  std::vector<std::vector<int64_t>> key_rows, value_rows, lr_rows;
  lk::PageSpace kv_space, lr_space;
  void* k_pages = nullptr;   // [n_layers][n_kv_local][kv_total_pages] pages; inside a page: page_layout.cuh
  void* v_pages = nullptr;
  void* lr_pages = nullptr;  // [n_layers][lr_total_pages][P][r_pad]
  // SelectiveRecompute (kvcache.hpp:53-58, 245-246, 289-305): one hidden-state cache of the trajectory (rows x d_model,
  // paged through the K / V page table) and the layers whose cached rows a returning agent may overwrite
  // key-side low-rank cache L_k = X A_k (an extension, kernels.hpp: KeyLowRank): one L x rank_k cache per layer shared by
  // every agent and kv head, laid out like the shared V_lr cache, own page table
  int64_t rk_pad = 0;                    // row width in HBM (rank_k zero-padded to 16 / 32 / 64); 0: no such cache
  void* lk_pages = nullptr;              // [n_layers][lk_total_pages][P][rk_pad]
  lk::PageSpace lk_space;
  std::vector<int64_t> lk_rows;          // [layer]
  int64_t lk_page_stride() const { return P * rk_pad; }
  int64_t lk_layer_stride() const { return lk_space.total_pages() * lk_page_stride(); }
  void* hidden_pages = nullptr;          // [kv_total_pages][P][d_model]
  // Which cached rows are certainly complete on the device (fla_decode_tma prefetches those before its programmatic-
  // dependent-launch wait).  Every call that writes pages records an event behind its kernels and the lowest row it
  // wrote; while that event has not completed, rows from `pending_row0` on may still be in flight.
  cudaEvent_t write_event = nullptr;
  bool write_recorded = false;
  int64_t pending_row0 = 0;
  int64_t hidden_rows = 0;
  std::vector<int64_t> recompute_layers;
  uint64_t reserved_bytes = 0;
  int64_t kv_sets() const { return dims.scheme == LORAKV_NONSHARED ? dims.n_agents : 1; }
  int64_t lr_sets() const {
    if (dims.scheme == LORAKV_BASESHARED) return dims.n_agents;
    if (dims.scheme == LORAKV_BASELRSHARED) return 1;
    return 0;
  }
  int64_t d_kv_local() const { return n_kv_local * dims.d_head; }
  // element strides of the page arrays
  int64_t kv_page_stride() const { return P * dims.d_head; }
  int64_t kv_head_stride() const { return kv_space.total_pages() * kv_page_stride(); }
  int64_t kv_layer_stride() const { return n_kv_local * kv_head_stride(); }
  int64_t lr_page_stride() const { return P * r_pad; }
  int64_t lr_layer_stride() const { return lr_space.total_pages() * lr_page_stride(); }
};

struct lorakv_adapters {
  lorakv_ctx* ctx = nullptr;
  int64_t n_layers = 0, n_agents = 0, d_model = 0, rank = 0, n_kv_heads = 0, d_head = 0;
  int64_t kv_head_begin = 0, n_kv_local = 0;
  int dtype = LORAKV_F32;
  float* a = nullptr;      // [n_layers][d_model][rank] float32 (values already representable in dtype)
  float* a_agent = nullptr; // [n_layers][n_agents][d_model][rank], allocated on the first per-agent upload (BaseShared)
  float* b = nullptr;      // [n_layers][n_agents][rank][n_kv_local*d_head] float32
  float* scale = nullptr;  // [n_layers][n_agents] device copy of alpha/rank
  std::vector<float> scale_host;
  std::vector<uint8_t> a_set, b_set, a_agent_set;
  // key-side adapter (extension): shared down-projection A_k per layer, B_k and alpha_k / rank_k per (layer, agent)
  int64_t rank_k = 0;
  float* a_k = nullptr;      // [n_layers][d_model][rank_k]
  float* b_k = nullptr;      // [n_layers][n_agents][rank_k][n_kv_local*d_head]
  float* scale_k = nullptr;  // [n_layers][n_agents]
  std::vector<float> scale_k_host;
  std::vector<uint8_t> a_k_set, b_k_set;
};

// End-of-step output gather of a kv-head-sharded run over peer memory (peer_gather.cu).  Every rank owns one
// allocation {flags, full output x 2} and maps every other rank's through CUDA IPC; the decode epilogue stores
// its slice of the output rows into all of them, a one-block kernel then publishes the step number to the
// peers' flag words and waits for theirs.
struct lorakv_gather {
  lorakv_ctx* ctx = nullptr;
  int rank = 0, world = 1;
  int64_t full_elems = 0;            // floats of one full output [layers][n_batch][n_q * d]
  size_t buf_bytes = 0;              // flags page + 2 * full output
  char* local = nullptr;             // this rank's allocation
  char* peer[8] = {};                // every rank's allocation as mapped here (peer[rank] == local)
  bool connected = false;
  uint32_t epoch = 0;                // steps gathered so far
  uint32_t* status_host = nullptr;   // pinned word the status flag is read back into
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  // Overlapped handshake (lorakv_gather_set_overlap): the handshake kernel runs on a side stream behind this step's epilogue
  // while the ctx stream goes on with the next step's attention; the ctx stream waits for it only before the NEXT epilogue
  // stores into the peers' buffers (the buffer-reuse guard) and in lorakv_gather_wait (before a consumer reads the rows)
  bool overlap = false;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_merged = nullptr, ev_synced = nullptr;
  bool sync_pending = false;         // ev_synced of the previous step has not been waited for on the ctx stream yet
};

namespace lk {
int gather_sync(lorakv_gather* g);                                         // peer_gather.cu
float* gather_buffer(const lorakv_gather* g, int rank, uint32_t epoch);
int gather_read_status(lorakv_gather* g);                                  // enqueue the status read-back
int gather_wait(lorakv_gather* g);                                         // ctx stream waits for an overlapped handshake
}  // namespace lk

// Projection weights of the step that feeds the cache (engine.hpp:376-403): Wk, Wv per layer, restricted to
// the kv heads this shard holds.  bf16 pools with d_head 128 keep them packed for the tcgen05 kernel
// (kv_project_umma.cu), every other case keeps the caller's float32 matrices.
struct lorakv_proj {
  lorakv_ctx* ctx = nullptr;
  int64_t n_layers = 0, d_model = 0, n_kv_heads = 0, d_head = 0, kv_head_begin = 0, n_kv_local = 0;
  int dtype = LORAKV_F32;
  bool fused = false;
  void* packed = nullptr;    // [n_layers][2 * n_kv_local * d_head / 64 blocks][d_model][64] bf16, SWIZZLE_128B
  float* wk = nullptr;       // [n_layers][d_model][n_kv_heads * d_head] float32 (exact path only)
  float* wv = nullptr;
  std::vector<uint8_t> set;
  // query projection (engine.hpp:362-373): Wq, the shared q-LoRA down-projection and per-agent up-projections
  int64_t n_q_heads = 0, q_rank = 0, q_agents = 0;
  bool q_fused = false;
  void* wq_packed = nullptr; // [n_layers][n_q_local * d_head / 64 blocks][d_model][64] bf16
  float* wq = nullptr;       // [n_layers][d_model][n_q_heads * d_head] float32 (exact path only)
  float* aq = nullptr;       // [n_layers][d_model][q_rank]
  float* bq = nullptr;       // [n_layers][q_agents][q_rank][n_q_heads * d_head]
  void* bq_extra = nullptr;  // [n_layers][q_agents][n_q_local * d_head / 64 blocks][64][64] bf16: B_q as one more k block (rank <= 32)
  std::vector<float> q_scale;          // [n_layers][q_agents] alpha / rank
  std::vector<uint8_t> q_set, q_lora_set;
};
