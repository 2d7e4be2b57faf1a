// api.cu -- the C ABI (include/lorakv_b200.h): context, memory helpers, the integer bookkeeping of
// the reference's KvStore (proj/include/lorakv/kvcache.hpp:112-142, 213-420) kept on the host, the
// adapter tables (proj/include/lorakv/lora.hpp:13-87) and the dispatch into the kernels.
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <new>

#include "kernels.hpp"
#include "state.hpp"

namespace lk {

std::string& err_slot() {
  thread_local std::string s;
  return s;
}

int fail(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  err_slot() = buf;
  return LORAKV_ERR;
}

int scratch_reserve(lorakv_ctx* ctx, Scratch& s, size_t bytes) {
  if (bytes <= s.bytes) return LORAKV_OK;
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (s.ptr) LK_CUDA(cudaFree(s.ptr));
  s.ptr = nullptr; s.bytes = 0;
  size_t want = std::max(bytes, (size_t)1 << 20);
  want = (want + ((size_t)1 << 20) - 1) & ~(((size_t)1 << 20) - 1);
  LK_CUDA(cudaMalloc(&s.ptr, want));
  s.bytes = want;
  return LORAKV_OK;
}

int pinned_reserve(lorakv_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->pinned_bytes) return LORAKV_OK;
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->pinned) LK_CUDA(cudaFreeHost(ctx->pinned));
  ctx->pinned = nullptr; ctx->pinned_bytes = 0;
  LK_CUDA(cudaMallocHost(&ctx->pinned, bytes));
  ctx->pinned_bytes = bytes;
  return LORAKV_OK;
}

int stage_agent_ids(lorakv_ctx* ctx, const int32_t* ids, int64_t n, const int32_t** dev) {
  for (IdSlot& s : ctx->id_slots)
    if (s.dev && (int64_t)s.ids.size() == n && std::memcmp(s.ids.data(), ids, (size_t)n * sizeof(int32_t)) == 0) {
      *dev = s.dev;
      return LORAKV_OK;
    }
  IdSlot& s = ctx->id_slots[ctx->id_next];
  ctx->id_next = (ctx->id_next + 1) % lorakv_ctx::kIdSlots;
  if (!s.copied) LK_CUDA(cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming));
  if ((size_t)n > s.cap) {
    LK_CUDA(cudaStreamSynchronize(ctx->stream));     // kernels reading the old device buffer are done
    if (s.host) LK_CUDA(cudaFreeHost(s.host));
    if (s.dev) LK_CUDA(cudaFree(s.dev));
    s.host = nullptr; s.dev = nullptr; s.cap = 0; s.ids.clear();
    const size_t cap = std::max<size_t>(64, (size_t)n * 2);
    LK_CUDA(cudaMallocHost(&s.host, cap * sizeof(int32_t)));
    LK_CUDA(cudaMalloc(&s.dev, cap * sizeof(int32_t)));
    s.cap = cap;
  } else {
    LK_CUDA(cudaEventSynchronize(s.copied));         // the previous copy out of this pinned buffer has completed
  }
  std::memcpy(s.host, ids, (size_t)n * sizeof(int32_t));
  s.ids.assign(ids, ids + n);
  // stream order protects the device buffer: kernels of earlier calls that read it run before this copy
  LK_CUDA(cudaMemcpyAsync(s.dev, s.host, (size_t)n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
  LK_CUDA(cudaEventRecord(s.copied, ctx->stream));
  *dev = s.dev;
  return LORAKV_OK;
}

int note_pages_written(lorakv_pool* pool, int64_t row0) {
  lorakv_ctx* ctx = pool->ctx;
  if (!pool->write_event) LK_CUDA(cudaEventCreateWithFlags(&pool->write_event, cudaEventDisableTiming));
  // still in flight from an earlier call? then the lowest pending row carries over
  const bool earlier_done = !pool->write_recorded || cudaEventQuery(pool->write_event) == cudaSuccess;
  pool->pending_row0 = earlier_done ? row0 : std::min(pool->pending_row0, row0);
  LK_CUDA(cudaEventRecord(pool->write_event, ctx->stream));
  pool->write_recorded = true;
  return LORAKV_OK;
}

int64_t stable_rows(lorakv_pool* pool, int64_t L) {
  if (!pool->write_recorded) return L;
  const cudaError_t e = cudaEventQuery(pool->write_event);
  if (e == cudaSuccess) { pool->write_recorded = false; return L; }
  if (e != cudaErrorNotReady) { (void)cudaGetLastError(); return 0; }
  return std::max<int64_t>(0, std::min(L, pool->pending_row0));
}

static const char* kSchemeName[5] = {"NonShared", "FullShared", "BaseShared", "BaseLRShared",
                                     "SelectiveRecompute"};
static const char* kWhat[3] = {"key", "value", "lr"};

// resolve (which, layer, agent) -> (set, row counter) the way append_* / *_view do
// (kvcache.hpp:268-288, 307-324); *none is set for the LR cache of a scheme that keeps none
static int resolve(const lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t* set,
                   bool* none) {
  *none = false; *set = 0;
  if (which == LORAKV_HIDDEN) {      // one hidden-state cache for the trajectory (kvcache.hpp:245-246); no layer, no agent
    if (pool->dims.scheme != LORAKV_SELECTIVE) return fail("KvStore: scheme %s has no hidden-state cache", kSchemeName[pool->dims.scheme]);
    return LORAKV_OK;
  }
  if (which == LORAKV_LK) {          // key-side low-rank cache (extension): one per layer, shared by all agents
    if (pool->rk_pad == 0) return fail("KvStore: this store keeps no key-side low-rank cache (rank_k = 0)");
    if (layer < 0 || layer >= pool->dims.n_layers) return fail("layer %lld out of range", (long long)layer);
    return LORAKV_OK;
  }
  if (which < LORAKV_KEY || which > LORAKV_LR) return fail("bad cache selector %d", which);
  const bool per_agent = (which != LORAKV_LR && pool->dims.scheme == LORAKV_NONSHARED) ||
                         (which == LORAKV_LR && pool->dims.scheme == LORAKV_BASESHARED);
  if (which == LORAKV_LR && pool->lr_sets() == 0) {
    *none = true;
    return LORAKV_OK;
  }
  if (per_agent) {
    if (agent < 0 || agent >= pool->dims.n_agents) return fail("unknown agent %lld", (long long)agent);
    *set = agent;
  }
  if (layer < 0 || layer >= pool->dims.n_layers) return fail("layer %lld out of range", (long long)layer);
  return LORAKV_OK;
}

// row counter of the buffer (which, set, layer)
static int64_t& row_counter(lorakv_pool* pool, int which, int64_t set, int64_t layer) {
  if (which == LORAKV_HIDDEN) return pool->hidden_rows;
  if (which == LORAKV_LK) return pool->lk_rows[(size_t)layer];
  auto& t = which == LORAKV_KEY ? pool->key_rows : which == LORAKV_VALUE ? pool->value_rows : pool->lr_rows;
  return t[(size_t)set][(size_t)layer];
}
static int64_t cache_cols_full(const lorakv_pool* pool, int which) {      // width of a caller's row
  if (which == LORAKV_LK) return pool->dims.rank_k;
  return which == LORAKV_HIDDEN ? pool->dims.d_model : which == LORAKV_LR ? pool->dims.rank : pool->dims.n_kv_heads * pool->dims.d_head;
}
static int64_t cache_cols_local(const lorakv_pool* pool, int which) {     // width of a stored / returned row
  if (which == LORAKV_LK) return pool->dims.rank_k;
  return which == LORAKV_HIDDEN ? pool->dims.d_model : which == LORAKV_LR ? pool->dims.rank : pool->d_kv_local();
}
static std::vector<std::vector<int64_t>>& rows_of(lorakv_pool* pool, int which) {
  return which == LORAKV_KEY ? pool->key_rows : which == LORAKV_VALUE ? pool->value_rows : pool->lr_rows;
}
static const std::vector<std::vector<int64_t>>& rows_of(const lorakv_pool* pool, int which) {
  return which == LORAKV_KEY ? pool->key_rows : which == LORAKV_VALUE ? pool->value_rows : pool->lr_rows;
}

// make sure logical pages covering rows [0, row_end) of `set` exist; ids in first-touch order
static int ensure_pages(lorakv_pool* pool, PageSpace& sp, int64_t set, int64_t row_end) {
  const int64_t need = (row_end + pool->P - 1) / pool->P;
  auto& tab = sp.table[(size_t)set];
  if ((int64_t)tab.size() >= need) return LORAKV_OK;
  if (need > sp.max_pages)
    return fail("KvStore: trajectory of %lld rows exceeds the pool capacity of %lld tokens",
                (long long)row_end, (long long)(sp.max_pages * pool->P));
  const size_t first = tab.size();
  while ((int64_t)tab.size() < need) tab.push_back(sp.next_free++);
  LK_CUDA(cudaMemcpyAsync(sp.dev_table + set * sp.max_pages + first, tab.data() + first,
                          (tab.size() - first) * sizeof(int32_t), cudaMemcpyHostToDevice,
                          pool->ctx->stream));
  // the host vector may be reallocated by a later push_back before the copy runs
  LK_CUDA(cudaStreamSynchronize(pool->ctx->stream));
  return LORAKV_OK;
}

template <class E>
static int stage_rows(lorakv_ctx* ctx, const E* rows, int64_t n, int64_t cols, int64_t ld,
                      int mem_kind, const E** dev, int64_t* dev_ld) {
  if (mem_kind == LORAKV_DEVICE) { *dev = rows; *dev_ld = ld; return LORAKV_OK; }
  if (mem_kind != LORAKV_HOST) return fail("bad mem_kind %d", mem_kind);
  LK_TRY(scratch_reserve(ctx, ctx->in, (size_t)std::max<int64_t>(n * cols, 1) * sizeof(E)));
  if (n > 0 && cols > 0)
    LK_CUDA(cudaMemcpy2DAsync(ctx->in.ptr, cols * sizeof(E), rows, ld * sizeof(E),
                              cols * sizeof(E), n, cudaMemcpyHostToDevice, ctx->stream));
  *dev = static_cast<const E*>(ctx->in.ptr);
  *dev_ld = cols;
  return LORAKV_OK;
}

}  // namespace lk

using namespace lk;

extern "C" {

int lorakv_abi_version(void) { return LORAKV_ABI_VERSION; }
const char* lorakv_last_error(void) { return err_slot().c_str(); }

// ---- context -------------------------------------------------------------------------------
int lorakv_ctx_create(int device, void* stream, lorakv_ctx** out) {
  if (!out) return fail("ctx_create: null out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail("lorakv_b200 needs a CUDA device (there is no CPU fallback): %s",
                e != cudaSuccess ? cudaGetErrorString(e) : "no device found");
  if (device < 0 || device >= n) return fail("ctx_create: device %d out of range [0,%d)", device, n);
  LK_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  LK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail("lorakv_b200 is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major,
                prop.minor);
  lorakv_ctx* ctx = new (std::nothrow) lorakv_ctx();
  if (!ctx) return fail("ctx_create: out of host memory");
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  ctx->l2_bytes = prop.l2CacheSize > 0 ? (int64_t)prop.l2CacheSize : (int64_t)126 << 20;
  const char* no_pdl = std::getenv("LORAKV_NO_PDL");       // A/B switch for the programmatic dependent launches
  ctx->pdl = !(no_pdl && no_pdl[0] == '1');
  const char* no_spec = std::getenv("LORAKV_NO_SPECULATION");
  ctx->speculate = ctx->pdl && !(no_spec && no_spec[0] == '1');
  if (stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t se = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (se != cudaSuccess) { delete ctx; return fail("ctx_create: %s", cudaGetErrorString(se)); }
    ctx->owns_stream = true;
  }
  *out = ctx;
  return LORAKV_OK;
}

void lorakv_ctx_destroy(lorakv_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (Scratch* s : {&ctx->in, &ctx->out, &ctx->work, &ctx->flush, &ctx->proj, &ctx->qrows, &ctx->qk, &ctx->planes})
    if (s->ptr) cudaFree(s->ptr);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  for (IdSlot& s : ctx->id_slots) {
    if (s.host) cudaFreeHost(s.host);
    if (s.dev) cudaFree(s.dev);
    if (s.copied) cudaEventDestroy(s.copied);
  }
  for (cudaEvent_t e : ctx->prof_ev) if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->prof_ring) if (e) cudaEventDestroy(e);
  if (ctx->owns_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int lorakv_ctx_synchronize(lorakv_ctx* ctx) {
  if (!ctx) return fail("null context");
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  return LORAKV_OK;
}
void* lorakv_ctx_stream(lorakv_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
int lorakv_ctx_sm_count(lorakv_ctx* ctx) { return ctx ? ctx->sm_count : 0; }
int64_t lorakv_ctx_launch_count(lorakv_ctx* ctx) { return ctx ? ctx->launches : 0; }

int lorakv_dev_alloc(lorakv_ctx* ctx, int64_t bytes, void** out) {
  if (!ctx || !out || bytes < 0) return fail("dev_alloc: bad arguments");
  LK_CUDA(cudaSetDevice(ctx->device));
  LK_CUDA(cudaMalloc(out, (size_t)std::max<int64_t>(bytes, 1)));
  return LORAKV_OK;
}
int lorakv_dev_free(lorakv_ctx* ctx, void* p) {
  if (!ctx) return fail("null context");
  if (p) LK_CUDA(cudaFree(p));
  return LORAKV_OK;
}
int lorakv_host_alloc(lorakv_ctx* ctx, int64_t bytes, void** out) {
  if (!ctx || !out || bytes < 0) return fail("host_alloc: bad arguments");
  LK_CUDA(cudaMallocHost(out, (size_t)std::max<int64_t>(bytes, 1)));
  return LORAKV_OK;
}
int lorakv_host_free(lorakv_ctx* ctx, void* p) {
  if (!ctx) return fail("null context");
  if (p) LK_CUDA(cudaFreeHost(p));
  return LORAKV_OK;
}
int lorakv_copy_h2d(lorakv_ctx* ctx, void* dst, const void* src, int64_t bytes) {
  if (!ctx) return fail("null context");
  LK_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, ctx->stream));
  return LORAKV_OK;
}
int lorakv_copy_d2h(lorakv_ctx* ctx, void* dst, const void* src, int64_t bytes) {
  if (!ctx) return fail("null context");
  LK_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return LORAKV_OK;
}
int lorakv_flush_l2(lorakv_ctx* ctx) {
  if (!ctx) return fail("null context");
  const size_t bytes = (size_t)256 << 20;   // 2x the 126 MB L2
  LK_TRY(scratch_reserve(ctx, ctx->flush, bytes));
  LK_CUDA(cudaMemsetAsync(ctx->flush.ptr, 0, bytes, ctx->stream));
  return LORAKV_OK;
}

struct lorakv_event { cudaEvent_t ev; };
int lorakv_event_create(lorakv_ctx* ctx, lorakv_event** out) {
  if (!ctx || !out) return fail("event_create: null argument");
  LK_CUDA(cudaSetDevice(ctx->device));
  lorakv_event* e = new (std::nothrow) lorakv_event();
  if (!e) return fail("event_create: out of host memory");
  cudaError_t ce = cudaEventCreate(&e->ev);
  if (ce != cudaSuccess) { delete e; return fail("event_create: %s", cudaGetErrorString(ce)); }
  *out = e;
  return LORAKV_OK;
}
int lorakv_event_record(lorakv_ctx* ctx, lorakv_event* ev) {
  if (!ctx || !ev) return fail("event_record: null argument");
  LK_CUDA(cudaEventRecord(ev->ev, ctx->stream));
  return LORAKV_OK;
}
int lorakv_event_elapsed_ms(lorakv_event* start, lorakv_event* stop, float* ms) {
  if (!start || !stop || !ms) return fail("event_elapsed_ms: null argument");
  LK_CUDA(cudaEventSynchronize(stop->ev));
  LK_CUDA(cudaEventElapsedTime(ms, start->ev, stop->ev));
  return LORAKV_OK;
}
void lorakv_event_destroy(lorakv_event* ev) {
  if (!ev) return;
  cudaEventDestroy(ev->ev);
  delete ev;
}

int lorakv_ctx_set_l2_bytes(lorakv_ctx* ctx, int64_t bytes) {
  if (!ctx || bytes < 1) return fail("ctx_set_l2_bytes: bad argument");
  ctx->l2_bytes = bytes;
  return LORAKV_OK;
}
int lorakv_ctx_set_prefill_split_keys(lorakv_ctx* ctx, int64_t keys) {
  if (!ctx || keys < 0 || keys > (int64_t)1 << 30) return fail("ctx_set_prefill_split_keys: bad argument");
  ctx->split_keys = (int)keys;
  return LORAKV_OK;
}
int lorakv_ctx_set_profiling(lorakv_ctx* ctx, int enabled) {
  if (!ctx) return fail("null context");
  LK_CUDA(cudaSetDevice(ctx->device));
  if (enabled && !ctx->prof_ev[0]) {
    LK_CUDA(cudaEventCreate(&ctx->prof_ev[0]));
    LK_CUDA(cudaEventCreate(&ctx->prof_ev[1]));
  }
  if (enabled && ctx->prof_ring.empty()) {
    ctx->prof_ring.resize(2 * lorakv_ctx::kProfPairs, nullptr);
    for (cudaEvent_t& e : ctx->prof_ring) LK_CUDA(cudaEventCreate(&e));
  }
  ctx->profiling = enabled != 0;
  ctx->prof_valid = false;
  ctx->prof_count = 0;
  return LORAKV_OK;
}
int lorakv_ctx_mean_kernel_ms(lorakv_ctx* ctx, float* ms, int* n_calls) {
  if (!ctx || !ms) return fail("null argument");
  if (ctx->prof_count < 1) return fail("mean_kernel_ms: no profiled fast-path call yet");
  LK_CUDA(cudaEventSynchronize(ctx->prof_ring[(size_t)(2 * ctx->prof_count - 1)]));
  double sum = 0.0;
  for (int i = 0; i < ctx->prof_count; ++i) {
    float t = 0.f;
    LK_CUDA(cudaEventElapsedTime(&t, ctx->prof_ring[(size_t)(2 * i)], ctx->prof_ring[(size_t)(2 * i + 1)]));
    sum += t;
  }
  *ms = (float)(sum / ctx->prof_count);
  if (n_calls) *n_calls = ctx->prof_count;
  ctx->prof_count = 0;
  return LORAKV_OK;
}
int lorakv_ctx_last_kernel_ms(lorakv_ctx* ctx, float* ms) {
  if (!ctx || !ms) return fail("null argument");
  if (!ctx->prof_valid) return fail("last_kernel_ms: no profiled fast-path call yet");
  LK_CUDA(cudaEventSynchronize(ctx->prof_ev[1]));
  LK_CUDA(cudaEventElapsedTime(ms, ctx->prof_ev[0], ctx->prof_ev[1]));
  return LORAKV_OK;
}

int lorakv_selftest_umma(lorakv_ctx* ctx, const float* a, const float* b, int N, int K, int b_mn_major, float alpha,
                         int rescale, int a_in_tmem, float* d) {
  return umma_selftest(ctx, a, b, N, K, b_mn_major, alpha, rescale, a_in_tmem, d);
}

int lorakv_set_kernel_policy(lorakv_ctx* ctx, int policy) {
  if (!ctx) return 0;
  const int old = ctx->policy;
  ctx->policy = policy;
  return old;
}
const char* lorakv_last_kernel(lorakv_ctx* ctx) { return ctx ? ctx->last_kernel : "none"; }

// ---- per-head operators ------------------------------------------------------------------------
#define LK_OPS(SUF, T)                                                                              \
  int lorakv_fla_forward_##SUF(lorakv_ctx* ctx, const T* q, int64_t ldq, const T* k, int64_t ldk,   \
                               const T* v, int64_t ldv, const T* vlr, int64_t ldlr, const T* b,     \
                               int64_t ldb, T s, int64_t Lc, int64_t L, int64_t d, int64_t r,       \
                               int64_t off, T* out, T* row_max, T* row_denom) {                     \
    return generic_forward<T>(ctx, "flash_lora_attention", 0, q, ldq, k, ldk, v, ldv, vlr, ldlr, b, \
                              ldb, s, Lc, L, 1, 1, d, r, off, out, row_max, row_denom);             \
  }                                                                                                 \
  int lorakv_expand_first_forward_##SUF(lorakv_ctx* ctx, const T* q, int64_t ldq, const T* k,       \
                                        int64_t ldk, const T* v, int64_t ldv, const T* vlr,         \
                                        int64_t ldlr, const T* b, int64_t ldb, T s, int64_t Lc,     \
                                        int64_t L, int64_t d, int64_t r, int64_t off, T* out) {     \
    return generic_forward<T>(ctx, "expand_first_attention", 1, q, ldq, k, ldk, v, ldv, vlr, ldlr,  \
                              b, ldb, s, Lc, L, 1, 1, d, r, off, out, nullptr, nullptr);            \
  }                                                                                                 \
  int lorakv_naive_forward_##SUF(lorakv_ctx* ctx, const T* q, int64_t ldq, const T* k, int64_t ldk, \
                                 const T* v, int64_t ldv, const T* vlr, int64_t ldlr, const T* b,   \
                                 int64_t ldb, T s, int64_t Lc, int64_t L, int64_t d, int64_t r,     \
                                 int64_t off, T* out) {                                             \
    return naive_forward<T>(ctx, q, ldq, k, ldk, v, ldv, vlr, ldlr, b, ldb, s, Lc, L, d, r, off,    \
                            out);                                                                   \
  }                                                                                                 \
  int lorakv_gqa_forward_##SUF(lorakv_ctx* ctx, const T* q, int64_t ldq, const T* k, int64_t ldk,   \
                               const T* v, int64_t ldv, const T* vlr, int64_t ldlr, const T* b,     \
                               int64_t ldb, T s, int64_t Lc, int64_t L, int64_t n_q, int64_t n_kv,  \
                               int64_t d, int64_t r, int64_t off, T* out) {                         \
    if (n_q < 1 || n_kv < 1 || n_q % n_kv != 0)                                                     \
      return fail("gqa_attention: n_q_heads %lld not divisible by n_kv_heads %lld", (long long)n_q, \
                  (long long)n_kv);                                                                 \
    return generic_forward<T>(ctx, "flash_lora_attention", 0, q, ldq, k, ldk, v, ldv, vlr, ldlr, b, \
                              ldb, s, Lc, L, (int)n_q, (int)n_kv, d, r, off, out, nullptr, nullptr);\
  }
LK_OPS(f32, float)
LK_OPS(f64, double)

// gqa_attention with the key-side low-rank term (KeyLowRank, kernels.hpp): n_q = n_kv = 1 is the per-head operator
#define LK_KEY_OPS(SUF, T)                                                                                             \
  int lorakv_gqa_forward_keylr_##SUF(lorakv_ctx* ctx, const T* q, int64_t ldq, const T* k, int64_t ldk, const T* v,    \
                                     int64_t ldv, const T* vlr, int64_t ldlr, const T* b, int64_t ldb, T s,            \
                                     const T* l_k, int64_t ld_lk, const T* b_k, int64_t ld_bk, T k_scale, int64_t Lc,  \
                                     int64_t L, int64_t n_q, int64_t n_kv, int64_t d, int64_t r, int64_t r_k,          \
                                     int64_t off, T* out) {                                                            \
    if (n_q < 1 || n_kv < 1 || n_q % n_kv != 0)                                                                        \
      return fail("gqa_attention: n_q_heads %lld not divisible by n_kv_heads %lld", (long long)n_q, (long long)n_kv);  \
    const KeyLowRank<T> key{l_k, ld_lk, b_k, ld_bk, k_scale, r_k};                                                     \
    return generic_forward<T>(ctx, "flash_lora_attention", 0, q, ldq, k, ldk, v, ldv, vlr, ldlr, b, ldb, s, Lc, L,     \
                              (int)n_q, (int)n_kv, d, r, off, out, nullptr, nullptr, r_k > 0 ? &key : nullptr);        \
  }
LK_KEY_OPS(f32, float)
LK_KEY_OPS(f64, double)

int lorakv_matmul_f32(lorakv_ctx* ctx, const float* a, int64_t lda, const float* b, int64_t ldb, int64_t M,
                      int64_t K, int64_t N, float* out) {
  return matmul_forward<float>(ctx, a, lda, b, ldb, M, K, N, out);
}
int lorakv_matmul_f64(lorakv_ctx* ctx, const double* a, int64_t lda, const double* b, int64_t ldb, int64_t M,
                      int64_t K, int64_t N, double* out) {
  return matmul_forward<double>(ctx, a, lda, b, ldb, M, K, N, out);
}

void lorakv_lr_mac_counts(int64_t total_len, int64_t cur_len, int64_t rank, int64_t d_head,
                          uint64_t* no_reorder, uint64_t* reorder) {
  const uint64_t L = (uint64_t)total_len, Lc = (uint64_t)cur_len, r = (uint64_t)rank, d = (uint64_t)d_head;
  if (no_reorder) *no_reorder = L * r * d + Lc * L * d;
  if (reorder) *reorder = Lc * L * r + Lc * r * d;
}

void lorakv_attn_macs(int64_t L_c, int64_t L, int64_t d, int64_t r, int expand_first, uint64_t macs[3]) {
  // Dense tile accounting of attention.hpp:229-243 / :286-307 summed over any tiling.
  const uint64_t Lc = (uint64_t)L_c, Lu = (uint64_t)L, du = (uint64_t)d, ru = (uint64_t)r;
  macs[0] = Lc * Lu * du;
  macs[1] = Lc * Lu * du;
  macs[2] = expand_first ? Lu * ru * du + Lc * Lu * (ru > 0 ? du : 0) : Lc * Lu * ru + Lc * ru * du;
}

// ---- planning ---------------------------------------------------------------------------------
int lorakv_plan_core(int scheme, int64_t first_recompute, int64_t length, int64_t seen,
                     int64_t new_tokens, int64_t out[9]) {
  if (new_tokens < 0) return fail("plan_core: new_tokens must be >= 0");
  if (seen < 0 || seen > length) return fail("plan_core: seen out of range");
  if (scheme < LORAKV_NONSHARED || scheme > LORAKV_SELECTIVE) return fail("plan_core: unknown scheme %d", scheme);
  const int64_t total = length + new_tokens;
  // every range starts as `fresh` = [length, total); the schemes that cannot reuse another
  // agent's work widen some of them to `unseen` = [seen, total)
  for (int i = 0; i < 3; ++i) { out[2 * i] = length; out[2 * i + 1] = total; }
  out[6] = out[7] = out[8] = 0;
  const bool widen_hidden = scheme == LORAKV_NONSHARED || scheme == LORAKV_BASESHARED || scheme == LORAKV_SELECTIVE;
  const bool widen_kv = scheme == LORAKV_NONSHARED;
  const bool widen_lr = scheme == LORAKV_NONSHARED || scheme == LORAKV_BASESHARED;
  if (widen_hidden) out[0] = seen;
  if (widen_kv) out[2] = seen;
  if (widen_lr) out[4] = seen;
  if (scheme == LORAKV_SELECTIVE) { out[6] = seen; out[7] = total; out[8] = first_recompute; }
  return LORAKV_OK;
}

// ---- pool ----------------------------------------------------------------------------------------
int lorakv_pool_create(lorakv_ctx* ctx, const lorakv_pool_dims* dims, lorakv_pool** out) {
  if (!ctx || !dims || !out) return fail("pool_create: null argument");
  *out = nullptr;
  if (dims->n_layers < 1 || dims->n_kv_heads < 1 || dims->d_head < 1 || dims->d_model < 1 || dims->n_agents < 1)
    return fail("KvStore: invalid dims");
  if (dims->rank < 0) return fail("KvStore: negative rank");
  // SelectiveRecompute is a baseline scheme outside the Flash-LoRA-Attention path; its store (shared K / V, the hidden-state
  // cache, the overwrite of recompute layers) exists so that the reference's callers and tests run against this library
  if (dims->scheme < LORAKV_NONSHARED || dims->scheme > LORAKV_SELECTIVE) return fail("KvStore: unknown scheme %d", dims->scheme);
  if (dims->dtype != LORAKV_F32 && dims->dtype != LORAKV_BF16 && dims->dtype != LORAKV_F64) return fail("KvStore: unknown dtype %d", dims->dtype);
  if (dims->max_tokens < 1) return fail("KvStore: max_tokens must be >= 1");
  lorakv_pool* p = new (std::nothrow) lorakv_pool();
  if (!p) return fail("pool_create: out of host memory");
  p->ctx = ctx;
  p->dims = *dims;
  p->P = dims->page_tokens > 0 ? dims->page_tokens : 64;
  p->dims.page_tokens = p->P;
  p->n_kv_local = dims->n_kv_local > 0 ? dims->n_kv_local : dims->n_kv_heads - dims->kv_head_begin;
  p->dims.n_kv_local = p->n_kv_local;
  if (dims->kv_head_begin < 0 || p->n_kv_local < 1 || dims->kv_head_begin + p->n_kv_local > dims->n_kv_heads) {
    delete p;
    return fail("KvStore: kv head shard [%lld,+%lld) outside [0,%lld)", (long long)dims->kv_head_begin,
                (long long)dims->n_kv_local, (long long)dims->n_kv_heads);
  }
  p->elem = dims->dtype == LORAKV_BF16 ? 2 : dims->dtype == LORAKV_F64 ? 8 : 4;
  const bool has_lr = p->lr_sets() > 0 && dims->rank > 0;
  // LR row width in HBM: the rank padded with zero columns (exact) to 16/32/64 or a multiple of
  // 64, the widths page_layout.cuh can swizzle
  p->r_pad = 0;
  if (has_lr) {
    p->r_pad = 16;   // one tcgen05 N-tile / one 32-byte swizzled row at least
    while (p->r_pad < dims->rank && p->r_pad < 64) p->r_pad *= 2;
    if (p->r_pad < dims->rank) p->r_pad = (dims->rank + 63) / 64 * 64;
  }
  if (dims->rank_k < 0 || dims->rank_k > 64) { delete p; return fail("KvStore: key rank %lld outside [0,64]", (long long)dims->rank_k); }
  if (dims->rank_k > 0) {
    p->rk_pad = 16;
    while (p->rk_pad < dims->rank_k) p->rk_pad *= 2;
  }
  p->seen.assign((size_t)dims->n_agents, 0);
  const int64_t max_pages = (dims->max_tokens + p->P - 1) / p->P;
  p->dims.max_tokens = max_pages * p->P;
  auto init_space = [&](PageSpace& sp, int64_t sets) {
    sp.n_sets = sets; sp.max_pages = max_pages; sp.next_free = 0;
    sp.table.assign((size_t)sets, {});
  };
  init_space(p->kv_space, p->kv_sets());
  init_space(p->lr_space, p->lr_sets());
  init_space(p->lk_space, p->rk_pad > 0 ? 1 : 0);
  p->lk_rows.assign((size_t)dims->n_layers, 0);
  p->key_rows.assign((size_t)p->kv_sets(), std::vector<int64_t>((size_t)dims->n_layers, 0));
  p->value_rows = p->key_rows;
  p->lr_rows.assign((size_t)std::max<int64_t>(p->lr_sets(), 1), std::vector<int64_t>((size_t)dims->n_layers, 0));

  auto cleanup = [&](int rc) { lorakv_pool_destroy(p); return rc; };
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cleanup(fail("pool_create: %s", cudaGetErrorString(e)));
  const size_t kv_bytes = (size_t)(dims->n_layers * p->kv_layer_stride()) * (size_t)p->elem;
  const size_t lr_bytes = (size_t)(dims->n_layers * p->lr_layer_stride()) * (size_t)p->elem;
  auto alloc_zero = [&](void** ptr, size_t bytes) -> int {
    if (bytes == 0) return LORAKV_OK;
    LK_CUDA(cudaMalloc(ptr, bytes));
    // pages are zero-filled so that the unused tail of the last page multiplies as exact zeros
    LK_CUDA(cudaMemsetAsync(*ptr, 0, bytes, ctx->stream));
    p->reserved_bytes += bytes;
    return LORAKV_OK;
  };
  int rc = alloc_zero(&p->k_pages, kv_bytes);
  if (rc == LORAKV_OK) rc = alloc_zero(&p->v_pages, kv_bytes);
  if (rc == LORAKV_OK) rc = alloc_zero(&p->lr_pages, lr_bytes);
  if (rc == LORAKV_OK) rc = alloc_zero(&p->lk_pages, (size_t)(dims->n_layers * p->lk_layer_stride()) * (size_t)p->elem);
  if (rc == LORAKV_OK && dims->scheme == LORAKV_SELECTIVE)
    rc = alloc_zero(&p->hidden_pages, (size_t)(p->kv_space.total_pages() * p->P * dims->d_model) * (size_t)p->elem);
  auto alloc_table = [&](PageSpace& sp) -> int {
    if (sp.total_pages() == 0) return LORAKV_OK;
    LK_CUDA(cudaMalloc(&sp.dev_table, (size_t)sp.total_pages() * sizeof(int32_t)));
    LK_CUDA(cudaMemsetAsync(sp.dev_table, 0, (size_t)sp.total_pages() * sizeof(int32_t), ctx->stream));
    return LORAKV_OK;
  };
  if (rc == LORAKV_OK) rc = alloc_table(p->kv_space);
  if (rc == LORAKV_OK) rc = alloc_table(p->lr_space);
  if (rc == LORAKV_OK) rc = alloc_table(p->lk_space);
  if (rc != LORAKV_OK) return cleanup(rc);
  *out = p;
  return LORAKV_OK;
}

void lorakv_pool_destroy(lorakv_pool* p) {
  if (!p) return;
  cudaSetDevice(p->ctx->device);
  cudaStreamSynchronize(p->ctx->stream);
  if (p->write_event) cudaEventDestroy(p->write_event);
  for (void* q : {p->k_pages, p->v_pages, p->lr_pages, p->hidden_pages, p->lk_pages, (void*)p->kv_space.dev_table,
                  (void*)p->lr_space.dev_table, (void*)p->lk_space.dev_table})
    if (q) cudaFree(q);
  delete p;
}

int lorakv_pool_dims_get(const lorakv_pool* pool, lorakv_pool_dims* out) {
  if (!pool || !out) return fail("null argument");
  *out = pool->dims;
  return LORAKV_OK;
}

int lorakv_pool_append_tokens(lorakv_pool* pool, int64_t n) {
  if (!pool) return fail("null pool");
  if (n < 0) return fail("append_tokens: negative count");
  pool->length += n;
  return LORAKV_OK;
}
int64_t lorakv_pool_length(const lorakv_pool* pool) { return pool ? pool->length : -1; }

int lorakv_pool_seen(const lorakv_pool* pool, int64_t agent, int64_t* out) {
  if (!pool || !out) return fail("null argument");
  if (agent < 0 || agent >= pool->dims.n_agents) return fail("unknown agent %lld", (long long)agent);
  *out = pool->seen[(size_t)agent];
  return LORAKV_OK;
}
int lorakv_pool_mark_seen(lorakv_pool* pool, int64_t agent) {
  if (!pool) return fail("null pool");
  if (agent < 0 || agent >= pool->dims.n_agents) return fail("unknown agent %lld", (long long)agent);
  if (pool->length < pool->seen[(size_t)agent]) return fail("KvStore: seen_upto may not decrease");
  pool->seen[(size_t)agent] = pool->length;
  return LORAKV_OK;
}
int lorakv_pool_plan_step(const lorakv_pool* pool, int64_t agent, int64_t new_tokens, int64_t out[9]) {
  int64_t seen = 0;
  LK_TRY(lorakv_pool_seen(pool, agent, &seen));
  return lorakv_plan_core(pool->dims.scheme, 0, pool->length, seen, new_tokens, out);
}

// first-writer-wins arithmetic of append_fww (kvcache.hpp:400-407)
static int fww(const char* what, int64_t rows, int64_t row_begin, int64_t n, int64_t* skip, int64_t* add) {
  if (row_begin > rows) return fail("KvStore: %s append leaves a gap at row %lld", what, (long long)rows);
  const int64_t present = rows - row_begin;
  if (present >= n) { *skip = n; *add = 0; return LORAKV_OK; }
  *skip = present;
  *add = n - present;
  return LORAKV_OK;
}

}  // extern "C"

static const char* kWhat4[5] = {"key", "value", "lr", "hidden", "key-lr"};

template <class E>
static int pool_append_impl(lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t row_begin,
                            const E* rows, int64_t n_rows, int64_t ld, int mem_kind, int64_t* appended) {
  if (!pool) return fail("null pool");
  if (appended) *appended = 0;
  int64_t set; bool none;
  LK_TRY(resolve(pool, which, layer, agent, &set, &none));
  if (none) return fail("KvStore: scheme %s has no LR cache", kSchemeName[pool->dims.scheme]);
  if (n_rows < 0) return fail("append: negative row count");
  if ((sizeof(E) == 8) != (pool->dims.dtype == LORAKV_F64))
    return fail("append: %s rows into a pool of another element type (fp64 pools take float64 rows, the others float32)",
                sizeof(E) == 8 ? "float64" : "float32");
  int64_t& have = row_counter(pool, which, set, layer);
  int64_t skip, add;
  LK_TRY(fww(kWhat4[which], have, row_begin, n_rows, &skip, &add));
  if (add == 0) return LORAKV_OK;
  const int64_t full_cols = cache_cols_full(pool, which);
  if (full_cols > 0) {
    if (!rows) return fail("append: null rows");
    lorakv_ctx* ctx = pool->ctx;
    LK_CUDA(cudaSetDevice(ctx->device));
    LK_TRY(ensure_pages(pool, which == LORAKV_LR ? pool->lr_space : which == LORAKV_LK ? pool->lk_space : pool->kv_space, set, have + add));
    const E* dev; int64_t dev_ld;
    LK_TRY(stage_rows(ctx, rows + skip * ld, add, full_cols, ld, mem_kind, &dev, &dev_ld));
    const int64_t col0 = (which == LORAKV_KEY || which == LORAKV_VALUE) ? pool->dims.kv_head_begin * pool->dims.d_head : 0;
    LK_TRY(launch_append_scatter(pool, which, layer, set, have, dev + col0, add, dev_ld));
    if (mem_kind == LORAKV_HOST) LK_CUDA(cudaStreamSynchronize(ctx->stream));  // staging is reused
    else LK_TRY(note_pages_written(pool, have));
  }
  have += add;
  if (appended) *appended = add;
  return LORAKV_OK;
}

// recompute_overwrite (kvcache.hpp:298-305): same scatter as an append, over rows that exist, counters untouched
template <class E>
static int pool_overwrite_impl(lorakv_pool* pool, int which, int64_t layer, int64_t row_begin, const E* rows, int64_t n_rows,
                               int64_t ld, int mem_kind) {
  if (!pool) return fail("null pool");
  if (which != LORAKV_KEY && which != LORAKV_VALUE) return fail("bad cache selector %d", which);
  const bool allowed = pool->dims.scheme == LORAKV_SELECTIVE &&
                       std::binary_search(pool->recompute_layers.begin(), pool->recompute_layers.end(), layer);
  if (!allowed)
    return fail("KvStore: overwrite of existing cache rows is forbidden (scheme %s, layer %lld)", kSchemeName[pool->dims.scheme], (long long)layer);
  if (layer < 0 || layer >= pool->dims.n_layers) return fail("layer %lld out of range", (long long)layer);
  if ((sizeof(E) == 8) != (pool->dims.dtype == LORAKV_F64)) return fail("overwrite: rows of another element type than the pool's");
  const int64_t have = row_counter(pool, which, 0, layer);
  if (row_begin < 0 || n_rows < 0 || row_begin + n_rows > have)
    return fail("GrowMat::overwrite: rows [%lld,%lld) not materialized", (long long)row_begin, (long long)(row_begin + n_rows));
  if (n_rows == 0) return LORAKV_OK;
  if (!rows) return fail("overwrite: null rows");
  lorakv_ctx* ctx = pool->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  const E* dev; int64_t dev_ld;
  LK_TRY(stage_rows(ctx, rows, n_rows, cache_cols_full(pool, which), ld, mem_kind, &dev, &dev_ld));
  LK_TRY(launch_append_scatter(pool, which, layer, 0, row_begin, dev + pool->dims.kv_head_begin * pool->dims.d_head, n_rows, dev_ld));
  if (mem_kind == LORAKV_HOST) LK_CUDA(cudaStreamSynchronize(ctx->stream));
  else LK_TRY(note_pages_written(pool, row_begin));
  return LORAKV_OK;
}

template <class E>
static int pool_read_impl(const lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t row_begin, int64_t n_rows, E* out) {
  if (!pool) return fail("null pool");
  int64_t set; bool none;
  LK_TRY(resolve(pool, which, layer, agent, &set, &none));
  if (none) return LORAKV_OK;   // zero columns
  if ((sizeof(E) == 8) != (pool->dims.dtype == LORAKV_F64)) return fail("read: rows of another element type than the pool's");
  const int64_t have = row_counter(const_cast<lorakv_pool*>(pool), which, set, layer);
  if (row_begin < 0 || n_rows < 0 || row_begin + n_rows > have)
    return fail("row_range [%lld,%lld) out of bounds for %lld rows", (long long)row_begin,
                (long long)(row_begin + n_rows), (long long)have);
  const int64_t cols = cache_cols_local(pool, which);
  if (n_rows == 0 || cols == 0) return LORAKV_OK;
  if (!out) return fail("read: null out");
  lorakv_ctx* ctx = pool->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  LK_TRY(scratch_reserve(ctx, ctx->out, (size_t)(n_rows * cols) * sizeof(E)));
  LK_TRY(launch_gather_rows(pool, which, layer, set, row_begin, n_rows, static_cast<E*>(ctx->out.ptr)));
  LK_CUDA(cudaMemcpyAsync(out, ctx->out.ptr, (size_t)(n_rows * cols) * sizeof(E), cudaMemcpyDeviceToHost, ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  return LORAKV_OK;
}

extern "C" {

int lorakv_pool_append(lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t row_begin,
                       const float* rows, int64_t n_rows, int64_t ld, int mem_kind, int64_t* appended) {
  return pool_append_impl(pool, which, layer, agent, row_begin, rows, n_rows, ld, mem_kind, appended);
}
int lorakv_pool_append_f64(lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t row_begin,
                           const double* rows, int64_t n_rows, int64_t ld, int mem_kind, int64_t* appended) {
  return pool_append_impl(pool, which, layer, agent, row_begin, rows, n_rows, ld, mem_kind, appended);
}
int lorakv_pool_overwrite(lorakv_pool* pool, int which, int64_t layer, int64_t row_begin, const float* rows, int64_t n_rows,
                          int64_t ld, int mem_kind) {
  return pool_overwrite_impl(pool, which, layer, row_begin, rows, n_rows, ld, mem_kind);
}
int lorakv_pool_overwrite_f64(lorakv_pool* pool, int which, int64_t layer, int64_t row_begin, const double* rows, int64_t n_rows,
                              int64_t ld, int mem_kind) {
  return pool_overwrite_impl(pool, which, layer, row_begin, rows, n_rows, ld, mem_kind);
}
int lorakv_pool_read_f64(const lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t row_begin, int64_t n_rows,
                         double* out) {
  return pool_read_impl(pool, which, layer, agent, row_begin, n_rows, out);
}
int lorakv_pool_get_recompute_layers(const lorakv_pool* pool, int64_t* out, int64_t cap, int64_t* n) {
  if (!pool) return fail("null pool");
  if (n) *n = (int64_t)pool->recompute_layers.size();
  for (int64_t i = 0; out && i < cap && i < (int64_t)pool->recompute_layers.size(); ++i) out[i] = pool->recompute_layers[(size_t)i];
  return LORAKV_OK;
}
int lorakv_pool_set_recompute_layers(lorakv_pool* pool, const int64_t* layers, int64_t n) {
  if (!pool || (n > 0 && !layers)) return fail("null argument");
  for (int64_t i = 0; i < n; ++i)
    if (layers[i] < 0 || layers[i] >= pool->dims.n_layers) return fail("KvStore: recompute layer %lld out of range", (long long)layers[i]);
  pool->recompute_layers.assign(layers, layers + n);
  std::sort(pool->recompute_layers.begin(), pool->recompute_layers.end());
  return LORAKV_OK;
}

int lorakv_pool_append_lr_project(lorakv_pool* pool, const lorakv_adapters* ad, int64_t layer,
                                  int64_t agent, int64_t row_begin, const float* x, int64_t n_rows,
                                  int64_t ld, int mem_kind, int64_t* appended) {
  if (!pool || !ad) return fail("null argument");
  if (appended) *appended = 0;
  if (pool->dims.dtype == LORAKV_F64) return fail("lr_append_project: fp64 pools are storage only (append_lr takes the rows)");
  int64_t set; bool none;
  LK_TRY(resolve(pool, LORAKV_LR, layer, agent, &set, &none));
  if (none) return fail("KvStore: scheme %s has no LR cache", kSchemeName[pool->dims.scheme]);
  if (ad->rank != pool->dims.rank || ad->d_model != pool->dims.d_model || layer >= ad->n_layers)
    return fail("lr_append_project: adapter table does not match the pool (rank %lld vs %lld)",
                (long long)ad->rank, (long long)pool->dims.rank);
  const bool own_a = ad->a_agent && agent >= 0 && agent < ad->n_agents && ad->a_agent_set[(size_t)(layer * ad->n_agents + agent)];
  if (pool->dims.rank > 0 && !own_a && !ad->a_set[(size_t)layer]) return fail("lr_append_project: A of layer %lld was never uploaded", (long long)layer);
  int64_t& have = pool->lr_rows[(size_t)set][(size_t)layer];
  int64_t skip, add;
  LK_TRY(fww("lr", have, row_begin, n_rows, &skip, &add));
  if (add == 0) return LORAKV_OK;
  if (pool->dims.rank > 0) {
    lorakv_ctx* ctx = pool->ctx;
    LK_CUDA(cudaSetDevice(ctx->device));
    LK_TRY(ensure_pages(pool, pool->lr_space, set, have + add));
    const float* dev; int64_t dev_ld;
    LK_TRY(stage_rows(ctx, x + skip * ld, add, pool->dims.d_model, ld, mem_kind, &dev, &dev_ld));
    const float* a_dev = own_a ? ad->a_agent + (size_t)(layer * ad->n_agents + agent) * (size_t)(ad->d_model * ad->rank)
                               : ad->a + layer * ad->d_model * ad->rank;
    LK_TRY(launch_lr_project(pool, a_dev, ad->d_model, ad->rank, layer, set, have, dev, add, dev_ld));
    if (mem_kind == LORAKV_HOST) LK_CUDA(cudaStreamSynchronize(ctx->stream));
    else LK_TRY(note_pages_written(pool, have));
  }
  have += add;
  if (appended) *appended = add;
  return LORAKV_OK;
}

// ---- K / V_base projection + RoPE + append (engine.hpp:376-403) --------------------------------------
int lorakv_proj_create(lorakv_ctx* ctx, int64_t n_layers, int64_t d_model, int64_t n_kv_heads, int64_t d_head,
                       int64_t kv_head_begin, int64_t n_kv_local, int dtype, lorakv_proj** out) {
  if (!ctx || !out) return fail("proj_create: null argument");
  *out = nullptr;
  if (n_layers < 1 || d_model < 1 || n_kv_heads < 1 || d_head < 1) return fail("proj_create: invalid shape");
  if (d_head % 2 != 0) return fail("proj_create: d_head %lld must be even (half-dim rotation)", (long long)d_head);
  if (n_kv_local <= 0) { kv_head_begin = 0; n_kv_local = n_kv_heads; }
  if (kv_head_begin < 0 || kv_head_begin + n_kv_local > n_kv_heads) return fail("proj_create: kv head shard out of range");
  if (dtype != LORAKV_F32 && dtype != LORAKV_BF16) return fail("proj_create: bad dtype %d", dtype);
  LK_CUDA(cudaSetDevice(ctx->device));
  lorakv_proj* pr = new (std::nothrow) lorakv_proj();
  if (!pr) return fail("proj_create: out of host memory");
  pr->ctx = ctx; pr->n_layers = n_layers; pr->d_model = d_model; pr->n_kv_heads = n_kv_heads; pr->d_head = d_head;
  pr->kv_head_begin = kv_head_begin; pr->n_kv_local = n_kv_local; pr->dtype = dtype;
  pr->fused = kv_project_fused_shape(dtype, d_head, d_model);
  pr->set.assign((size_t)n_layers, 0);
  cudaError_t e;
  if (pr->fused) {
    e = cudaMalloc(&pr->packed, (size_t)(n_layers * kv_project_packed_elems(d_model, n_kv_local, d_head)) * 2);
  } else {
    const size_t bytes = (size_t)(n_layers * d_model * n_kv_heads * d_head) * sizeof(float);
    e = cudaMalloc(&pr->wk, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&pr->wv, bytes);
  }
  if (e != cudaSuccess) { lorakv_proj_destroy(pr); return fail("proj_create: %s", cudaGetErrorString(e)); }
  *out = pr;
  return LORAKV_OK;
}

void lorakv_proj_destroy(lorakv_proj* pr) {
  if (!pr) return;
  cudaSetDevice(pr->ctx->device);
  cudaStreamSynchronize(pr->ctx->stream);
  if (pr->packed) cudaFree(pr->packed);
  if (pr->wk) cudaFree(pr->wk);
  if (pr->wv) cudaFree(pr->wv);
  for (void* q : {pr->wq_packed, (void*)pr->wq, (void*)pr->aq, (void*)pr->bq, pr->bq_extra}) if (q) cudaFree(q);
  delete pr;
}

int lorakv_proj_set_kv(lorakv_proj* pr, int64_t layer, const float* wk, const float* wv) {
  if (!pr || !wk || !wv) return fail("null argument");
  if (layer < 0 || layer >= pr->n_layers) return fail("layer %lld out of range", (long long)layer);
  lorakv_ctx* ctx = pr->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  const int64_t dkv_full = pr->n_kv_heads * pr->d_head, dkv = pr->n_kv_local * pr->d_head;
  const size_t one = (size_t)(pr->d_model * dkv_full) * sizeof(float);
  if (pr->fused) {
    LK_TRY(scratch_reserve(ctx, ctx->in, 2 * one));
    float* sk = static_cast<float*>(ctx->in.ptr);
    float* sv = reinterpret_cast<float*>(static_cast<char*>(ctx->in.ptr) + one);
    LK_CUDA(cudaMemcpyAsync(sk, wk, one, cudaMemcpyHostToDevice, ctx->stream));
    LK_CUDA(cudaMemcpyAsync(sv, wv, one, cudaMemcpyHostToDevice, ctx->stream));
    char* dst = static_cast<char*>(pr->packed) + (size_t)(layer * kv_project_packed_elems(pr->d_model, pr->n_kv_local, pr->d_head)) * 2;
    LK_TRY(launch_pack_w(ctx, sk, dkv_full, pr->kv_head_begin * pr->d_head, dkv, pr->d_model, 0, dst));
    LK_TRY(launch_pack_w(ctx, sv, dkv_full, pr->kv_head_begin * pr->d_head, dkv, pr->d_model, dkv / 64, dst));
  } else {
    LK_CUDA(cudaMemcpyAsync(pr->wk + (size_t)layer * (one / sizeof(float)), wk, one, cudaMemcpyHostToDevice, ctx->stream));
    LK_CUDA(cudaMemcpyAsync(pr->wv + (size_t)layer * (one / sizeof(float)), wv, one, cudaMemcpyHostToDevice, ctx->stream));
  }
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  pr->set[(size_t)layer] = 1;
  return LORAKV_OK;
}

// ---- query projection (engine.hpp:362-373, :422) ----------------------------------------------------
int lorakv_proj_set_q(lorakv_proj* pr, int64_t layer, int64_t n_q_heads, const float* wq) {
  if (!pr || !wq) return fail("null argument");
  if (layer < 0 || layer >= pr->n_layers) return fail("layer %lld out of range", (long long)layer);
  if (n_q_heads < 1 || n_q_heads % pr->n_kv_heads != 0)
    return fail("gqa_attention: n_q_heads %lld not divisible by n_kv_heads %lld", (long long)n_q_heads, (long long)pr->n_kv_heads);
  if (pr->n_q_heads != 0 && pr->n_q_heads != n_q_heads) return fail("proj_set_q: n_q_heads changed from %lld to %lld", (long long)pr->n_q_heads, (long long)n_q_heads);
  lorakv_ctx* ctx = pr->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  const int64_t group = n_q_heads / pr->n_kv_heads, n_q_local = group * pr->n_kv_local;
  const int64_t dq_full = n_q_heads * pr->d_head, dq = n_q_local * pr->d_head;
  const size_t one = (size_t)(pr->d_model * dq_full) * sizeof(float);
  if (pr->n_q_heads == 0) {
    pr->q_fused = pr->fused && dq % 256 == 0;
    if (pr->q_fused) LK_CUDA(cudaMalloc(&pr->wq_packed, (size_t)(pr->n_layers * pr->d_model * dq) * 2));
    else LK_CUDA(cudaMalloc(&pr->wq, (size_t)pr->n_layers * one));
    pr->n_q_heads = n_q_heads;
    pr->q_set.assign((size_t)pr->n_layers, 0);
  }
  if (pr->q_fused) {
    LK_TRY(scratch_reserve(ctx, ctx->in, one));
    float* sq = static_cast<float*>(ctx->in.ptr);
    LK_CUDA(cudaMemcpyAsync(sq, wq, one, cudaMemcpyHostToDevice, ctx->stream));
    LK_TRY(launch_pack_w(ctx, sq, dq_full, pr->kv_head_begin * group * pr->d_head, dq, pr->d_model, 0,
                         static_cast<char*>(pr->wq_packed) + (size_t)(layer * pr->d_model * dq) * 2));
  } else {
    LK_CUDA(cudaMemcpyAsync(pr->wq + (size_t)layer * (one / sizeof(float)), wq, one, cudaMemcpyHostToDevice, ctx->stream));
  }
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  pr->q_set[(size_t)layer] = 1;
  return LORAKV_OK;
}

int lorakv_proj_set_q_lora(lorakv_proj* pr, int64_t layer, int64_t agent, int64_t n_agents, int64_t rank, const float* a_q,
                           const float* b_q, double alpha) {
  if (!pr || !a_q || !b_q) return fail("null argument");
  if (pr->n_q_heads == 0) return fail("proj_set_q_lora: upload Wq first (lorakv_proj_set_q)");
  if (layer < 0 || layer >= pr->n_layers) return fail("layer %lld out of range", (long long)layer);
  if (rank < 1) return fail("LoraAdapter: rank must be >= 1, got %lld", (long long)rank);
  if (rank > 64) return fail("proj_set_q_lora: rank %lld > 64 is not supported", (long long)rank);
  if (agent < 0 || agent >= n_agents) return fail("agent index %lld out of range [0,%lld)", (long long)agent, (long long)n_agents);
  const double sc = alpha / (double)rank;
  if (!(std::isfinite(sc) && sc > 0.0)) return fail("LoraAdapter: effective scale alpha/rank must be finite and positive");
  lorakv_ctx* ctx = pr->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  const int64_t dq_full = pr->n_q_heads * pr->d_head;
  if (!pr->aq) {
    LK_CUDA(cudaMalloc(&pr->aq, (size_t)(pr->n_layers * pr->d_model * rank) * sizeof(float)));
    LK_CUDA(cudaMalloc(&pr->bq, (size_t)(pr->n_layers * n_agents * rank * dq_full) * sizeof(float)));
    pr->q_rank = rank; pr->q_agents = n_agents;
    if (pr->q_fused && rank <= 32) {
      const int64_t dq_local = (pr->n_q_heads / pr->n_kv_heads) * pr->n_kv_local * pr->d_head;
      LK_CUDA(cudaMalloc(&pr->bq_extra, (size_t)(pr->n_layers * n_agents * dq_local * 64) * 2));
    }
    pr->q_scale.assign((size_t)(pr->n_layers * n_agents), 0.f);
    pr->q_lora_set.assign((size_t)(pr->n_layers * n_agents), 0);
  }
  if (rank != pr->q_rank || n_agents != pr->q_agents) return fail("proj_set_q_lora: rank / agent count changed");
  // shared-A multi-LoRA (lora.hpp:69-73): every agent's down-projection is the same matrix, the last upload stays
  LK_CUDA(cudaMemcpyAsync(pr->aq + (size_t)(layer * pr->d_model * rank), a_q, (size_t)(pr->d_model * rank) * sizeof(float),
                          cudaMemcpyHostToDevice, ctx->stream));
  LK_CUDA(cudaMemcpyAsync(pr->bq + (size_t)((layer * n_agents + agent) * rank * dq_full), b_q, (size_t)(rank * dq_full) * sizeof(float),
                          cudaMemcpyHostToDevice, ctx->stream));
  if (pr->bq_extra) {
    const int64_t group = pr->n_q_heads / pr->n_kv_heads, dq_local = group * pr->n_kv_local * pr->d_head;
    LK_TRY(launch_pack_lora_b(ctx, pr->bq + (size_t)((layer * n_agents + agent) * rank * dq_full), dq_full,
                              pr->kv_head_begin * group * pr->d_head, dq_local, rank,
                              static_cast<char*>(pr->bq_extra) + (size_t)((layer * n_agents + agent) * dq_local * 64) * 2));
  }
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  pr->q_scale[(size_t)(layer * n_agents + agent)] = (float)sc;
  pr->q_lora_set[(size_t)(layer * n_agents + agent)] = 1;
  return LORAKV_OK;
}

int lorakv_proj_query(lorakv_proj* pr, int64_t layer, int64_t agent, int64_t pos_begin, const float* x, int64_t n_rows,
                      int64_t ld, int rope, float* q_out, int mem_kind) {
  if (!pr || !q_out) return fail("null argument");
  if (layer < 0 || layer >= pr->n_layers) return fail("layer %lld out of range", (long long)layer);
  if (pr->n_q_heads == 0 || !pr->q_set[(size_t)layer]) return fail("proj_query: Wq of layer %lld was never uploaded", (long long)layer);
  if (n_rows < 0 || pos_begin < 0) return fail("proj_query: negative row count or position");
  if (n_rows == 0) return LORAKV_OK;
  if (!x) return fail("proj_query: null rows");
  const bool lora = agent >= 0;
  if (lora) {
    if (!pr->aq || agent >= pr->q_agents) return fail("agent index %lld out of range [0,%lld)", (long long)agent, (long long)pr->q_agents);
    if (!pr->q_lora_set[(size_t)(layer * pr->q_agents + agent)]) return fail("proj_query: q adapter of layer %lld agent %lld was never uploaded", (long long)layer, (long long)agent);
  }
  const bool host = mem_kind == LORAKV_HOST;
  if (!host && mem_kind != LORAKV_DEVICE) return fail("bad mem_kind %d", mem_kind);
  lorakv_ctx* ctx = pr->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  const int64_t group = pr->n_q_heads / pr->n_kv_heads, n_q_local = group * pr->n_kv_local;
  const int64_t dq_full = pr->n_q_heads * pr->d_head, dq = n_q_local * pr->d_head;
  const int64_t col0 = pr->kv_head_begin * group * pr->d_head;
  const float* dev; int64_t dev_ld;
  LK_TRY(stage_rows(ctx, x, n_rows, pr->d_model, ld, mem_kind, &dev, &dev_ld));
  float* q_dev = q_out;
  const size_t q_bytes = (size_t)(n_rows * dq) * sizeof(float);
  if (host) { LK_TRY(scratch_reserve(ctx, ctx->out, q_bytes)); q_dev = static_cast<float*>(ctx->out.ptr); }
  const int64_t rank = lora ? pr->q_rank : 0;
  const float* aq = lora ? pr->aq + (size_t)(layer * pr->d_model * rank) : nullptr;
  const float* bq = lora ? pr->bq + (size_t)((layer * pr->q_agents + agent) * rank * dq_full) : nullptr;
  const float sc = lora ? pr->q_scale[(size_t)(layer * pr->q_agents + agent)] : 0.f;
  const bool fused = pr->q_fused && (dev_ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(dev) & 15) == 0);
  if (!fused && pr->q_fused) return fail("proj_query: rows must be 16-byte aligned with a stride that is a multiple of 4");
  float* down = nullptr;
  const bool small = fused && ctx->policy != 1 && rows_project_supported(n_rows, pr->d_model, rank);
  if (fused && lora) {
    LK_TRY(scratch_reserve(ctx, ctx->proj, (size_t)(n_rows * rank) * sizeof(float)));
    down = static_cast<float*>(ctx->proj.ptr);
    if (small) LK_TRY(launch_rows_xa(ctx, aq, pr->d_model, rank, dev, n_rows, dev_ld, down));
    else LK_TRY(launch_xa_dense(ctx, aq, pr->d_model, rank, dev, n_rows, dev_ld, down));
  }
  const void* packed = fused ? static_cast<const char*>(pr->wq_packed) + (size_t)(layer * pr->d_model * dq) * 2 : nullptr;
  if (small) {
    LK_TRY(launch_rows_q_project(ctx, packed, pr->d_model, dq, pr->d_head, down, bq ? bq + col0 : nullptr, dq_full, rank, sc, pos_begin,
                                 dev, n_rows, dev_ld, rope != 0, q_dev));
    if (host) {
      LK_CUDA(cudaMemcpyAsync(q_out, q_dev, q_bytes, cudaMemcpyDeviceToHost, ctx->stream));
      LK_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return LORAKV_OK;
  }
  const float* wq = fused ? nullptr : pr->wq + (size_t)(layer * pr->d_model * dq_full);
  // the packed matrix already holds only this shard's columns: its column origin is 0, B_q keeps the full width
  const void* bq_extra = (fused && lora && pr->bq_extra) ? static_cast<const char*>(pr->bq_extra) + (size_t)((layer * pr->q_agents + agent) * dq * 64) * 2
                                                         : nullptr;
  LK_TRY(launch_q_project(ctx, fused, packed, wq, dq_full, col0, pr->d_model, dq, pr->d_head, down, aq, bq, dq_full, rank, sc,
                          pos_begin, dev, n_rows, dev_ld, rope != 0, q_dev, bq_extra));
  if (host) {
    LK_CUDA(cudaMemcpyAsync(q_out, q_dev, q_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return LORAKV_OK;
}

static int append_kv_project_impl(lorakv_pool* pool, const lorakv_proj* pr, const lorakv_adapters* merge, int64_t layer, int64_t agent,
                                  int64_t row_begin, const float* x, int64_t n_rows, int64_t ld, int mem_kind, int rope,
                                  int64_t* appended);

int lorakv_pool_append_kv_project(lorakv_pool* pool, const lorakv_proj* pr, int64_t layer, int64_t agent, int64_t row_begin,
                                  const float* x, int64_t n_rows, int64_t ld, int mem_kind, int rope, int64_t* appended) {
  return append_kv_project_impl(pool, pr, nullptr, layer, agent, row_begin, x, n_rows, ld, mem_kind, rope, appended);
}

int lorakv_pool_append_kv_project_full(lorakv_pool* pool, const lorakv_proj* pr, const lorakv_adapters* ad, int64_t layer,
                                       int64_t agent, int64_t row_begin, const float* x, int64_t n_rows, int64_t ld,
                                       int mem_kind, int rope, int64_t* appended) {
  if (!ad) return fail("append_kv_project_full: null adapter table");
  return append_kv_project_impl(pool, pr, ad, layer, agent, row_begin, x, n_rows, ld, mem_kind, rope, appended);
}

static int append_kv_project_impl(lorakv_pool* pool, const lorakv_proj* pr, const lorakv_adapters* merge, int64_t layer, int64_t agent,
                                  int64_t row_begin, const float* x, int64_t n_rows, int64_t ld, int mem_kind, int rope,
                                  int64_t* appended) {
  if (!pool || !pr) return fail("null argument");
  if (appended) *appended = 0;
  int64_t set; bool none;
  LK_TRY(resolve(pool, LORAKV_KEY, layer, agent, &set, &none));
  if (pr->d_model != pool->dims.d_model || pr->n_kv_heads != pool->dims.n_kv_heads || pr->d_head != pool->dims.d_head ||
      pr->kv_head_begin != pool->dims.kv_head_begin || pr->n_kv_local != pool->n_kv_local || pr->dtype != pool->dims.dtype ||
      layer >= pr->n_layers)
    return fail("append_kv_project: projection weights do not match the pool (d_model %lld vs %lld, d_kv %lld vs %lld)",
                (long long)pr->d_model, (long long)pool->dims.d_model, (long long)(pr->n_kv_heads * pr->d_head),
                (long long)(pool->dims.n_kv_heads * pool->dims.d_head));
  if (!pr->set[(size_t)layer]) return fail("append_kv_project: Wk / Wv of layer %lld were never uploaded", (long long)layer);
  if (n_rows < 0) return fail("append: negative row count");
  int64_t& have_k = pool->key_rows[(size_t)set][(size_t)layer];
  int64_t& have_v = pool->value_rows[(size_t)set][(size_t)layer];
  int64_t skip_k, add_k, skip_v, add_v;
  LK_TRY(fww("key", have_k, row_begin, n_rows, &skip_k, &add_k));
  LK_TRY(fww("value", have_v, row_begin, n_rows, &skip_v, &add_v));
  const int64_t add = std::max(add_k, add_v);
  if (add == 0) return LORAKV_OK;
  if (!x) return fail("append: null rows");
  const int64_t skip = n_rows - add;
  lorakv_ctx* ctx = pool->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  LK_TRY(ensure_pages(pool, pool->kv_space, set, row_begin + n_rows));
  const float* dev; int64_t dev_ld;
  LK_TRY(stage_rows(ctx, x + skip * ld, add, pool->dims.d_model, ld, mem_kind, &dev, &dev_ld));
  const size_t w_off = (size_t)(layer * pr->d_model * pr->n_kv_heads * pr->d_head);
  const void* packed = pr->fused ? static_cast<const char*>(pr->packed) +
                                       (size_t)(layer * kv_project_packed_elems(pr->d_model, pr->n_kv_local, pr->d_head)) * 2
                                 : nullptr;
  // "full values" (engine.hpp:385-393): the value rows carry the agent's LoRA contribution
  const float *av = nullptr, *bv = nullptr, *down = nullptr;
  int64_t rank = 0; float v_scale = 0.f;
  if (merge) {
    if (merge->rank < 1 || merge->d_model != pr->d_model || merge->n_kv_local != pr->n_kv_local || merge->d_head != pr->d_head ||
        layer >= merge->n_layers)
      return fail("append_kv_project_full: adapter table does not match the projection (rank %lld)", (long long)merge->rank);
    if (agent < 0 || agent >= merge->n_agents) return fail("agent index %lld out of range [0,%lld)", (long long)agent, (long long)merge->n_agents);
    const bool has_a = merge->a_set[(size_t)layer] ||
                       (merge->a_agent && merge->a_agent_set[(size_t)(layer * merge->n_agents + agent)]);
    if (!has_a || !merge->b_set[(size_t)(layer * merge->n_agents + agent)])
      return fail("append_kv_project_full: A / B of layer %lld agent %lld were never uploaded", (long long)layer, (long long)agent);
    rank = merge->rank;
    if (rank > 64) return fail("append_kv_project_full: rank %lld > 64 is not supported", (long long)rank);
    // the agent's own down-projection when one was uploaded (engine.hpp:375-379 uses v_lora->adapter(agent).a: NonShared
    // and FullShared adapters need not share A), else the layer's shared A
    const bool own_a = merge->a_agent && merge->a_agent_set[(size_t)(layer * merge->n_agents + agent)];
    av = own_a ? merge->a_agent + (size_t)(layer * merge->n_agents + agent) * (size_t)(merge->d_model * rank)
               : merge->a + layer * merge->d_model * rank;
    bv = merge->b + ((layer * merge->n_agents + agent) * rank) * (merge->n_kv_local * merge->d_head);
    v_scale = merge->scale_host[(size_t)(layer * merge->n_agents + agent)];
    if (pr->fused) {
      LK_TRY(scratch_reserve(ctx, ctx->proj, (size_t)(add * rank) * sizeof(float)));
      float* dn = static_cast<float*>(ctx->proj.ptr);
      if (rows_project_supported(add, pr->d_model, rank)) LK_TRY(launch_rows_xa(ctx, av, pr->d_model, rank, dev, add, dev_ld, dn));
      else LK_TRY(launch_xa_dense(ctx, av, pr->d_model, rank, dev, add, dev_ld, dn));
      down = dn;
    }
  }
  if (pr->fused && ctx->policy != 1 && rows_project_supported(add, pr->d_model, rank)) {
    // a decode step's handful of rows: weight-streaming GEMVs over all SMs instead of one 128-row tcgen05 tile
    LK_TRY(launch_rows_kv_project(pool, packed, layer, set, row_begin + skip, row_begin + skip_k, row_begin + skip_v, dev, add, dev_ld,
                                  rope != 0, down, bv, rank, v_scale));
    if (mem_kind == LORAKV_HOST) LK_CUDA(cudaStreamSynchronize(ctx->stream));
    else LK_TRY(note_pages_written(pool, row_begin + skip));
    have_k += add_k; have_v += add_v;
    if (appended) *appended = add;
    return LORAKV_OK;
  }
  LK_TRY(launch_kv_project(pool, packed, pr->fused ? nullptr : pr->wk + w_off, pr->fused ? nullptr : pr->wv + w_off, layer, set,
                           row_begin + skip, row_begin + skip_k, row_begin + skip_v, dev, add, dev_ld, rope != 0, down, av, bv, rank,
                           v_scale));
  if (mem_kind == LORAKV_HOST) LK_CUDA(cudaStreamSynchronize(ctx->stream));
  else LK_TRY(note_pages_written(pool, row_begin + skip));
  have_k += add_k; have_v += add_v;
  if (appended) *appended = add;
  return LORAKV_OK;
}

int lorakv_pool_rows(const lorakv_pool* pool, int which, int64_t layer, int64_t agent, int64_t* rows) {
  if (!pool || !rows) return fail("null argument");
  int64_t set; bool none;
  LK_TRY(resolve(pool, which, layer, agent, &set, &none));
  if (none) {   // lr_view on a scheme without LR: L x 0 with L = key rows (kvcache.hpp:323)
    LK_TRY(resolve(pool, LORAKV_KEY, layer, agent, &set, &none));
    *rows = pool->key_rows[(size_t)set][(size_t)layer];
    return LORAKV_OK;
  }
  *rows = row_counter(const_cast<lorakv_pool*>(pool), which, set, layer);
  return LORAKV_OK;
}

int lorakv_pool_read(const lorakv_pool* pool, int which, int64_t layer, int64_t agent,
                     int64_t row_begin, int64_t n_rows, float* out) {
  return pool_read_impl(pool, which, layer, agent, row_begin, n_rows, out);
}

int lorakv_pool_bytes(const lorakv_pool* pool, uint64_t out[4]) {
  if (!pool || !out) return fail("null argument");
  // elements x sizeof(T), exactly as CacheBytes counts them (kvcache.hpp:330-344): logical rows,
  // not page capacity; a kv-head shard counts its own columns
  const uint64_t sz = (uint64_t)pool->elem, dkv = (uint64_t)pool->d_kv_local(), r = (uint64_t)pool->dims.rank;
  uint64_t k = 0, v = 0, l = 0;
  for (const auto& per : pool->key_rows) for (int64_t n : per) k += (uint64_t)n * dkv;
  for (const auto& per : pool->value_rows) for (int64_t n : per) v += (uint64_t)n * dkv;
  if (pool->lr_sets() > 0)
    for (const auto& per : pool->lr_rows) for (int64_t n : per) l += (uint64_t)n * r;
  for (int64_t n : pool->lk_rows) l += (uint64_t)n * (uint64_t)pool->dims.rank_k;     // key-side low-rank rows count as low-rank bytes
  out[0] = k * sz; out[1] = v * sz; out[2] = l * sz;
  out[3] = (uint64_t)pool->hidden_rows * (uint64_t)pool->dims.d_model * sz;
  return LORAKV_OK;
}
uint64_t lorakv_pool_allocated_elements(const lorakv_pool* pool) {
  uint64_t b[4];
  if (lorakv_pool_bytes(pool, b) != LORAKV_OK) return 0;
  return (b[0] + b[1] + b[2] + b[3]) / (uint64_t)pool->elem;
}
uint64_t lorakv_pool_reserved_bytes(const lorakv_pool* pool) { return pool ? pool->reserved_bytes : 0; }

int lorakv_pool_page_table(const lorakv_pool* pool, int which, int64_t agent, int32_t* out, int64_t cap,
                           int64_t* n_pages) {
  if (!pool) return fail("null pool");
  int64_t set; bool none;
  LK_TRY(resolve(pool, which, 0, agent, &set, &none));
  if (none) { if (n_pages) *n_pages = 0; return LORAKV_OK; }
  const auto& tab = (which == LORAKV_LR ? pool->lr_space : which == LORAKV_LK ? pool->lk_space : pool->kv_space).table[(size_t)set];
  if (n_pages) *n_pages = (int64_t)tab.size();
  for (int64_t i = 0; i < cap && i < (int64_t)tab.size(); ++i) out[i] = tab[(size_t)i];
  return LORAKV_OK;
}

// ---- adapters ---------------------------------------------------------------------------------------
int lorakv_adapters_create(lorakv_ctx* ctx, int64_t n_layers, int64_t n_agents, int64_t d_model,
                           int64_t rank, int64_t n_kv_heads, int64_t d_head, int64_t kv_head_begin,
                           int64_t n_kv_local, int dtype, lorakv_adapters** out) {
  if (!ctx || !out) return fail("adapters_create: null argument");
  *out = nullptr;
  if (n_layers < 1 || n_agents < 1 || d_model < 1 || n_kv_heads < 1 || d_head < 1) return fail("adapters: invalid dims");
  if (rank < 1) return fail("LoraAdapter: rank must be >= 1, got %lld", (long long)rank);
  if (rank > std::min(d_model, n_kv_heads * d_head))
    return fail("LoraAdapter: rank %lld exceeds min(d_in, d_out)", (long long)rank);
  if (n_kv_local <= 0) n_kv_local = n_kv_heads - kv_head_begin;
  if (kv_head_begin < 0 || kv_head_begin + n_kv_local > n_kv_heads) return fail("adapters: bad kv head shard");
  lorakv_adapters* ad = new (std::nothrow) lorakv_adapters();
  if (!ad) return fail("adapters_create: out of host memory");
  ad->ctx = ctx; ad->n_layers = n_layers; ad->n_agents = n_agents; ad->d_model = d_model; ad->rank = rank;
  ad->n_kv_heads = n_kv_heads; ad->d_head = d_head; ad->kv_head_begin = kv_head_begin; ad->n_kv_local = n_kv_local;
  ad->dtype = dtype;
  ad->scale_host.assign((size_t)(n_layers * n_agents), 0.f);
  ad->a_set.assign((size_t)n_layers, 0);
  ad->b_set.assign((size_t)(n_layers * n_agents), 0);
  cudaSetDevice(ctx->device);
  const size_t a_bytes = (size_t)(n_layers * d_model * rank) * sizeof(float);
  const size_t b_bytes = (size_t)(n_layers * n_agents * rank * n_kv_local * d_head) * sizeof(float);
  cudaError_t e = cudaMalloc(&ad->a, a_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&ad->b, b_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&ad->scale, (size_t)(n_layers * n_agents) * sizeof(float));
  if (e == cudaSuccess) e = cudaMemsetAsync(ad->a, 0, a_bytes, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(ad->b, 0, b_bytes, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(ad->scale, 0, (size_t)(n_layers * n_agents) * sizeof(float), ctx->stream);
  if (e != cudaSuccess) {
    lorakv_adapters_destroy(ad);
    return fail("adapters_create: %s", cudaGetErrorString(e));
  }
  *out = ad;
  return LORAKV_OK;
}

void lorakv_adapters_destroy(lorakv_adapters* ad) {
  if (!ad) return;
  cudaSetDevice(ad->ctx->device);
  cudaStreamSynchronize(ad->ctx->stream);
  if (ad->a) cudaFree(ad->a);
  if (ad->a_agent) cudaFree(ad->a_agent);
  if (ad->b) cudaFree(ad->b);
  if (ad->scale) cudaFree(ad->scale);
  for (float* q : {ad->a_k, ad->b_k, ad->scale_k})
    if (q) cudaFree(q);
  delete ad;
}

int lorakv_adapters_set_a(lorakv_adapters* ad, int64_t layer, const float* a) {
  if (!ad || !a) return fail("null argument");
  if (layer < 0 || layer >= ad->n_layers) return fail("layer %lld out of range", (long long)layer);
  LK_CUDA(cudaSetDevice(ad->ctx->device));
  LK_CUDA(cudaMemcpyAsync(ad->a + layer * ad->d_model * ad->rank, a, (size_t)(ad->d_model * ad->rank) * sizeof(float),
                          cudaMemcpyHostToDevice, ad->ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ad->ctx->stream));
  ad->a_set[(size_t)layer] = 1;
  return LORAKV_OK;
}

int lorakv_adapters_set_a_agent(lorakv_adapters* ad, int64_t layer, int64_t agent, const float* a) {
  if (!ad || !a) return fail("null argument");
  if (layer < 0 || layer >= ad->n_layers) return fail("layer %lld out of range", (long long)layer);
  if (agent < 0 || agent >= ad->n_agents)
    return fail("agent index %lld out of range [0,%lld)", (long long)agent, (long long)ad->n_agents);
  LK_CUDA(cudaSetDevice(ad->ctx->device));
  const size_t one = (size_t)(ad->d_model * ad->rank);
  if (!ad->a_agent) {
    LK_CUDA(cudaMalloc(&ad->a_agent, (size_t)(ad->n_layers * ad->n_agents) * one * sizeof(float)));
    ad->a_agent_set.assign((size_t)(ad->n_layers * ad->n_agents), 0);
  }
  LK_CUDA(cudaMemcpyAsync(ad->a_agent + (size_t)(layer * ad->n_agents + agent) * one, a, one * sizeof(float),
                          cudaMemcpyHostToDevice, ad->ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ad->ctx->stream));
  ad->a_agent_set[(size_t)(layer * ad->n_agents + agent)] = 1;
  return LORAKV_OK;
}

int lorakv_adapters_set_b(lorakv_adapters* ad, int64_t layer, int64_t agent, const float* b, double alpha) {
  if (!ad || !b) return fail("null argument");
  if (layer < 0 || layer >= ad->n_layers) return fail("layer %lld out of range", (long long)layer);
  if (agent < 0 || agent >= ad->n_agents)
    return fail("agent index %lld out of range [0,%lld)", (long long)agent, (long long)ad->n_agents);
  const double s = alpha / (double)ad->rank;
  if (!(std::isfinite(s) && s > 0.0)) return fail("LoraAdapter: effective scale alpha/rank must be finite and positive");
  LK_CUDA(cudaSetDevice(ad->ctx->device));
  const int64_t dkv_full = ad->n_kv_heads * ad->d_head, dkv = ad->n_kv_local * ad->d_head;
  float* dst = ad->b + ((layer * ad->n_agents + agent) * ad->rank) * dkv;
  LK_CUDA(cudaMemcpy2DAsync(dst, dkv * sizeof(float), b + ad->kv_head_begin * ad->d_head, dkv_full * sizeof(float),
                            dkv * sizeof(float), ad->rank, cudaMemcpyHostToDevice, ad->ctx->stream));
  const float sf = (float)s;
  ad->scale_host[(size_t)(layer * ad->n_agents + agent)] = sf;
  LK_CUDA(cudaMemcpyAsync(ad->scale + layer * ad->n_agents + agent, &ad->scale_host[(size_t)(layer * ad->n_agents + agent)],
                          sizeof(float), cudaMemcpyHostToDevice, ad->ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ad->ctx->stream));
  ad->b_set[(size_t)(layer * ad->n_agents + agent)] = 1;
  return LORAKV_OK;
}

// ---- key-side adapter tables (extension; kernels.hpp: KeyLowRank) ------------------------------------------------------
int lorakv_adapters_enable_key(lorakv_adapters* ad, int64_t rank_k) {
  if (!ad) return fail("null argument");
  if (rank_k < 1 || rank_k > 64) return fail("LoraAdapter: key rank must be in [1,64], got %lld", (long long)rank_k);
  if (ad->rank_k == rank_k) return LORAKV_OK;
  if (ad->rank_k != 0) return fail("adapters: the key-side tables were already created with rank %lld", (long long)ad->rank_k);
  LK_CUDA(cudaSetDevice(ad->ctx->device));
  const size_t a_bytes = (size_t)(ad->n_layers * ad->d_model * rank_k) * sizeof(float);
  const size_t b_bytes = (size_t)(ad->n_layers * ad->n_agents * rank_k * ad->n_kv_local * ad->d_head) * sizeof(float);
  LK_CUDA(cudaMalloc(&ad->a_k, a_bytes));
  LK_CUDA(cudaMalloc(&ad->b_k, b_bytes));
  LK_CUDA(cudaMalloc(&ad->scale_k, (size_t)(ad->n_layers * ad->n_agents) * sizeof(float)));
  LK_CUDA(cudaMemsetAsync(ad->a_k, 0, a_bytes, ad->ctx->stream));
  LK_CUDA(cudaMemsetAsync(ad->b_k, 0, b_bytes, ad->ctx->stream));
  LK_CUDA(cudaMemsetAsync(ad->scale_k, 0, (size_t)(ad->n_layers * ad->n_agents) * sizeof(float), ad->ctx->stream));
  ad->rank_k = rank_k;
  ad->scale_k_host.assign((size_t)(ad->n_layers * ad->n_agents), 0.f);
  ad->a_k_set.assign((size_t)ad->n_layers, 0);
  ad->b_k_set.assign((size_t)(ad->n_layers * ad->n_agents), 0);
  return LORAKV_OK;
}

int lorakv_adapters_set_a_k(lorakv_adapters* ad, int64_t layer, const float* a_k) {
  if (!ad || !a_k) return fail("null argument");
  if (ad->rank_k == 0) return fail("adapters: no key-side tables (lorakv_adapters_enable_key)");
  if (layer < 0 || layer >= ad->n_layers) return fail("layer %lld out of range", (long long)layer);
  LK_CUDA(cudaSetDevice(ad->ctx->device));
  LK_CUDA(cudaMemcpyAsync(ad->a_k + layer * ad->d_model * ad->rank_k, a_k, (size_t)(ad->d_model * ad->rank_k) * sizeof(float),
                          cudaMemcpyHostToDevice, ad->ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ad->ctx->stream));
  ad->a_k_set[(size_t)layer] = 1;
  return LORAKV_OK;
}

int lorakv_adapters_set_b_k(lorakv_adapters* ad, int64_t layer, int64_t agent, const float* b_k, double alpha_k) {
  if (!ad || !b_k) return fail("null argument");
  if (ad->rank_k == 0) return fail("adapters: no key-side tables (lorakv_adapters_enable_key)");
  if (layer < 0 || layer >= ad->n_layers) return fail("layer %lld out of range", (long long)layer);
  if (agent < 0 || agent >= ad->n_agents)
    return fail("agent index %lld out of range [0,%lld)", (long long)agent, (long long)ad->n_agents);
  const double s = alpha_k / (double)ad->rank_k;
  if (!(std::isfinite(s) && s > 0.0)) return fail("LoraAdapter: effective scale alpha/rank must be finite and positive");
  LK_CUDA(cudaSetDevice(ad->ctx->device));
  const int64_t dkv_full = ad->n_kv_heads * ad->d_head, dkv = ad->n_kv_local * ad->d_head;
  const size_t la = (size_t)(layer * ad->n_agents + agent);
  float* dst = ad->b_k + (la * ad->rank_k) * dkv;
  LK_CUDA(cudaMemcpy2DAsync(dst, dkv * sizeof(float), b_k + ad->kv_head_begin * ad->d_head, dkv_full * sizeof(float),
                            dkv * sizeof(float), ad->rank_k, cudaMemcpyHostToDevice, ad->ctx->stream));
  ad->scale_k_host[la] = (float)s;
  LK_CUDA(cudaMemcpyAsync(ad->scale_k + la, &ad->scale_k_host[la], sizeof(float), cudaMemcpyHostToDevice, ad->ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ad->ctx->stream));
  ad->b_k_set[la] = 1;
  return LORAKV_OK;
}

int lorakv_pool_append_lk_project(lorakv_pool* pool, const lorakv_adapters* ad, int64_t layer, int64_t row_begin, const float* x,
                                  int64_t n_rows, int64_t ld, int mem_kind, int64_t* appended) {
  if (!pool || !ad) return fail("null argument");
  if (appended) *appended = 0;
  if (pool->dims.dtype == LORAKV_F64) return fail("lk_append_project: fp64 pools are storage only");
  int64_t set; bool none;
  LK_TRY(resolve(pool, LORAKV_LK, layer, 0, &set, &none));
  if (ad->rank_k != pool->dims.rank_k || ad->d_model != pool->dims.d_model || layer >= ad->n_layers)
    return fail("lk_append_project: adapter table does not match the pool (key rank %lld vs %lld)", (long long)ad->rank_k,
                (long long)pool->dims.rank_k);
  if (!ad->a_k_set[(size_t)layer]) return fail("lk_append_project: A_k of layer %lld was never uploaded", (long long)layer);
  if (n_rows < 0) return fail("append: negative row count");
  int64_t& have = pool->lk_rows[(size_t)layer];
  int64_t skip, add;
  LK_TRY(fww("key-lr", have, row_begin, n_rows, &skip, &add));
  if (add == 0) return LORAKV_OK;
  if (!x) return fail("append: null rows");
  lorakv_ctx* ctx = pool->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  LK_TRY(ensure_pages(pool, pool->lk_space, 0, have + add));
  const float* dev; int64_t dev_ld;
  LK_TRY(stage_rows(ctx, x + skip * ld, add, pool->dims.d_model, ld, mem_kind, &dev, &dev_ld));
  LK_TRY(launch_lr_project(pool, ad->a_k + layer * ad->d_model * ad->rank_k, ad->d_model, ad->rank_k, layer, 0, have, dev, add, dev_ld,
                           LORAKV_LK));
  if (mem_kind == LORAKV_HOST) LK_CUDA(cudaStreamSynchronize(ctx->stream));
  else LK_TRY(note_pages_written(pool, have));
  have += add;
  if (appended) *appended = add;
  return LORAKV_OK;
}

// ---- fast paths ---------------------------------------------------------------------------------------
static int check_adapters(const lorakv_pool* pool, const lorakv_adapters* ad) {
  if (pool->r_pad == 0) return LORAKV_OK;
  if (!ad) return fail("attention: the pool keeps a rank-%lld cache but no adapter tables were given", (long long)pool->dims.rank);
  if (ad->rank != pool->dims.rank || ad->n_layers != pool->dims.n_layers || ad->n_kv_local != pool->n_kv_local ||
      ad->kv_head_begin != pool->dims.kv_head_begin || ad->d_head != pool->dims.d_head)
    return fail("attention: adapter tables do not match the pool");
  return LORAKV_OK;
}

// rows every buffer the call reads has materialised (K, V and -- when present -- LR)
// validate_attention_inputs (attention.hpp:58-76) rejects k, v_base and v_lr views of different row counts; so does this
// (a cache that lags -- e.g. a BaseShared agent whose LR prefill is pending -- is an error, never a silently shorter context)
static int visible_rows(const lorakv_pool* pool, int64_t layer, int64_t kv_set, int64_t lr_set, int64_t* L, bool with_lr = true) {
  const int64_t nk = pool->key_rows[(size_t)kv_set][(size_t)layer], nv = pool->value_rows[(size_t)kv_set][(size_t)layer];
  if (nk != nv) return fail("attention: k is %lldx%lld but v_base has %lld rows (layer %lld)", (long long)nk,
                            (long long)pool->d_kv_local(), (long long)nv, (long long)layer);
  if (pool->r_pad > 0 && with_lr) {     // (a batch over per-agent low-rank caches checks every entry's own cache instead)
    const int64_t nl = pool->lr_rows[(size_t)lr_set][(size_t)layer];
    if (nl != nk) return fail("attention: v_lr has %lld rows, k has %lld (layer %lld; the low-rank cache of this agent lags: its LR prefill "
                              "is pending)", (long long)nl, (long long)nk, (long long)layer);
  }
  *L = nk;
  return LORAKV_OK;
}

static int run_paged(lorakv_pool* pool, const lorakv_adapters* ad, int64_t layer_begin, int64_t layer_end,
                     int64_t kv_set, int64_t lr_set, const int32_t* agent_ids, int64_t n_batch,
                     int64_t rows_per_entry, int64_t query_offset, int64_t n_q_heads, const float* q,
                     float* out, int mem_kind, const lk::PeerOut* peers = nullptr, bool per_entry_lr = false) {
  lorakv_ctx* ctx = pool->ctx;
  LK_CUDA(cudaSetDevice(ctx->device));
  if (pool->dims.dtype == LORAKV_F64)
    return fail("attention: fp64 pages are storage only; attend over the views with gqa_attention<double> (lorakv_gqa_forward_f64), "
                "as the reference's step() does");
  if (layer_begin < 0 || layer_end > pool->dims.n_layers || layer_begin >= layer_end) return fail("attention: bad layer range");
  if (n_q_heads < 1 || n_q_heads % pool->dims.n_kv_heads != 0)
    return fail("gqa_attention: n_q_heads %lld not divisible by n_kv_heads %lld", (long long)n_q_heads, (long long)pool->dims.n_kv_heads);
  LK_TRY(check_adapters(pool, ad));
  const int64_t group = n_q_heads / pool->dims.n_kv_heads;
  const int64_t n_q_local = group * pool->n_kv_local;
  int64_t L = -1;
  for (int64_t l = layer_begin; l < layer_end; ++l) {
    int64_t Ll;
    LK_TRY(visible_rows(pool, l, kv_set, lr_set, &Ll, !per_entry_lr));
    if (per_entry_lr) {   // every entry reads its own agent's low-rank cache: all of them must have caught up
      Ll = std::min(pool->key_rows[(size_t)kv_set][(size_t)l], pool->value_rows[(size_t)kv_set][(size_t)l]);
      for (int64_t i = 0; i < n_batch; ++i) {
        const int64_t a = agent_ids ? agent_ids[i] : 0;
        if (a < 0 || a >= pool->dims.n_agents) return fail("unknown agent %lld", (long long)a);
        if (pool->lr_rows[(size_t)a][(size_t)l] < Ll)
          return fail("fla_decode_batched: the per-agent low-rank cache of agent %lld holds %lld of %lld rows on layer %lld (its LR prefill "
                      "is pending)", (long long)a, (long long)pool->lr_rows[(size_t)a][(size_t)l], (long long)Ll, (long long)l);
      }
    }
    if (L >= 0 && Ll != L) return fail("attention: layers %lld..%lld hold different row counts", (long long)layer_begin, (long long)layer_end);
    L = Ll;
  }
  if (query_offset < 0 || query_offset + rows_per_entry > L)
    return fail("attention: query_offset %lld with L_c %lld exceeds L %lld", (long long)query_offset,
                (long long)rows_per_entry, (long long)L);
  const int64_t n_layers = layer_end - layer_begin;
  const int64_t n_elems = n_layers * n_batch * rows_per_entry * n_q_local * pool->dims.d_head;
  if (n_elems == 0) return LORAKV_OK;

  // agent ids -> device: staged once per distinct list (stage_agent_ids), no copy when the batch repeats
  std::vector<int32_t> ids_host((size_t)n_batch);
  for (int64_t i = 0; i < n_batch; ++i) {
    const int32_t a = agent_ids ? agent_ids[i] : 0;
    if (a < 0 || a >= pool->dims.n_agents) return fail("unknown agent %d", a);
    if (ad && pool->r_pad > 0)
      for (int64_t l = layer_begin; l < layer_end; ++l)
        if (!ad->b_set[(size_t)(l * ad->n_agents + a)]) return fail("attention: B of layer %lld agent %d was never uploaded", (long long)l, a);
    ids_host[(size_t)i] = a;
  }
  const size_t q_bytes = (size_t)n_elems * sizeof(float);
  const bool host = mem_kind == LORAKV_HOST;
  if (!host && mem_kind != LORAKV_DEVICE) return fail("bad mem_kind %d", mem_kind);
  // with a peer gather the rows go to the gather buffers; the local slab only serves the paths without a merge epilogue
  const bool local_slab = host || peers;
  if (local_slab) LK_TRY(scratch_reserve(ctx, ctx->out, 2 * ((q_bytes + 255) / 256 * 256)));
  char* base = static_cast<char*>(ctx->out.ptr);
  const size_t ids_bytes = 0;
  const int32_t* ids_dev = nullptr;
  LK_TRY(stage_agent_ids(ctx, ids_host.data(), n_batch, &ids_dev));
  const float* q_dev = q;
  float* out_dev = out;
  if (local_slab) out_dev = reinterpret_cast<float*>(base + ids_bytes + (q_bytes + 255) / 256 * 256);
  if (host) {
    float* qd = reinterpret_cast<float*>(base + ids_bytes);
    LK_CUDA(cudaMemcpyAsync(qd, q, q_bytes, cudaMemcpyHostToDevice, ctx->stream));
    q_dev = qd;
  }

  // key-side low-rank term: every layer's L_k must have caught up, the agents' B_k must be there; the queries are projected
  // through B_k once (r_k numbers per row and head) before the attention kernel
  if (pool->rk_pad > 0) {
    if (!ad || ad->rank_k != pool->dims.rank_k)
      return fail("attention: the pool keeps a rank-%lld key-side cache but the adapter tables carry key rank %lld", (long long)pool->dims.rank_k,
                  (long long)(ad ? ad->rank_k : 0));
    for (int64_t l = layer_begin; l < layer_end; ++l) {
      if (pool->lk_rows[(size_t)l] != L)
        return fail("attention: l_k has %lld rows, k has %lld (layer %lld)", (long long)pool->lk_rows[(size_t)l], (long long)L, (long long)l);
      for (int64_t i = 0; i < n_batch; ++i)
        if (!ad->b_k_set[(size_t)(l * ad->n_agents + ids_host[(size_t)i])])
          return fail("attention: B_k of layer %lld agent %d was never uploaded", (long long)l, ids_host[(size_t)i]);
    }
  }

  PagedAttnCall call;
  call.pool = pool; call.adapters = ad; call.layer_begin = layer_begin; call.layer_end = layer_end;
  call.kv_set = kv_set; call.lr_set = lr_set; call.agent_ids_dev = ids_dev; call.n_batch = n_batch;
  call.rows_per_entry = rows_per_entry; call.query_offset = query_offset; call.n_q_local = n_q_local;
  call.L = L; call.q_dev = q_dev; call.out_dev = out_dev;
  call.agent_host = ids_host[0];
  call.peers = peers;
  call.per_entry_lr = per_entry_lr;
  if (pool->rk_pad > 0) {
    LK_TRY(scratch_reserve(ctx, ctx->qk, (size_t)(n_layers * n_batch * rows_per_entry * n_q_local * pool->rk_pad) * sizeof(float)));
    LK_TRY(launch_qk_project(call, static_cast<float*>(ctx->qk.ptr)));
    call.qk_dev = static_cast<const float*>(ctx->qk.ptr);
  }
  bool rows_at_peers = false;    // the decode kernels' merge epilogue stores straight into the gather buffers
  if (per_entry_lr) {
    if (ctx->policy == 1 || !decode_tma_per_entry_lr_supported(call))
      return fail("fla_decode_batched: scheme %s keeps per-agent caches; this shape has no batched kernel, batch one agent per call",
                  kSchemeName[pool->dims.scheme]);
    LK_TRY(launch_decode_tma(call));
    rows_at_peers = true;
  } else if (ctx->policy == 0 && decode_umma_supported(call)) { LK_TRY(launch_decode_umma(call)); rows_at_peers = true; }
  else if (ctx->policy != 1 && decode_tma_supported(call)) { LK_TRY(launch_decode_tma(call)); rows_at_peers = true; }
  else if (ctx->policy != 1 && decode_f32_supported(call)) { LK_TRY(launch_decode_f32(call)); rows_at_peers = true; }
  else if (ctx->policy != 1 && prefill_umma_supported(call)) LK_TRY(launch_prefill_umma(call));
  else if (ctx->policy == 0 && prefill_split_supported(call)) LK_TRY(launch_prefill_split(call));
  else if (ctx->policy != 1 && prefill_f32_supported(call)) LK_TRY(launch_prefill_f32(call));
  else LK_TRY(launch_paged_simt(call));
  if (peers) {
    if (!rows_at_peers)
      LK_TRY(launch_peer_scatter(ctx, out_dev, n_layers * n_batch * rows_per_entry, n_q_local, pool->dims.d_head, *peers));
    return LORAKV_OK;      // the caller publishes the step and reads the gathered rows
  }

  if (host) {
    LK_CUDA(cudaMemcpyAsync(out, out_dev, q_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return LORAKV_OK;
}

int lorakv_fla_decode_batched(lorakv_pool* pool, const lorakv_adapters* ad, int64_t layer_begin,
                              int64_t layer_end, const int32_t* agent_ids, int64_t n_batch,
                              int64_t n_q_heads, const float* q, float* out, int mem_kind) {
  if (!pool || !q || !out) return fail("fla_decode_batched: null argument");
  if (n_batch < 1) return fail("fla_decode_batched: empty batch");
  // per-agent caches (NonShared K/V, BaseShared LR) can only serve one agent per launch
  int64_t kv_set = 0, lr_set = 0;
  const bool per_agent = pool->dims.scheme == LORAKV_NONSHARED || (pool->dims.scheme == LORAKV_BASESHARED && pool->r_pad > 0);
  bool per_entry_lr = false;
  if (per_agent) {
    bool mixed = false;
    for (int64_t i = 1; i < n_batch; ++i)
      if (agent_ids && agent_ids[i] != agent_ids[0]) mixed = true;
    // BaseShared shares K / V_base: a batch of different agents still streams them once, every entry reading its own
    // agent's V_lr page set (fla_decode_tma, PA).  NonShared has nothing to share between agents.
    if (mixed && pool->dims.scheme == LORAKV_NONSHARED)
      return fail("fla_decode_batched: scheme %s keeps per-agent caches; batch one agent per call", kSchemeName[pool->dims.scheme]);
    per_entry_lr = mixed;
    const int64_t a = agent_ids ? agent_ids[0] : 0;
    if (a < 0 || a >= pool->dims.n_agents) return fail("unknown agent %lld", (long long)a);
    if (pool->dims.scheme == LORAKV_NONSHARED) kv_set = a; else lr_set = a;
  }
  int64_t L;
  LK_TRY(visible_rows(pool, layer_begin, kv_set, lr_set, &L, !per_entry_lr));
  if (L < 1) return fail("attention: query_offset 0 with L_c 1 exceeds L 0");
  return run_paged(pool, ad, layer_begin, layer_end, kv_set, lr_set, agent_ids, n_batch, 1, L - 1, n_q_heads, q, out, mem_kind, nullptr,
                   per_entry_lr);
}

// Sharded decode step ending in the output gather over peer memory (peer_gather.cu).
int lorakv_fla_decode_batched_gather(lorakv_pool* pool, const lorakv_adapters* ad, lorakv_gather* g, int64_t layer_begin,
                                     int64_t layer_end, const int32_t* agent_ids, int64_t n_batch, int64_t n_q_heads,
                                     const float* q, int q_mem_kind, float* out_host, float** out_dev) {
  if (!pool || !g || !q) return fail("fla_decode_batched_gather: null argument");
  if (n_batch < 1) return fail("fla_decode_batched: empty batch");
  if (g->ctx != pool->ctx) return fail("fla_decode_batched_gather: the gather and the pool belong to different contexts");
  if (!g->connected) return fail("fla_decode_batched_gather: the gather is not connected to its peers (lorakv_gather_connect)");
  if (pool->dims.scheme == LORAKV_NONSHARED || (pool->dims.scheme == LORAKV_BASESHARED && pool->r_pad > 0))
    return fail("fla_decode_batched_gather: scheme %s keeps per-agent caches; batch one agent per call", kSchemeName[pool->dims.scheme]);
  if (n_q_heads < 1 || n_q_heads % pool->dims.n_kv_heads != 0)
    return fail("gqa_attention: n_q_heads %lld not divisible by n_kv_heads %lld", (long long)n_q_heads, (long long)pool->dims.n_kv_heads);
  const int64_t n_layers = layer_end - layer_begin;
  const int64_t full = n_layers * n_batch * n_q_heads * pool->dims.d_head;
  if (full != g->full_elems)
    return fail("fla_decode_batched_gather: the step produces %lld output floats, the gather was created for %lld", (long long)full,
                (long long)g->full_elems);
  int64_t L;
  LK_TRY(visible_rows(pool, layer_begin, 0, 0, &L));
  if (L < 1) return fail("attention: query_offset 0 with L_c 1 exceeds L 0");
  const uint32_t epoch = g->epoch + 1;
  lk::PeerOut peers;
  peers.n = g->world;
  for (int i = 0; i < g->world; ++i) peers.dst[i] = lk::gather_buffer(g, i, epoch);
  peers.n_q_total = n_q_heads;
  peers.q_head_begin = pool->dims.kv_head_begin * (n_q_heads / pool->dims.n_kv_heads);
  // overlapped handshake: the previous step's handshake still runs beside this step's attention kernel; only the kernel
  // that stores into the peers' buffers (the reuse of the buffer pair) has to wait for it
  if (g->overlap && g->sync_pending) { peers.wait_event = g->ev_synced; g->sync_pending = false; }
  LK_TRY(run_paged(pool, ad, layer_begin, layer_end, 0, 0, agent_ids, n_batch, 1, L - 1, n_q_heads, q, nullptr, q_mem_kind, &peers));
  g->epoch = epoch;
  LK_TRY(lk::gather_sync(g));
  float* mine = lk::gather_buffer(g, g->rank, epoch);
  if (out_dev) *out_dev = mine;
  if (out_host) {
    lorakv_ctx* ctx = pool->ctx;
    LK_TRY(lk::gather_wait(g));
    LK_CUDA(cudaMemcpyAsync(out_host, mine, (size_t)full * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    LK_TRY(lk::gather_read_status(g));
    LK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (*g->status_host != 0) return fail("peer gather: rank %d waited %.1f s for a peer that never published step %u", g->rank,
                                          g->timeout_ns * 1e-9, epoch);
  }
  return LORAKV_OK;
}

/* Status of the gathers enqueued so far (synchronises the ctx stream): fails if a handshake timed out. */
int lorakv_gather_check(lorakv_gather* g) {
  if (!g) return fail("gather_check: null argument");
  LK_TRY(lk::gather_read_status(g));
  LK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  if (*g->status_host != 0) return fail("peer gather: rank %d waited %.1f s for a peer that never arrived", g->rank, g->timeout_ns * 1e-9);
  return LORAKV_OK;
}

int lorakv_fla_prefill(lorakv_pool* pool, const lorakv_adapters* ad, int64_t layer, int64_t agent,
                       int64_t n_q_heads, const float* q, int64_t L_c, int64_t query_offset, float* out,
                       int mem_kind) {
  if (!pool || !q || !out) return fail("fla_prefill: null argument");
  if (agent < 0 || agent >= pool->dims.n_agents) return fail("unknown agent %lld", (long long)agent);
  if (L_c < 0) return fail("fla_prefill: negative L_c");
  if (L_c == 0) return LORAKV_OK;
  int64_t kv_set = pool->dims.scheme == LORAKV_NONSHARED ? agent : 0;
  int64_t lr_set = pool->dims.scheme == LORAKV_BASESHARED ? agent : 0;
  const int32_t id = (int32_t)agent;
  return run_paged(pool, ad, layer, layer + 1, kv_set, lr_set, &id, 1, L_c, query_offset, n_q_heads, q, out, mem_kind);
}

// ---- one decode layer-step of step() on the attention sublayer (engine.hpp:331-443) ----------------------------------
// == lorakv_pool_append_kv_project[_full] + lorakv_pool_append_lr_project + lorakv_proj_query + lorakv_fla_prefill on rows
// [row_begin, row_begin + n_rows).  A decode step's handful of fresh rows on a bf16 pool runs as FOUR chained launches
// (step_layer.cu: all projections in two; attention; merge epilogue); anything else goes through those entry points.
int lorakv_step_layer(lorakv_pool* pool, const lorakv_proj* pr, const lorakv_adapters* ad, int64_t layer, int64_t agent,
                      int64_t row_begin, const float* x, int64_t n_rows, int64_t ld, int rope, int64_t n_q_heads, float* q_scratch,
                      float* out, int mem_kind) {
  if (!pool || !pr || !x || !out) return fail("step_layer: null argument");
  if (n_rows < 1) return fail("step_layer: no rows");
  if (layer < 0 || layer >= pool->dims.n_layers) return fail("layer %lld out of range", (long long)layer);
  if (agent < 0 || agent >= pool->dims.n_agents) return fail("unknown agent %lld", (long long)agent);
  const int scheme = pool->dims.scheme;
  const bool full_values = scheme == LORAKV_NONSHARED || scheme == LORAKV_FULLSHARED;
  const bool lr_cached = pool->lr_sets() > 0 && pool->r_pad > 0;
  if (lr_cached && !ad) return fail("step_layer: the pool keeps a rank-%lld cache but no adapter tables were given", (long long)pool->dims.rank);
  const bool merge_v = full_values && ad != nullptr;
  const bool q_lora = pr->aq != nullptr && agent < pr->q_agents && layer < pr->n_layers &&
                      pr->q_lora_set[(size_t)(layer * pr->q_agents + agent)];
  lorakv_ctx* ctx = pool->ctx;
  const int64_t r_q = q_lora ? pr->q_rank : 0, r_v = (merge_v || lr_cached) ? ad->rank : 0;
  int64_t kv_set = 0, lr_set = 0; bool none;
  LK_TRY(resolve(pool, LORAKV_KEY, layer, agent, &kv_set, &none));
  if (lr_cached) LK_TRY(resolve(pool, LORAKV_LR, layer, agent, &lr_set, &none));
  // the fused path wants fresh rows only (every cache of the step ends exactly at row_begin): the decode case
  const bool fresh = pool->key_rows[(size_t)kv_set][(size_t)layer] == row_begin && pool->value_rows[(size_t)kv_set][(size_t)layer] == row_begin &&
                     (!lr_cached || pool->lr_rows[(size_t)lr_set][(size_t)layer] == row_begin);
  const bool fast = mem_kind == LORAKV_DEVICE && ctx->policy != 1 && fresh && pr->fused && pr->q_fused && pool->rk_pad == 0 &&
                    pool->dims.dtype == LORAKV_BF16 && step_layer_supported(n_rows, pr->d_model, pr->d_head, r_q, r_v) &&
                    n_q_heads == pr->n_q_heads && layer < pr->n_layers && pr->set[(size_t)layer] && pr->q_set[(size_t)layer];
  const int64_t group = pr->n_kv_heads > 0 ? n_q_heads / pr->n_kv_heads : 0;
  const int64_t dq = group * pr->n_kv_local * pr->d_head;
  if (!fast) {
    int64_t added = 0;
    if (merge_v) LK_TRY(lorakv_pool_append_kv_project_full(pool, pr, ad, layer, agent, row_begin, x, n_rows, ld, mem_kind, rope, &added));
    else LK_TRY(lorakv_pool_append_kv_project(pool, pr, layer, agent, row_begin, x, n_rows, ld, mem_kind, rope, &added));
    if (lr_cached) LK_TRY(lorakv_pool_append_lr_project(pool, ad, layer, agent, row_begin, x, n_rows, ld, mem_kind, &added));
    if (pool->rk_pad > 0) {      // key-side low-rank cache (extension): L_k rows = x A_k
      if (!ad) return fail("step_layer: the pool keeps a key-side low-rank cache but no adapter tables were given");
      LK_TRY(lorakv_pool_append_lk_project(pool, ad, layer, row_begin, x, n_rows, ld, mem_kind, &added));
    }
    float* q = q_scratch;
    std::vector<float> q_host;
    if (!q) {
      if (mem_kind == LORAKV_HOST) { q_host.resize((size_t)(n_rows * dq)); q = q_host.data(); }
      else { LK_TRY(scratch_reserve(ctx, ctx->qrows, (size_t)(n_rows * dq) * sizeof(float))); q = static_cast<float*>(ctx->qrows.ptr); }
    }
    LK_TRY(lorakv_proj_query(const_cast<lorakv_proj*>(pr), layer, q_lora ? agent : -1, row_begin, x, n_rows, ld, rope, q, mem_kind));
    return lorakv_fla_prefill(pool, (lr_cached || pool->rk_pad > 0) ? ad : nullptr, layer, agent, n_q_heads, q, n_rows, row_begin, out, mem_kind);
  }
  // ---- fused path ----
  if (pr->d_model != pool->dims.d_model || pr->n_kv_heads != pool->dims.n_kv_heads || pr->d_head != pool->dims.d_head ||
      pr->kv_head_begin != pool->dims.kv_head_begin || pr->n_kv_local != pool->n_kv_local || pr->dtype != pool->dims.dtype)
    return fail("append_kv_project: projection weights do not match the pool (d_model %lld vs %lld, d_kv %lld vs %lld)",
                (long long)pr->d_model, (long long)pool->dims.d_model, (long long)(pr->n_kv_heads * pr->d_head),
                (long long)(pool->dims.n_kv_heads * pool->dims.d_head));
  const float *a_v = nullptr, *b_v = nullptr; float s_v = 0.f;
  if (merge_v || lr_cached) {
    if (ad->d_model != pr->d_model || ad->n_kv_local != pr->n_kv_local || ad->d_head != pr->d_head || layer >= ad->n_layers ||
        agent >= ad->n_agents)
      return fail("step_layer: adapter table does not match the projection (rank %lld)", (long long)ad->rank);
    const size_t la = (size_t)(layer * ad->n_agents + agent);
    const bool own_a = ad->a_agent && ad->a_agent_set[la];
    if (!own_a && !ad->a_set[(size_t)layer]) return fail("lr_append_project: A of layer %lld was never uploaded", (long long)layer);
    if (!ad->b_set[la]) return fail("attention: B of layer %lld agent %lld was never uploaded", (long long)layer, (long long)agent);
    a_v = own_a ? ad->a_agent + la * (size_t)(ad->d_model * ad->rank) : ad->a + layer * ad->d_model * ad->rank;
    b_v = ad->b + (la * ad->rank) * (size_t)(ad->n_kv_local * ad->d_head);
    s_v = ad->scale_host[la];
  }
  LK_CUDA(cudaSetDevice(ctx->device));
  LK_TRY(ensure_pages(pool, pool->kv_space, kv_set, row_begin + n_rows));
  if (lr_cached) LK_TRY(ensure_pages(pool, pool->lr_space, lr_set, row_begin + n_rows));
  float* q_dev = q_scratch;
  if (!q_dev) { LK_TRY(scratch_reserve(ctx, ctx->qrows, (size_t)(n_rows * dq) * sizeof(float))); q_dev = static_cast<float*>(ctx->qrows.ptr); }
  const int64_t dq_full = pr->n_q_heads * pr->d_head, col0 = pr->kv_head_begin * group * pr->d_head;
  StepLayerCall c;
  c.layer = layer; c.kv_set = kv_set; c.lr_set = lr_set; c.row0 = row_begin; c.n_rows = n_rows; c.x_dev = x; c.ld = ld;
  c.wq_packed = static_cast<const char*>(pr->wq_packed) + (size_t)(layer * pr->d_model * dq) * 2;
  c.wkv_packed = static_cast<const char*>(pr->packed) + (size_t)(layer * kv_project_packed_elems(pr->d_model, pr->n_kv_local, pr->d_head)) * 2;
  c.dq = dq;
  c.a_q = q_lora ? pr->aq + (size_t)(layer * pr->d_model * r_q) : nullptr;
  c.b_q = q_lora ? pr->bq + (size_t)((layer * pr->q_agents + agent) * r_q * dq_full) + col0 : nullptr;
  c.ldb_q = dq_full; c.r_q = r_q; c.s_q = q_lora ? pr->q_scale[(size_t)(layer * pr->q_agents + agent)] : 0.f;
  c.a_v = a_v; c.b_v = b_v; c.r_v = r_v; c.s_v = s_v;
  c.merge_v = merge_v; c.append_lr = lr_cached; c.rope = rope != 0; c.q_dev = q_dev;
  LK_TRY(launch_step_layer(pool, c));
  LK_TRY(note_pages_written(pool, row_begin));
  pool->key_rows[(size_t)kv_set][(size_t)layer] += n_rows;
  pool->value_rows[(size_t)kv_set][(size_t)layer] += n_rows;
  if (lr_cached) pool->lr_rows[(size_t)lr_set][(size_t)layer] += n_rows;
  const int32_t id = (int32_t)agent;
  return run_paged(pool, lr_cached ? ad : nullptr, layer, layer + 1, kv_set, lr_set, &id, 1, n_rows, row_begin, n_q_heads, q_dev, out,
                   LORAKV_DEVICE);
}

}  // extern "C"
