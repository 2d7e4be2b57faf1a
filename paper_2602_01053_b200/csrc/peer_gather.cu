// peer_gather.cu -- the end-of-step output gather of a kv-head-sharded decode, over NVLink peer memory.
//
// q head h reads only kv head h/g (proj/include/lorakv/attention.hpp:348-354), so a rank that holds a
// kv-head shard produces the column slice [q_head_begin*d, (q_head_begin+n_q_local)*d) of every output row
// (gqa_attention's L_c x (n_q*d) result, attention.hpp:346,359-360) and the only exchange of the step is putting
// the slices side by side.  Instead of writing a local slab and calling a collective on it, the merge epilogue of
// the decode kernels (fla_decode_tma.cu: store_out) stores every finished row into the gather buffer of EVERY rank
// -- plain st.global to addresses mapped with cudaIpcOpenMemHandle, carried by NVLink / NVSwitch -- while other CTAs
// are still merging.  What is left is a handshake: gather_sync_kernel (one block) publishes this rank's step
// number in the peers' flag words with a system-scope release and spins until every peer's number has arrived
// here (system-scope acquire).  Kernel completion orders the epilogue's peer stores before the release.
//
// Two output buffers alternate by step parity.  A rank can be at most one step ahead of a peer (it cannot pass
// step s+1's handshake before the peer entered step s+1's), and a peer enters step s+1's handshake only after its
// own stream has finished everything it enqueued before -- including whatever consumed step s's buffer.  So a
// buffer is rewritten (step s+2) only after every rank's stream-ordered readers of step s are done.
#include <cstring>

#include "kernels.hpp"
#include "state.hpp"

namespace lk {
namespace {

constexpr size_t kFlagBytes = 256;     // [0..7] arrival step of rank p, [8] status (0 ok, 1 timed out)

struct SyncParams {
  uint32_t* peer_flags[kMaxPeers];   // flag page of every rank as mapped here
  uint32_t* my_flags;
  int rank, world;
  uint32_t epoch;
  unsigned long long timeout_ns;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void gather_sync_kernel(const SyncParams p) {
  const int pe = threadIdx.x;
  if (pe >= p.world) return;
  uint32_t* remote = nullptr;
#pragma unroll
  for (int i = 0; i < kMaxPeers; ++i)
    if (i == pe) remote = p.peer_flags[i];
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote + p.rank), "r"(p.epoch) : "memory");
  const uint32_t* mine = p.my_flags + pe;
  const unsigned long long t0 = global_ns();
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if ((int32_t)(v - p.epoch) >= 0) break;
    if (global_ns() - t0 > p.timeout_ns) { p.my_flags[8] = 1u; break; }     // a peer never arrived: report, do not hang
    __nanosleep(200);
  }
}

__global__ void peer_scatter_kernel(const float* __restrict__ slab, int64_t rows, int64_t w_local, int64_t w_full, int64_t col0,
                                    const PeerOut peers) {
  const int64_t n4 = rows * (w_local / 4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / (w_local / 4), c4 = i % (w_local / 4);
    const float4 v = reinterpret_cast<const float4*>(slab)[i];
    const int64_t off = row * w_full + col0 + c4 * 4;
#pragma unroll
    for (int pe = 0; pe < kMaxPeers; ++pe)
      if (pe < peers.n) *reinterpret_cast<float4*>(peers.dst[pe] + off) = v;
  }
}

}  // namespace

int launch_peer_scatter(lorakv_ctx* ctx, const float* slab_dev, int64_t rows, int64_t n_q_local, int64_t d, const PeerOut& peers) {
  const int64_t w_local = n_q_local * d, w_full = peers.n_q_total * d;
  if (w_local % 4 != 0) return fail("peer gather: a slice of %lld floats per row is not 16-byte granular", (long long)w_local);
  const int64_t n4 = rows * (w_local / 4);
  if (n4 == 0) return LORAKV_OK;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 4 * ctx->sm_count) blocks = 4 * ctx->sm_count;
  if (peers.wait_event) LK_CUDA(cudaStreamWaitEvent(ctx->stream, static_cast<cudaEvent_t>(peers.wait_event), 0));
  peer_scatter_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(slab_dev, rows, w_local, w_full, peers.q_head_begin * d, peers);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

// publish this step to the peers and wait for theirs (on the ctx stream)
int gather_sync(lorakv_gather* g) {
  SyncParams sp{};
  for (int i = 0; i < g->world; ++i) sp.peer_flags[i] = reinterpret_cast<uint32_t*>(g->peer[i]);
  sp.my_flags = reinterpret_cast<uint32_t*>(g->local);
  sp.rank = g->rank; sp.world = g->world; sp.epoch = g->epoch; sp.timeout_ns = g->timeout_ns;
  if (g->overlap) {
    // side stream: behind this step's epilogue (ev_merged), beside whatever the ctx stream does next
    LK_CUDA(cudaEventRecord(g->ev_merged, g->ctx->stream));
    LK_CUDA(cudaStreamWaitEvent(g->side, g->ev_merged, 0));
    gather_sync_kernel<<<1, 32, 0, g->side>>>(sp);
    LK_CUDA(cudaGetLastError());
    LK_CUDA(cudaEventRecord(g->ev_synced, g->side));
    g->sync_pending = true;
  } else {
    gather_sync_kernel<<<1, 32, 0, g->ctx->stream>>>(sp);
    LK_CUDA(cudaGetLastError());
  }
  g->ctx->launches++;
  return LORAKV_OK;
}

// the ctx stream waits for the last handshake (no-op when none is outstanding)
int gather_wait(lorakv_gather* g) {
  if (g->overlap && g->sync_pending) {
    LK_CUDA(cudaStreamWaitEvent(g->ctx->stream, g->ev_synced, 0));
    g->sync_pending = false;
  }
  return LORAKV_OK;
}

int gather_read_status(lorakv_gather* g) {
  LK_TRY(gather_wait(g));
  LK_CUDA(cudaMemcpyAsync(g->status_host, g->local + 8 * sizeof(uint32_t), sizeof(uint32_t), cudaMemcpyDeviceToHost, g->ctx->stream));
  return LORAKV_OK;
}

float* gather_buffer(const lorakv_gather* g, int rank, uint32_t epoch) {
  return reinterpret_cast<float*>(g->peer[rank] + kFlagBytes) + (size_t)(epoch & 1u) * (size_t)g->full_elems;
}

}  // namespace lk

using lk::fail;

extern "C" {

int lorakv_gather_create(lorakv_ctx* ctx, int rank, int world, int64_t full_elems, lorakv_gather** out) {
  if (!ctx || !out) return fail("gather_create: null argument");
  if (world < 1 || world > lk::kMaxPeers) return fail("gather_create: world size %d outside [1, %d]", world, lk::kMaxPeers);
  if (rank < 0 || rank >= world) return fail("gather_create: rank %d outside [0, %d)", rank, world);
  if (full_elems < 1) return fail("gather_create: empty output");
  LK_CUDA(cudaSetDevice(ctx->device));
  auto* g = new lorakv_gather;
  g->ctx = ctx; g->rank = rank; g->world = world; g->full_elems = full_elems;
  g->buf_bytes = lk::kFlagBytes + 2 * (size_t)full_elems * sizeof(float);
  // cudaMalloc, not a stream-ordered pool: only plain device allocations can be exported through CUDA IPC
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&g->local), g->buf_bytes);
  if (e != cudaSuccess) { delete g; return fail("gather_create: cudaMalloc(%zu): %s", g->buf_bytes, cudaGetErrorString(e)); }
  e = cudaMemset(g->local, 0, g->buf_bytes);
  if (e != cudaSuccess) { cudaFree(g->local); delete g; return fail("gather_create: cudaMemset: %s", cudaGetErrorString(e)); }
  e = cudaMallocHost(reinterpret_cast<void**>(&g->status_host), 64);
  if (e != cudaSuccess) { cudaFree(g->local); delete g; return fail("gather_create: cudaMallocHost: %s", cudaGetErrorString(e)); }
  *g->status_host = 0;
  g->peer[rank] = g->local;
  g->connected = world == 1;
  *out = g;
  return LORAKV_OK;
}

int lorakv_gather_disconnect(lorakv_gather* g) {
  if (!g) return fail("gather_disconnect: null argument");
  LK_CUDA(cudaSetDevice(g->ctx->device));
  if (g->side) LK_CUDA(cudaStreamSynchronize(g->side));
  LK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  for (int i = 0; i < g->world; ++i)
    if (i != g->rank && g->peer[i]) { cudaIpcCloseMemHandle(g->peer[i]); g->peer[i] = nullptr; }
  g->connected = false;
  return LORAKV_OK;
}

void lorakv_gather_destroy(lorakv_gather* g) {
  if (!g) return;
  lorakv_gather_disconnect(g);
  if (g->side) { cudaStreamSynchronize(g->side); cudaStreamDestroy(g->side); }
  if (g->ev_merged) cudaEventDestroy(g->ev_merged);
  if (g->ev_synced) cudaEventDestroy(g->ev_synced);
  cudaFree(g->local);
  cudaFreeHost(g->status_host);
  delete g;
}

int lorakv_gather_export(lorakv_gather* g, unsigned char* handle) {
  if (!g || !handle) return fail("gather_export: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == LORAKV_GATHER_HANDLE_BYTES, "handle size");
  LK_CUDA(cudaSetDevice(g->ctx->device));
  cudaIpcMemHandle_t h;
  LK_CUDA(cudaIpcGetMemHandle(&h, g->local));
  std::memcpy(handle, &h, sizeof h);
  return LORAKV_OK;
}

int lorakv_gather_connect(lorakv_gather* g, const unsigned char* handles) {
  if (!g || !handles) return fail("gather_connect: null argument");
  if (g->connected) return g->world == 1 ? LORAKV_OK : fail("gather_connect: already connected");
  LK_CUDA(cudaSetDevice(g->ctx->device));
  for (int i = 0; i < g->world; ++i) {
    if (i == g->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)i * LORAKV_GATHER_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int j = 0; j < i; ++j)
        if (j != g->rank && g->peer[j]) { cudaIpcCloseMemHandle(g->peer[j]); g->peer[j] = nullptr; }
      return fail("gather_connect: rank %d cannot map the buffer of rank %d: %s", g->rank, i, cudaGetErrorString(e));
    }
    g->peer[i] = static_cast<char*>(p);
  }
  g->connected = true;
  return LORAKV_OK;
}

int lorakv_gather_set_timeout_ms(lorakv_gather* g, int64_t ms) {
  if (!g || ms < 1) return fail("gather_set_timeout_ms: bad argument");
  g->timeout_ns = (uint64_t)ms * 1000000ull;
  return LORAKV_OK;
}

int lorakv_gather_set_overlap(lorakv_gather* g, int enabled) {
  if (!g) return fail("gather_set_overlap: null argument");
  LK_CUDA(cudaSetDevice(g->ctx->device));
  if (enabled && !g->side) {
    LK_CUDA(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
    LK_CUDA(cudaEventCreateWithFlags(&g->ev_merged, cudaEventDisableTiming));
    LK_CUDA(cudaEventCreateWithFlags(&g->ev_synced, cudaEventDisableTiming));
  }
  if (!enabled) LK_TRY(lk::gather_wait(g));     // an outstanding handshake joins the ctx stream first
  g->overlap = enabled != 0;
  return LORAKV_OK;
}

int lorakv_gather_wait(lorakv_gather* g) {
  if (!g) return fail("gather_wait: null argument");
  return lk::gather_wait(g);
}

int lorakv_gather_steps(const lorakv_gather* g, int64_t* steps) {
  if (!g || !steps) return fail("gather_steps: null argument");
  *steps = g->epoch;
  return LORAKV_OK;
}

}  // extern "C"
