// fla_decode_tma.cu -- batched Flash-LoRA-Attention decode over the paged bf16 cache, tuned for HBM
// bandwidth: K / V_base / V_lr tiles are streamed from HBM into shared memory by the TMA engine
// (cp.async.bulk + mbarrier rings, one ring per worker), the contractions run on the tensor cores
// (mma.sync m16n8k16 bf16 -> fp32) and the softmax bookkeeping uses warp-level reductions.
//
// What it computes: one gqa_attention call (proj/include/lorakv/attention.hpp:332-363) per (layer,
// batch entry) with query_offset = L-1 (engine.hpp:440-443), i.e. per q head the blocked
// flash_lora_attention of attention.hpp:210-268 -- but reordered so that the cache is read ONCE:
// the g q heads of a kv head and all batch entries (agents) are rows of the same MMA tile, where the
// reference's per-head loop (:347-361) re-streams K/V for every q head and every agent.
//
//   worker   = MW warps (MW = 1/2/4/8 for <= 16/32/64/128 query rows per kv head); warp i of a worker
//              owns rows [16 i, 16 i + 16) and every worker owns its own ring of shared-memory stages
//   work     = the (unit, 16-key tile) pairs in unit-major order, cut into equal contiguous ranges,
//              one per worker (unit = layer x kv head [x 128-row block]); a worker emits one partial
//              (m, l, O, O_lr) per unit its range touches and fla_decode_merge combines them
//   per tile = S = Q K^T (8 k-steps), online softmax in the exp2 domain with lazy rescaling,
//              O += P V_base and O_lr += P V_lr with the same P (attention.hpp:185-198)
//   epilogue = fla_decode_merge: split merge, o += (lr_scale * o_lr[p]) * B[agent][p,:], out = o / l
//              (attention.hpp:244-259)
//
// Pages arrive pre-swizzled (page_layout.cuh), so a contiguous bulk copy of 16 tokens lands as a
// bank-conflict-free ldmatrix tile.  Masking: key j contributes iff j < L; masked scores are never
// exponentiated (p = 0 exactly), matching attention.hpp:154-171.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <limits>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kWarps = 8;           // warps per CTA
// single-warp workers per CTA when they take 32-key tiles: three at d_head 128, four at d_head 64 (half the bytes per
// key for the same softmax work: 3 x 32 loses there, 0.253 vs 0.204 ms on a 16-layer probe, 4 x 32 gains 4 %)
constexpr int wide_workers(int d) { return d == 128 ? 3 : 4; }
constexpr int kKeyStep = 16;        // keys per MMA k-step; a tile is KT of them
constexpr int kMaxStages = 24;      // ring depth limit per worker
constexpr int kRingBudget = 216 * 1024;   // of the 227 KB a CTA may own
constexpr float kRescaleThreshold = 8.0f;   // log2 units: p stays <= 2^8 between rescales

#ifdef LK_DECODE_TRACE
// debug build only (make EXTRA=-DLK_DECODE_TRACE): per-warp phase timestamps of the last launch, tools/probe_decode_trace.py
__device__ unsigned long long g_decode_trace[1024 * 16];
__device__ __forceinline__ void trace_mark(int64_t warp_global, int slot) {
  if ((threadIdx.x & 31) == 0 && warp_global < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_decode_trace[warp_global * 16 + slot] = t;
  }
}
#define LK_TRACE(slot) trace_mark((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), slot)
__device__ unsigned long long g_merge_trace[512 * 4];
#define LK_MTRACE(slot)                                                                              \
  do {                                                                                               \
    if (threadIdx.x == 0) {                                                                          \
      unsigned long long t_;                                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                         \
      const int b_ = blockIdx.x + gridDim.x * blockIdx.y;                                            \
      if (b_ < 512) g_merge_trace[b_ * 4 + slot] = t_;                                               \
    }                                                                                                \
  } while (0)
#else
#define LK_MTRACE(slot)
#define LK_TRACE(slot)
#endif

struct DecodeParams {
  const __nv_bfloat16 *k_pages, *v_pages, *lr_pages;
  const int32_t *kv_table, *lr_table;
  int64_t kv_layer_stride, kv_head_stride, kv_page_stride, lr_layer_stride, lr_page_stride;  // elements
  int P, group, n_kv_local, n_batch, rows_total, row_blocks, n_pages;
  int64_t L, layer_begin, n_q_local;
  int64_t T;             // tiles per unit
  int64_t total_tiles;   // units * T of ONE layer chunk
  int64_t G;             // tiles per worker and chunk
  int n_chunks;          // equal layer chunks walked one after the other (1 = the whole launch at once)
  int64_t n_workers;     // workers of the launch (partials are laid out [chunk][worker][segment])
  int max_seg, n_stages;
  float scale_log2;      // (1/sqrt(d)) * log2(e)
  uint64_t l2_policy;    // cache-hint operand of the K / V bulk copies (0 = none)
  uint64_t lr_policy;    // ... and of the V_lr copies (evict-last while the launch's low-rank cache fits in L2)
  const float* q;        // [layers][n_batch][n_q_local * d]
  float* part;           // [workers * max_seg][16 * MW][4 + D + RP]
  // per-entry low-rank caches (template flag PA; BaseShared batches): entry i reads page set agent_ids[i]
  const int32_t* lr_tables;   // [sets][lr_max_pages]
  const int32_t* agent_ids;   // [n_batch]
  int lr_max_pages;
  int lr_per_block;           // entries of one row block = V_lr tiles per stage (16 * MW / group)
  int identity;               // bit 0 / 1 / 2: the K-V / V_lr / L_k page table is the identity (PageSpace::identity): no table load
  // key-side low-rank term (template RK > 0; kernels.hpp: KeyLowRank): L_k tiles ride in the stage behind V_lr, the queries
  // projected through B_k (launch_qk_project) extend the Q fragments, S = Q K^T + Qk L_k^T in the same accumulators
  const __nv_bfloat16* lk_pages; const int32_t* lk_table; int64_t lk_layer_stride, lk_page_stride;
  const float* qk;            // [layers][n_batch][n_q_local][RK]
  int64_t stable_rows;        // cache rows [0, stable_rows) are complete whatever the predecessor kernel is doing (0: none)
};

// The cache is streamed exactly once per step, so the copies carry an L2 evict-first policy: the lines
// should not displace the small reused operands (page tables, partials, B).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  if (policy != 0)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)), "l"(policy)
                 : "memory");
  else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// D = d_head (64 / 128), RP = padded rank (0 / 16 / 32 / 64), MW = warps per worker, KT = 16-key
// steps per tile (1 for single-warp workers whose eight rings must share the SM's shared memory; 2 for
// the multi-warp workers, which halves their per-tile synchronisation and doubles the MMA ILP)
// PA: every batch entry has its own V_lr page set (BaseShared).  A stage then holds K, V_base and one V_lr tile per
// entry of the row block; the lanes of the producer warp issue the V_lr copies in parallel (lane e -> entry e), and
// a consumer warp runs the O_lr MMA once per entry its 16 rows touch with P masked to that entry's rows.
// NW = warps per CTA.  Eight, except for single-warp workers (wide_workers): at d_head 128 three workers with 32-key tiles
// and four-stage rings stream faster than eight with 16-key tiles and three-stage rings (cfg 2: 0.695 -> 0.617 ms per
// step, 7.1 TB/s) -- the bulk copies are twice as large and every worker prefetches deeper, and three warps still cover
// the few MMAs a <= 16-row tile needs.  d_head 64 wants four (three lose there) and the multi-warp workers keep eight warps
// (fewer lose: cfg 4 with 6 warps 1.87 ms vs 1.41 ms).
template <int D, int RP, int MW, int KT, bool PA = false, int NW = kWarps, int RK = 0>
__global__ void __launch_bounds__(NW * 32, 1) fla_decode_tma_kernel(const DecodeParams p) {
  static_assert(RK == 0 || (MW == 1 && !PA), "the key-side low-rank term is built for single-warp workers");
  constexpr uint32_t kLkBytes = kKeyStep * KT * RK * 2;
  constexpr int kTK = kKeyStep * KT;                    // keys per tile
  constexpr int kWorkers = NW / MW;
  constexpr int kBlocks = D / 64;                       // 64-column blocks of a K / V page
  constexpr uint32_t kBlockBytes = kTK * 128;           // one block of one tile
  constexpr uint32_t kKvBytes = kBlocks * kBlockBytes;  // K (or V) tile
  constexpr uint32_t kLrBytes = kTK * RP * 2;
  constexpr int kNO = D / 8, kNL = RP / 8;              // n8 tiles of O and O_lr
  constexpr int PS = 4 + D + RP;                        // floats per partial row
  const uint32_t kStageBytes = 2 * kKvBytes + (PA ? (uint32_t)p.lr_per_block : 1u) * kLrBytes + kLkBytes;

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kWorkers][kMaxStages];
  __shared__ uint64_t empty_bar[kWorkers][kMaxStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wk = warp / MW, wi = warp % MW;
  const int g = lane >> 2, t = lane & 3;
  const int NS = p.n_stages;
  LK_TRACE(0);

  if (threadIdx.x == 0) {
    for (int a = 0; a < kWorkers; ++a)
      for (int s = 0; s < NS; ++s) {
        ptx::mbar_init(&full_bar[a][s], 1);
        ptx::mbar_init(&empty_bar[a][s], MW);
      }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  LK_TRACE(1);

  // (unit, tile) arithmetic in 32 bits: the launcher checks that the tile count of the launch fits.  The 64-bit divisions
  // of the first version cost a lone warp ~2 us before its first bulk copy went out (a one-layer launch lasts ~25).
  const int w = (int)blockIdx.x * kWorkers + wk;
  const int T32 = (int)p.T, G32 = (int)p.G, total32 = (int)p.total_tiles;
  // A launch whose low-rank cache does not fit in L2 is cut into p.n_chunks equal LAYER CHUNKS that every worker walks
  // through one after the other (no grid barrier: all workers get the same share of every chunk and stay in step), so
  // that at any time the kv heads of only a few layers are in flight and their shared V_lr tiles are served by L2.
  // Inside a chunk the (unit, tile) pairs are cut into equal contiguous ranges as before (p.total_tiles per chunk).
  int g0 = 0, first_unit = 0;
  int n = 0, chunk = 0;

  const uint32_t ring = ptx::smem_u32(smem) + (uint32_t)wk * (uint32_t)NS * kStageBytes;
  uint64_t* full = full_bar[wk];
  uint64_t* empty = empty_bar[wk];
  const bool producer = wi == 0;
  const int units_per_layer = p.n_kv_local * p.row_blocks;

  // page-table window held across the lanes of the producer warp: lane i caches logical page base + i
  int win_base = -(1 << 30), win_kv = 0, win_lr = 0, win_lk = 0;

  // Producer cursor.  Everything the per-tile path needs is carried incrementally (unit, tile, page,
  // token, stage, wrap count): the only divisions happen here and at unit changes, never per tile.
  int p_unit = 0;
  int p_tl = 0, p_page = 0, p_tok = 0, p_layer = 0, p_kvh = 0;
  int p_stage = 0, p_wrap = 0, p_issued = 0;      // stage and wrap count run on across chunks, like the consumer's

  auto issue_next = [&]() {       // whole producer warp; lane 0 talks to the TMA engine
    // the stage must have been released by every warp of the worker (a fresh barrier passes the parity-1 wait)
    ptx::mbar_wait(&empty[p_stage], (uint32_t)((p_wrap & 1) ^ 1));
    if (p_issued == 1) LK_TRACE(11);
    const bool id_kv = (p.identity & 1) != 0, id_lr = (p.identity & 2) != 0 || RP == 0 || PA, id_lk = (p.identity & 4) != 0 || RK == 0;
    if (!(id_kv && id_lr && id_lk) && (p_page < win_base || p_page >= win_base + 32)) {
      win_base = p_page;
      const int pg = p_page + lane;
      if (!id_kv) win_kv = pg < p.n_pages ? p.kv_table[pg] : 0;
      if (!id_lr) win_lr = pg < p.n_pages ? p.lr_table[pg] : 0;
      if (!id_lk) win_lk = pg < p.n_pages ? p.lk_table[pg] : 0;
    }
    const int phys_kv = id_kv ? p_page : __shfl_sync(0xffffffffu, win_kv, p_page - win_base);
    const int phys_lr = id_lr ? p_page : __shfl_sync(0xffffffffu, win_lr, p_page - win_base);
    const int phys_lk = id_lk ? p_page : __shfl_sync(0xffffffffu, win_lk, p_page - win_base);
    int pa_entries = 0;         // PA: entries of this row block that exist (the last block may be ragged)
    if (PA) {
      const int e0 = (int)(p_unit % p.row_blocks) * p.lr_per_block;
      pa_entries = min(p.lr_per_block, p.n_batch - e0);
      if (lane < pa_entries) {  // lane e streams the V_lr tile of entry e0 + e from that entry's own page set
        const int set = p.agent_ids[e0 + lane];
        const int phys = p.lr_tables[(int64_t)set * p.lr_max_pages + p_page];
        const int64_t lr_off = (p.layer_begin + p_layer) * p.lr_layer_stride + (int64_t)phys * p.lr_page_stride + (int64_t)p_tok * RP;
        bulk_g2s(ring + (uint32_t)p_stage * kStageBytes + 2 * kKvBytes + (uint32_t)lane * kLrBytes, p.lr_pages + lr_off, kLrBytes,
                 &full[p_stage], p.lr_policy);
      }
    }
    if (ptx::elect_one()) {     // not `lane == 0`: no ELECT / BRA.U.ANY waterfall loop around each UBLKCP
      const uint32_t dst = ring + (uint32_t)p_stage * kStageBytes;
      const int64_t layer = p.layer_begin + p_layer;
      const int64_t kv_off = layer * p.kv_layer_stride + (int64_t)p_kvh * p.kv_head_stride +
                             (int64_t)phys_kv * p.kv_page_stride + (int64_t)p_tok * 64;
      ptx::mbar_arrive_expect_tx(&full[p_stage], PA ? 2 * kKvBytes + (uint32_t)pa_entries * kLrBytes : kStageBytes);
      if (p_issued == 1) LK_TRACE(12);
#pragma unroll
      for (int b = 0; b < kBlocks; ++b) {
        bulk_g2s(dst + b * kBlockBytes, p.k_pages + kv_off + (int64_t)b * p.P * 64, kBlockBytes, &full[p_stage], p.l2_policy);
        bulk_g2s(dst + kKvBytes + b * kBlockBytes, p.v_pages + kv_off + (int64_t)b * p.P * 64, kBlockBytes, &full[p_stage], p.l2_policy);
      }
      if (RP > 0 && !PA) {
        const int64_t lr_off = layer * p.lr_layer_stride + (int64_t)phys_lr * p.lr_page_stride + (int64_t)p_tok * RP;
        // V_lr is per layer, not per head: the same tile is read once per kv head, at different times of the launch.
        // Kept with evict-last while K / V stream through with evict-first, the whole low-rank cache of the step
        // (33 MB at cfg 2) stays in L2 and DRAM serves it once instead of n_kv times.
        bulk_g2s(dst + 2 * kKvBytes, p.lr_pages + lr_off, kLrBytes, &full[p_stage], p.lr_policy);
      }
      if (RK > 0) {     // L_k is per layer like V_lr: every kv head of the layer reads the same tile, so it gets the same L2 hint
        const int64_t lk_off = layer * p.lk_layer_stride + (int64_t)phys_lk * p.lk_page_stride + (int64_t)p_tok * RK;
        bulk_g2s(dst + 2 * kKvBytes + kLrBytes, p.lk_pages + lk_off, kLkBytes, &full[p_stage], p.lr_policy);
      }
    }
    if (p_issued == 1) LK_TRACE(13);
    // advance the cursor
    ++p_issued;
    if (++p_stage == NS) { p_stage = 0; ++p_wrap; }
    p_tok += kTK;
    if (p_tok == p.P) { p_tok = 0; ++p_page; }
    if (++p_tl == T32) {
      p_tl = 0; p_page = 0; p_tok = 0;
      ++p_unit;
      p_layer = p_unit / units_per_layer;
      p_kvh = (p_unit / p.row_blocks) % p.n_kv_local;
    }
  };

  const float ninf = -std::numeric_limits<float>::infinity();
  uint32_t qa[D / 16][4];
  uint32_t qka[RK > 0 ? RK / 16 : 1][4];          // the queries through B_k: RK / 16 more k-steps of the score product
  float o[kNO][4];
  float olr[kNL > 0 ? kNL : 1][4];
  float m_used[2], l_run[2];
  int cur_unit = -1;

  auto flush = [&]() {            // partial of the unit just finished
    const int64_t slot = ((int64_t)chunk * p.n_workers + w) * p.max_seg + (cur_unit - first_unit);
    float* base = p.part + (slot * (16 * MW) + wi * 16) * PS;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float l = l_run[h];
      l += __shfl_xor_sync(0xffffffffu, l, 1);
      l += __shfl_xor_sync(0xffffffffu, l, 2);
      float* row = base + (g + 8 * h) * PS;
      if (t == 0) { row[0] = m_used[h]; row[1] = l; }
#pragma unroll
      for (int nt = 0; nt < kNO; ++nt)
        *reinterpret_cast<float2*>(row + 4 + 8 * nt + 2 * t) = make_float2(o[nt][2 * h], o[nt][2 * h + 1]);
#pragma unroll
      for (int nt = 0; nt < kNL; ++nt)
        *reinterpret_cast<float2*>(row + 4 + D + 8 * nt + 2 * t) = make_float2(olr[nt][2 * h], olr[nt][2 * h + 1]);
    }
  };

  // ldmatrix lane roles
  const int mi = lane >> 3, rr = lane & 7;

  // first rows of a unit: Q fragments (bf16, registers) and empty accumulators.  Two phases, so that the launch's first
  // bulk copies can be issued while the query loads are in flight: load_q only ISSUES the loads (volatile asm keeps them
  // ahead of the copies in program order), pack_q consumes them.
  float2 qraw[2][D / 16][2];
  float2 qkraw[2][RK > 0 ? RK / 16 : 1][2];
  auto load_q = [&](int u) {
    const int layer_rel = u / units_per_layer;
    const int kvh = (u / p.row_blocks) % p.n_kv_local;
    const int rb = u % p.row_blocks;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rho = rb * 16 * MW + wi * 16 + g + 8 * h;
      const bool real = rho < p.rows_total;
      const int entry = real ? rho / p.group : 0, gi = real ? rho % p.group : 0;
      const float* src = p.q + (((int64_t)layer_rel * p.n_batch + entry) * p.n_q_local + (int64_t)kvh * p.group + gi) * D;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          float2 v = make_float2(0.f, 0.f);
          if (real)
            asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(src + 16 * kk + 8 * part + 2 * t));
          qraw[h][kk][part] = v;
        }
      if (RK > 0) {
        const float* srck = p.qk + (((int64_t)layer_rel * p.n_batch + entry) * p.n_q_local + (int64_t)kvh * p.group + gi) * RK;
#pragma unroll
        for (int kk = 0; kk < RK / 16; ++kk)
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            float2 v = make_float2(0.f, 0.f);
            if (real)
              asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(srck + 16 * kk + 8 * part + 2 * t));
            qkraw[h][kk][part] = v;
          }
      }
    }
  };
  auto pack_q = [&]() {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        qa[kk][h] = pack_bf16(qraw[h][kk][0].x, qraw[h][kk][0].y);
        qa[kk][2 + h] = pack_bf16(qraw[h][kk][1].x, qraw[h][kk][1].y);
      }
      if (RK > 0) {
#pragma unroll
        for (int kk = 0; kk < RK / 16; ++kk) {
          qka[kk][h] = pack_bf16(qkraw[h][kk][0].x, qkraw[h][kk][0].y);
          qka[kk][2 + h] = pack_bf16(qkraw[h][kk][1].x, qkraw[h][kk][1].y);
        }
      }
      m_used[h] = ninf; l_run[h] = 0.f;
    }
#pragma unroll
    for (int nt = 0; nt < kNO; ++nt) { o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f; }
#pragma unroll
    for (int nt = 0; nt < (kNL > 0 ? kNL : 1); ++nt) { olr[nt][0] = olr[nt][1] = olr[nt][2] = olr[nt][3] = 0.f; }
  };

  // start of this worker's range in a layer chunk: producer cursor, tile count; false when the range is empty
  int tl0 = 0;
  auto setup_chunk = [&](int ch) -> bool {
    const int chunk_base = ch * total32;
    g0 = chunk_base + w * G32;
    const int g1 = min(g0 + G32, chunk_base + total32);
    n = g1 > g0 ? g1 - g0 : 0;
    if (n == 0) return false;
    p_unit = g0 / T32;
    first_unit = p_unit;
    p_tl = g0 - p_unit * T32;
    tl0 = p_tl;
    p_page = (p_tl * kTK) / p.P; p_tok = (p_tl * kTK) % p.P;
    p_layer = p_unit / units_per_layer; p_kvh = (p_unit / p.row_blocks) % p.n_kv_local;
    p_issued = 0;
    return true;
  };

  // Launched as a programmatic dependent, everything up to pdl_wait() overlaps the tail of the previous kernel of the stream
  // (the merge of the previous layer, the projections of this one).  That includes the first bulk copies of the cache rows
  // that are CERTAINLY complete: p.stable_rows comes from the host, which tracks every page write of the pool with an
  // event (state.hpp: lorakv_pool::write_event) -- rows below it were written by work the host has seen complete, so no
  // assumption about the predecessor is needed.  A decode step appends one row: everything but the last tile of a unit
  // is prefetched while the predecessor is still finishing, and the first tile is consumed ~2 us earlier.
  const bool have0 = setup_chunk(0);
  if (have0 && producer && !PA) {
    const int pre = n < NS ? n : NS;
    while (p_issued < pre && (int64_t)(p_tl + 1) * kTK <= p.stable_rows) issue_next();
  }
  // from here on the predecessor's results are read (q, the newest cache rows, the page table entries of new pages)
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  LK_TRACE(8);

  // consumer cursor, carried incrementally like the producer's
  int c_stage = 0, c_wrap = 0;
  for (chunk = 0; chunk < p.n_chunks; ++chunk) {
  if (chunk == 0 ? !have0 : !setup_chunk(chunk)) continue;
  int u = first_unit;
  int tl = tl0;
  // Start-up order (measured with the phase trace of tools/probe_decode_trace.py): the query loads go out first -- once
  // every SM's bulk copies are in flight the memory system is saturated and a plain load waits ~2.4 us behind them, 1.1 us
  // on an idle one --, two stages are issued while they fly (0.4 us of issue work per stage: five bulk copies), then the
  // fragments are packed and the rest of the ring goes out.  First tile consumed ~1 us earlier than "Q, then four stages".
  cur_unit = u;
  load_q(u);
  LK_TRACE(14);
  const int pre = n < NS ? n : NS;
  if (producer)
    while (p_issued < (pre < 2 ? pre : 2)) { issue_next(); LK_TRACE(10); }
  pack_q();
  LK_TRACE(9);
  if (producer)
    while (p_issued < pre) issue_next();
  LK_TRACE(2);
  for (int i = 0; i < n; ++i) {
    // refill the stage released one iteration ago (tile p_issued goes where tile p_issued - NS was)
    if (producer && i >= 1 && p_issued < n) issue_next();
    const int s = c_stage;
    if (i == 0) LK_TRACE(3);
    ptx::mbar_wait(&full[s], (uint32_t)(c_wrap & 1));
    if (i == 0) LK_TRACE(4);

    const uint32_t sK = ring + (uint32_t)s * kStageBytes, sV = sK + kKvBytes, sLR = sV + kKvBytes;

    // ---- S = Q K^T : 16 rows x 16 KT keys ---------------------------------------------------
    constexpr int NT = 2 * KT;      // n8 tiles of S
    float sc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
    {
      const int key = (mi >> 1) * 8 + rr;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int chunk = 2 * kk + (mi & 1);
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const uint32_t addr = sK + (uint32_t)(chunk >> 3) * kBlockBytes + (uint32_t)(key + 16 * kt) * 128u +
                                (uint32_t)(((chunk & 7) ^ rr) << 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(addr, b0, b1, b2, b3);
          mma_bf16(sc[2 * kt], qa[kk], b0, b1);
          mma_bf16(sc[2 * kt + 1], qa[kk], b2, b3);
        }
      }
      if (RK > 0) {     // + Qk L_k^T: the L_k tile is [keys][RK] with 2 RK-byte rows, swizzled like every narrow page row
        const uint32_t sLK = sLR + kLrBytes;
#pragma unroll
        for (int kk = 0; kk < RK / 16; ++kk) {
          const int chunk = 2 * kk + (mi & 1);
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            uint32_t off = (uint32_t)(key + 16 * kt) * (2u * RK) + (uint32_t)chunk * 16u;
            off ^= ((off >> 7) & (uint32_t)(RK / 8 - 1)) << 4;
            uint32_t b0, b1, b2, b3;
            ldsm_x4(sLK + off, b0, b1, b2, b3);
            mma_bf16(sc[2 * kt], qka[kk], b0, b1);
            mma_bf16(sc[2 * kt + 1], qka[kk], b2, b3);
          }
        }
      }
    }

    // ---- online softmax (exp2 domain), rows g and g + 8 ------------------------------------------
    const int64_t key_base = (int64_t)tl * kTK + 2 * t;
    bool valid[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) valid[nt][e] = key_base + 8 * nt + e < p.L;
    float tmax[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float mx = ninf;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float v = valid[nt][e] ? sc[nt][2 * h + e] * p.scale_log2 : ninf;
          sc[nt][2 * h + e] = v;
          mx = fmaxf(mx, v);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      tmax[h] = mx;
    }
    const bool grow = tmax[0] > m_used[0] + kRescaleThreshold || tmax[1] > m_used[1] + kRescaleThreshold;
    if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float m_new = fmaxf(m_used[h], tmax[h]);
        const float alpha = (m_used[h] == ninf) ? 0.f : ex2(m_used[h] - m_new);
        m_used[h] = m_new;
        l_run[h] *= alpha;
#pragma unroll
        for (int nt = 0; nt < kNO; ++nt) { o[nt][2 * h] *= alpha; o[nt][2 * h + 1] *= alpha; }
#pragma unroll
        for (int nt = 0; nt < kNL; ++nt) { olr[nt][2 * h] *= alpha; olr[nt][2 * h + 1] *= alpha; }
      }
    }
    uint32_t pa[KT][4];
    {
      float pv[NT][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float x = valid[nt][e] ? ex2(sc[nt][2 * h + e] - m_used[h]) : 0.f;
            pv[nt][2 * h + e] = x;
            l_run[h] += x;
          }
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        pa[kt][0] = pack_bf16(pv[2 * kt][0], pv[2 * kt][1]);
        pa[kt][1] = pack_bf16(pv[2 * kt][2], pv[2 * kt][3]);
        pa[kt][2] = pack_bf16(pv[2 * kt + 1][0], pv[2 * kt + 1][1]);
        pa[kt][3] = pack_bf16(pv[2 * kt + 1][2], pv[2 * kt + 1][3]);
      }
    }

    // ---- O += P V_base, O_lr += P V_lr ---------------------------------------------------------------
    {
      const int key = (mi & 1) * 8 + rr;
#pragma unroll
      for (int np = 0; np < D / 16; ++np) {
        const int chunk = 2 * np + (mi >> 1);
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const uint32_t addr = sV + (uint32_t)(chunk >> 3) * kBlockBytes + (uint32_t)(key + 16 * kt) * 128u +
                                (uint32_t)(((chunk & 7) ^ rr) << 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(addr, b0, b1, b2, b3);
          mma_bf16(o[2 * np], pa[kt], b0, b1);
          mma_bf16(o[2 * np + 1], pa[kt], b2, b3);
        }
      }
      if (RP >= 16 && !PA) {
#pragma unroll
        for (int np = 0; np < RP / 16; ++np) {
          const int chunk = 2 * np + (mi >> 1);
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            uint32_t off = (uint32_t)(key + 16 * kt) * (2u * RP) + (uint32_t)chunk * 16u;
            off ^= ((off >> 7) & (uint32_t)(RP / 8 - 1)) << 4;
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(sLR + off, b0, b1, b2, b3);
            mma_bf16(olr[2 * np], pa[kt], b0, b1);
            mma_bf16(olr[2 * np + 1], pa[kt], b2, b3);
          }
        }
      }
      if (RP >= 16 && PA) {
        // rows g and g + 8 of this warp belong to entries ent_lo / ent_hi of the row block; one masked MMA pass per entry
        const int ent_lo = (wi * 16 + g) / p.group, ent_hi = (wi * 16 + g + 8) / p.group;
        const int e_first = (wi * 16) / p.group, e_last = min((wi * 16 + 15) / p.group, p.lr_per_block - 1);
        for (int e = e_first; e <= e_last; ++e) {
          const uint32_t sE = sLR + (uint32_t)e * kLrBytes;
          const uint32_t m_lo = ent_lo == e ? 0xffffffffu : 0u, m_hi = ent_hi == e ? 0xffffffffu : 0u;
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            const uint32_t pe[4] = {pa[kt][0] & m_lo, pa[kt][1] & m_hi, pa[kt][2] & m_lo, pa[kt][3] & m_hi};
#pragma unroll
            for (int np = 0; np < RP / 16; ++np) {
              const int chunk = 2 * np + (mi >> 1);
              uint32_t off = (uint32_t)(key + 16 * kt) * (2u * RP) + (uint32_t)chunk * 16u;
              off ^= ((off >> 7) & (uint32_t)(RP / 8 - 1)) << 4;
              uint32_t b0, b1, b2, b3;
              ldsm_x4_t(sE + off, b0, b1, b2, b3);
              mma_bf16(olr[2 * np], pe, b0, b1);
              mma_bf16(olr[2 * np + 1], pe, b2, b3);
            }
          }
        }
      }
    }

    // this warp is done with the stage
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (++c_stage == NS) { c_stage = 0; ++c_wrap; }
    if (++tl == T32) {
      tl = 0; ++u;
      if (i + 1 < n) { flush(); cur_unit = u; load_q(u); pack_q(); }
    }
    if (i == 0) LK_TRACE(5);
  }
  LK_TRACE(6);
  flush();
  LK_TRACE(7);
  }   // layer chunks
}

// ---- merge of the per-worker partials + up-projection epilogue -----------------------------------
struct DecodeMergeParams {
  const float* part;
  int D, RP, r, MW, group, n_kv_local, n_batch, rows_total, row_blocks;
  int64_t T, G, layer_begin, n_q_local;
  int max_seg;
  const int32_t* agent_ids;
  const float* b;        // [n_layers][n_agents][r][n_kv_local * d]
  const float* scale;    // [n_layers][n_agents]
  int64_t n_agents;
  float* out;            // [layers][n_batch][n_q_local * d]
  PeerOut peers;         // n > 0: the row goes to every rank's [layers][n_batch][n_q_total * d] buffer instead
  int agent_fixed;       // >= 0: every row belongs to this agent (prefill blocks: the batch axis is the position)
  int64_t units_per_chunk, n_workers;   // layer chunks of fla_decode_tma: partials are [chunk][worker][segment]
};

// Address of the output row of (layer, batch entry, local q head): the local slab, or -- when the step ends in the
// output gather -- the same row of the full-width buffer (the stores then fan out to every peer, store_row).
__device__ __forceinline__ int64_t merge_row_offset(const DecodeMergeParams& p, int64_t layer_rel, int entry, int64_t head) {
  if (p.peers.n == 0) return ((layer_rel * p.n_batch + entry) * p.n_q_local + head) * p.D;
  return ((layer_rel * p.n_batch + entry) * p.peers.n_q_total + p.peers.q_head_begin + head) * p.D;
}
__device__ __forceinline__ void store_out(const DecodeMergeParams& p, int64_t off, float v) {
  if (p.peers.n == 0) { p.out[off] = v; return; }
#pragma unroll
  for (int pe = 0; pe < kMaxPeers; ++pe)          // constant indices: the table stays in the parameter bank
    if (pe < p.peers.n) p.peers.dst[pe][off] = v;
}

constexpr int kMergeWarps = 8;

// One CTA per (query row, layer x kv head): the latency-optimised merge of a launch with few rows (one layer per launch:
// ~55 splits per row at cfg 2).  ONE global round trip after the attention kernel completes: warp w takes splits w, w + 8,
// ... and issues the loads of up to eight of them -- (m, l) and its lanes' columns of O / O_lr -- before using any; it
// reduces them relative to its own maximum, the warps' results meet in shared memory.  Everything that does not depend on
// the attention kernel happens BEFORE pdl_wait(): address arithmetic and this thread's column of B[agent] (static data), so
// under a programmatic dependent launch the CTA is resident and set up when the partials arrive.
// RMAX: rank bucket (the thread's B column lives in RMAX registers), COLS: ceil((D + RP) / 32).  Two CTAs per SM's worth of
// registers (<= 128 per thread): a merge CTA has to fit beside a 24K-register attention CTA -- beside the one it waits for and
// beside the next layer's, which sets itself up under this epilogue.  With 179 registers it did not, and two thirds of the
// next launch's CTAs started only after the merge had left their SM (phase trace, profiles/r2_decode_phase_trace.txt).
template <int RMAX, int COLS>
__global__ void __launch_bounds__(kMergeWarps * 32, 2) fla_decode_merge_kernel(const DecodeMergeParams p) {
  constexpr int kMaxCols = COLS;         // (D + RP) <= 192 columns / 32 lanes
  constexpr int kBatch = 8;              // splits of a warp in flight together
  constexpr int kMaxRank = RMAX;
  __shared__ float m_s[kMergeWarps], l_s[kMergeWarps];
  __shared__ float acc_s[kMergeWarps][192];
  __shared__ float tot_s[192];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  LK_MTRACE(0);
  const int rho = blockIdx.x;
  const int kvh = blockIdx.y % p.n_kv_local;
  const int64_t layer_rel = blockIdx.y / p.n_kv_local;
  const int rows_blk = 16 * p.MW;
  const int rb = rho / rows_blk, r_in = rho % rows_blk;
  const int64_t u = (layer_rel * p.n_kv_local + kvh) * p.row_blocks + rb;
  const int64_t ch = u / p.units_per_chunk, u_loc = u % p.units_per_chunk;    // layer chunk of the unit, unit inside it
  const int64_t w_lo = (u_loc * p.T) / p.G, w_hi = ((u_loc + 1) * p.T - 1) / p.G;
  const int ns = (int)(w_hi - w_lo + 1);
  const int PS = 4 + p.D + p.RP, C = p.D + p.RP;
  const float ninf = -std::numeric_limits<float>::infinity();
  // partial of split s: worker w_lo + s, segment = unit minus the worker's first unit.  Only the FIRST worker of a unit can
  // have started in an earlier unit (every later one starts inside it: segment 0), so one 64-bit division serves the row
  const int64_t seg_lo = u_loc - (w_lo * p.G) / p.T;
  const float* part0 = p.part + ((ch * p.n_workers + w_lo) * p.max_seg * rows_blk + r_in) * PS;
  const int64_t split_stride = (int64_t)p.max_seg * rows_blk * PS;
  const int64_t seg_off = seg_lo * rows_blk * PS;
  auto row_of = [&](int s) -> const float* { return part0 + s * split_stride + (s == 0 ? seg_off : 0); };
  // ---- epilogue operands that do not depend on the attention kernel ----
  const int gi = rho % p.group, entry = rho / p.group;
  const int64_t layer = p.layer_begin + layer_rel;
  const int64_t dkv = (int64_t)p.n_kv_local * p.D;
  const int agent = p.agent_fixed >= 0 ? p.agent_fixed : (p.agent_ids ? p.agent_ids[entry] : 0);
  const float* b = p.r > 0 ? p.b + ((layer * p.n_agents + agent) * p.r) * dkv + (int64_t)kvh * p.D : nullptr;
  const float scale = p.r > 0 ? p.scale[layer * p.n_agents + agent] : 0.f;
  const int64_t dst = merge_row_offset(p, layer_rel, entry, (int64_t)kvh * p.group + gi);
  // B[agent][k][tid] for the output column this thread finishes, in registers (r <= 64, launcher).  Not in shared memory: the
  // CTA must fit beside a 209 KB attention CTA to be resident while it waits (8 KB more and the overlap is lost: 27.7 -> 29.5 us)
  float bcol[kMaxRank];
  if (tid < p.D) {
#pragma unroll
    for (int k = 0; k < kMaxRank; ++k) bcol[k] = k < p.r ? __ldg(b + (int64_t)k * dkv + tid) : 0.f;
  }
  ptx::pdl_launch_dependents();          // the next layer's kernels may set themselves up under this epilogue
  LK_MTRACE(1);
  ptx::pdl_wait();                       // the partials of the attention kernel are complete and visible from here on
  LK_MTRACE(2);
  // ---- this warp's splits, kBatch at a time, all loads first ----
  float m_w = ninf, l_w = 0.f;
  float acc[kMaxCols];
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) acc[i] = 0.f;
  for (int s0 = warp; s0 < ns; s0 += kBatch * kMergeWarps) {
    float2 ml[kBatch];
    float v[kBatch][kMaxCols];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int sidx = s0 + j * kMergeWarps;
      const float* row = row_of(sidx < ns ? sidx : s0);
      ml[j] = sidx < ns ? *reinterpret_cast<const float2*>(row) : make_float2(ninf, 0.f);
#pragma unroll
      for (int i = 0; i < kMaxCols; ++i) {
        const int c = lane + 32 * i;
        v[j][i] = (sidx < ns && c < C) ? row[4 + c] : 0.f;
      }
    }
    float m_new = m_w;
#pragma unroll
    for (int j = 0; j < kBatch; ++j) m_new = fmaxf(m_new, ml[j].x);
    if (m_new == ninf) continue;         // only empty splits so far
    const float keep = (m_w == ninf) ? 0.f : exp2f(m_w - m_new);
    l_w *= keep;
#pragma unroll
    for (int i = 0; i < kMaxCols; ++i) acc[i] *= keep;
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      if (ml[j].x == ninf) continue;     // an empty split carries no accumulators: its values are never used
      const float wgt = exp2f(ml[j].x - m_new);
      l_w = fmaf(wgt, ml[j].y, l_w);
#pragma unroll
      for (int i = 0; i < kMaxCols; ++i) acc[i] = fmaf(wgt, v[j][i], acc[i]);
    }
    m_w = m_new;
  }
  if (lane == 0) { m_s[warp] = m_w; l_s[warp] = l_w; }
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) {
    const int c = lane + 32 * i;
    if (c < C) acc_s[warp][c] = acc[i];
  }
  __syncthreads();
  // ---- the warps' results relative to the row maximum ----
  float mx = m_s[0];
#pragma unroll
  for (int i = 1; i < kMergeWarps; ++i) mx = fmaxf(mx, m_s[i]);
  float wq[kMergeWarps], lsum = 0.f;
#pragma unroll
  for (int i = 0; i < kMergeWarps; ++i) {
    wq[i] = (m_s[i] == ninf) ? 0.f : exp2f(m_s[i] - mx);
    lsum = fmaf(wq[i], l_s[i], lsum);
  }
  if (tid < C) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kMergeWarps; ++i) t = fmaf(wq[i], acc_s[i][tid], t);
    tot_s[tid] = t;
  }
  __syncthreads();
  // ---- epilogue: o += (lr_scale * o_lr[k]) * B[agent][k,:], out = o / l (attention.hpp:244-259) ----
  if (tid < p.D) {
    float o = tot_s[tid];
#pragma unroll
    for (int k = 0; k < kMaxRank; ++k)
      if (k < p.r) o = fmaf(scale * tot_s[p.D + k], bcol[k], o);
    store_out(p, dst + tid, o / lsum);
  }
  LK_MTRACE(3);
}

template <int D, int RP, int MW, int KT, bool PA = false, int NW = kWarps, int RK = 0>
int launch_t(lorakv_ctx* ctx, const DecodeParams& dp, unsigned grid, size_t smem) {
  auto kern = fla_decode_tma_kernel<D, RP, MW, KT, PA, NW, RK>;
  static int attr_device = -1;         // once per instantiation: the attribute call costs more than the launch
  if (attr_device != ctx->device) {
    LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBudget));
    attr_device = ctx->device;
  }
  prof_mark(ctx, 0);
  LK_CUDA(launch_kernel(ctx, kern, dim3(grid), dim3(NW * 32), smem, true, dp));
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

// per-entry V_lr tiles (BaseShared batches): 16-key tiles for every worker width (the stage already carries one V_lr tile
// per entry)
template <int D, int RP>
int launch_mw_pa(lorakv_ctx* ctx, const DecodeParams& dp, unsigned grid, size_t smem, int mw, int kt = 1) {
  if (kt == 2) {           // 32-key tiles for the multi-warp workers when two stages of them fit (half the barrier round trips)
    switch (mw) {
      case 2: return launch_t<D, RP, 2, 2, true>(ctx, dp, grid, smem);
      case 4: return launch_t<D, RP, 4, 2, true>(ctx, dp, grid, smem);
      default: return launch_t<D, RP, 8, 2, true>(ctx, dp, grid, smem);
    }
  }
  switch (mw) {
    case 1: return launch_t<D, RP, 1, 1, true>(ctx, dp, grid, smem);
    case 2: return launch_t<D, RP, 2, 1, true>(ctx, dp, grid, smem);
    case 4: return launch_t<D, RP, 4, 1, true>(ctx, dp, grid, smem);
    default: return launch_t<D, RP, 8, 1, true>(ctx, dp, grid, smem);
  }
}
template <int D>
int launch_rp_pa(lorakv_ctx* ctx, const DecodeParams& dp, unsigned grid, size_t smem, int mw, int rp, int kt) {
  switch (rp) {
    case 16: return launch_mw_pa<D, 16>(ctx, dp, grid, smem, mw, kt);
    case 32: return launch_mw_pa<D, 32>(ctx, dp, grid, smem, mw, kt);
    default: return launch_mw_pa<D, 64>(ctx, dp, grid, smem, mw, kt);
  }
}

template <int D, int RP>
int launch_mw(lorakv_ctx* ctx, const DecodeParams& dp, unsigned grid, size_t smem, int mw, int kt, int rk = 0) {
  if (rk == 16) return launch_t<D, RP, 1, 2, false, wide_workers(D), 16>(ctx, dp, grid, smem);     // key-side low-rank term:
  if (rk == 32) return launch_t<D, RP, 1, 2, false, wide_workers(D), 32>(ctx, dp, grid, smem);     // single-warp wide workers only
  if (mw == 1) {
    if (kt == 2) return launch_t<D, RP, 1, 2, false, wide_workers(D)>(ctx, dp, grid, smem);
    return launch_t<D, RP, 1, 1>(ctx, dp, grid, smem);
  }
  if (kt == 2) {
    switch (mw) {
      case 2: return launch_t<D, RP, 2, 2>(ctx, dp, grid, smem);
      case 4: return launch_t<D, RP, 4, 2>(ctx, dp, grid, smem);
      default: return launch_t<D, RP, 8, 2>(ctx, dp, grid, smem);
    }
  }
  switch (mw) {
    case 2: return launch_t<D, RP, 2, 1>(ctx, dp, grid, smem);
    case 4: return launch_t<D, RP, 4, 1>(ctx, dp, grid, smem);
    default: return launch_t<D, RP, 8, 1>(ctx, dp, grid, smem);
  }
}

template <int D>
int launch_rp(lorakv_ctx* ctx, const DecodeParams& dp, unsigned grid, size_t smem, int mw, int kt, int rp, int rk) {
  switch (rp) {
    case 0: return launch_mw<D, 0>(ctx, dp, grid, smem, mw, kt, rk);
    case 16: return launch_mw<D, 16>(ctx, dp, grid, smem, mw, kt, rk);
    case 32: return launch_mw<D, 32>(ctx, dp, grid, smem, mw, kt, rk);
    default: return launch_mw<D, 64>(ctx, dp, grid, smem, mw, kt, rk);
  }
}

}  // namespace

// The same merge when a row has at most 32 partials (a whole decode step in one launch: ~5 per row): one WARP per
// (query row, layer x kv head) and no block-level barrier -- lanes over the splits for the maximum and the
// denominator, then lanes over the columns for the weighted sums.  A CTA per row spent its time in four
// __syncthreads with 250 of its 256 threads idle (31 us per cfg-2 step for 13 MB of partials).
__global__ void __launch_bounds__(kMergeWarps * 32) fla_decode_merge_warp_kernel(const DecodeMergeParams p, int64_t n_rows_units) {
  __shared__ float olr_s[kMergeWarps][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kMergeWarps + warp;
  if (gw >= n_rows_units) return;
  const int rho = (int)(gw % p.rows_total);
  const int64_t y = gw / p.rows_total;
  const int kvh = (int)(y % p.n_kv_local);
  const int64_t layer_rel = y / p.n_kv_local;
  const int rows_blk = 16 * p.MW;
  const int rb = rho / rows_blk, r_in = rho % rows_blk;
  const int64_t u = (layer_rel * p.n_kv_local + kvh) * p.row_blocks + rb;
  const int64_t ch = u / p.units_per_chunk, u_loc = u % p.units_per_chunk;    // layer chunk of the unit, unit inside it
  const int64_t w_lo = (u_loc * p.T) / p.G, w_hi = ((u_loc + 1) * p.T - 1) / p.G;
  const int ns = (int)(w_hi - w_lo + 1);                     // <= 32, checked by the launcher
  const int PS = 4 + p.D + p.RP, C = p.D + p.RP;
  const float ninf = -std::numeric_limits<float>::infinity();
  // partial of split s: worker w_lo + s, segment = unit minus the worker's first unit.  Only the FIRST worker of a unit can
  // have started in an earlier unit (every later one starts inside it: segment 0), so one 64-bit division serves the row
  // instead of one per split (they were half of the instructions this kernel executed)
  const int64_t seg_lo = u_loc - (w_lo * p.G) / p.T;
  const float* part0 = p.part + ((ch * p.n_workers + w_lo) * p.max_seg * rows_blk + r_in) * PS;
  const int64_t split_stride = (int64_t)p.max_seg * rows_blk * PS;
  const int64_t seg_off = seg_lo * rows_blk * PS;
  auto row_of = [&](int s) -> const float* { return part0 + s * split_stride + (s == 0 ? seg_off : 0); };
  ptx::pdl_launch_dependents();          // the next layer's kernels may set themselves up under this epilogue
  ptx::pdl_wait();                       // the partials of the attention kernel are complete and visible from here on
  float m = ninf, l = 0.f;
  if (lane < ns) { const float2 ml = *reinterpret_cast<const float2*>(row_of(lane)); m = ml.x; l = ml.y; }
  float mx = m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const float wgt = (m == ninf) ? 0.f : exp2f(m - mx);
  float lsum = wgt * l;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  constexpr int kMaxCols = 6;            // (D + RP) <= 192 columns / 32 lanes
  float acc[kMaxCols];
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) acc[i] = 0.f;
  // four splits per round so that their loads are in flight together (one at a time cost ~0.7 us of latency each);
  // an empty split carries no accumulators, so its values are never read (weight 0, predicate off)
  for (int s0 = 0; s0 < ns; s0 += 4) {
    float ws[4], v[4][kMaxCols];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int sidx = s0 + u;
      ws[u] = __shfl_sync(0xffffffffu, wgt, sidx & 31);
      if (sidx >= ns) ws[u] = 0.f;
      const float* row = row_of(sidx < ns ? sidx : 0) + 4;
#pragma unroll
      for (int i = 0; i < kMaxCols; ++i) {
        const int c = lane + 32 * i;
        v[u][i] = (ws[u] != 0.f && c < C) ? row[c] : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < kMaxCols; ++i) acc[i] = fmaf(ws[u], v[u][i], acc[i]);
  }
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) {
    const int c = lane + 32 * i;
    if (c >= p.D && c < C) olr_s[warp][c - p.D] = acc[i];
  }
  __syncwarp();
  // ---- epilogue: o += (lr_scale * o_lr[k]) * B[agent][k,:], out = o / l (attention.hpp:244-259) ----
  const int gi = rho % p.group, entry = rho / p.group;
  const int64_t layer = p.layer_begin + layer_rel;
  const int64_t dkv = (int64_t)p.n_kv_local * p.D;
  const int agent = p.agent_fixed >= 0 ? p.agent_fixed : (p.agent_ids ? p.agent_ids[entry] : 0);
  const float* b = p.r > 0 ? p.b + ((layer * p.n_agents + agent) * p.r) * dkv + (int64_t)kvh * p.D : nullptr;
  const float scale = p.r > 0 ? p.scale[layer * p.n_agents + agent] : 0.f;
  const int64_t dst = merge_row_offset(p, layer_rel, entry, (int64_t)kvh * p.group + gi);
  const float inv_l = 1.0f / lsum;
  // k outermost: one shared-memory read and one multiply per rank index, the (up to four) columns of a lane as
  // independent loads of the same B row -- the column-outer form re-read olr_s and recomputed the 64-bit row address per
  // (column, k) and was most of the ~5000 instructions a warp executed at rank 64
  const float* bp = b + lane;
  for (int k = 0; k < p.r; ++k, bp += dkv) {
    const float sk = scale * olr_s[warp][k];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < p.D) acc[i] = fmaf(sk, __ldg(bp + 32 * i), acc[i]);
  }
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) {
    const int c = lane + 32 * i;
    if (c < p.D) store_out(p, dst + c, acc[i] * inv_l);
  }
}

int launch_decode_merge(lorakv_ctx* ctx, const float* part, int d, int rp, int r, int mw, int group, int n_kv_local, int n_batch,
                        int rows_total, int row_blocks, int64_t T, int64_t G, int64_t layer_begin, int64_t n_q_local, int max_seg,
                        const int32_t* agent_ids_dev, const lorakv_adapters* adapters, float* out_dev, int64_t n_layers,
                        const PeerOut* peers, int agent_fixed, int64_t units_per_chunk, int64_t n_workers) {
  DecodeMergeParams mp;
  if (peers) mp.peers = *peers;
  mp.agent_fixed = agent_fixed;
  mp.units_per_chunk = units_per_chunk > 0 ? units_per_chunk : (int64_t)n_layers * n_kv_local * row_blocks;   // one chunk
  mp.n_workers = n_workers;
  mp.part = part; mp.D = d; mp.RP = rp; mp.r = r; mp.MW = mw; mp.group = group;
  mp.n_kv_local = n_kv_local; mp.n_batch = n_batch; mp.rows_total = rows_total;
  mp.row_blocks = row_blocks; mp.T = T; mp.G = G; mp.layer_begin = layer_begin; mp.n_q_local = n_q_local;
  mp.max_seg = max_seg; mp.agent_ids = agent_ids_dev;
  mp.b = adapters ? adapters->b : nullptr; mp.scale = adapters ? adapters->scale : nullptr;
  mp.n_agents = adapters ? adapters->n_agents : 1;
  mp.out = out_dev;
  const int ns_max = (int)((T - 1) / G + 2);
  dim3 mgrid((unsigned)rows_total, (unsigned)(n_layers * n_kv_local));
  if (d + rp > 192) return fail("decode merge: d_head + padded rank %d exceeds 192 columns", d + rp);
  // the same shared-memory carve-out as the attention kernels, so that the SMs are not reconfigured between the two
  // launches of every layer-step (and the merge CTAs can become resident beside the attention CTAs they wait for)
  static int carve_device = -1;
  if (carve_device != ctx->device) {
    LK_CUDA(cudaFuncSetAttribute(fla_decode_merge_warp_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    LK_CUDA(cudaFuncSetAttribute(fla_decode_merge_kernel<16, 5>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    LK_CUDA(cudaFuncSetAttribute(fla_decode_merge_kernel<16, 6>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    LK_CUDA(cudaFuncSetAttribute(fla_decode_merge_kernel<32, 6>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    LK_CUDA(cudaFuncSetAttribute(fla_decode_merge_kernel<64, 6>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    carve_device = ctx->device;
  }
  if (r > 64) return fail("decode merge: rank %d exceeds 64", r);
  // the output gather's overlapped handshake of the previous step guards the peers' buffers this epilogue stores into
  if (peers && peers->wait_event) LK_CUDA(cudaStreamWaitEvent(ctx->stream, static_cast<cudaEvent_t>(peers->wait_event), 0));
  // many rows (a whole step per launch): one warp per row, throughput; few rows (a layer per launch) or many splits: one CTA
  // per row, one global round trip
  if (ns_max <= 32 && rp <= 64 && (int64_t)rows_total * n_layers * n_kv_local > 1024) {
    const int64_t n = (int64_t)rows_total * n_layers * n_kv_local;
    LK_CUDA(launch_kernel(ctx, fla_decode_merge_warp_kernel, dim3((unsigned)((n + kMergeWarps - 1) / kMergeWarps)), dim3(kMergeWarps * 32), 0,
                          true, mp, n));
  } else {
    if (r <= 16 && d + rp <= 160) LK_CUDA(launch_kernel(ctx, fla_decode_merge_kernel<16, 5>, mgrid, dim3(kMergeWarps * 32), 0, true, mp));
    else if (r <= 16) LK_CUDA(launch_kernel(ctx, fla_decode_merge_kernel<16, 6>, mgrid, dim3(kMergeWarps * 32), 0, true, mp));
    else if (r <= 32) LK_CUDA(launch_kernel(ctx, fla_decode_merge_kernel<32, 6>, mgrid, dim3(kMergeWarps * 32), 0, true, mp));
    else LK_CUDA(launch_kernel(ctx, fla_decode_merge_kernel<64, 6>, mgrid, dim3(kMergeWarps * 32), 0, true, mp));
  }
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

bool lr_fits_l2(const PagedAttnCall& c, int64_t lr_bytes_per_layer) {
  return (c.layer_end - c.layer_begin) * lr_bytes_per_layer <= c.pool->ctx->l2_bytes * 6 / 10;
}
int64_t lr_chunk_budget(const PagedAttnCall& c) { return c.pool->ctx->l2_bytes * 28 / 100; }

bool decode_tma_per_entry_lr_supported(const PagedAttnCall& c) {
  if (!decode_tma_supported(c) || c.pool->r_pad < 16) return false;
  const int64_t group = c.n_q_local / c.pool->n_kv_local;
  return group >= 1 && (16 % group == 0 || group % 16 == 0) && group <= 128;   // a batch entry's rows never straddle a 16-row warp tile unevenly
}

bool decode_tma_supported(const PagedAttnCall& c) {
  const lorakv_pool* pool = c.pool;
  if (pool->rk_pad > 0) {      // key-side low-rank term: built for the single-warp wide workers (<= 16 query rows per kv head)
    const int64_t group = pool->n_kv_local > 0 ? c.n_q_local / pool->n_kv_local : 0;
    if (c.per_entry_lr || c.n_batch * group > 16 || pool->P % (2 * kKeyStep) != 0 || (pool->rk_pad != 16 && pool->rk_pad != 32)) return false;
  }
  const int64_t d = pool->dims.d_head, rp = pool->r_pad;
  if (pool->dims.dtype != LORAKV_BF16) return false;       // fp32 pages keep the 1e-4 contract on FFMA
  if (c.rows_per_entry != 1 || c.query_offset != c.L - 1) return false;   // decode only
  if (d != 64 && d != 128) return false;
  if (!(rp == 0 || rp == 16 || rp == 32 || rp == 64)) return false;
  if (pool->P % kKeyStep != 0) return false;             // a tile (16 or 32 keys) never straddles a page
  if (c.L < 1 || c.n_batch < 1) return false;
  return true;
}

int launch_decode_tma(const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const int d = (int)pool->dims.d_head, r = (int)pool->dims.rank, rp = (int)pool->r_pad;
  const int64_t n_layers = c.layer_end - c.layer_begin;
  const int group = (int)(c.n_q_local / pool->n_kv_local);
  const int64_t rows_total = c.n_batch * group;
  if (r > 0 && !c.adapters) return fail("paged attention: rank %lld cache needs adapter tables", (long long)r);
  int mw = 1;
  while (16 * mw < rows_total && mw < 8) mw *= 2;
  const int rows_blk = 16 * mw;
  const int row_blocks = (int)((rows_total + rows_blk - 1) / rows_blk);
  const bool pa = c.per_entry_lr && rp > 0;
  const int lr_per_block = pa ? (int)std::min<int64_t>(rows_blk / group, c.n_batch) : 1;   // V_lr tiles per stage
  // 32-key tiles whenever a page holds them; single-warp workers then run three (d_head 128) or four (64) per CTA
  // per-entry V_lr tiles: 32-key tiles for the multi-warp workers too whenever two stages of them fit -- half the barrier round
  // trips per key and twice the MMAs between them (cfg-5 shard, 16 agents x rank 32: 1.76 -> 1.10 ms per step, 0.57 -> 0.91 of
  // the HBM peak; LORAKV_PA_KT1=1 keeps 16-key tiles for A/B runs)
  static const bool pa_kt1 = std::getenv("LORAKV_PA_KT1") && std::getenv("LORAKV_PA_KT1")[0] == '1';
  const bool pa_wide = pa && !pa_kt1 && mw >= 2 && pool->P % (2 * kKeyStep) == 0 &&
                       (size_t)(kWarps / mw) * 2 * (2 * kKeyStep * (4 * d + 2 * rp * lr_per_block)) <= (size_t)kRingBudget;
  const int kt = ((!pa && pool->P % (2 * kKeyStep) == 0) || pa_wide) ? 2 : 1;
  const int workers_per_cta = (mw == 1 && kt == 2) ? wide_workers(d) : kWarps / mw;
  const int tk = kKeyStep * kt;
  const int rk = (int)pool->rk_pad;
  const uint32_t stage_bytes = tk * (4 * d + 2 * rp * lr_per_block + 2 * rk);
  if (pa && (size_t)workers_per_cta * 2 * stage_bytes > (size_t)kRingBudget)
    return fail("decode over per-agent low-rank caches: %d entries x rank %d do not fit two stages per worker", lr_per_block, rp);
  int n_stages = (int)(kRingBudget / (workers_per_cta * stage_bytes));
  if (n_stages > kMaxStages) n_stages = kMaxStages;
  const size_t smem = (size_t)workers_per_cta * n_stages * stage_bytes;

  const int64_t T = (c.L + tk - 1) / tk;
  // V_lr is shared by the kv heads of a layer (kernels.hpp: lr_fits_l2).  When the launch's low-rank cache does not
  // fit in L2, the layers are cut into the fewest equal chunks whose share does; every worker walks the chunks in
  // order, so only a chunk's V_lr is live at a time and DRAM serves it once instead of once per kv head.
  int n_chunks = 1;
  // (per-entry V_lr: every agent of the batch has its own cache, all of them are shared by the kv heads of the layer)
  const int64_t lr_layer_bytes = c.L * rp * 2 * (pa ? c.n_batch : 1);
  // (worth it from four kv heads per GPU on -- with two, the re-read it saves is ~5 % of the bytes and the pipeline
  // restart per chunk costs as much: cfg 4 on 4 GPUs 0.478 ms chunked vs 0.434 ms not -- and while a worker still
  // gets a few dozen tiles per chunk)
  if (!pa && rp > 0 && pool->n_kv_local >= 4 && !lr_fits_l2(c, lr_layer_bytes)) {
    int nc_pick = (int)n_layers;
    for (int64_t nc = 2; nc <= n_layers; ++nc)
      if (n_layers % nc == 0 && (n_layers / nc) * lr_layer_bytes <= lr_chunk_budget(c)) { nc_pick = (int)nc; break; }
    const int64_t tiles_per_worker = (n_layers / nc_pick) * pool->n_kv_local * row_blocks * T / ((int64_t)ctx->sm_count * workers_per_cta);
    if (tiles_per_worker >= 32) n_chunks = nc_pick;
  }
  const int64_t units = n_layers * pool->n_kv_local * row_blocks;
  const int64_t units_per_chunk = units / n_chunks;
  const int64_t total = units_per_chunk * T;             // tiles of one chunk
  const int64_t max_workers = (int64_t)ctx->sm_count * workers_per_cta;
  int64_t G = (total + max_workers - 1) / max_workers;
  if (G < 4) G = 4;
  const int64_t n_workers = (total + G - 1) / G;
  const unsigned grid = (unsigned)((n_workers + workers_per_cta - 1) / workers_per_cta);
  const int max_seg = (int)((G + T - 2) / T + 1);
  if ((total + G) * n_chunks >= ((int64_t)1 << 31)) return fail("decode: %lld key tiles in one launch exceed the kernel's 32-bit tile arithmetic", (long long)(total * n_chunks));
  const int PS = 4 + d + rp;
  const size_t part_bytes = (size_t)n_chunks * n_workers * max_seg * rows_blk * PS * sizeof(float);
  LK_TRY(scratch_reserve(ctx, ctx->work, part_bytes));

  DecodeParams dp;
  dp.k_pages = static_cast<const __nv_bfloat16*>(pool->k_pages);
  dp.v_pages = static_cast<const __nv_bfloat16*>(pool->v_pages);
  dp.lr_pages = static_cast<const __nv_bfloat16*>(pool->lr_pages);
  dp.kv_table = pool->kv_space.dev_table + c.kv_set * pool->kv_space.max_pages;
  dp.lr_table = rp > 0 ? pool->lr_space.dev_table + c.lr_set * pool->lr_space.max_pages : nullptr;
  dp.kv_layer_stride = pool->kv_layer_stride(); dp.kv_head_stride = pool->kv_head_stride();
  dp.kv_page_stride = pool->kv_page_stride();
  dp.lr_layer_stride = pool->lr_layer_stride(); dp.lr_page_stride = pool->lr_page_stride();
  dp.P = (int)pool->P; dp.group = group; dp.n_kv_local = (int)pool->n_kv_local; dp.n_batch = (int)c.n_batch;
  dp.rows_total = (int)rows_total; dp.row_blocks = row_blocks;
  dp.n_pages = (int)((c.L + pool->P - 1) / pool->P);
  dp.L = c.L; dp.layer_begin = c.layer_begin; dp.n_q_local = c.n_q_local;
  dp.T = T; dp.total_tiles = total; dp.G = G; dp.max_seg = max_seg; dp.n_stages = n_stages;
  dp.n_chunks = n_chunks; dp.n_workers = n_workers;
  dp.scale_log2 = (float)((1.0 / sqrt((double)d)) * 1.4426950408889634);
  dp.l2_policy = ptx::kEvictFirst;      // the cache is streamed once per step: do not let it push the partials and q out of L2
  dp.lr_policy = (n_chunks > 1 || lr_fits_l2(c, lr_layer_bytes)) ? ptx::kEvictLast : ptx::kEvictFirst;
  dp.q = c.q_dev; dp.part = static_cast<float*>(ctx->work.ptr);
  dp.lr_tables = pool->lr_space.dev_table; dp.agent_ids = c.agent_ids_dev;
  dp.lr_max_pages = (int)pool->lr_space.max_pages; dp.lr_per_block = lr_per_block;
  dp.identity = (pool->kv_space.identity(c.kv_set, dp.n_pages) ? 1 : 0) | ((rp > 0 && !pa && pool->lr_space.identity(c.lr_set, dp.n_pages)) ? 2 : 0) |
                ((rk > 0 && pool->lk_space.identity(0, dp.n_pages)) ? 4 : 0);
  dp.lk_pages = static_cast<const __nv_bfloat16*>(pool->lk_pages); dp.lk_table = pool->lk_space.dev_table;
  dp.lk_layer_stride = pool->lk_layer_stride(); dp.lk_page_stride = pool->lk_page_stride(); dp.qk = c.qk_dev;
  if (rk > 0 && !c.qk_dev) return fail("decode: the key-side low-rank term needs the projected queries (launch_qk_project)");
  if (const char* e = std::getenv("LORAKV_NO_PAGE_IDENTITY")) if (e[0] == '1') dp.identity = 0;
  // rows the kernel may prefetch before its dependent-launch wait: needs the identity tables (a new page's table entry
  // arrives with the predecessor's work) and a host-verified completion of every earlier page write
  dp.stable_rows = (ctx->speculate && !pa && (dp.identity & 1) && (rp == 0 || (dp.identity & 2)) && (rk == 0 || (dp.identity & 4)))
                       ? stable_rows(pool, c.L) : 0;
  if (pa) {
    // an entry's V_lr tile is read once per kv head of the layer: with one kv head per GPU it streams (evict-first); with
    // several, the policy chosen above keeps the batch's low-rank caches L2-resident when the launch's share fits (cfg 2 under
    // BaseShared: 0.93 -> 0.97 of the HBM peak)
    if (pool->n_kv_local == 1) dp.lr_policy = ptx::kEvictFirst;
    if (d == 128) LK_TRY(launch_rp_pa<128>(ctx, dp, grid, smem, mw, rp, kt));
    else LK_TRY(launch_rp_pa<64>(ctx, dp, grid, smem, mw, rp, kt));
  } else if (d == 128) LK_TRY(launch_rp<128>(ctx, dp, grid, smem, mw, kt, rp, rk));
  else LK_TRY(launch_rp<64>(ctx, dp, grid, smem, mw, kt, rp, rk));

  LK_TRY(launch_decode_merge(ctx, dp.part, d, rp, r, mw, group, (int)pool->n_kv_local, (int)c.n_batch, (int)rows_total, row_blocks,
                             T, G, c.layer_begin, c.n_q_local, max_seg, c.agent_ids_dev, c.adapters, c.out_dev, n_layers, c.peers, -1,
                             units_per_chunk, n_workers));
  ctx->last_kernel = n_chunks > 1 ? "fla_decode_tma (layer chunks)" : "fla_decode_tma";
  return LORAKV_OK;
}

}  // namespace lk

#ifdef LK_DECODE_TRACE
extern "C" int lorakv_debug_merge_trace(unsigned long long* out, int n_words) {
  return cudaMemcpyFromSymbol(out, lk::g_merge_trace, sizeof(unsigned long long) * (size_t)n_words) == cudaSuccess ? 0 : 1;
}
extern "C" int lorakv_debug_decode_trace(unsigned long long* out, int n_words) {
  return cudaMemcpyFromSymbol(out, lk::g_decode_trace, sizeof(unsigned long long) * (size_t)n_words) == cudaSuccess ? 0 : 1;
}
#endif
