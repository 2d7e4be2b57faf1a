// fla_prefill_umma.cu -- Flash-LoRA-Attention prefill / append-step attention on the 5th-generation
// tensor cores: tcgen05.mma with accumulators in TMEM, K / V_base / V_lr tiles staged by the TMA
// engine (cp.async.bulk) straight from the pre-swizzled bf16 pages (page_layout.cuh).
//
// What it computes: gqa_attention (proj/include/lorakv/attention.hpp:332-363) for ONE agent on ONE layer
// with L_c query rows at positions [query_offset, query_offset + L_c) of the cached trajectory
// (engine.hpp:440-443 in StepMode::Prefill), i.e. per q head flash_lora_attention (:210-268):
//   S = mask(Q K^T) / sqrt(d), online softmax, O += P V_base (d wide), O_lr += P V_lr (r wide),
//   epilogue o += (lr_scale * o_lr[p]) * B[p,:], out = o / l                       (:244-259)
//
// Mapping.  One CTA owns the g q heads of one kv head for PB = 128 / g consecutive query positions:
// the 128 MMA rows are (head-in-group, position), so a K/V tile is fetched once for the whole group
// (the reference re-reads it per q head, :347-361).  Keys are visited up to the causal boundary of the
// CTA's last row; only the boundary tiles pay for the mask.
//
// Roles (352 threads):
//   warps 0-7  softmax + correction + epilogue.  A softmax tile is 128 rows x 64 keys; thread (w, lane)
//              owns the whole row 32 (w % 4) + lane of it (64 scores in registers, no cross-thread
//              reduction).  Warps 0-3 take the even tiles, warps 4-7 the odd ones: the two warps that
//              share a scheduler (w and w + 4: same TMEM lanes) are always half a tile apart, so one
//              warp's TMEM load / row max / bookkeeping runs under the other's exp phase and the MUFU
//              (16 ex2 / clk / SM -- the longest per-tile resource next to the tensor pipe) never idles.
//              The running row maximum is handed from tile j to tile j + 1 through shared memory, ordered by an
//              mbarrier per (warp pair, direction): 32 arrivals by the owner of j, a parity wait by the owner of j + 1.
//   warp 8/10  TMA producers: bulk copies of K (warp 8) and of V_base + V_lr (warp 10) into 3-stage rings
//              of 128-key stages, mbarrier tracked, independent of each other
//   warp 9     MMA issuer (one elected thread): S(j) = Q K_j^T (N = 64) into one of FOUR TMEM S buffers,
//              O += P_j V_j and O_lr += P_j V_lr_j; issue order S0 S1 S2 | PV0 S3 | PV1 S4 | ... so three
//              score tiles are always in flight ahead of the softmax warps
// TMEM (512 columns): S0..S3 [0,256) 64 each | O [256,256+D) | O_lr [384,384+RP) | Q [448,448+D/2)
// Q and P never touch shared memory: both are written to TMEM as packed bf16 pairs (tcgen05.st) and fed
// to tcgen05.mma as the A operand from TMEM; P(j) overwrites the first 32 columns of the S buffer it was
// computed from.  Shared memory then carries only the K / V / V_lr tiles -- with A in shared memory a
// 128x128x16 MMA needs 8 KB per 64 cycles, the whole 128 B/clk of the SM, and the kernel was bound by
// shared-memory bandwidth (ncu, profiles/r1_ncu_prefill_umma_v1.txt).  Masked entries are exact zeros
// and never exponentiated (attention.hpp:171).  Rescaling of O / O_lr is lazy: only when a row's running
// max grows by more than 8 (log2 units), which leaves the result unchanged; the thread that sees the
// growth waits for PV(j-1), rescales its row and only then hands the new maximum on.
#include <cuda_bf16.h>

#include <limits>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kBM = 128;            // MMA rows per CTA
constexpr int kBN = 128;            // keys per K / V stage in shared memory
constexpr int kSN = 64;             // keys per softmax tile (one S buffer in TMEM)
constexpr int kThreads = 352;        // 8 softmax warps + K producer + MMA issuer + V producer
constexpr int kMaxStages = 3;
constexpr float kRescaleThreshold = 8.0f;

struct PrefillParams {
  const __nv_bfloat16 *k_pages, *v_pages, *lr_pages;
  const int32_t *kv_table, *lr_table;
  int64_t kv_layer_off, kv_head_stride, kv_page_stride, lr_layer_off, lr_page_stride;   // elements
  int P, group, n_kv_local, n_pages, r;
  int64_t L, L_c, query_offset, n_q_local;
  int n_qblocks;
  // decode mode (kDecode): one CTA = (layer, kv head, key split); rows = (batch entry, head in group)
  int n_batch, rows_total, splits, tiles_per_split;
  int64_t kv_layer_stride, lr_layer_stride, layer_begin_rel;
  float* part;          // [units * splits][128][4 + D + RP] partial (m, l, O, O_lr), merged by fla_decode_merge
  float scale_log2, lr_scale;
  const float* q;       // [L_c][n_q_local * D]
  const float* b;       // [r][n_kv_local * D] of this (layer, agent)
  // key-side low-rank term (template RK > 0; kernels.hpp: KeyLowRank): L_k tiles ride in the K stage, the queries projected
  // through B_k (launch_qk_project) sit in TMEM beside Q: RK / 16 more k steps of the score chain, S = Q K^T + Qk L_k^T
  const __nv_bfloat16* lk_pages; const int32_t* lk_table; int64_t lk_layer_off, lk_layer_stride, lk_page_stride;
  const float* qk;      // [layers][n_batch][rows][n_q_local][RK]
  float* out;           // [L_c][n_q_local * D]
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// (a, b) <- (a, b) * s + c and (x, y) += (a, b) as ONE packed instruction each (fma.rn.f32x2 / add.rn.f32x2, sm_100): the same
// roundings as the scalar forms, half the instructions -- the softmax warps execute ~290 instructions per thread and tile, and
// under the power cap an instruction not issued is time
__device__ __forceinline__ void ffma2(float& a, float& b, float s, float c) {
  asm("{\n\t.reg .b64 x, y, z;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 y, {%2, %2};\n\tmov.b64 z, {%3, %3};\n\t"
      "fma.rn.f32x2 x, x, y, z;\n\tmov.b64 {%0, %1}, x;\n\t}"
      : "+f"(a), "+f"(b) : "f"(s), "f"(c));
}
__device__ __forceinline__ void fadd2(float& x, float& y, float a, float b) {
  asm("{\n\t.reg .b64 u, v;\n\tmov.b64 u, {%0, %1};\n\tmov.b64 v, {%2, %3};\n\tadd.rn.f32x2 u, u, v;\n\tmov.b64 {%0, %1}, u;\n\t}"
      : "+f"(x), "+f"(y) : "f"(a), "f"(b));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

#ifdef LK_PREFILL_TRACE
// debug build only (make EXTRA=-DLK_PREFILL_TRACE): clock64 stamps of ONE CTA (blockIdx.x == gridDim.x / 2) per softmax tile,
// tools/probe_prefill_trace.py.  Slots: 0 score chain about to be issued (MMA thread, K stage there), 1 P V about to be issued
// (P and V there, fence done), 8 its MMAs issued, 9 its commits issued, 10 / 11 the same for the score chain; softmax warp 0 / 4
// lane 0: 2 S seen, 3 row maximum done, 4 partner's maximum seen, 5 exponentials done, 6 P stored and published
__device__ long long g_prefill_trace[2048 * 16];
#define LK_PTRACE(tile, slot)                                                                           \
  do {                                                                                                  \
    if (blockIdx.x == gridDim.x / 2 && (tile) < 2048) g_prefill_trace[(tile) * 16 + (slot)] = clock64(); \
  } while (0)
#else
#define LK_PTRACE(tile, slot)
#endif

struct Barriers {
  uint64_t q_full, p_full[4], pv_done[4], all_done;
  uint64_t k_full[kMaxStages], k_empty[kMaxStages], v_full[kMaxStages], v_empty[kMaxStages], s_full[4], hand[8];
};

// kDecode = false: prefill block (rows = head x position, causal mask, final output)
// kDecode = true : batched decode for many rows per kv head (rows = batch entry x head, all at position L-1);
//                  a CTA streams one split of one (layer, kv head) and writes an un-normalised partial
template <int D, int RP, bool kDecode, int RK = 0>
__global__ void __launch_bounds__(kThreads, 1) fla_prefill_umma_kernel(const PrefillParams p) {
  static_assert(RK == 0 || RK == 16 || RK == 32, "key-side rank: one or two k steps");
  static_assert(RK == 0 || D == 64 || RP <= 32, "TMEM: Qk sits behind O_lr at d_head 128");
  constexpr int kQBlocks = D / 64;                           // 64-column K-blocks of Q / K; 64-column N-blocks of V
  constexpr uint32_t kBlkBytes = kBN * 128;                  // one [128 rows][64] bf16 block = 16 KB
  constexpr uint32_t kKBytes = kQBlocks * kBlkBytes;         // K stage == V stage bytes
  constexpr uint32_t kLrRow = 2 * RP;                        // bytes of one V_lr row
  constexpr uint32_t kLrBytes = kBN * kLrRow;
  constexpr uint32_t kLkRow = 2 * RK;                        // bytes of one L_k row
  constexpr uint32_t kLkBytes = kBN * kLkRow;
  constexpr uint32_t kTmemS = 0, kTmemO = 256, kTmemLr = 384, kTmemQ = 448;
  constexpr uint32_t kTmemQk = D == 64 ? 480 : 384 + RP;     // 16 columns: Qk as packed bf16 pairs, zero padded
  // K / V ring depth: three stages hide the L2 latency of a stage behind two stages of work; the widest
  // configuration (d 128, rank 64) only has room for two
  constexpr int kStages = (2 * 3 * kKBytes + 3 * kLrBytes + 3 * kLkBytes + 1024 <= 227 * 1024 - 4096) ? 3 : 2;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ Barriers bars;
  __shared__ uint32_t tmem_base_s;
  __shared__ float m_s[kBM];            // running row maximum: owner of tile j -> owner of tile j + 1 (bars.hand orders it)
  __shared__ float l_s[2][kBM];         // [softmax warpgroup][row]: partial row sums for the epilogue ...
  __shared__ float mref_s[2][kBM];      // ... and the maximum each of them is relative to
  unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sK = smem;                          // kStages stages each
  unsigned char* sV = sK + kStages * kKBytes;
  unsigned char* sLR = sV + kStages * kKBytes;
  unsigned char* sLK = sLR + kStages * kLrBytes;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) LK_PTRACE(2047, 0);          // CTA-level stamps live in row 2047: 0 entry, 1 set-up done, 2 predecessor complete,
                                             // 3 Q in TMEM, 4 last P V complete, 5 epilogue operands staged, 6 rows stored, 7 exit
  // ---- what this CTA owns: n_tiles softmax tiles of kSN keys starting at key tile_begin * kSN ----
  int PB, kvh, n_tiles, tile_begin;
  int64_t q0, rows_here, kv_layer_off, lr_layer_off, lk_layer_off, mask_from;   // mask_from: first key that some row cannot see
  int unit = 0, split = 0, layer_rel = 0;
  if constexpr (!kDecode) {
    PB = kBM / p.group;                                           // query positions per CTA
    // one kv head at a time, heavy (late) blocks first inside it: the CTAs in flight share ONE head's K / V, which stays in
    // L2 (with the head index fastest all heads streamed at once: 3.0 GB of DRAM reads per layer for 134 MB of cache)
    kvh = (int)(blockIdx.x / p.n_qblocks);
    const int qb = p.n_qblocks - 1 - (int)(blockIdx.x % p.n_qblocks);
    q0 = (int64_t)qb * PB;
    rows_here = min((int64_t)PB, p.L_c - q0);                     // real positions in this block
    const int64_t last_visible_cta = p.query_offset + q0 + rows_here - 1;
    n_tiles = (int)(last_visible_cta / kSN) + 1;
    tile_begin = 0;
    kv_layer_off = p.kv_layer_off; lr_layer_off = p.lr_layer_off; lk_layer_off = p.lk_layer_off;
    mask_from = p.query_offset + q0 + 1;
  } else {
    PB = 1; q0 = 0; rows_here = p.rows_total;
    unit = (int)(blockIdx.x / p.splits); split = (int)(blockIdx.x % p.splits);
    layer_rel = unit / p.n_kv_local; kvh = unit % p.n_kv_local;
    const int total_tiles = (int)((p.L + kSN - 1) / kSN);
    tile_begin = split * p.tiles_per_split * (kBN / kSN);         // the host splits in stages of kBN keys
    n_tiles = min(p.tiles_per_split * (kBN / kSN), total_tiles - tile_begin);
    if (n_tiles < 0) n_tiles = 0;
    kv_layer_off = p.kv_layer_off + (int64_t)layer_rel * p.kv_layer_stride;
    lr_layer_off = p.lr_layer_off + (int64_t)layer_rel * p.lr_layer_stride;
    lk_layer_off = p.lk_layer_off + (int64_t)layer_rel * p.lk_layer_stride;
    mask_from = p.L;
  }
  const int n_stages_needed = (n_tiles + 1) / 2;                  // kBN-key stages the producers stream

  if (tid == 0) {
    ptx::mbar_init(&bars.q_full, 256);
    for (int s = 0; s < 4; ++s) ptx::mbar_init(&bars.p_full[s], 128);
    for (int s = 0; s < 4; ++s) ptx::mbar_init(&bars.pv_done[s], 1);
    ptx::mbar_init(&bars.all_done, 1);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&bars.k_full[s], 1); ptx::mbar_init(&bars.k_empty[s], 1);
      ptx::mbar_init(&bars.v_full[s], 1); ptx::mbar_init(&bars.v_empty[s], 1);
    }
    for (int s = 0; s < 4; ++s) ptx::mbar_init(&bars.s_full[s], 1);
    for (int s = 0; s < 8; ++s) ptx::mbar_init(&bars.hand[s], 32);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc(&tmem_base_s, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  if (tid == 0) LK_PTRACE(2047, 1);
  // launched as a programmatic dependent (decode mode: one launch per layer; prefill: behind the projections): barrier
  // set-up and the TMEM allocation above ran under the predecessor's tail; its results (q, fresh cache rows) are read below
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  if (tid == 0) LK_PTRACE(2047, 2);

  if (warp == 8 || warp == 10) {
    // ===================== TMA producers: warp 8 streams K, warp 10 streams V_base + V_lr =====================
    if (ptx::elect_one()) {
      const bool is_k = warp == 8;
      const int tpc = p.P < kBN ? p.P : kBN;           // tokens per bulk copy
      const int n_copies = kBN / tpc;
      uint64_t* full = is_k ? bars.k_full : bars.v_full;
      uint64_t* empty = is_k ? bars.k_empty : bars.v_empty;
      unsigned char* ring = is_k ? sK : sV;
      const __nv_bfloat16* pages = is_k ? p.k_pages : p.v_pages;
      const int64_t stage_key0 = (int64_t)tile_begin * kSN;
      for (int j = 0; j < n_stages_needed; ++j) {
        const int s = j % kStages;
        if (j >= kStages) ptx::mbar_wait(&empty[s], (uint32_t)(((j / kStages) & 1) ^ 1));   // the phase that freed the stage
        ptx::mbar_arrive_expect_tx(&full[s], is_k ? kKBytes + kLkBytes : kKBytes + kLrBytes);
        for (int i = 0; i < n_copies; ++i) {
          const int64_t key0 = stage_key0 + (int64_t)j * kBN + (int64_t)i * tpc;
          int page = (int)(key0 / p.P);
          const int tok0 = (int)(key0 % p.P);
          if (page >= p.n_pages) page = p.n_pages - 1;  // wholly masked keys: any finite rows will do
          const int64_t base = kv_layer_off + (int64_t)kvh * p.kv_head_stride + (int64_t)p.kv_table[page] * p.kv_page_stride +
                               (int64_t)tok0 * 64;
#pragma unroll
          for (int b = 0; b < kQBlocks; ++b)
            bulk_g2s(ptx::smem_u32(ring + s * kKBytes + b * kBlkBytes + i * tpc * 128), pages + base + (int64_t)b * p.P * 64,
                     (uint32_t)tpc * 128u, &full[s]);
          if (RP > 0 && !is_k) {
            const int64_t lr_base = lr_layer_off + (int64_t)p.lr_table[page] * p.lr_page_stride + (int64_t)tok0 * RP;
            bulk_g2s(ptx::smem_u32(sLR + s * kLrBytes + i * tpc * kLrRow), p.lr_pages + lr_base, (uint32_t)tpc * kLrRow, &full[s]);
          }
          if (RK > 0 && is_k) {
            const int64_t lk_base = lk_layer_off + (int64_t)p.lk_table[page] * p.lk_page_stride + (int64_t)tok0 * RK;
            bulk_g2s(ptx::smem_u32(sLK + s * kLkBytes + i * tpc * kLkRow), p.lk_pages + lk_base, (uint32_t)tpc * kLkRow, &full[s]);
          }
        }
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer =====================
    // elect.sync (not `lane == 0`): the compiler then knows one thread of a converged warp runs this
    // block and emits straight-line UTCHMMA / UTCBAR; under `lane == 0` every tcgen05 instruction was
    // wrapped in an ELECT / BRA.U.ANY waterfall loop (~80 cycles per MMA, the issue thread became the
    // bottleneck of the whole CTA: ncu source view, profiles/r1_ncu_prefill_umma_v5_elect.txt)
    if (ptx::elect_one()) {
      // The issue thread is the scarcest resource of the CTA (one instruction every few cycles): everything
      // that does not change per tile is folded into descriptor words computed once, a tile only adds its
      // stage offset to the low word (the 14-bit start-address field, units of 16 bytes).
      const uint32_t idesc_s = ptx::instr_desc_bf16(kBM, kBN, ptx::kMajorK, ptx::kMajorK);     // S of TWO tiles at once
      const uint32_t idesc_o = ptx::instr_desc_bf16(kBM, D, ptx::kMajorK, ptx::kMajorMN);
      const uint32_t idesc_lr = ptx::instr_desc_bf16(kBM, RP > 0 ? RP : 16, ptx::kMajorK, ptx::kMajorMN);
      const uint32_t lr_mode = RP == 64 ? ptx::kSw128 : RP == 32 ? ptx::kSw64 : ptx::kSw32;
      const uint64_t kd = ptx::smem_desc(ptx::smem_u32(sK), 16u, 1024u, ptx::kSw128);
      const uint64_t vd = ptx::smem_desc(ptx::smem_u32(sV), kBlkBytes, 1024u, ptx::kSw128);
      const uint64_t ld = ptx::smem_desc(ptx::smem_u32(sLR), kBN * kLrRow, 8u * kLrRow, lr_mode);
      // an L_k tile is K-major with narrow rows: one swizzle atom (32 / 64 bytes) along the rank, 8-key groups 8 rows apart
      const uint64_t lkd = ptx::smem_desc(ptx::smem_u32(sLK), 16u, 8u * kLkRow, RK == 32 ? ptx::kSw64 : ptx::kSw32);
      const uint32_t kd_hi = (uint32_t)(kd >> 32), vd_hi = (uint32_t)(vd >> 32), ld_hi = (uint32_t)(ld >> 32), lkd_hi = (uint32_t)(lkd >> 32);
      auto desc = [](uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 32) | lo; };
      // S of tiles (j, j + 1), j even: one N = 128 MMA chain over the whole K stage (j / 2) % kStages into the
      // adjacent S buffers j % 4 and j % 4 + 1
      auto issue_s2 = [&](int j, bool k_there = false) {
        const int st = j >> 1, ks_stage = st % kStages;
        // no tcgen05 fence here: the stage was filled by the TMA engine (its mbarrier completion makes the bytes visible to the
        // tensor cores), and the S buffers being overwritten were handed back through p_full + the fence of the P V step, which
        // precedes this chain in program order
        if (!k_there) ptx::mbar_wait(&bars.k_full[ks_stage], (uint32_t)((st / kStages) & 1));
        const uint32_t k_lo = (uint32_t)kd + (uint32_t)ks_stage * (kKBytes >> 4);
        const uint32_t s_tmem = tmem + kTmemS + (uint32_t)(j & 3) * kSN;
        LK_PTRACE(j, 0); LK_PTRACE(j + 1, 0);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          ptx::umma_bf16_ts(s_tmem, tmem + kTmemQ + 8u * ks, desc(kd_hi, k_lo + (uint32_t)(((ks / 4) * kBlkBytes + (ks % 4) * 32u) >> 4)),
                            idesc_s, ks > 0 ? 1u : 0u);
        if (RK > 0) {
          const uint32_t lk_lo = (uint32_t)lkd + (uint32_t)ks_stage * (kLkBytes >> 4);
#pragma unroll
          for (int kk = 0; kk < RK / 16; ++kk)
            ptx::umma_bf16_ts(s_tmem, tmem + kTmemQk + 8u * kk, desc(lkd_hi, lk_lo + (uint32_t)(kk * 32u >> 4)), idesc_s, 1u);
        }
        LK_PTRACE(j, 10);
        ptx::umma_commit(&bars.k_empty[ks_stage]);
        ptx::umma_commit(&bars.s_full[j & 3]);       // ONE arrival for the pair: the owner of the odd tile waits on this barrier too
      };
      if (n_tiles > 0) {
        ptx::mbar_wait(&bars.q_full, 0);
        ptx::tc_fence_after();
        issue_s2(0);
      }
      if (n_tiles > 2) issue_s2(2);
      // O += P(j) V(j), O_lr += P(j) V_lr(j): the 64 keys [64 (j & 1), +64) of V stage vs, P(j) in the S(j) buffer
      auto issue_pv = [&](int j, int vs) {
        const int h = j & 1;
        const uint32_t v_lo = (uint32_t)vd + (uint32_t)vs * (kKBytes >> 4) + (uint32_t)h * ((kSN / 16) * 2048u >> 4);
        const uint32_t l_lo = (uint32_t)ld + (uint32_t)vs * (kLrBytes >> 4) + (uint32_t)h * ((kSN / 16) * 16u * kLrRow >> 4);
        const uint32_t p_tmem = tmem + kTmemS + (uint32_t)(j & 3) * kSN;
#pragma unroll
        for (int ks = 0; ks < kSN / 16; ++ks) {
          ptx::umma_bf16_ts(tmem + kTmemO, p_tmem + 8u * ks, desc(vd_hi, v_lo + (uint32_t)ks * (2048u >> 4)), idesc_o,
                            (j > 0 || ks > 0) ? 1u : 0u);
          if (RP > 0)
            ptx::umma_bf16_ts(tmem + kTmemLr, p_tmem + 8u * ks, desc(ld_hi, l_lo + (uint32_t)ks * (16u * kLrRow >> 4)), idesc_lr,
                              (j > 0 || ks > 0) ? 1u : 0u);
        }
        ptx::umma_commit(&bars.pv_done[j & 3]);
      };
      // This thread's own instruction stream is long: a barrier wait costs it ~75 clocks even when the phase completed long ago, a
      // fence ~90, a commit ~60 (per-tile clock stamps of one CTA, profiles/r2_prefill_tile_trace.txt).  Hence no fence behind the
      // K wait, one s_full arrival per pair, and the stage waits ahead of the P wait.
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j >> 1, vs = st % kStages, h = j & 1;
        // one P barrier per S buffer (not per warpgroup): a warpgroup can finish tile j + 2 before this thread
        // has looked at tile j (S(j+2) is issued ahead of PV(j)), and a parity wait two phases late never returns;
        // P(j+4) needs S(j+4), which is only issued behind PV(j+1)
        // the stage waits first: V of this pair and K of the pair whose scores go out behind it landed long ago, and a wait
        // costs this thread ~75 clocks even then -- better spent before P arrives than between P and its MMAs
        if (h == 0) {
          ptx::mbar_wait(&bars.v_full[vs], (uint32_t)((st / kStages) & 1));
          if (j + 4 < n_tiles) ptx::mbar_wait(&bars.k_full[(st + 2) % kStages], (uint32_t)(((st + 2) / kStages) & 1));
        }
        ptx::mbar_wait(&bars.p_full[j & 3], (uint32_t)((j >> 2) & 1));
        ptx::tc_fence_after();
        LK_PTRACE(j, 1);
        issue_pv(j, vs);
        LK_PTRACE(j, 8);
        if (h == 1 || j == n_tiles - 1) ptx::umma_commit(&bars.v_empty[vs]);
        if (j == n_tiles - 1) ptx::umma_commit(&bars.all_done);
        LK_PTRACE(j, 9);
        // S of tiles (j + 3, j + 4) into the buffers of tiles (j - 1, j), both of whose PV are issued by now
        if (h == 1 && j + 3 < n_tiles) issue_s2(j + 3, true);
      }
    }
  } else {
    // ===================== softmax / correction / epilogue =====================
    // thread (w, lane) owns MMA row 32 (w % 4) + lane (= its TMEM lane); warpgroup wg = w / 4 takes the
    // tiles j with j % 2 == wg
    const int row = (warp & 3) * 32 + lane;
    const int wg = warp >> 2;
    // row -> (query row of the call, q head): prefill rows are (head in group, position); decode rows are
    // (batch entry, head in group), every one at position L - 1
    bool real_row;
    int64_t last_visible;
    const float* q_src;
    const float* qk_src = nullptr;
    float* dst = nullptr;
    if constexpr (!kDecode) {
      const int hg = row / PB;                                 // q head within the group
      int64_t pos_local = row % PB;
      if (pos_local >= rows_here) pos_local = rows_here - 1;   // padding rows shadow the last real one
      real_row = (row % PB) < rows_here;
      const int64_t pos = q0 + pos_local;
      last_visible = p.query_offset + pos;
      q_src = p.q + pos * (p.n_q_local * D) + ((int64_t)kvh * p.group + hg) * D;
      dst = p.out + pos * (p.n_q_local * D) + ((int64_t)kvh * p.group + hg) * D;
      if (RK > 0) qk_src = p.qk + (pos * p.n_q_local + (int64_t)kvh * p.group + hg) * RK;
    } else {
      real_row = row < p.rows_total;
      const int rho = real_row ? row : p.rows_total - 1;
      const int entry = rho / p.group, gi = rho % p.group;
      last_visible = p.L - 1;
      q_src = p.q + (((int64_t)(p.layer_begin_rel + layer_rel) * p.n_batch + entry) * p.n_q_local + (int64_t)kvh * p.group + gi) * D;
      if (RK > 0) qk_src = p.qk + (((int64_t)(p.layer_begin_rel + layer_rel) * p.n_batch + entry) * p.n_q_local + (int64_t)kvh * p.group + gi) * RK;
    }
    const float ninf = -std::numeric_limits<float>::infinity();

    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    // ---- Q tile -> TMEM: this thread's half of its row, fp32 -> packed bf16 pairs ----
    {
      const float* src = q_src + wg * (D / 2);
#pragma unroll
      for (int c0 = 0; c0 < D / 4; c0 += 16) {          // D/4 packed columns per thread, 16 per store
        uint32_t r16[16];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(src + 2 * (c0 + i)));
          r16[i] = pack_bf16(v.x, v.y);
          r16[i + 1] = pack_bf16(v.z, v.w);
        }
        ptx::tmem_st16(tmem + lane_base + kTmemQ + (uint32_t)wg * (D / 4) + c0, r16);
      }
      if (RK > 0 && wg == 0) {        // the row's queries through B_k: RK numbers -> RK / 2 packed columns, zero padded to 16
        uint32_t r16[16];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (2 * i < RK) v = __ldg(reinterpret_cast<const float4*>(qk_src + 2 * i));
          r16[i] = pack_bf16(v.x, v.y);
          r16[i + 1] = pack_bf16(v.z, v.w);
        }
        ptx::tmem_st16(tmem + lane_base + kTmemQk, r16);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars.q_full);
      if (tid == 0) LK_PTRACE(2047, 3);
    }

    float m_mine = ninf;          // the maximum this thread's row sum is relative to (scaled, log2 units)
    float l_run = 0.f;            // row sum over this warpgroup's tiles
    for (int j = wg; j < n_tiles; j += 2) {
      const int sb = j & 3;
      ptx::mbar_wait(&bars.s_full[sb & 2], (uint32_t)((j >> 2) & 1));        // one arrival per tile pair, on the even tile's barrier
      ptx::tc_fence_after();
      if ((warp & 3) == 0 && lane == 0) LK_PTRACE(j, 2);
      float sc[kSN];
      {
        uint32_t raw[kSN];
        ptx::tmem_ld64_wait(tmem + lane_base + kTmemS + (uint32_t)sb * kSN, raw);
#pragma unroll
        for (int c = 0; c < kSN; ++c) sc[c] = __uint_as_float(raw[c]);
      }

      const int64_t key0 = (int64_t)(tile_begin + j) * kSN;
      const bool tile_needs_mask = key0 + kSN - 1 >= mask_from;   // CTA-uniform
      if (tile_needs_mask) {
#pragma unroll
        for (int c = 0; c < kSN; ++c)
          if (key0 + c > last_visible) sc[c] = ninf;
      }
      // row max of the raw scores: 8 independent chains
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = sc[u];
#pragma unroll
      for (int c = 8; c < kSN; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], sc[c]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])), fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) *
                       p.scale_log2;                       // scale > 0 commutes with max; -inf stays -inf

      // the running maximum after tile j - 1, published by the partner warp
      float m_prev = ninf;
      if ((warp & 3) == 0 && lane == 0) LK_PTRACE(j, 3);
      if (j > 0) {                  // the partner warp (same rows, other warpgroup) published after tile j - 1
        ptx::mbar_wait(&bars.hand[(warp & 3) * 2 + (wg ^ 1)], (uint32_t)(((j - 1) >> 1) & 1));
        m_prev = *reinterpret_cast<volatile float*>(&m_s[row]);
      }
      if ((warp & 3) == 0 && lane == 0) LK_PTRACE(j, 4);
      float m_used = m_prev;
      const float m_cand = fmaxf(m_prev, mx);
      if (j == 0) {
        m_used = m_cand;          // key 0 is visible to every row, so this is finite
      } else {
        const bool grow = m_cand > m_prev + kRescaleThreshold;
        if (__any_sync(0xffffffffu, grow)) {
          // correction: O and O_lr of this row are final for tile j-1 once PV(j-1) has completed, and PV(j)
          // cannot start before this thread delivers P(j).  A parity wait is only meaningful while the barrier
          // is at most one phase away from the one asked for, so PV completion is tracked by FOUR barriers
          // (tile % 4), each advancing once per four tiles: S(j) having arrived guarantees PV(j-4) (S of an
          // odd tile is issued with its even neighbour, behind PV(j-4)), hence PV(j-5), and PV(j+3) cannot
          // have been issued.
          ptx::mbar_wait(&bars.pv_done[(j - 1) & 3], (uint32_t)(((j - 1) >> 2) & 1));
          ptx::tc_fence_after();
          // tcgen05.ld / st are warp-collective (.sync.aligned): every lane takes part, lanes whose row did not
          // grow scale by 1
          const float alpha = grow ? ex2(m_prev - m_cand) : 1.f;
          if (grow) m_used = m_cand;
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 16) {
            uint32_t r16[16];
            const uint32_t addr = tmem + lane_base + kTmemO + c0;
            ptx::tmem_ld16(addr, r16);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) r16[i] = __float_as_uint(__uint_as_float(r16[i]) * alpha);
            ptx::tmem_st16(addr, r16);
          }
#pragma unroll
          for (int c0 = 0; c0 < RP; c0 += 16) {
            uint32_t r16[16];
            ptx::tmem_ld16(tmem + lane_base + kTmemLr + c0, r16);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) r16[i] = __float_as_uint(__uint_as_float(r16[i]) * alpha);
            ptx::tmem_st16(tmem + lane_base + kTmemLr + c0, r16);
          }
          ptx::tmem_wait_st();
        }
      }
      // hand the maximum to the owner of tile j + 1
      if (j + 1 < n_tiles) {        // mbarrier.arrive releases the store; one barrier per (warp pair, direction), 32 arrivals
        m_s[row] = m_used;
        ptx::mbar_arrive(&bars.hand[(warp & 3) * 2 + wg]);
      }
      // bring this warpgroup's row sum to the new reference (its last tile was j - 2)
      if (m_used != m_mine) {
        l_run *= (m_mine == ninf) ? 0.f : ex2(m_mine - m_used);
        m_mine = m_used;
      }
      // P = exp2(s * scale - m) in one FFMA + MUFU; masked entries (-inf) come out as exact zeros
      float ls4[4] = {0.f, 0.f, 0.f, 0.f};
      const float neg_m = -m_used;
#pragma unroll
      for (int c = 0; c < kSN; c += 2) {
        ffma2(sc[c], sc[c + 1], p.scale_log2, neg_m);
        sc[c] = ex2(sc[c]);
        sc[c + 1] = ex2(sc[c + 1]);
        fadd2(ls4[c & 3], ls4[(c & 3) + 1], sc[c], sc[c + 1]);
      }
      l_run += (ls4[0] + ls4[1]) + (ls4[2] + ls4[3]);
      if ((warp & 3) == 0 && lane == 0) LK_PTRACE(j, 5);
      // P(j) -> TMEM, over the first 32 columns of the S(j) buffer (this thread has its scores in registers;
      // S(j+4) is issued behind PV(j) on the in-order pipe)
#pragma unroll
      for (int c0 = 0; c0 < kSN / 2; c0 += 16) {
        uint32_t r16[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) r16[i] = pack_bf16(sc[2 * (c0 + i)], sc[2 * (c0 + i) + 1]);
        ptx::tmem_st16(tmem + lane_base + kTmemS + (uint32_t)sb * kSN + c0, r16);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars.p_full[sb]);
      if ((warp & 3) == 0 && lane == 0) LK_PTRACE(j, 6);
    }

    // ---- both warpgroups: wait for the last PV, bring the two partial row sums to the final maximum ----
    if (n_tiles > 0) {
      ptx::mbar_wait(&bars.all_done, 0);
      ptx::tc_fence_after();
    }
    if (tid == 0) LK_PTRACE(2047, 4);
    l_s[wg][row] = l_run;
    mref_s[wg][row] = m_mine;
    named_bar_sync(9, 256);
    const float m_fin = fmaxf(mref_s[0][row], mref_s[1][row]);     // the maximum never decreases: the later tile holds it
    float l_tot = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < 2; ++w2) {
      const float mr = mref_s[w2][row];
      if (mr != ninf) l_tot += l_s[w2][row] * ex2(mr - m_fin);
    }

    if constexpr (kDecode) {
      // ---- partial of this split: (m, l, O, O_lr) un-normalised, merged (+ B epilogue) by fla_decode_merge ----
      constexpr int PS = 4 + D + RP;
      float* prow = p.part + ((int64_t)blockIdx.x * kBM + row) * PS;
      if (wg == 0) { prow[0] = m_fin; prow[1] = l_tot; }
      if (n_tiles > 0) {
#pragma unroll
        for (int cc = 0; cc < D / 2; cc += 16) {
          const int c0 = wg * (D / 2) + cc;
          uint32_t r16[16];
          ptx::tmem_ld16(tmem + lane_base + kTmemO + c0, r16);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(prow + 4 + c0 + i) = make_float4(__uint_as_float(r16[i]), __uint_as_float(r16[i + 1]),
                                                                        __uint_as_float(r16[i + 2]), __uint_as_float(r16[i + 3]));
        }
        if (wg == 0) {
#pragma unroll
          for (int c0 = 0; c0 < RP; c0 += 16) {
            uint32_t r16[16];
            ptx::tmem_ld16(tmem + lane_base + kTmemLr + c0, r16);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              *reinterpret_cast<float4*>(prow + 4 + D + c0 + i) = make_float4(__uint_as_float(r16[i]), __uint_as_float(r16[i + 1]),
                                                                              __uint_as_float(r16[i + 2]), __uint_as_float(r16[i + 3]));
          }
        }
      }
    } else {
      // ---- epilogue: o += (lr_scale * o_lr[p]) * B[p,:], out = o / l ----
      float* b_s = reinterpret_cast<float*>(sK);            // K stages are idle now: stage B[r][D] of this kv head
      for (int idx = tid; idx < p.r * D; idx += 256)
        b_s[idx] = p.b[(int64_t)(idx / D) * ((int64_t)p.n_kv_local * D) + (int64_t)kvh * D + idx % D];
      named_bar_sync(9, 256);
      if (tid == 0) LK_PTRACE(2047, 5);
      const float inv_l = 1.0f / l_tot;
      float w[RP > 0 ? RP : 1];
#pragma unroll
      for (int c0 = 0; c0 < RP; c0 += 16) {
        uint32_t r16[16];
        ptx::tmem_ld16(tmem + lane_base + kTmemLr + c0, r16);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) w[c0 + i] = p.lr_scale * __uint_as_float(r16[i]);
      }
#pragma unroll
      for (int cc = 0; cc < D / 2; cc += 16) {
        const int c0 = wg * (D / 2) + cc;
        uint32_t r16[16];
        ptx::tmem_ld16(tmem + lane_base + kTmemO + c0, r16);
        ptx::tmem_wait_ld();
        float acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = __uint_as_float(r16[i]);
        // B rows as 16-byte broadcast reads from shared memory
#pragma unroll
        for (int k = 0; k < RP; ++k) {
          if (k < p.r) {
            const float4* bp = reinterpret_cast<const float4*>(b_s + k * D + c0);
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              const float4 bv = bp[i4];
              acc[4 * i4] = fmaf(w[k], bv.x, acc[4 * i4]);
              acc[4 * i4 + 1] = fmaf(w[k], bv.y, acc[4 * i4 + 1]);
              acc[4 * i4 + 2] = fmaf(w[k], bv.z, acc[4 * i4 + 2]);
              acc[4 * i4 + 3] = fmaf(w[k], bv.w, acc[4 * i4 + 3]);
            }
          }
        }
        // the finished row goes through shared memory (the V stages are idle: every stage was consumed before all_done): a thread
        // owns a ROW, and 16-byte stores of 32 lanes into rows 16 KB apart cost the CTA ~9 000 clocks (clock trace); staged, a warp
        // stores whole 512-byte rows.  Row stride D + 4 floats: the 16-byte stores of eight lanes fall into eight bank groups.
        float* o_row = reinterpret_cast<float*>(sV) + (size_t)row * (D + 4) + c0;
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(o_row + i) = make_float4(acc[i] * inv_l, acc[i + 1] * inv_l, acc[i + 2] * inv_l, acc[i + 3] * inv_l);
      }
      named_bar_sync(9, 256);
      for (int r2 = warp; r2 < kBM; r2 += 8) {                 // warp w stores rows w, w + 8, ...: lane = 16 bytes of the row
        const int hg2 = r2 / PB, pl2 = r2 % PB;
        if (pl2 >= rows_here) continue;
        float* d2 = p.out + (q0 + pl2) * (p.n_q_local * D) + ((int64_t)kvh * p.group + hg2) * D;
        const float* s2 = reinterpret_cast<const float*>(sV) + (size_t)r2 * (D + 4);
        for (int c = lane * 4; c < D; c += 128) *reinterpret_cast<float4*>(d2 + c) = *reinterpret_cast<const float4*>(s2 + c);
      }
    }
  }

  if (tid == 0) LK_PTRACE(2047, 6);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
  if (tid == 0) LK_PTRACE(2047, 7);
}

template <int D, int RP, bool kDecode, int RK = 0>
int launch_t(lorakv_ctx* ctx, const PrefillParams& pp, unsigned grid) {
  const size_t blk = (size_t)kBN * 128;
  const size_t kv = (D / 64) * blk, lr = (size_t)kBN * 2 * RP, lk = (size_t)kBN * 2 * RK;
  const int stages = (2 * 3 * kv + 3 * lr + 3 * lk + 1024 <= (size_t)227 * 1024 - 4096) ? 3 : 2;   // mirrors kStages in the kernel
  const size_t smem = stages * (2 * kv + lr + lk) + 1024;
  auto kern = fla_prefill_umma_kernel<D, RP, kDecode, RK>;
  static int attr_device = -1;         // once per instantiation: smem depends on the template parameters only
  if (attr_device != ctx->device) {
    LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_device = ctx->device;
  }
  prof_mark(ctx, 0);
  LK_CUDA(launch_kernel(ctx, kern, dim3(grid), dim3(kThreads), smem, true, pp));
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

// key-side rank 16 / 32 beside value-side rank 0 / 16 / 32 (rank 64 at d_head 128 leaves no TMEM columns for Qk: the caller
// keeps those on the CUDA-core kernel, key_lowrank_umma_ok)
template <int D, bool kDecode, int RK>
int launch_rp_rk(lorakv_ctx* ctx, const PrefillParams& pp, unsigned grid, int rp) {
  switch (rp) {
    case 0: return launch_t<D, 0, kDecode, RK>(ctx, pp, grid);
    case 16: return launch_t<D, 16, kDecode, RK>(ctx, pp, grid);
    case 32: return launch_t<D, 32, kDecode, RK>(ctx, pp, grid);
    default:
      if constexpr (D == 64) return launch_t<D, 64, kDecode, RK>(ctx, pp, grid);
      else return fail("fla_prefill_umma: key-side term beside a rank-64 value side at d_head 128 (no TMEM columns left)");
  }
}

template <int D, bool kDecode>
int launch_rp(lorakv_ctx* ctx, const PrefillParams& pp, unsigned grid, int rp, int rk = 0) {
  if (rk == 16) return launch_rp_rk<D, kDecode, 16>(ctx, pp, grid, rp);
  if (rk == 32) return launch_rp_rk<D, kDecode, 32>(ctx, pp, grid, rp);
  switch (rp) {
    case 0: return launch_t<D, 0, kDecode>(ctx, pp, grid);
    case 16: return launch_t<D, 16, kDecode>(ctx, pp, grid);
    case 32: return launch_t<D, 32, kDecode>(ctx, pp, grid);
    default: return launch_t<D, 64, kDecode>(ctx, pp, grid);
  }
}

void fill_common(PrefillParams& pp, const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  const int d = (int)pool->dims.d_head, rp = (int)pool->r_pad;
  pp.k_pages = static_cast<const __nv_bfloat16*>(pool->k_pages);
  pp.v_pages = static_cast<const __nv_bfloat16*>(pool->v_pages);
  pp.lr_pages = static_cast<const __nv_bfloat16*>(pool->lr_pages);
  pp.kv_table = pool->kv_space.dev_table + c.kv_set * pool->kv_space.max_pages;
  pp.lr_table = rp > 0 ? pool->lr_space.dev_table + c.lr_set * pool->lr_space.max_pages : nullptr;
  pp.kv_layer_off = c.layer_begin * pool->kv_layer_stride(); pp.kv_head_stride = pool->kv_head_stride();
  pp.kv_page_stride = pool->kv_page_stride();
  pp.lr_layer_off = c.layer_begin * pool->lr_layer_stride(); pp.lr_page_stride = pool->lr_page_stride();
  pp.kv_layer_stride = pool->kv_layer_stride(); pp.lr_layer_stride = pool->lr_layer_stride();
  pp.P = (int)pool->P; pp.group = (int)(c.n_q_local / pool->n_kv_local); pp.n_kv_local = (int)pool->n_kv_local;
  pp.n_pages = (int)((c.L + pool->P - 1) / pool->P); pp.r = (int)pool->dims.rank;
  pp.L = c.L; pp.L_c = c.rows_per_entry; pp.query_offset = c.query_offset; pp.n_q_local = c.n_q_local;
  pp.scale_log2 = (float)((1.0 / sqrt((double)d)) * 1.4426950408889634);
  pp.q = c.q_dev; pp.out = c.out_dev;
  pp.n_qblocks = 0; pp.n_batch = (int)c.n_batch; pp.rows_total = 0; pp.splits = 1; pp.tiles_per_split = 0;
  pp.layer_begin_rel = 0; pp.part = nullptr; pp.lr_scale = 0.f; pp.b = nullptr;
  const bool rk = pool->rk_pad > 0;
  pp.lk_pages = static_cast<const __nv_bfloat16*>(pool->lk_pages);
  pp.lk_table = rk ? pool->lk_space.dev_table : nullptr;
  pp.lk_layer_stride = rk ? pool->lk_layer_stride() : 0; pp.lk_layer_off = c.layer_begin * pp.lk_layer_stride;
  pp.lk_page_stride = rk ? pool->lk_page_stride() : 0; pp.qk = c.qk_dev;
}

// the key-side low-rank term on this kernel: rank_k padded to 16 / 32 (one or two more k steps of the score chain) and
// 16 free TMEM columns for Qk (d_head 128 with a rank-64 value side has none)
bool key_lowrank_umma_ok(const lorakv_pool* pool) {
  if (pool->rk_pad == 0) return true;
  if (pool->rk_pad != 16 && pool->rk_pad != 32) return false;
  return pool->dims.d_head == 64 || pool->r_pad <= 32;
}

bool umma_shape_ok(const lorakv_pool* pool) {
  const int64_t d = pool->dims.d_head, rp = pool->r_pad, P = pool->P;
  if (pool->dims.dtype != LORAKV_BF16) return false;
  if (d != 64 && d != 128) return false;
  if (!(rp == 0 || rp == 16 || rp == 32 || rp == 64)) return false;
  if (P < 16 || (P & (P - 1)) != 0) return false;           // power-of-two pages: tiles are made of whole runs
  return true;
}

}  // namespace

bool prefill_umma_supported(const PagedAttnCall& c) {
  const lorakv_pool* pool = c.pool;
  if (!key_lowrank_umma_ok(pool) || (pool->rk_pad > 0 && !c.qk_dev)) return false;
  if (!umma_shape_ok(pool)) return false;
  if (c.n_batch != 1 || c.rows_per_entry < 2 || c.layer_end - c.layer_begin != 1) return false;
  const int64_t group = c.n_q_local / pool->n_kv_local;
  if (group < 1 || group > kBM || kBM % group != 0) return false;
  if (c.L < 1) return false;
  return true;
}

int launch_prefill_umma(const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const int d = (int)pool->dims.d_head, r = (int)pool->dims.rank, rp = (int)pool->r_pad;
  if (r > 0 && !c.adapters) return fail("paged attention: rank %lld cache needs adapter tables", (long long)r);
  PrefillParams pp;
  fill_common(pp, c);
  const int PB = kBM / pp.group;
  const int64_t layer = c.layer_begin, agent = c.agent_host;
  pp.n_qblocks = (int)((c.rows_per_entry + PB - 1) / PB);
  pp.lr_scale = (r > 0) ? c.adapters->scale_host[(size_t)(layer * c.adapters->n_agents + agent)] : 0.f;
  pp.b = (r > 0) ? c.adapters->b + ((layer * c.adapters->n_agents + agent) * r) * (pool->n_kv_local * (int64_t)d) : nullptr;
  const unsigned grid = (unsigned)((int64_t)pp.n_qblocks * pool->n_kv_local);
  if (d == 128) LK_TRY((launch_rp<128, false>(ctx, pp, grid, rp, (int)pool->rk_pad)));
  else LK_TRY((launch_rp<64, false>(ctx, pp, grid, rp, (int)pool->rk_pad)));
  ctx->last_kernel = "fla_prefill_umma";
  return LORAKV_OK;
}

// Batched decode with many query rows per kv head (more than 32 = agents x group): the tcgen05 kernel in
// decode mode.  One CTA streams one split of one (layer, kv head); rows (batch entry, head) fill the 128 MMA
// rows (blocks of 128 when there are more).  Partials go through the same merge + epilogue kernel as
// fla_decode_tma.
bool decode_umma_supported(const PagedAttnCall& c) {
  const lorakv_pool* pool = c.pool;
  if (!key_lowrank_umma_ok(pool) || (pool->rk_pad > 0 && !c.qk_dev)) return false;
  if (!umma_shape_ok(pool)) return false;
  if (c.rows_per_entry != 1 || c.query_offset != c.L - 1 || c.L < 1 || c.n_batch < 1) return false;
  const int64_t rows_total = c.n_batch * (c.n_q_local / pool->n_kv_local);
  // (with the key-side low-rank term the streaming kernel carries up to 16 rows per kv head: this kernel takes over from 17)
  return rows_total > (pool->rk_pad > 0 ? 16 : 32) && rows_total <= kBM;
}

int launch_decode_umma(const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const int d = (int)pool->dims.d_head, r = (int)pool->dims.rank, rp = (int)pool->r_pad;
  if (r > 0 && !c.adapters) return fail("paged attention: rank %lld cache needs adapter tables", (long long)r);
  PrefillParams pp;
  fill_common(pp, c);
  const int64_t n_layers = c.layer_end - c.layer_begin;
  const int64_t units = n_layers * pool->n_kv_local;
  const int64_t total_tiles = (c.L + kBN - 1) / kBN;
  // splits: enough CTAs for ~4 waves of the machine, at least 4 tiles each
  int64_t splits = (4 * (int64_t)ctx->sm_count + units - 1) / units;
  // ... but a CTA pays ~17 us before and after its stream (TMEM allocation, Q, pipeline fill, drain, partial store): with one
  // layer per launch (8 units) four waves of 14-tile CTAs spent as long on that as on streaming (cfg 5: 177 us per layer, 0.48
  // of the HBM roofline).  At least 48 stages of 128 keys per CTA, and no nearly-empty second wave.
  if (splits > total_tiles / 48) splits = total_tiles / 48;
  if (splits < 1) splits = 1;
  if (units * splits > ctx->sm_count && units * splits < 2 * (int64_t)ctx->sm_count && ctx->sm_count / units >= 1) splits = ctx->sm_count / units;
  const int64_t tiles_per_split = (total_tiles + splits - 1) / splits;
  splits = (total_tiles + tiles_per_split - 1) / tiles_per_split;
  pp.rows_total = (int)(c.n_batch * pp.group);
  pp.splits = (int)splits; pp.tiles_per_split = (int)tiles_per_split;
  const int PS = 4 + d + rp;
  const size_t part_bytes = (size_t)(units * splits) * kBM * PS * sizeof(float);
  LK_TRY(scratch_reserve(ctx, ctx->work, part_bytes));
  pp.part = static_cast<float*>(ctx->work.ptr);
  const unsigned grid = (unsigned)(units * splits);
  if (d == 128) LK_TRY((launch_rp<128, true>(ctx, pp, grid, rp, (int)pool->rk_pad)));
  else LK_TRY((launch_rp<64, true>(ctx, pp, grid, rp, (int)pool->rk_pad)));
  // merge + B epilogue: the partial slots are [unit][split], i.e. fla_decode_merge's closed form with
  // T = splits * G tiles per unit and G tiles per worker, one segment per worker
  LK_TRY(launch_decode_merge(ctx, pp.part, d, rp, r, /*MW=*/8, pp.group, (int)pool->n_kv_local, (int)c.n_batch, pp.rows_total,
                             /*row_blocks=*/1, /*T=*/splits * tiles_per_split, /*G=*/tiles_per_split, c.layer_begin, c.n_q_local,
                             /*max_seg=*/1, c.agent_ids_dev, c.adapters, c.out_dev, n_layers, c.peers));
  ctx->last_kernel = "fla_decode_umma";
  return LORAKV_OK;
}

}  // namespace lk

#ifdef LK_PREFILL_TRACE
extern "C" int lorakv_debug_prefill_trace(long long* out, int n_words) {
  return cudaMemcpyFromSymbol(out, lk::g_prefill_trace, sizeof(long long) * (size_t)n_words) == cudaSuccess ? 0 : 1;
}
#endif
