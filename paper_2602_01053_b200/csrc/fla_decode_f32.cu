// fla_decode_f32.cu -- batched Flash-LoRA-Attention decode over the paged FP32 cache ("fp32 mode": results within
// 1e-4 of the reference on max_rel_error), HBM-bound like its bf16 sibling fla_decode_tma.cu.
//
// What it computes is the same: one gqa_attention call (proj/include/lorakv/attention.hpp:332-363) per (layer,
// batch entry) with query_offset = L-1 (engine.hpp:440-443), the g q heads of a kv head and all batch entries
// stacked as rows of one MMA tile so that the cache is read once per step; partials (m, l, O, O_lr) per worker
// and unit, merged and up-projected by fla_decode_merge (attention.hpp:244-259).
//
// How it keeps fp32 accuracy on the tensor cores: every product runs as three mma.sync.m16n8k8 TF32 MMAs over
// operands split into two TF32 halves,  a*b ~= a_hi*b_hi + a_lo*b_hi + a_hi*b_lo  with  x_hi = x & 0xffffe000
// (exactly representable in TF32) and x_lo = x - x_hi (exact in fp32; its own truncation to TF32 and the dropped
// a_lo*b_lo term are both ~2^-22 relative).  Accumulation is fp32.  The CUDA-core kernel this replaces for the
// shape (fla_paged_simt) ran the cfg-2 step at 0.14 of the HBM roofline; the MACs of a decode step are few
// enough that 3x the tensor work still hides behind the cache stream.
//
// Data movement is the bf16 kernel's: per worker a ring of shared-memory stages filled by cp.async.bulk (TMA
// engine) against mbarriers, L2 evict-first.  A stage is 8 keys: 8 * (2 * D + RP) * 4 bytes (8.5 KB at d = 128,
// r = 16 -- the same bytes as the bf16 kernel's 16-key stage, so the same three stages per single-warp worker).
// FP32 pages are row-major with the 16-byte chunks of a row XOR-swizzled by the token index (page_layout.cuh),
// which makes both fragment patterns below bank-conflict-free with plain 32-bit shared loads:
//   S = Q K^T : B fragment (k = dim, n = key): lane (g, t) reads K[key g][8 kk + t], K[key g][8 kk + 4 + t]
//   O += P V  : B fragment (k = key, n = dim): lane (g, t) reads V[key 2t][8 nt + g], V[key 2t + 1][8 nt + g]
// The k slots of the P V step are assigned to keys as (slot t, slot t + 4) = (key 2t, key 2t + 1), which is
// exactly how the S accumulator fragment holds them: P moves from the softmax to the A operand without a shuffle.
#include <cstdlib>
#include <limits>

#include "kernels.hpp"
#include "page_layout.cuh"
#include <cuda_bf16.h>

#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kTK = 8;                      // keys per tile = one n8 tile of S = one k8 step of P V
constexpr int kMaxStages = 24;
constexpr int kRingBudget = 216 * 1024;
constexpr float kRescaleThreshold = 8.0f;   // log2 units

// 12 warps of 168 registers spill and leave two stages per ring: 2.2 ms vs 1.6 ms at cfg 2; six / four single-warp workers with deeper
// rings (the bf16 kernel's wide-worker layout) lose here, the kernel being bound by the tensor pipe: 1.60 / 1.64 vs 1.49 ms
constexpr int warps_per_cta(int mw) { return mw <= 8 ? 8 : 8; }

struct DecodeF32Params {
  const float *k_pages, *v_pages, *lr_pages;
  const int32_t *kv_table, *lr_table;
  int64_t kv_layer_stride, kv_head_stride, kv_page_stride, lr_layer_stride, lr_page_stride;  // elements
  int P, group, n_kv_local, n_batch, rows_total, row_blocks, n_pages;
  int64_t L, layer_begin, n_q_local;
  int64_t T, total_tiles, G;
  int max_seg, n_stages;
  float scale_log2;
  uint64_t l2_policy, lr_policy;   // K / V stream evict-first; V_lr evict-last while the launch's low-rank cache fits in L2
  const float* q;
  float* part;           // [workers * max_seg][16 * MW][4 + D + RP]
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lds32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// x = hi + lo with hi exactly a TF32 number
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
// acc += a * b with the running sum kept OUT of the tensor-core accumulator: the MMA adds its products into C with
// truncation, a bias of up to 2^-24 per instruction that grows linearly with the length of the chain (4096 key tiles of a
// 32K-token row: 2e-4 -- measured, and over the 1e-4 contract).  The tile's product therefore starts from zero and
// is added to the running sum with an ordinary round-to-nearest FADD, whose error grows only as the square root.
__device__ __forceinline__ void mma_3x_add(float (&acc)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint32_t bh0, uint32_t bh1,
                                           uint32_t bl0, uint32_t bl1) {
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  mma_tf32(d, al[0], al[1], al[2], al[3], bh0, bh1);
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
  // two packed adds (add.rn.f32x2, sm_100) instead of four scalar ones: the adds are pure issue pressure here
  asm("{\n\t.reg .b64 a, b;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%4, %5};\n\tadd.rn.f32x2 a, a, b;\n\tmov.b64 {%0, %1}, a;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%6, %7};\n\tadd.rn.f32x2 a, a, b;\n\tmov.b64 {%2, %3}, a;\n\t}"
      : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
      : "f"(d[0]), "f"(d[1]), "f"(d[2]), "f"(d[3]));
}
// c += a * b for full-precision fragments: small terms first
__device__ __forceinline__ void mma_3x(float (&c)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint32_t bh0, uint32_t bh1,
                                       uint32_t bl0, uint32_t bl1) {
  mma_tf32(c, al[0], al[1], al[2], al[3], bh0, bh1);
  mma_tf32(c, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
  mma_tf32(c, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
}

// W = warps per CTA: 12 where the worker width divides it (their ~168 registers each still hold the Q fragments and
// the O accumulators; four more warps per SM hide more of the MMA and shared-memory latency), else 8
template <int D, int RP, int MW, int W>
__global__ void __launch_bounds__(W * 32, 1) fla_decode_f32_kernel(const DecodeF32Params p) {
  constexpr int kWorkers = W / MW;
  constexpr uint32_t kRowBytes = D * 4;
  constexpr uint32_t kKvBytes = kTK * kRowBytes;
  constexpr uint32_t kLrRowBytes = RP * 4;
  constexpr uint32_t kLrBytes = kTK * kLrRowBytes;
  constexpr uint32_t kStageBytes = 2 * kKvBytes + kLrBytes;
  constexpr int kLrSwz = RP >= 32 ? 7 : (RP / 4 - 1);   // chunks per LR row - 1, capped at one 128-byte line
  constexpr int kNO = D / 8, kNL = RP / 8;
  constexpr int PS = 4 + D + RP;

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kWorkers][kMaxStages];
  __shared__ uint64_t empty_bar[kWorkers][kMaxStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wk = warp / MW, wi = warp % MW;
  const int g = lane >> 2, t = lane & 3;
  const int NS = p.n_stages;

  if (threadIdx.x == 0) {
    for (int a = 0; a < kWorkers; ++a)
      for (int s = 0; s < NS; ++s) {
        ptx::mbar_init(&full_bar[a][s], 1);
        ptx::mbar_init(&empty_bar[a][s], MW);
      }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  ptx::pdl_wait();                  // launched as a programmatic dependent: the set-up above ran under the predecessor's tail
  ptx::pdl_launch_dependents();

  const int64_t w = (int64_t)blockIdx.x * kWorkers + wk;
  const int64_t g0 = w * p.G;
  const int64_t g1 = min(g0 + p.G, p.total_tiles);
  const int n = g1 > g0 ? (int)(g1 - g0) : 0;
  if (n == 0) return;

  const uint32_t ring = ptx::smem_u32(smem) + (uint32_t)wk * (uint32_t)NS * kStageBytes;
  uint64_t* full = full_bar[wk];
  uint64_t* empty = empty_bar[wk];
  const bool producer = wi == 0;
  const int units_per_layer = p.n_kv_local * p.row_blocks;

  // producer cursor, carried incrementally (no per-tile division); page-table window across the lanes
  int win_base = -(1 << 30), win_kv = 0, win_lr = 0;
  const int T32 = (int)p.T;
  int64_t p_unit = g0 / p.T;
  int p_tl = (int)(g0 - p_unit * p.T);
  int p_page = (p_tl * kTK) / p.P, p_tok = (p_tl * kTK) % p.P;
  int p_layer = (int)(p_unit / units_per_layer), p_kvh = (int)((p_unit / p.row_blocks) % p.n_kv_local);
  int p_stage = 0, p_wrap = 0, p_issued = 0;

  auto issue_next = [&]() {
    if (p_page < win_base || p_page >= win_base + 32) {
      win_base = p_page;
      const int pg = p_page + lane;
      win_kv = pg < p.n_pages ? p.kv_table[pg] : 0;
      if (RP > 0) win_lr = pg < p.n_pages ? p.lr_table[pg] : 0;
    }
    const int phys_kv = __shfl_sync(0xffffffffu, win_kv, p_page - win_base);
    const int phys_lr = RP > 0 ? __shfl_sync(0xffffffffu, win_lr, p_page - win_base) : 0;
    if (ptx::elect_one()) {
      const uint32_t dst = ring + (uint32_t)p_stage * kStageBytes;
      const int64_t layer = p.layer_begin + p_layer;
      const int64_t kv_off = layer * p.kv_layer_stride + (int64_t)p_kvh * p.kv_head_stride +
                             (int64_t)phys_kv * p.kv_page_stride + (int64_t)p_tok * D;
      ptx::mbar_arrive_expect_tx(&full[p_stage], kStageBytes);
      bulk_g2s(dst, p.k_pages + kv_off, kKvBytes, &full[p_stage], p.l2_policy);
      bulk_g2s(dst + kKvBytes, p.v_pages + kv_off, kKvBytes, &full[p_stage], p.l2_policy);
      if (RP > 0) {
        const int64_t lr_off = layer * p.lr_layer_stride + (int64_t)phys_lr * p.lr_page_stride + (int64_t)p_tok * RP;
        bulk_g2s(dst + 2 * kKvBytes, p.lr_pages + lr_off, kLrBytes, &full[p_stage], p.lr_policy);   // re-read by every kv head
      }
    }
    ++p_issued;
    if (++p_stage == NS) { p_stage = 0; ++p_wrap; }
    p_tok += kTK;
    if (p_tok == p.P) { p_tok = 0; ++p_page; }
    if (++p_tl == T32) {
      p_tl = 0; p_page = 0; p_tok = 0;
      ++p_unit;
      p_layer = (int)(p_unit / units_per_layer);
      p_kvh = (int)((p_unit / p.row_blocks) % p.n_kv_local);
    }
  };

  if (producer) {
    const int pre = n < NS ? n : NS;
    for (int i = 0; i < pre; ++i) issue_next();
  }

  const float ninf = -std::numeric_limits<float>::infinity();
  float qf[D / 8][4];          // A fragments of Q in full fp32: (g, t), (g + 8, t), (g, t + 4), (g + 8, t + 4) of every k8 step
  float o[kNO][4];
  float olr[kNL > 0 ? kNL : 1][4];
  float m_used[2], l_run[2];
  int64_t cur_unit = -1;

  auto flush = [&]() {
    const int64_t first_unit = g0 / p.T;
    const int64_t slot = w * p.max_seg + (cur_unit - first_unit);
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

  // shared-memory byte offsets of this lane's fragment elements inside a K / V tile (the swizzle term is folded in)
  //   K: row g, chunk (2 kk + j) ^ g, word t           -> kOff + ((2 kk + j) ^ g) * 16
  //   V: row 2t + j, chunk (2 nt + (g >> 2)) ^ (2t + j), word g & 3
  const uint32_t k_row = (uint32_t)g * kRowBytes + (uint32_t)t * 4u;
  const uint32_t v_row0 = (uint32_t)(2 * t) * kRowBytes + (uint32_t)(g & 3) * 4u;
  const uint32_t v_row1 = v_row0 + kRowBytes;
  const uint32_t v_c0 = (uint32_t)((g >> 2) ^ (2 * t)), v_c1 = (uint32_t)((g >> 2) ^ (2 * t + 1));   // low chunk bits, pre-XORed

  int64_t u = g0 / p.T;
  int tl = (int)(g0 - u * p.T);
  int c_stage = 0, c_wrap = 0;
  for (int i = 0; i < n; ++i) {
    if (u != cur_unit) {
      if (cur_unit >= 0) flush();
      cur_unit = u;
      const int layer_rel = (int)(u / units_per_layer);
      const int kvh = (int)((u / p.row_blocks) % p.n_kv_local);
      const int rb = (int)(u % p.row_blocks);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rho = rb * 16 * MW + wi * 16 + g + 8 * h;
        const bool real = rho < p.rows_total;
        const int entry = real ? rho / p.group : 0, gi = real ? rho % p.group : 0;
        const float* src = p.q + (((int64_t)layer_rel * p.n_batch + entry) * p.n_q_local + (int64_t)kvh * p.group + gi) * D;
#pragma unroll
        for (int kk = 0; kk < D / 8; ++kk) {
          qf[kk][h] = real ? __ldg(src + 8 * kk + t) : 0.f;
          qf[kk][2 + h] = real ? __ldg(src + 8 * kk + 4 + t) : 0.f;
        }
        m_used[h] = ninf; l_run[h] = 0.f;
      }
#pragma unroll
      for (int nt = 0; nt < kNO; ++nt) { o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f; }
#pragma unroll
      for (int nt = 0; nt < (kNL > 0 ? kNL : 1); ++nt) { olr[nt][0] = olr[nt][1] = olr[nt][2] = olr[nt][3] = 0.f; }
    }

    if (producer && i >= 1 && p_issued < n) {
      ptx::mbar_wait(&empty[p_stage], (uint32_t)((p_wrap & 1) ^ 1));
      issue_next();
    }
    const int s = c_stage;
    ptx::mbar_wait(&full[s], (uint32_t)(c_wrap & 1));
    const uint32_t sK = ring + (uint32_t)s * kStageBytes, sV = sK + kKvBytes, sLR = sV + kKvBytes;

    // ---- S = Q K^T : 16 rows x 8 keys, 3 x TF32 ------------------------------------------------------
    // three accumulators (hi*hi, lo*hi, hi*lo) so that the 3 * D / 8 MMAs form three chains, not one
    float sc[4] = {0.f, 0.f, 0.f, 0.f}, sc_a[4] = {0.f, 0.f, 0.f, 0.f}, sc_b[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < D / 8; ++kk) {
      const uint32_t line = sK + k_row + (uint32_t)((2 * kk) >> 3) * 128u;
      const float k0 = lds32(line + ((uint32_t)(((2 * kk) & 7) ^ g) << 4));
      const float k1 = lds32(line + ((uint32_t)(((2 * kk + 1) & 7) ^ g) << 4));
      uint32_t ah[4], al[4], bh0, bl0, bh1, bl1;
#pragma unroll
      for (int e = 0; e < 4; ++e) split_tf32(qf[kk][e], ah[e], al[e]);
      split_tf32(k0, bh0, bl0);
      split_tf32(k1, bh1, bl1);
      mma_tf32(sc_a, al[0], al[1], al[2], al[3], bh0, bh1);
      mma_tf32(sc_b, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
      mma_tf32(sc, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) sc[e] += sc_a[e] + sc_b[e];

    // ---- online softmax (exp2 domain), rows g and g + 8; this lane holds keys 2t, 2t + 1 -----------------
    const int64_t key_base = (int64_t)tl * kTK + 2 * t;
    const bool valid0 = key_base < p.L, valid1 = key_base + 1 < p.L;
    float tmax[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float v0 = valid0 ? sc[2 * h] * p.scale_log2 : ninf;
      const float v1 = valid1 ? sc[2 * h + 1] * p.scale_log2 : ninf;
      sc[2 * h] = v0; sc[2 * h + 1] = v1;
      float mx = fmaxf(v0, v1);
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
    // P as the A operand of the k8 step over this tile's keys: slot t = key 2t, slot t + 4 = key 2t + 1
    uint32_t ph[4], pl[4];
    {
      const float p00 = valid0 ? ex2(sc[0] - m_used[0]) : 0.f;   // row g,     key 2t
      const float p01 = valid1 ? ex2(sc[1] - m_used[0]) : 0.f;   // row g,     key 2t + 1
      const float p10 = valid0 ? ex2(sc[2] - m_used[1]) : 0.f;   // row g + 8, key 2t
      const float p11 = valid1 ? ex2(sc[3] - m_used[1]) : 0.f;   // row g + 8, key 2t + 1
      l_run[0] += p00 + p01;
      l_run[1] += p10 + p11;
      split_tf32(p00, ph[0], pl[0]);
      split_tf32(p10, ph[1], pl[1]);
      split_tf32(p01, ph[2], pl[2]);
      split_tf32(p11, ph[3], pl[3]);
    }

    // ---- O += P V_base, O_lr += P V_lr ---------------------------------------------------------------
#pragma unroll
    for (int nt = 0; nt < kNO; ++nt) {
      const uint32_t line = (uint32_t)((2 * nt) >> 3) * 128u;
      const float v0 = lds32(sV + v_row0 + line + ((((uint32_t)(2 * nt) & 7u) ^ v_c0) << 4));
      const float v1 = lds32(sV + v_row1 + line + ((((uint32_t)(2 * nt) & 7u) ^ v_c1) << 4));
      uint32_t bh0, bl0, bh1, bl1;
      split_tf32(v0, bh0, bl0);
      split_tf32(v1, bh1, bl1);
      mma_3x_add(o[nt], ph, pl, bh0, bh1, bl0, bl1);
    }
    if (RP > 0) {
#pragma unroll
      for (int nt = 0; nt < kNL; ++nt) {
        const uint32_t chunk = (uint32_t)(2 * nt + (g >> 2));
        const uint32_t a0 = sLR + (uint32_t)(2 * t) * kLrRowBytes + ((chunk ^ ((uint32_t)(2 * t) & (uint32_t)kLrSwz)) << 4) + (uint32_t)(g & 3) * 4u;
        const uint32_t a1 = sLR + (uint32_t)(2 * t + 1) * kLrRowBytes + ((chunk ^ ((uint32_t)(2 * t + 1) & (uint32_t)kLrSwz)) << 4) +
                            (uint32_t)(g & 3) * 4u;
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(lds32(a0), bh0, bl0);
        split_tf32(lds32(a1), bh1, bl1);
        mma_3x_add(olr[nt], ph, pl, bh0, bh1, bl0, bl1);
      }
    }

    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (++c_stage == NS) { c_stage = 0; ++c_wrap; }
    if (++tl == T32) { tl = 0; ++u; }
  }
  flush();
}

// (x, y) -> two packed bf16 planes: hi = (bf16(x), bf16(y)), lo = (bf16(x - hi.x), bf16(y - hi.y)); x in the low half
__device__ __forceinline__ void split_bf16x2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x - __uint_as_float(hi << 16), y - __uint_as_float(hi & 0xffff0000u));
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void mma_bf16_k16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// acc += P V over 16 keys from the bf16 planes (p1 v0 + p0 v1 + p0 v0), the tile's product started from zero and added to the
// running sum with round-to-nearest adds (see mma_3x_add)
__device__ __forceinline__ void mma_bf16_3x_add(float (&acc)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint32_t bh0, uint32_t bh1,
                                                uint32_t bl0, uint32_t bl1) {
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  mma_bf16_k16(d, al, bh0, bh1);
  mma_bf16_k16(d, ah, bl0, bl1);
  mma_bf16_k16(d, ah, bh0, bh1);
  asm("{\n\t.reg .b64 a, b;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%4, %5};\n\tadd.rn.f32x2 a, a, b;\n\tmov.b64 {%0, %1}, a;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%6, %7};\n\tadd.rn.f32x2 a, a, b;\n\tmov.b64 {%2, %3}, a;\n\t}"
      : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
      : "f"(d[0]), "f"(d[1]), "f"(d[2]), "f"(d[3]));
}

// The same decode with 16-KEY TILES and the P V products on bf16 planes (round 2).  ncu on the kernel above: one stall per issue
// on the legacy tensor pipe ("math pipe throttle") -- the TF32 MMAs bound it, not HBM.  Per 16 keys it issues 96 (S) + 108 (P V,
// V_lr) HMMA.1688.TF32.  P V only has to meet 1e-4 on the output, and P in [0, 1] / V are exact sums of two bf16 numbers to
// 2^-17 (fla_prefill_split.cu), so here P V = p0 v0 + p1 v0 + p0 v1 as THREE m16n8k16 bf16 MMAs per 16 keys and n8 tile instead
// of six k8 TF32 ones: 96 + 54 MMAs per 16 keys.  The scores keep the split-TF32 products (they sit in the exponent).  A
// 16-key stage also halves the barrier round trips per key and lets both 8-key halves share one split of the Q fragments.
// Needs pages of a multiple of 16 tokens; other pools (and LORAKV_F32_NARROW=1) keep the kernel above.
template <int D, int RP, int MW, int W>
__global__ void __launch_bounds__(W * 32, 1) fla_decode_f32w_kernel(const DecodeF32Params p) {
  constexpr int kTK = 16;
  constexpr int kWorkers = W / MW;
  constexpr uint32_t kRowBytes = D * 4;
  constexpr uint32_t kKvBytes = kTK * kRowBytes;
  constexpr uint32_t kLrRowBytes = RP * 4;
  constexpr uint32_t kLrBytes = kTK * kLrRowBytes;
  constexpr uint32_t kStageBytes = 2 * kKvBytes + kLrBytes;
  constexpr int kLrSwz = RP >= 32 ? 7 : (RP / 4 - 1);   // chunks per LR row - 1, capped at one 128-byte line
  constexpr int kNO = D / 8, kNL = RP / 8;
  constexpr int PS = 4 + D + RP;

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kWorkers][kMaxStages];
  __shared__ uint64_t empty_bar[kWorkers][kMaxStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wk = warp / MW, wi = warp % MW;
  const int g = lane >> 2, t = lane & 3;
  const int NS = p.n_stages;

  if (threadIdx.x == 0) {
    for (int a = 0; a < kWorkers; ++a)
      for (int s = 0; s < NS; ++s) {
        ptx::mbar_init(&full_bar[a][s], 1);
        ptx::mbar_init(&empty_bar[a][s], MW);
      }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  ptx::pdl_wait();                  // launched as a programmatic dependent: the set-up above ran under the predecessor's tail
  ptx::pdl_launch_dependents();

  const int64_t w = (int64_t)blockIdx.x * kWorkers + wk;
  const int64_t g0 = w * p.G;
  const int64_t g1 = min(g0 + p.G, p.total_tiles);
  const int n = g1 > g0 ? (int)(g1 - g0) : 0;
  if (n == 0) return;

  const uint32_t ring = ptx::smem_u32(smem) + (uint32_t)wk * kStageBytes;        // one 16-key buffer per worker
  uint64_t* full = full_bar[wk];
  uint64_t* empty = empty_bar[wk];
  const bool producer = wi == 0;
  const int units_per_layer = p.n_kv_local * p.row_blocks;

  // producer cursor, carried incrementally (no per-tile division); page-table window across the lanes
  int win_base = -(1 << 30), win_kv = 0, win_lr = 0;
  const int T32 = (int)p.T;
  int64_t p_unit = g0 / p.T;
  int p_tl = (int)(g0 - p_unit * p.T);
  int p_page = (p_tl * kTK) / p.P, p_tok = (p_tl * kTK) % p.P;
  int p_layer = (int)(p_unit / units_per_layer), p_kvh = (int)((p_unit / p.row_blocks) % p.n_kv_local);
  // ONE 16-key buffer per worker (a second one does not fit: 8 workers x 17.4 KB), but K and V / V_lr have their own barrier
  // pairs (full[0] / empty[0]: K, full[1] / empty[1]: V + V_lr): the K tile is free once the scores are done, so the next
  // tile's K flies during this tile's softmax and P V, and the next V / V_lr -- issued behind this tile's P V -- during the next
  // tile's score product.  Both copies of a tile come from the same cursor: issue_k computes the addresses, issue_v advances.
  int64_t cur_kv_off = 0, cur_lr_off = 0;
  auto issue_k = [&]() {
    if (p_page < win_base || p_page >= win_base + 32) {
      win_base = p_page;
      const int pg = p_page + lane;
      win_kv = pg < p.n_pages ? p.kv_table[pg] : 0;
      if (RP > 0) win_lr = pg < p.n_pages ? p.lr_table[pg] : 0;
    }
    const int phys_kv = __shfl_sync(0xffffffffu, win_kv, p_page - win_base);
    const int phys_lr = RP > 0 ? __shfl_sync(0xffffffffu, win_lr, p_page - win_base) : 0;
    const int64_t layer = p.layer_begin + p_layer;
    cur_kv_off = layer * p.kv_layer_stride + (int64_t)p_kvh * p.kv_head_stride + (int64_t)phys_kv * p.kv_page_stride + (int64_t)p_tok * D;
    cur_lr_off = RP > 0 ? layer * p.lr_layer_stride + (int64_t)phys_lr * p.lr_page_stride + (int64_t)p_tok * RP : 0;
    if (ptx::elect_one()) {
      ptx::mbar_arrive_expect_tx(&full[0], kKvBytes);
      bulk_g2s(ring, p.k_pages + cur_kv_off, kKvBytes, &full[0], p.l2_policy);
    }
  };
  auto issue_v = [&]() {
    if (ptx::elect_one()) {
      ptx::mbar_arrive_expect_tx(&full[1], kKvBytes + kLrBytes);
      bulk_g2s(ring + kKvBytes, p.v_pages + cur_kv_off, kKvBytes, &full[1], p.l2_policy);
      if (RP > 0) bulk_g2s(ring + 2 * kKvBytes, p.lr_pages + cur_lr_off, kLrBytes, &full[1], p.lr_policy);   // re-read by every kv head
    }
    p_tok += kTK;
    if (p_tok == p.P) { p_tok = 0; ++p_page; }
    if (++p_tl == T32) {
      p_tl = 0; p_page = 0; p_tok = 0;
      ++p_unit;
      p_layer = (int)(p_unit / units_per_layer);
      p_kvh = (int)((p_unit / p.row_blocks) % p.n_kv_local);
    }
  };

  if (producer) { issue_k(); issue_v(); }

  const float ninf = -std::numeric_limits<float>::infinity();
  float qf[D / 8][4];          // A fragments of Q in full fp32: (g, t), (g + 8, t), (g, t + 4), (g + 8, t + 4) of every k8 step
  float o[kNO][4];
  float olr[kNL > 0 ? kNL : 1][4];
  float m_used[2], l_run[2];
  int64_t cur_unit = -1;

  auto flush = [&]() {
    const int64_t first_unit = g0 / p.T;
    const int64_t slot = w * p.max_seg + (cur_unit - first_unit);
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

  // shared-memory byte offsets of this lane's fragment elements inside a K / V tile (the swizzle term is folded in)
  //   K: row g, chunk (2 kk + j) ^ g, word t           -> kOff + ((2 kk + j) ^ g) * 16
  //   V: row 2t + j, chunk (2 nt + (g >> 2)) ^ (2t + j), word g & 3
  const uint32_t k_row = (uint32_t)g * kRowBytes + (uint32_t)t * 4u;
  const uint32_t v_row0 = (uint32_t)(2 * t) * kRowBytes + (uint32_t)(g & 3) * 4u;
  const uint32_t v_row1 = v_row0 + kRowBytes;
  const uint32_t v_c0 = (uint32_t)((g >> 2) ^ (2 * t)), v_c1 = (uint32_t)((g >> 2) ^ (2 * t + 1));   // low chunk bits, pre-XORed

  int64_t u = g0 / p.T;
  int tl = (int)(g0 - u * p.T);
  for (int i = 0; i < n; ++i) {
    if (u != cur_unit) {
      if (cur_unit >= 0) flush();
      cur_unit = u;
      const int layer_rel = (int)(u / units_per_layer);
      const int kvh = (int)((u / p.row_blocks) % p.n_kv_local);
      const int rb = (int)(u % p.row_blocks);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rho = rb * 16 * MW + wi * 16 + g + 8 * h;
        const bool real = rho < p.rows_total;
        const int entry = real ? rho / p.group : 0, gi = real ? rho % p.group : 0;
        const float* src = p.q + (((int64_t)layer_rel * p.n_batch + entry) * p.n_q_local + (int64_t)kvh * p.group + gi) * D;
#pragma unroll
        for (int kk = 0; kk < D / 8; ++kk) {
          qf[kk][h] = real ? __ldg(src + 8 * kk + t) : 0.f;
          qf[kk][2 + h] = real ? __ldg(src + 8 * kk + 4 + t) : 0.f;
        }
        m_used[h] = ninf; l_run[h] = 0.f;
      }
#pragma unroll
      for (int nt = 0; nt < kNO; ++nt) { o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f; }
#pragma unroll
      for (int nt = 0; nt < (kNL > 0 ? kNL : 1); ++nt) { olr[nt][0] = olr[nt][1] = olr[nt][2] = olr[nt][3] = 0.f; }
    }

    const uint32_t sK = ring, sV = sK + kKvBytes, sLR = sV + kKvBytes;
    ptx::mbar_wait(&full[0], (uint32_t)(i & 1));

    // ---- S = Q K^T : 16 rows x 8 keys, 3 x TF32 ------------------------------------------------------
    // three accumulators (hi*hi, lo*hi, hi*lo) so that the 3 * D / 8 MMAs form three chains, not one
    // sc[u]: keys 8 u + {2t, 2t + 1} of rows g (elements 0, 1) and g + 8 (2, 3); the cross terms of both halves share sx[u]
    float sc[2][4], sx[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) { sc[u][e] = 0.f; sx[u][e] = 0.f; }
#pragma unroll
    for (int kk = 0; kk < D / 8; ++kk) {
      uint32_t ah[4], al[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) split_tf32(qf[kk][e], ah[e], al[e]);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t line = sK + k_row + (uint32_t)u * 8u * kRowBytes + (uint32_t)((2 * kk) >> 3) * 128u;
        const float k0 = lds32(line + ((uint32_t)(((2 * kk) & 7) ^ g) << 4));
        const float k1 = lds32(line + ((uint32_t)(((2 * kk + 1) & 7) ^ g) << 4));
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(k0, bh0, bl0);
        split_tf32(k1, bh1, bl1);
        mma_tf32(sx[u], al[0], al[1], al[2], al[3], bh0, bh1);
        mma_tf32(sx[u], ah[0], ah[1], ah[2], ah[3], bl0, bl1);
        mma_tf32(sc[u], ah[0], ah[1], ah[2], ah[3], bh0, bh1);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[u][e] += sx[u][e];
    // the K tile is free: the next tile's K goes out now
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[0]);
    if (producer && i + 1 < n) {
      ptx::mbar_wait(&empty[0], (uint32_t)(i & 1));
      issue_k();
    }

    // ---- online softmax (exp2 domain), rows g and g + 8; this lane holds keys 2t, 2t + 1 -----------------
    const int64_t key_base = (int64_t)tl * kTK + 2 * t;
    bool valid[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) { valid[u][0] = key_base + 8 * u < p.L; valid[u][1] = key_base + 8 * u + 1 < p.L; }
    float tmax[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float mx = ninf;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float v0 = valid[u][0] ? sc[u][2 * h] * p.scale_log2 : ninf;
        const float v1 = valid[u][1] ? sc[u][2 * h + 1] * p.scale_log2 : ninf;
        sc[u][2 * h] = v0; sc[u][2 * h + 1] = v1;
        mx = fmaxf(mx, fmaxf(v0, v1));
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
    // P as the A operand of ONE k16 step over the tile's 16 keys, two bf16 planes: a0 / a1 = rows g / g + 8, keys 2t, 2t + 1;
    // a2 / a3 = the same rows, keys 2t + 8, 2t + 9 -- exactly where the two score halves hold them
    uint32_t ph[4], pl[4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float pa = valid[u][0] ? ex2(sc[u][2 * h] - m_used[h]) : 0.f;
        const float pb = valid[u][1] ? ex2(sc[u][2 * h + 1] - m_used[h]) : 0.f;
        l_run[h] += pa + pb;
        split_bf16x2(pa, pb, ph[2 * u + h], pl[2 * u + h]);
      }

    // ---- O += P V_base, O_lr += P V_lr ---------------------------------------------------------------
    ptx::mbar_wait(&full[1], (uint32_t)(i & 1));
    // B fragments of the k16 step: b0 = (keys 2t, 2t + 1), b1 = (keys 2t + 8, 2t + 9) at column g of the n8 tile -- the rows the
    // k8 fragments already address, and the same rows eight keys further down (the page swizzle repeats every eight tokens)
#pragma unroll
    for (int nt = 0; nt < kNO; ++nt) {
      const uint32_t line = (uint32_t)((2 * nt) >> 3) * 128u;
      const uint32_t a0 = sV + v_row0 + line + ((((uint32_t)(2 * nt) & 7u) ^ v_c0) << 4);
      const uint32_t a1 = sV + v_row1 + line + ((((uint32_t)(2 * nt) & 7u) ^ v_c1) << 4);
      uint32_t bh0, bl0, bh1, bl1;
      split_bf16x2(lds32(a0), lds32(a1), bh0, bl0);
      split_bf16x2(lds32(a0 + 8u * kRowBytes), lds32(a1 + 8u * kRowBytes), bh1, bl1);
      mma_bf16_3x_add(o[nt], ph, pl, bh0, bh1, bl0, bl1);
    }
    if (RP > 0) {
#pragma unroll
      for (int nt = 0; nt < kNL; ++nt) {
        const uint32_t chunk = (uint32_t)(2 * nt + (g >> 2));
        const uint32_t a0 = sLR + (uint32_t)(2 * t) * kLrRowBytes + ((chunk ^ ((uint32_t)(2 * t) & (uint32_t)kLrSwz)) << 4) + (uint32_t)(g & 3) * 4u;
        const uint32_t a1 = sLR + (uint32_t)(2 * t + 1) * kLrRowBytes + ((chunk ^ ((uint32_t)(2 * t + 1) & (uint32_t)kLrSwz)) << 4) +
                            (uint32_t)(g & 3) * 4u;
        uint32_t bh0, bl0, bh1, bl1;
        split_bf16x2(lds32(a0), lds32(a1), bh0, bl0);
        split_bf16x2(lds32(a0 + 8u * kLrRowBytes), lds32(a1 + 8u * kLrRowBytes), bh1, bl1);
        mma_bf16_3x_add(olr[nt], ph, pl, bh0, bh1, bl0, bl1);
      }
    }

    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[1]);
    if (producer && i + 1 < n) {
      ptx::mbar_wait(&empty[1], (uint32_t)(i & 1));
      issue_v();
    }
    if (++tl == T32) { tl = 0; ++u; }
  }
  flush();
}

// ---- prefill blocks over fp32 pages ---------------------------------------------------------------------
// gqa_attention for L_c rows of one agent on one layer (attention.hpp:332-363) with the causal rule of :44-46: key j is
// hidden from the row at position query_offset + i iff j > query_offset + i.  Same fragments, same split-TF32
// products and the same stage ring as the decode kernel, arranged as a flash-attention forward: one CTA = eight
// warps = 128 query rows of one kv head (row = position * group + q head within the group), all eight warps consume
// every 8-key stage of the ring warp 0 fills.  CTAs are ordered kv head by kv head (one head's K / V_base, 33 MB at
// 32K tokens, stays in L2 while its row blocks run) and, inside a head, longest causal range first.  A CTA covers its
// rows' whole key range, so it writes exactly one partial per row and fla_decode_merge (one "split") applies
// B[agent] and the division by l.
struct PrefillF32Params {
  const float *k_pages, *v_pages, *lr_pages;
  const int32_t *kv_table, *lr_table;
  int64_t kv_head_stride, kv_page_stride, lr_page_stride;   // elements; layer offsets already applied to the page pointers
  int P, group, n_kv_local, rows_total, row_blocks, n_pages, n_stages;
  int64_t L_c, query_offset, n_q_local;
  float scale_log2;
  const float* q;        // [L_c][n_q_local * D]
  float* part;           // [n_kv_local * row_blocks][128][4 + D + RP]
};

template <int D, int RP>
__global__ void __launch_bounds__(256, 1) fla_prefill_f32_kernel(const PrefillF32Params p) {
  constexpr int MW = 8;
  constexpr uint32_t kRowBytes = D * 4;
  constexpr uint32_t kKvBytes = kTK * kRowBytes;
  constexpr uint32_t kLrRowBytes = RP * 4;
  constexpr uint32_t kLrBytes = kTK * kLrRowBytes;
  constexpr uint32_t kStageBytes = 2 * kKvBytes + kLrBytes;
  constexpr int kLrSwz = RP >= 32 ? 7 : (RP / 4 - 1);
  constexpr int kNO = D / 8, kNL = RP / 8;
  constexpr int PS = 4 + D + RP;

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[kMaxStages];
  __shared__ uint64_t empty[kMaxStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wi = warp;
  const int g = lane >> 2, t = lane & 3;
  const int NS = p.n_stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], MW); }
    ptx::fence_barrier_init();
  }
  __syncthreads();

  const int kvh = (int)(blockIdx.x / p.row_blocks);
  const int rb = p.row_blocks - 1 - (int)(blockIdx.x % p.row_blocks);     // longest key range first
  const int64_t i_last = min(p.L_c - 1, (int64_t)((rb * 128 + 127) / p.group));
  const int n = (int)((p.query_offset + i_last) / kTK + 1);                 // tiles holding keys 0 .. query_offset + i_last
  const uint32_t ring = ptx::smem_u32(smem);
  const bool producer = wi == 0;

  int win_base = -(1 << 30), win_kv = 0, win_lr = 0;
  int p_page = 0, p_tok = 0, p_stage = 0, p_wrap = 0, p_issued = 0;
  auto issue_next = [&]() {
    if (p_page < win_base || p_page >= win_base + 32) {
      win_base = p_page;
      const int pg = p_page + lane;
      win_kv = pg < p.n_pages ? p.kv_table[pg] : 0;
      if (RP > 0) win_lr = pg < p.n_pages ? p.lr_table[pg] : 0;
    }
    const int phys_kv = __shfl_sync(0xffffffffu, win_kv, p_page - win_base);
    const int phys_lr = RP > 0 ? __shfl_sync(0xffffffffu, win_lr, p_page - win_base) : 0;
    if (ptx::elect_one()) {
      const uint32_t dst = ring + (uint32_t)p_stage * kStageBytes;
      const int64_t kv_off = (int64_t)kvh * p.kv_head_stride + (int64_t)phys_kv * p.kv_page_stride + (int64_t)p_tok * D;
      ptx::mbar_arrive_expect_tx(&full[p_stage], kStageBytes);
      bulk_g2s(dst, p.k_pages + kv_off, kKvBytes, &full[p_stage], ptx::kEvictLast);
      bulk_g2s(dst + kKvBytes, p.v_pages + kv_off, kKvBytes, &full[p_stage], ptx::kEvictLast);
      if (RP > 0) {
        const int64_t lr_off = (int64_t)phys_lr * p.lr_page_stride + (int64_t)p_tok * RP;
        bulk_g2s(dst + 2 * kKvBytes, p.lr_pages + lr_off, kLrBytes, &full[p_stage], ptx::kEvictLast);
      }
    }
    ++p_issued;
    if (++p_stage == NS) { p_stage = 0; ++p_wrap; }
    p_tok += kTK;
    if (p_tok == p.P) { p_tok = 0; ++p_page; }
  };
  if (producer) {
    const int pre = n < NS ? n : NS;
    for (int i = 0; i < pre; ++i) issue_next();
  }

  const float ninf = -std::numeric_limits<float>::infinity();
  float qf[D / 8][4];
  float o[kNO][4];
  float olr[kNL > 0 ? kNL : 1][4];
  float m_used[2], l_run[2];
  int64_t vis[2];                  // last visible key of rows g and g + 8
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int rho = rb * 128 + wi * 16 + g + 8 * h;
    const bool real = rho < p.rows_total;
    const int64_t pos = real ? rho / p.group : i_last;
    const int gi = real ? rho % p.group : 0;
    const float* src = p.q + (pos * p.n_q_local + (int64_t)kvh * p.group + gi) * D;
#pragma unroll
    for (int kk = 0; kk < D / 8; ++kk) {
      qf[kk][h] = real ? __ldg(src + 8 * kk + t) : 0.f;
      qf[kk][2 + h] = real ? __ldg(src + 8 * kk + 4 + t) : 0.f;
    }
    vis[h] = p.query_offset + pos;
    m_used[h] = ninf; l_run[h] = 0.f;
  }
#pragma unroll
  for (int nt = 0; nt < kNO; ++nt) { o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f; }
#pragma unroll
  for (int nt = 0; nt < (kNL > 0 ? kNL : 1); ++nt) { olr[nt][0] = olr[nt][1] = olr[nt][2] = olr[nt][3] = 0.f; }
  // keys beyond the last one any row of this warp may see are skipped (the stage is still released)
  const int64_t warp_vis = p.query_offset + min(i_last, (int64_t)((rb * 128 + wi * 16 + 15) / p.group));

  const uint32_t k_row = (uint32_t)g * kRowBytes + (uint32_t)t * 4u;
  const uint32_t v_row0 = (uint32_t)(2 * t) * kRowBytes + (uint32_t)(g & 3) * 4u;
  const uint32_t v_row1 = v_row0 + kRowBytes;
  const uint32_t v_c0 = (uint32_t)((g >> 2) ^ (2 * t)), v_c1 = (uint32_t)((g >> 2) ^ (2 * t + 1));

  int c_stage = 0, c_wrap = 0;
  for (int i = 0; i < n; ++i) {
    if (producer && i >= 1 && p_issued < n) {
      ptx::mbar_wait(&empty[p_stage], (uint32_t)((p_wrap & 1) ^ 1));
      issue_next();
    }
    const int s = c_stage;
    ptx::mbar_wait(&full[s], (uint32_t)(c_wrap & 1));
    const uint32_t sK = ring + (uint32_t)s * kStageBytes, sV = sK + kKvBytes, sLR = sV + kKvBytes;
    const int64_t key_base = (int64_t)i * kTK + 2 * t;

    if ((int64_t)i * kTK <= warp_vis) {
      float sc[4] = {0.f, 0.f, 0.f, 0.f}, sc_a[4] = {0.f, 0.f, 0.f, 0.f}, sc_b[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < D / 8; ++kk) {
        const uint32_t line = sK + k_row + (uint32_t)((2 * kk) >> 3) * 128u;
        const float k0 = lds32(line + ((uint32_t)(((2 * kk) & 7) ^ g) << 4));
        const float k1 = lds32(line + ((uint32_t)(((2 * kk + 1) & 7) ^ g) << 4));
        uint32_t ah[4], al[4], bh0, bl0, bh1, bl1;
#pragma unroll
        for (int e = 0; e < 4; ++e) split_tf32(qf[kk][e], ah[e], al[e]);
        split_tf32(k0, bh0, bl0);
        split_tf32(k1, bh1, bl1);
        mma_tf32(sc_a, al[0], al[1], al[2], al[3], bh0, bh1);
        mma_tf32(sc_b, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
        mma_tf32(sc, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[e] += sc_a[e] + sc_b[e];

      // causal mask per row (attention.hpp:149-154); masked scores are never exponentiated (:171)
      bool valid[2][2];
      float tmax[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        valid[h][0] = key_base <= vis[h];
        valid[h][1] = key_base + 1 <= vis[h];
        const float v0 = valid[h][0] ? sc[2 * h] * p.scale_log2 : ninf;
        const float v1 = valid[h][1] ? sc[2 * h + 1] * p.scale_log2 : ninf;
        sc[2 * h] = v0; sc[2 * h + 1] = v1;
        float mx = fmaxf(v0, v1);
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
      uint32_t ph[4], pl[4];
      {
        const float p00 = valid[0][0] ? ex2(sc[0] - m_used[0]) : 0.f;
        const float p01 = valid[0][1] ? ex2(sc[1] - m_used[0]) : 0.f;
        const float p10 = valid[1][0] ? ex2(sc[2] - m_used[1]) : 0.f;
        const float p11 = valid[1][1] ? ex2(sc[3] - m_used[1]) : 0.f;
        l_run[0] += p00 + p01;
        l_run[1] += p10 + p11;
        split_tf32(p00, ph[0], pl[0]);
        split_tf32(p10, ph[1], pl[1]);
        split_tf32(p01, ph[2], pl[2]);
        split_tf32(p11, ph[3], pl[3]);
      }
#pragma unroll
      for (int nt = 0; nt < kNO; ++nt) {
        const uint32_t line = (uint32_t)((2 * nt) >> 3) * 128u;
        const float v0 = lds32(sV + v_row0 + line + ((((uint32_t)(2 * nt) & 7u) ^ v_c0) << 4));
        const float v1 = lds32(sV + v_row1 + line + ((((uint32_t)(2 * nt) & 7u) ^ v_c1) << 4));
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(v0, bh0, bl0);
        split_tf32(v1, bh1, bl1);
        mma_3x_add(o[nt], ph, pl, bh0, bh1, bl0, bl1);
      }
      if (RP > 0) {
#pragma unroll
        for (int nt = 0; nt < kNL; ++nt) {
          const uint32_t chunk = (uint32_t)(2 * nt + (g >> 2));
          const uint32_t a0 = sLR + (uint32_t)(2 * t) * kLrRowBytes + ((chunk ^ ((uint32_t)(2 * t) & (uint32_t)kLrSwz)) << 4) + (uint32_t)(g & 3) * 4u;
          const uint32_t a1 = sLR + (uint32_t)(2 * t + 1) * kLrRowBytes + ((chunk ^ ((uint32_t)(2 * t + 1) & (uint32_t)kLrSwz)) << 4) +
                              (uint32_t)(g & 3) * 4u;
          uint32_t bh0, bl0, bh1, bl1;
          split_tf32(lds32(a0), bh0, bl0);
          split_tf32(lds32(a1), bh1, bl1);
          mma_3x_add(olr[nt], ph, pl, bh0, bh1, bl0, bl1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (++c_stage == NS) { c_stage = 0; ++c_wrap; }
  }

  // one partial per row: slot = unit (fla_decode_merge with a single split per row)
  const int64_t unit = (int64_t)kvh * p.row_blocks + rb;
  float* base = p.part + (unit * 128 + wi * 16) * PS;
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
}

template <int D, int RP>
int launch_prefill_t(lorakv_ctx* ctx, const PrefillF32Params& pp, unsigned grid, size_t smem) {
  auto kern = fla_prefill_f32_kernel<D, RP>;
  LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prof_mark(ctx, 0);
  kern<<<grid, 256, smem, ctx->stream>>>(pp);
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

template <int D>
int launch_prefill_rp(lorakv_ctx* ctx, const PrefillF32Params& pp, unsigned grid, size_t smem, int rp) {
  switch (rp) {
    case 0: return launch_prefill_t<D, 0>(ctx, pp, grid, smem);
    case 16: return launch_prefill_t<D, 16>(ctx, pp, grid, smem);
    case 32: return launch_prefill_t<D, 32>(ctx, pp, grid, smem);
    default: return launch_prefill_t<D, 64>(ctx, pp, grid, smem);
  }
}

template <int D, int RP, int MW, bool kWide = false>
int launch_t(lorakv_ctx* ctx, const DecodeF32Params& dp, unsigned grid, size_t smem) {
  constexpr int W = warps_per_cta(MW);
  auto kern = kWide ? fla_decode_f32w_kernel<D, RP, MW, W> : fla_decode_f32_kernel<D, RP, MW, W>;
  static size_t attr_smem = 0;         // the attribute call costs more than the launch: only when the ring grows
  static int attr_device = -1;
  if (attr_device != ctx->device || smem > attr_smem) {
    LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_device = ctx->device; attr_smem = smem;
  }
  prof_mark(ctx, 0);
  LK_CUDA(launch_kernel(ctx, kern, dim3(grid), dim3(W * 32), smem, true, dp));
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

template <int D, int RP>
int launch_mw(lorakv_ctx* ctx, const DecodeF32Params& dp, unsigned grid, size_t smem, int mw, bool wide) {
  if (wide) {
    switch (mw) {
      case 1: return launch_t<D, RP, 1, true>(ctx, dp, grid, smem);
      case 2: return launch_t<D, RP, 2, true>(ctx, dp, grid, smem);
      case 4: return launch_t<D, RP, 4, true>(ctx, dp, grid, smem);
      default: return launch_t<D, RP, 8, true>(ctx, dp, grid, smem);
    }
  }
  switch (mw) {
    case 1: return launch_t<D, RP, 1>(ctx, dp, grid, smem);
    case 2: return launch_t<D, RP, 2>(ctx, dp, grid, smem);
    case 4: return launch_t<D, RP, 4>(ctx, dp, grid, smem);
    default: return launch_t<D, RP, 8>(ctx, dp, grid, smem);
  }
}

template <int D>
int launch_rp(lorakv_ctx* ctx, const DecodeF32Params& dp, unsigned grid, size_t smem, int mw, int rp, bool wide) {
  switch (rp) {
    case 0: return launch_mw<D, 0>(ctx, dp, grid, smem, mw, wide);
    case 16: return launch_mw<D, 16>(ctx, dp, grid, smem, mw, wide);
    case 32: return launch_mw<D, 32>(ctx, dp, grid, smem, mw, wide);
    default: return launch_mw<D, 64>(ctx, dp, grid, smem, mw, wide);
  }
}

}  // namespace

bool decode_f32_supported(const PagedAttnCall& c) {
  const lorakv_pool* pool = c.pool;
  if (pool->rk_pad > 0) return false;          // the key-side low-rank term runs on fla_paged_simt (and fla_decode_tma where built)
  const int64_t d = pool->dims.d_head, rp = pool->r_pad;
  if (pool->dims.dtype != LORAKV_F32) return false;
  if (c.rows_per_entry != 1 || c.query_offset != c.L - 1) return false;   // decode only
  if (d != 64 && d != 128) return false;
  if (!(rp == 0 || rp == 16 || rp == 32 || rp == 64)) return false;
  if (pool->P % kTK != 0) return false;                                    // a tile never straddles a page
  if (c.L < 1 || c.n_batch < 1) return false;
  return true;
}

int launch_decode_f32(const PagedAttnCall& c) {
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
  const int workers_per_cta = warps_per_cta(mw) / mw;
  // 16-key tiles with the P V products on bf16 planes (fla_decode_f32w_kernel) whenever a page holds whole tiles
  static const bool narrow = std::getenv("LORAKV_F32_NARROW") && std::getenv("LORAKV_F32_NARROW")[0] == '1';
  const bool wide = !narrow && pool->P % 16 == 0;
  const int tk = wide ? 16 : kTK;
  const uint32_t stage_bytes = tk * (2 * d + rp) * 4;
  int n_stages = (int)(kRingBudget / (workers_per_cta * stage_bytes));
  if (n_stages > kMaxStages) n_stages = kMaxStages;
  if (wide) n_stages = 1;                 // one buffer per worker, K and V / V_lr released separately (fla_decode_f32w_kernel)
  const size_t smem = (size_t)workers_per_cta * n_stages * stage_bytes;
  if (wide) n_stages = 2;                 // ... with two barrier pairs

  const int64_t T = (c.L + tk - 1) / tk;
  const int64_t units = n_layers * pool->n_kv_local * row_blocks;
  const int64_t total = units * T;
  const int64_t max_workers = (int64_t)ctx->sm_count * workers_per_cta;
  int64_t G = (total + max_workers - 1) / max_workers;
  if (G < 8) G = 8;
  const int64_t n_workers = (total + G - 1) / G;
  const unsigned grid = (unsigned)((n_workers + workers_per_cta - 1) / workers_per_cta);
  const int max_seg = (int)((G + T - 2) / T + 1);
  const int PS = 4 + d + rp;
  const size_t part_bytes = (size_t)grid * workers_per_cta * max_seg * rows_blk * PS * sizeof(float);
  LK_TRY(scratch_reserve(ctx, ctx->work, part_bytes));

  DecodeF32Params dp;
  dp.k_pages = static_cast<const float*>(pool->k_pages);
  dp.v_pages = static_cast<const float*>(pool->v_pages);
  dp.lr_pages = static_cast<const float*>(pool->lr_pages);
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
  dp.scale_log2 = (float)((1.0 / sqrt((double)d)) * 1.4426950408889634);
  dp.l2_policy = ptx::kEvictFirst;
  dp.lr_policy = lr_fits_l2(c, c.L * rp * 4) ? ptx::kEvictLast : ptx::kEvictFirst;
  dp.q = c.q_dev; dp.part = static_cast<float*>(ctx->work.ptr);
  if (d == 128) LK_TRY(launch_rp<128>(ctx, dp, grid, smem, mw, rp, wide));
  else LK_TRY(launch_rp<64>(ctx, dp, grid, smem, mw, rp, wide));

  LK_TRY(launch_decode_merge(ctx, dp.part, d, rp, r, mw, group, (int)pool->n_kv_local, (int)c.n_batch, (int)rows_total, row_blocks,
                             T, G, c.layer_begin, c.n_q_local, max_seg, c.agent_ids_dev, c.adapters, c.out_dev, n_layers, c.peers));
  ctx->last_kernel = "fla_decode_f32";
  return LORAKV_OK;
}

bool prefill_f32_supported(const PagedAttnCall& c) {
  const lorakv_pool* pool = c.pool;
  if (pool->rk_pad > 0) return false;          // the key-side low-rank term runs on fla_paged_simt (and fla_decode_tma where built)
  const int64_t d = pool->dims.d_head, rp = pool->r_pad;
  if (pool->dims.dtype != LORAKV_F32) return false;
  if (c.n_batch != 1 || c.rows_per_entry < 2 || c.layer_end - c.layer_begin != 1) return false;   // prefill blocks only
  if (d != 64 && d != 128) return false;
  if (!(rp == 0 || rp == 16 || rp == 32 || rp == 64)) return false;
  if (pool->P % kTK != 0) return false;
  if (c.L < 1 || c.n_q_local % pool->n_kv_local != 0) return false;
  return true;
}

int launch_prefill_f32(const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const int d = (int)pool->dims.d_head, r = (int)pool->dims.rank, rp = (int)pool->r_pad;
  if (r > 0 && !c.adapters) return fail("paged attention: rank %lld cache needs adapter tables", (long long)r);
  const int group = (int)(c.n_q_local / pool->n_kv_local);
  const int64_t rows_total = c.rows_per_entry * group;
  const int row_blocks = (int)((rows_total + 127) / 128);
  const uint32_t stage_bytes = kTK * (2 * d + rp) * 4;
  int n_stages = (int)(kRingBudget / stage_bytes);
  if (n_stages > kMaxStages) n_stages = kMaxStages;
  const size_t smem = (size_t)n_stages * stage_bytes;
  const int64_t units = pool->n_kv_local * row_blocks;
  const int PS = 4 + d + rp;
  LK_TRY(scratch_reserve(ctx, ctx->work, (size_t)units * 128 * PS * sizeof(float)));

  PrefillF32Params pp;
  const int64_t layer = c.layer_begin;
  pp.k_pages = static_cast<const float*>(pool->k_pages) + layer * pool->kv_layer_stride();
  pp.v_pages = static_cast<const float*>(pool->v_pages) + layer * pool->kv_layer_stride();
  pp.lr_pages = rp > 0 ? static_cast<const float*>(pool->lr_pages) + layer * pool->lr_layer_stride() : nullptr;
  pp.kv_table = pool->kv_space.dev_table + c.kv_set * pool->kv_space.max_pages;
  pp.lr_table = rp > 0 ? pool->lr_space.dev_table + c.lr_set * pool->lr_space.max_pages : nullptr;
  pp.kv_head_stride = pool->kv_head_stride(); pp.kv_page_stride = pool->kv_page_stride(); pp.lr_page_stride = pool->lr_page_stride();
  pp.P = (int)pool->P; pp.group = group; pp.n_kv_local = (int)pool->n_kv_local;
  pp.rows_total = (int)rows_total; pp.row_blocks = row_blocks;
  pp.n_pages = (int)((c.L + pool->P - 1) / pool->P); pp.n_stages = n_stages;
  pp.L_c = c.rows_per_entry; pp.query_offset = c.query_offset; pp.n_q_local = c.n_q_local;
  pp.scale_log2 = (float)((1.0 / sqrt((double)d)) * 1.4426950408889634);
  pp.q = c.q_dev; pp.part = static_cast<float*>(ctx->work.ptr);
  const unsigned grid = (unsigned)units;
  if (d == 128) LK_TRY(launch_prefill_rp<128>(ctx, pp, grid, smem, rp));
  else LK_TRY(launch_prefill_rp<64>(ctx, pp, grid, smem, rp));

  // one partial per row: the merge's closed form with T = G = 1 tile per unit, one segment per worker
  LK_TRY(launch_decode_merge(ctx, pp.part, d, rp, r, /*MW=*/8, group, (int)pool->n_kv_local, /*n_batch=*/(int)c.rows_per_entry,
                             (int)rows_total, row_blocks, /*T=*/1, /*G=*/1, c.layer_begin, c.n_q_local, /*max_seg=*/1,
                             /*agent_ids_dev=*/nullptr, c.adapters, c.out_dev, /*n_layers=*/1, nullptr, /*agent_fixed=*/(int)c.agent_host));
  ctx->last_kernel = "fla_prefill_f32";
  return LORAKV_OK;
}

}  // namespace lk
