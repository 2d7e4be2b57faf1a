// fla_prefill_split.cu -- fp32-mode prefill (fp32 pages, <= 1e-4 on max_rel_error) on the 5th-generation tensor cores.
//
// What it computes: the same operator as fla_prefill_umma.cu -- gqa_attention (proj/include/lorakv/attention.hpp:332-363)
// for ONE agent on ONE layer with L_c query rows at positions [query_offset, query_offset + L_c), i.e. per q head
// flash_lora_attention (:210-268) with the epilogue o += (lr_scale * o_lr[p]) * B[p,:], out = o / l (:244-259) -- but over a
// pool that stores float32 rows, to the north star's fp32-mode tolerance.
//
// How fp32 accuracy gets onto a bf16 tensor pipe: every fp32 number is an exact sum of bf16 terms,
//     x = x0 + x1 + x2 (+ 2^-27 |x|),   x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1),
// and a product of two such sums is the sum of the pairwise plane products the tensor cores accumulate in fp32:
//     scores   q . k = q0k0 + q0k1 + q1k0 + q0k2 + q2k0 + q1k1        six bf16 MMAs, dropped terms <= 2^-25
//     P V            = p0v0 + p1v0 + p0v1                              three bf16 MMAs, dropped terms <= 2^-17
// The scores sit in the exponent (an absolute error d in s is a relative error d in p; the reference's fuzz grid goes to
// amplitude 25, |s| in the hundreds), so they get three planes; P V only has to meet 1e-4 relative, two planes do.  4.5 times
// the MMA work of the bf16 kernel at bf16 rate -- against three TF32 mma.sync products at an eighth of that rate in
// fla_prefill_f32 (fla_decode_f32.cu), which this kernel replaces for blocks of >= 128 query rows.
//
// Two kernels:
//   split_planes_kernel    one pass over the visible rows of the layer's fp32 pages: K -> three bf16 planes, V_base and V_lr ->
//                          two, written as 64-key STAGE IMAGES (the canonical SWIZZLE_128B / 64B / 32B operand tiles, K-major
//                          for K, MN-major for V and V_lr), so that the attention kernel's producers fill a stage with one
//                          contiguous bulk copy per plane and the tensor cores consume it in place.  HBM-bound, ~1 % of the call.
//   fla_prefill_split_kernel<D, RP>   one CTA = 128 query rows (row = position * g + head) of one kv head x one KEY SPLIT;
//                          warps 0-7 softmax (two warpgroups alternate 64-key tiles), warp 8 / 10 bulk-copy producers (K planes;
//                          V + V_lr planes), warp 9 one elected thread issuing tcgen05.mma.  TMEM (512 columns):
//                          S0 S1 [0,128) | O [128,128+D) | O_lr [256,256+RP) | Q planes [320, 320 + 3 D/2).  P is written back
//                          over its S buffer as two packed planes (hi: columns 0-31, lo: 32-63) and feeds the P V MMAs from TMEM.
//                          The CTA writes an un-normalised partial (m, l, O, O_lr); fla_decode_merge combines the splits of a
//                          row with round-to-nearest fp32 adds and applies B and 1 / l.
// Why key splits: a tensor-core accumulate truncates (measured on the mma.sync path, fla_decode_f32.cu: the running sums shrink
// by ~3e-8 per accumulate step, 2e-4 over a 32K-key row; measured on this kernel: -4.9e-6 / -2.4e-5 / -9.5e-5 for chains of
// 2K / 8K / 32K keys).  A split bounds the chain (4096 keys = 768 accumulate steps, ~1e-5); the combination across splits is
// exact-rounded.  Row sums are fp32 adds of the unrounded P in the softmax threads.
#include <cuda_bf16.h>

#include <cstdlib>
#include <limits>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kBM = 128;            // MMA rows per CTA
constexpr int kTN = 64;             // keys per stage = keys per softmax tile
constexpr int kThreads = 352;       // 8 softmax warps + K producer + MMA issuer + V producer
constexpr int kKStages = 2, kVStages = 2;
constexpr float kRescaleThreshold = 8.0f;

struct SplitPlanes {                 // where the stage images live (elements of bf16 from `base`)
  const __nv_bfloat16* base;
  int64_t k_plane, v_plane, lr_plane;       // offsets of plane 0 of each operand
  int64_t kv_plane_stride, lr_plane_stride; // between planes of one operand
  int64_t kv_head_stride;                   // between kv heads inside a plane
};

struct SplitParams {
  SplitPlanes pl;
  int group, n_kv_local, r;
  int64_t L_c, query_offset, n_q_local;
  int rows_total, row_blocks, splits, tiles_per_split;
  float scale_log2;
  const float* q;       // [L_c][n_q_local * D]
  float* part;          // [(kvh * row_blocks + rb) * splits + split][128][4 + D + RP]
};

struct PlaneSrc {                    // the fp32 pages the planes are cut from
  const float *k_pages, *v_pages, *lr_pages;          // at the layer
  const int32_t *kv_table, *lr_table;
  int64_t kv_head_stride, kv_page_stride, lr_page_stride;
  int P, n_kv_local, D, RP;
  int64_t L_vis;                     // rows [0, L_vis) are cut; the tail of the last stage is zero-filled
  int n_tiles;
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// x[0..8) -> NP bf16 planes of eight values (one 16-byte chunk each): plane p holds bf16(x - sum of the planes before it)
template <int NP>
__device__ __forceinline__ void split8(const float (&x)[8], uint4 (&out)[NP]) {
  float r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = x[i];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[i] = pack_bf16(r[2 * i], r[2 * i + 1]);
      r[2 * i] -= bf16_lo(w[i]);              // exact: the difference of an fp32 number and its bf16 rounding is an fp32 number
      r[2 * i + 1] -= bf16_hi(w[i]);
    }
    out[p] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// grid-stride over (operand, kv head, key, 8-column chunk); operand 0 = K (3 planes), 1 = V_base (2 planes), 2 = V_lr (2 planes)
__global__ void __launch_bounds__(256) split_planes_kernel(const PlaneSrc s, const SplitPlanes pl, __nv_bfloat16* dst) {
  const int cd = s.D / 8, cr = s.RP / 8;
  const int64_t keys = (int64_t)s.n_tiles * kTN;
  const int64_t n_kv = (int64_t)s.n_kv_local * keys * cd;          // chunks of K (and of V)
  const int64_t n_lr = keys * cr;
  const int64_t total = 2 * n_kv + n_lr;
  const PageLayout src_kv = make_page_layout(s.P, s.D, 4);
  const PageLayout src_lr = make_page_layout(s.P, s.RP > 0 ? s.RP : 4, 4);
  const PageLayout dst_lr = make_page_layout(kTN, s.RP > 0 ? s.RP : 8, 2);
  ptx::pdl_wait();                    // the rows may have been appended by the previous kernel on the stream
  ptx::pdl_launch_dependents();
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    float x[8];
    if (idx < 2 * n_kv) {
      const bool is_k = idx < n_kv;
      const int64_t i = is_k ? idx : idx - n_kv;
      const int chunk = (int)(i % cd);
      const int64_t key = (i / cd) % keys;
      const int kvh = (int)(i / (cd * keys));
      if (key < s.L_vis) {
        const int page = (int)(key / s.P), tok = (int)(key % s.P);
        const float* row = (is_k ? s.k_pages : s.v_pages) + (int64_t)kvh * s.kv_head_stride + (int64_t)s.kv_table[page] * s.kv_page_stride;
        const float4 a = *reinterpret_cast<const float4*>(row + page_offset(src_kv, tok, 8 * chunk));
        const float4 b = *reinterpret_cast<const float4*>(row + page_offset(src_kv, tok, 8 * chunk + 4));
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = 0.f;
      }
      // stage image: [tile][D / 64 column blocks][64 keys][64 columns], 128-byte rows, SWIZZLE_128B
      const int tile = (int)(key / kTN), kr = (int)(key % kTN), c = 8 * chunk;
      const int64_t off = (int64_t)kvh * pl.kv_head_stride + ((int64_t)tile * (s.D / 64) + c / 64) * (kTN * 64) +
                          (ptx::sw128_offset((uint32_t)kr, (uint32_t)(c % 64)) >> 1);
      if (is_k) {
        uint4 o[3];
        split8<3>(x, o);
#pragma unroll
        for (int p = 0; p < 3; ++p) *reinterpret_cast<uint4*>(dst + pl.k_plane + p * pl.kv_plane_stride + off) = o[p];
      } else {
        uint4 o[2];
        split8<2>(x, o);
#pragma unroll
        for (int p = 0; p < 2; ++p) *reinterpret_cast<uint4*>(dst + pl.v_plane + p * pl.kv_plane_stride + off) = o[p];
      }
    } else {
      const int64_t i = idx - 2 * n_kv;
      const int chunk = (int)(i % cr);
      const int64_t key = i / cr;
      if (key < s.L_vis) {
        const int page = (int)(key / s.P), tok = (int)(key % s.P);
        const float* row = s.lr_pages + (int64_t)s.lr_table[page] * s.lr_page_stride;
        const float4 a = *reinterpret_cast<const float4*>(row + page_offset(src_lr, tok, 8 * chunk));
        const float4 b = *reinterpret_cast<const float4*>(row + page_offset(src_lr, tok, 8 * chunk + 4));
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = 0.f;
      }
      const int tile = (int)(key / kTN), kr = (int)(key % kTN);
      const int64_t off = (int64_t)tile * (kTN * s.RP) + page_offset(dst_lr, kr, 8 * chunk);
      uint4 o[2];
      split8<2>(x, o);
#pragma unroll
      for (int p = 0; p < 2; ++p) *reinterpret_cast<uint4*>(dst + pl.lr_plane + p * pl.lr_plane_stride + off) = o[p];
    }
  }
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)), "l"(policy)
               : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

struct Barriers {
  uint64_t q_full, s_full[2], p_full[2], pv_done[2], all_done;
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages], hand[8];
};

template <int D, int RP>
__global__ void __launch_bounds__(kThreads, 1) fla_prefill_split_kernel(const SplitParams p) {
  constexpr int kQBlocks = D / 64;
  constexpr uint32_t kBlkBytes = kTN * 128;                   // one [64 keys][64 columns] bf16 block = 8 KB
  constexpr uint32_t kPlaneBytes = kQBlocks * kBlkBytes;      // one plane of a K or V stage
  constexpr uint32_t kKStage = 3 * kPlaneBytes, kVStage = 2 * kPlaneBytes;
  constexpr uint32_t kLrRow = 2 * RP, kLrPlane = kTN * kLrRow, kLrStage = 2 * kLrPlane;
  constexpr uint32_t kTmemS = 0, kTmemO = 128, kTmemLr = 256, kTmemQ = 320;
  constexpr uint32_t kQPlane = D / 2;                         // packed columns of one Q plane
  constexpr int PS = 4 + D + RP;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ Barriers bars;
  __shared__ uint32_t tmem_base_s;
  __shared__ float m_s[kBM];
  __shared__ float l_s[2][kBM];
  __shared__ float mref_s[2][kBM];
  unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sK = smem;
  unsigned char* sV = sK + kKStages * kKStage;
  unsigned char* sLR = sV + kVStages * kVStage;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // ---- what this CTA owns: heavy (late) row blocks first inside a kv head, the splits of a block next to each other ----
  const int split = (int)(blockIdx.x % p.splits);
  const int rb = p.row_blocks - 1 - (int)((blockIdx.x / p.splits) % p.row_blocks);
  const int kvh = (int)(blockIdx.x / ((unsigned)p.splits * p.row_blocks));
  const int64_t rho0 = (int64_t)rb * kBM;
  const int64_t rho_last = min(rho0 + kBM, (int64_t)p.rows_total) - 1;
  const int64_t pos_lo = rho0 / p.group, pos_hi = rho_last / p.group;
  const int n_tiles_blk = (int)((p.query_offset + pos_hi) / kTN) + 1;
  const int tile_begin = split * p.tiles_per_split;
  const int n_tiles = max(0, min(p.tiles_per_split, n_tiles_blk - tile_begin));
  const int64_t mask_from = p.query_offset + pos_lo + 1;       // first key that some row of the block cannot see
  float* part = p.part + (((int64_t)kvh * p.row_blocks + rb) * p.splits + split) * (int64_t)kBM * PS;

  if (n_tiles == 0) {                  // a split beyond the block's causal range: an empty partial (weight 0 in the merge)
    ptx::pdl_wait();
    if (tid < kBM) { part[(int64_t)tid * PS] = -std::numeric_limits<float>::infinity(); part[(int64_t)tid * PS + 1] = 0.f; }
    return;
  }

  if (tid == 0) {
    ptx::mbar_init(&bars.q_full, 256);
    for (int s = 0; s < 2; ++s) { ptx::mbar_init(&bars.s_full[s], 1); ptx::mbar_init(&bars.p_full[s], 128); ptx::mbar_init(&bars.pv_done[s], 1); }
    ptx::mbar_init(&bars.all_done, 1);
    for (int s = 0; s < kKStages; ++s) { ptx::mbar_init(&bars.k_full[s], 1); ptx::mbar_init(&bars.k_empty[s], 1); }
    for (int s = 0; s < kVStages; ++s) { ptx::mbar_init(&bars.v_full[s], 1); ptx::mbar_init(&bars.v_empty[s], 1); }
    for (int s = 0; s < 8; ++s) ptx::mbar_init(&bars.hand[s], 32);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc(&tmem_base_s, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  ptx::pdl_wait();                     // the planes are written by split_planes_kernel, the predecessor on the stream
  ptx::pdl_launch_dependents();

  if (warp == 8 || warp == 10) {
    // ===================== producers: one contiguous bulk copy per plane and stage =====================
    if (ptx::elect_one()) {
      const bool is_k = warp == 8;
      const __nv_bfloat16* base = p.pl.base + (int64_t)kvh * p.pl.kv_head_stride;
      if (is_k) {
        for (int j = 0; j < n_tiles; ++j) {
          const int s = j % kKStages;
          if (j >= kKStages) ptx::mbar_wait(&bars.k_empty[s], (uint32_t)(((j / kKStages) & 1) ^ 1));
          ptx::mbar_arrive_expect_tx(&bars.k_full[s], kKStage);
          const int64_t tile_off = (int64_t)(tile_begin + j) * (kPlaneBytes / 2);
#pragma unroll
          for (int pln = 0; pln < 3; ++pln)
            bulk_g2s(ptx::smem_u32(sK + s * kKStage + pln * kPlaneBytes), base + p.pl.k_plane + pln * p.pl.kv_plane_stride + tile_off,
                     kPlaneBytes, &bars.k_full[s], ptx::kEvictLast);
        }
      } else {
        for (int j = 0; j < n_tiles; ++j) {
          const int s = j % kVStages;
          if (j >= kVStages) ptx::mbar_wait(&bars.v_empty[s], (uint32_t)(((j / kVStages) & 1) ^ 1));
          ptx::mbar_arrive_expect_tx(&bars.v_full[s], kVStage + kLrStage);
          const int64_t tile_off = (int64_t)(tile_begin + j) * (kPlaneBytes / 2);
#pragma unroll
          for (int pln = 0; pln < 2; ++pln) {
            bulk_g2s(ptx::smem_u32(sV + s * kVStage + pln * kPlaneBytes), base + p.pl.v_plane + pln * p.pl.kv_plane_stride + tile_off,
                     kPlaneBytes, &bars.v_full[s], ptx::kEvictLast);
            if (RP > 0)
              bulk_g2s(ptx::smem_u32(sLR + s * kLrStage + pln * kLrPlane),
                       p.pl.base + p.pl.lr_plane + pln * p.pl.lr_plane_stride + (int64_t)(tile_begin + j) * (kLrPlane / 2), kLrPlane,
                       &bars.v_full[s], ptx::kEvictLast);
          }
        }
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer =====================
    if (ptx::elect_one()) {
      const uint32_t idesc_s = ptx::instr_desc_bf16(kBM, kTN, ptx::kMajorK, ptx::kMajorK);
      const uint32_t idesc_o = ptx::instr_desc_bf16(kBM, D, ptx::kMajorK, ptx::kMajorMN);
      const uint32_t idesc_lr = ptx::instr_desc_bf16(kBM, RP > 0 ? RP : 16, ptx::kMajorK, ptx::kMajorMN);
      const uint32_t lr_mode = RP == 64 ? ptx::kSw128 : RP == 32 ? ptx::kSw64 : ptx::kSw32;
      const uint64_t kd = ptx::smem_desc(ptx::smem_u32(sK), 16u, 1024u, ptx::kSw128);
      const uint64_t vd = ptx::smem_desc(ptx::smem_u32(sV), kBlkBytes, 1024u, ptx::kSw128);
      const uint64_t ld = ptx::smem_desc(ptx::smem_u32(sLR), kTN * kLrRow, 8u * kLrRow, lr_mode);
      const uint32_t kd_hi = (uint32_t)(kd >> 32), vd_hi = (uint32_t)(vd >> 32), ld_hi = (uint32_t)(ld >> 32);
      auto desc = [](uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 32) | lo; };
      // S(j) = sum over the six (Q plane, K plane) pairs, smallest terms first
      auto issue_s = [&](int j) {
        const int ks_stage = j % kKStages;
        ptx::mbar_wait(&bars.k_full[ks_stage], (uint32_t)((j / kKStages) & 1));
        ptx::tc_fence_after();
        const uint32_t k_lo = (uint32_t)kd + (uint32_t)ks_stage * (kKStage >> 4);
        const uint32_t s_tmem = tmem + kTmemS + (uint32_t)(j & 1) * kTN;
        constexpr int qa[6] = {1, 0, 2, 0, 1, 0}, kb[6] = {1, 2, 0, 1, 0, 0};
#pragma unroll
        for (int t = 0; t < 6; ++t) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks)
            ptx::umma_bf16_ts(s_tmem, tmem + kTmemQ + (uint32_t)qa[t] * kQPlane + 8u * ks,
                              desc(kd_hi, k_lo + (uint32_t)((kb[t] * kPlaneBytes + (ks / 4) * kBlkBytes + (ks % 4) * 32u) >> 4)), idesc_s,
                              (t > 0 || ks > 0) ? 1u : 0u);
        }
        ptx::umma_commit(&bars.k_empty[ks_stage]);
        ptx::umma_commit(&bars.s_full[j & 1]);
      };
      ptx::mbar_wait(&bars.q_full, 0);
      ptx::tc_fence_after();
      issue_s(0);
      if (n_tiles > 1) issue_s(1);
      for (int j = 0; j < n_tiles; ++j) {
        const int vs = j % kVStages;
        ptx::mbar_wait(&bars.p_full[j & 1], (uint32_t)((j >> 1) & 1));
        ptx::mbar_wait(&bars.v_full[vs], (uint32_t)((j / kVStages) & 1));
        ptx::tc_fence_after();
        const uint32_t v_lo = (uint32_t)vd + (uint32_t)vs * (kVStage >> 4);
        const uint32_t l_lo = (uint32_t)ld + (uint32_t)vs * (kLrStage >> 4);
        const uint32_t p_tmem = tmem + kTmemS + (uint32_t)(j & 1) * kTN;
        constexpr int pa[3] = {1, 0, 0}, vb[3] = {0, 1, 0};         // p1 v0, p0 v1, p0 v0
#pragma unroll
        for (int t = 0; t < 3; ++t) {
#pragma unroll
          for (int ks = 0; ks < kTN / 16; ++ks) {
            const uint32_t first = (j > 0 || t > 0 || ks > 0) ? 1u : 0u;
            ptx::umma_bf16_ts(tmem + kTmemO, p_tmem + (uint32_t)pa[t] * 32u + 8u * ks,
                              desc(vd_hi, v_lo + (uint32_t)((vb[t] * kPlaneBytes + ks * 2048u) >> 4)), idesc_o, first);
            if (RP > 0)
              ptx::umma_bf16_ts(tmem + kTmemLr, p_tmem + (uint32_t)pa[t] * 32u + 8u * ks,
                                desc(ld_hi, l_lo + (uint32_t)((vb[t] * kLrPlane + ks * 16u * kLrRow) >> 4)), idesc_lr, first);
          }
        }
        ptx::umma_commit(&bars.v_empty[vs]);
        ptx::umma_commit(&bars.pv_done[j & 1]);
        if (j == n_tiles - 1) ptx::umma_commit(&bars.all_done);
        if (j + 2 < n_tiles) issue_s(j + 2);       // into the buffer P(j) was read from: behind PV(j) on the in-order pipe
      }
    }
  } else {
    // ===================== softmax / correction / partial =====================
    const int row = (warp & 3) * 32 + lane;
    const int wg = warp >> 2;
    const int64_t rho = min(rho0 + row, (int64_t)p.rows_total - 1);       // padding rows shadow the last real one
    const int64_t pos = rho / p.group;
    const int hg = (int)(rho % p.group);
    const int64_t last_visible = p.query_offset + pos;
    const float* q_src = p.q + pos * (p.n_q_local * D) + ((int64_t)kvh * p.group + hg) * D;
    const float ninf = -std::numeric_limits<float>::infinity();
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;

    // ---- Q -> TMEM: this thread's half of its row as three bf16 planes of packed pairs ----
    {
      const float* src = q_src + wg * (D / 2);
#pragma unroll
      for (int c0 = 0; c0 < D / 4; c0 += 16) {           // D / 4 packed columns per thread and plane, 16 per store
        uint32_t h0[16], h1[16], h2[16];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(src + 2 * (c0 + i)));
          float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            float a = x[2 * u], b = x[2 * u + 1];
            h0[i + u] = pack_bf16(a, b); a -= bf16_lo(h0[i + u]); b -= bf16_hi(h0[i + u]);
            h1[i + u] = pack_bf16(a, b); a -= bf16_lo(h1[i + u]); b -= bf16_hi(h1[i + u]);
            h2[i + u] = pack_bf16(a, b);
          }
        }
        const uint32_t col = tmem + lane_base + kTmemQ + (uint32_t)wg * (D / 4) + c0;
        ptx::tmem_st16(col, h0);
        ptx::tmem_st16(col + kQPlane, h1);
        ptx::tmem_st16(col + 2 * kQPlane, h2);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars.q_full);
    }

    float m_mine = ninf, l_run = 0.f;
    for (int j = wg; j < n_tiles; j += 2) {
      const int sb = j & 1;
      ptx::mbar_wait(&bars.s_full[sb], (uint32_t)((j >> 1) & 1));
      ptx::tc_fence_after();
      float sc[kTN];
      {
        uint32_t raw[kTN];
        ptx::tmem_ld64_wait(tmem + lane_base + kTmemS + (uint32_t)sb * kTN, raw);
#pragma unroll
        for (int c = 0; c < kTN; ++c) sc[c] = __uint_as_float(raw[c]);
      }
      const int64_t key0 = (int64_t)(tile_begin + j) * kTN;
      if (key0 + kTN - 1 >= mask_from) {                   // CTA-uniform
#pragma unroll
        for (int c = 0; c < kTN; ++c)
          if (key0 + c > last_visible) sc[c] = ninf;
      }
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = sc[u];
#pragma unroll
      for (int c = 8; c < kTN; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], sc[c]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])), fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) *
                       p.scale_log2;

      float m_prev = ninf;
      if (j > 0) {
        ptx::mbar_wait(&bars.hand[(warp & 3) * 2 + (wg ^ 1)], (uint32_t)(((j - 1) >> 1) & 1));
        m_prev = *reinterpret_cast<volatile float*>(&m_s[row]);
      }
      float m_used = m_prev;
      const float m_cand = fmaxf(m_prev, mx);
      // a split that starts beyond a row's causal range sees only masked keys in its first tiles: the maximum stays -inf and
      // every p is an exact zero until the first visible key arrives
      const bool grow = (m_prev == ninf) ? (m_cand != ninf) : (m_cand > m_prev + kRescaleThreshold);
      if (j == 0) {
        m_used = m_cand;
      } else if (__any_sync(0xffffffffu, grow)) {
        ptx::mbar_wait(&bars.pv_done[(j - 1) & 1], (uint32_t)(((j - 1) >> 1) & 1));
        ptx::tc_fence_after();
        const float alpha = grow ? (m_prev == ninf ? 0.f : ex2(m_prev - m_cand)) : 1.f;
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
      if (j + 1 < n_tiles) {
        m_s[row] = m_used;
        ptx::mbar_arrive(&bars.hand[(warp & 3) * 2 + wg]);
      }
      if (m_used != m_mine) {
        l_run *= (m_mine == ninf) ? 0.f : ex2(m_mine - m_used);
        m_mine = m_used;
      }
      // P = exp2(s * scale - m); a row with nothing visible yet (m = -inf) gets exact zeros, not exp2(nan)
      const float m_sub = (m_used == ninf) ? 0.f : m_used;
      float ls4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < kTN; ++c) {
        const float e = ex2(fmaf(sc[c], p.scale_log2, -m_sub));
        sc[c] = e;
        ls4[c & 3] += e;
      }
      l_run += (ls4[0] + ls4[1]) + (ls4[2] + ls4[3]);
      // P(j) -> TMEM over its S buffer: plane 0 in columns [0, 32), plane 1 (the bf16 rounding residual) in [32, 64)
#pragma unroll
      for (int c0 = 0; c0 < kTN / 2; c0 += 16) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float a = sc[2 * (c0 + i)], b = sc[2 * (c0 + i) + 1];
          hi[i] = pack_bf16(a, b);
          lo[i] = pack_bf16(a - bf16_lo(hi[i]), b - bf16_hi(hi[i]));
        }
        ptx::tmem_st16(tmem + lane_base + kTmemS + (uint32_t)sb * kTN + c0, hi);
        ptx::tmem_st16(tmem + lane_base + kTmemS + (uint32_t)sb * kTN + 32u + c0, lo);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars.p_full[sb]);
    }

    ptx::mbar_wait(&bars.all_done, 0);
    ptx::tc_fence_after();
    l_s[wg][row] = l_run;
    mref_s[wg][row] = m_mine;
    named_bar_sync(9, 256);
    const float m_fin = fmaxf(mref_s[0][row], mref_s[1][row]);
    float l_tot = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < 2; ++w2) {
      const float mr = mref_s[w2][row];
      if (mr != ninf) l_tot += l_s[w2][row] * ex2(mr - m_fin);
    }
    // ---- partial of this split: (m, l, O, O_lr) un-normalised ----
    float* prow = part + (int64_t)row * PS;
    if (wg == 0) { prow[0] = m_fin; prow[1] = l_tot; }
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
    if (wg == 1) {
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

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int D, int RP>
int launch_t(lorakv_ctx* ctx, const SplitParams& sp, unsigned grid) {
  const size_t plane = (size_t)(D / 64) * kTN * 128;
  const size_t smem = kKStages * 3 * plane + kVStages * 2 * plane + kVStages * 2 * (size_t)kTN * 2 * RP + 1024;
  auto kern = fla_prefill_split_kernel<D, RP>;
  static int attr_device = -1;
  if (attr_device != ctx->device) {
    LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_device = ctx->device;
  }
  prof_mark(ctx, 0);
  LK_CUDA(launch_kernel(ctx, kern, dim3(grid), dim3(kThreads), smem, true, sp));
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

template <int D>
int launch_rp(lorakv_ctx* ctx, const SplitParams& sp, unsigned grid, int rp) {
  switch (rp) {
    case 0: return launch_t<D, 0>(ctx, sp, grid);
    case 16: return launch_t<D, 16>(ctx, sp, grid);
    case 32: return launch_t<D, 32>(ctx, sp, grid);
    default: return launch_t<D, 64>(ctx, sp, grid);
  }
}

int split_keys() {                     // keys per split: bounds the truncating accumulate chain (see the header)
  static int v = 0;
  if (v == 0) {
    const char* e = std::getenv("LORAKV_SPLIT_KEYS");
    v = e ? atoi(e) : 4096;
    if (v < kTN) v = kTN;
    v = (v + kTN - 1) / kTN * kTN;
  }
  return v;
}

}  // namespace

bool prefill_split_supported(const PagedAttnCall& c) {
  const lorakv_pool* pool = c.pool;
  if (pool->rk_pad > 0) return false;
  const int64_t d = pool->dims.d_head, rp = pool->r_pad;
  if (pool->dims.dtype != LORAKV_F32) return false;
  if (c.n_batch != 1 || c.layer_end - c.layer_begin != 1) return false;
  if (d != 64 && d != 128) return false;
  if (!(rp == 0 || rp == 16 || rp == 32 || rp == 64)) return false;
  if (c.L < 1 || pool->n_kv_local < 1 || c.n_q_local % pool->n_kv_local != 0) return false;
  const int64_t group = c.n_q_local / pool->n_kv_local;
  // the plane pass costs one sweep over the visible cache: it pays from a full 128-row tile per kv head on
  return c.rows_per_entry * group >= kBM;
}

int launch_prefill_split(const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const int d = (int)pool->dims.d_head, r = (int)pool->dims.rank, rp = (int)pool->r_pad;
  if (r > 0 && !c.adapters) return fail("paged attention: rank %lld cache needs adapter tables", (long long)r);
  const int group = (int)(c.n_q_local / pool->n_kv_local);
  const int64_t rows_total = c.rows_per_entry * group;
  const int row_blocks = (int)((rows_total + kBM - 1) / kBM);
  const int64_t L_vis = c.query_offset + c.rows_per_entry;
  const int n_tiles = (int)((L_vis + kTN - 1) / kTN);
  const int64_t layer = c.layer_begin;

  // ---- planes: [K x 3 | V x 2][kv head][tile][D / 64][64][64] and [V_lr x 2][tile][64][RP], bf16 ----
  const int64_t kv_head_stride = (int64_t)n_tiles * kTN * d;
  const int64_t kv_plane = pool->n_kv_local * kv_head_stride;
  const int64_t lr_plane = (int64_t)n_tiles * kTN * rp;
  SplitPlanes pl;
  pl.k_plane = 0; pl.v_plane = 3 * kv_plane; pl.lr_plane = 5 * kv_plane;
  pl.kv_plane_stride = kv_plane; pl.lr_plane_stride = lr_plane; pl.kv_head_stride = kv_head_stride;
  LK_TRY(scratch_reserve(ctx, ctx->planes, (size_t)(5 * kv_plane + 2 * lr_plane) * sizeof(__nv_bfloat16)));
  pl.base = static_cast<const __nv_bfloat16*>(ctx->planes.ptr);

  PlaneSrc src;
  src.k_pages = static_cast<const float*>(pool->k_pages) + layer * pool->kv_layer_stride();
  src.v_pages = static_cast<const float*>(pool->v_pages) + layer * pool->kv_layer_stride();
  src.lr_pages = rp > 0 ? static_cast<const float*>(pool->lr_pages) + layer * pool->lr_layer_stride() : nullptr;
  src.kv_table = pool->kv_space.dev_table + c.kv_set * pool->kv_space.max_pages;
  src.lr_table = rp > 0 ? pool->lr_space.dev_table + c.lr_set * pool->lr_space.max_pages : nullptr;
  src.kv_head_stride = pool->kv_head_stride(); src.kv_page_stride = pool->kv_page_stride(); src.lr_page_stride = pool->lr_page_stride();
  src.P = (int)pool->P; src.n_kv_local = (int)pool->n_kv_local; src.D = d; src.RP = rp;
  src.L_vis = L_vis; src.n_tiles = n_tiles;
  {
    const int64_t chunks = 2 * pool->n_kv_local * (int64_t)n_tiles * kTN * (d / 8) + (int64_t)n_tiles * kTN * (rp / 8);
    int64_t blocks = (chunks + 255) / 256;
    if (blocks > (int64_t)ctx->sm_count * 16) blocks = (int64_t)ctx->sm_count * 16;
    LK_CUDA(launch_kernel(ctx, split_planes_kernel, dim3((unsigned)blocks), dim3(256), 0, true, src, pl,
                          static_cast<__nv_bfloat16*>(ctx->planes.ptr)));
    ctx->launches++;
  }

  SplitParams sp;
  sp.pl = pl; sp.group = group; sp.n_kv_local = (int)pool->n_kv_local; sp.r = r;
  sp.L_c = c.rows_per_entry; sp.query_offset = c.query_offset; sp.n_q_local = c.n_q_local;
  sp.rows_total = (int)rows_total; sp.row_blocks = row_blocks;
  sp.tiles_per_split = (ctx->split_keys > 0 ? (ctx->split_keys + kTN - 1) / kTN : split_keys() / kTN);
  sp.splits = (n_tiles + sp.tiles_per_split - 1) / sp.tiles_per_split;
  // equal splits rather than a short last one
  sp.tiles_per_split = (n_tiles + sp.splits - 1) / sp.splits;
  sp.scale_log2 = (float)((1.0 / sqrt((double)d)) * 1.4426950408889634);
  sp.q = c.q_dev;
  const int PS = 4 + d + rp;
  const int64_t units = pool->n_kv_local * row_blocks;
  LK_TRY(scratch_reserve(ctx, ctx->work, (size_t)(units * sp.splits) * kBM * PS * sizeof(float)));
  sp.part = static_cast<float*>(ctx->work.ptr);
  const unsigned grid = (unsigned)(units * sp.splits);
  if (d == 128) LK_TRY(launch_rp<128>(ctx, sp, grid, rp));
  else LK_TRY(launch_rp<64>(ctx, sp, grid, rp));

  // the merge's closed form: T = splits tiles per unit, G = 1 tile per worker -> the partials of unit u are slots
  // [u * splits, (u + 1) * splits), unit = kv head x row block, rows = (position, head in group)
  LK_TRY(launch_decode_merge(ctx, sp.part, d, rp, r, /*MW=*/8, group, (int)pool->n_kv_local, /*n_batch=*/(int)c.rows_per_entry,
                             (int)rows_total, row_blocks, /*T=*/sp.splits, /*G=*/1, c.layer_begin, c.n_q_local, /*max_seg=*/1,
                             /*agent_ids_dev=*/nullptr, c.adapters, c.out_dev, /*n_layers=*/1, nullptr, /*agent_fixed=*/(int)c.agent_host));
  ctx->last_kernel = "fla_prefill_split";
  return LORAKV_OK;
}

}  // namespace lk
