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
// (the reference re-reads it per q head, :347-361).  Key tiles of 128 are visited up to the causal
// boundary of the CTA's last row; only the boundary tiles pay for the mask.
//
// Roles (192 threads):
//   warps 0-3  softmax + correction + epilogue; thread t owns MMA row t == TMEM lane t
//   warp 4     TMA producer: bulk copies of K (2 stages) and V_base + V_lr (2 stages), mbarrier tracked
//   warp 5     MMA issuer (one thread): S(j) = Q K_j^T into one of two TMEM S buffers, then
//              O += P_j V_j and O_lr += P_j V_lr_j; issue order S0 S1 PV0 S2 PV1 S3 ... so the tensor
//              pipe computes S(j+1) while the softmax warps work on S(j)
// TMEM (512 columns): S0 [0,128) | S1 [128,256) | O [256,256+D) | O_lr [384,384+RP)
// P goes through shared memory as a K-major SWIZZLE_128B A operand; masked entries are written as
// exact zeros and never exponentiated (attention.hpp:171).  Rescaling of O / O_lr is lazy: only when a
// row's running max grows by more than 8 (log2 units), which leaves the result unchanged.
#include <cuda_bf16.h>

#include <limits>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kBM = 128;            // MMA rows per CTA
constexpr int kBN = 128;            // keys per tile
constexpr int kThreads = 192;
constexpr float kRescaleThreshold = 8.0f;

struct PrefillParams {
  const __nv_bfloat16 *k_pages, *v_pages, *lr_pages;
  const int32_t *kv_table, *lr_table;
  int64_t kv_layer_off, kv_head_stride, kv_page_stride, lr_layer_off, lr_page_stride;   // elements
  int P, group, n_kv_local, n_pages, r;
  int64_t L, L_c, query_offset, n_q_local;
  int n_qblocks;
  float scale_log2, lr_scale;
  const float* q;       // [L_c][n_q_local * D]
  const float* b;       // [r][n_kv_local * D] of this (layer, agent)
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
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

struct Barriers {
  uint64_t q_full, p_full, pv_done;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2];
};

template <int D, int RP>
__global__ void __launch_bounds__(kThreads, 1) fla_prefill_umma_kernel(const PrefillParams p) {
  constexpr int kQBlocks = D / 64;                           // 64-column K-blocks of Q / K; 64-column N-blocks of V
  constexpr uint32_t kBlkBytes = kBN * 128;                  // one [128 rows][64] bf16 block = 16 KB
  constexpr uint32_t kQBytes = kQBlocks * kBlkBytes;
  constexpr uint32_t kKBytes = kQBlocks * kBlkBytes;         // K tile == V tile bytes
  constexpr uint32_t kLrRow = 2 * RP;                        // bytes of one V_lr row
  constexpr uint32_t kLrBytes = kBN * kLrRow;
  constexpr uint32_t kPBytes = 2 * kBlkBytes;                // [2 key blocks][128 rows][64 keys]
  constexpr uint32_t kTmemS = 0, kTmemO = 256, kTmemLr = 384;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ Barriers bars;
  __shared__ uint32_t tmem_base_s;
  unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sQ = smem;
  unsigned char* sK = sQ + kQBytes;                  // 2 stages
  unsigned char* sV = sK + 2 * kKBytes;              // 2 stages
  unsigned char* sP = sV + 2 * kKBytes;
  unsigned char* sLR = sP + kPBytes;                 // 2 stages

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int PB = kBM / p.group;                                  // query positions per CTA
  const int qb = p.n_qblocks - 1 - (int)(blockIdx.x / p.n_kv_local);   // heavy (late) blocks first
  const int kvh = (int)(blockIdx.x % p.n_kv_local);
  const int64_t q0 = (int64_t)qb * PB;
  const int64_t rows_here = min((int64_t)PB, p.L_c - q0);       // real positions in this block
  const int64_t last_visible_cta = p.query_offset + q0 + rows_here - 1;
  const int n_tiles = (int)(last_visible_cta / kBN) + 1;

  if (tid == 0) {
    ptx::mbar_init(&bars.q_full, 128);
    ptx::mbar_init(&bars.p_full, 128);
    ptx::mbar_init(&bars.pv_done, 1);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&bars.k_full[s], 1); ptx::mbar_init(&bars.k_empty[s], 1);
      ptx::mbar_init(&bars.v_full[s], 1); ptx::mbar_init(&bars.v_empty[s], 1);
      ptx::mbar_init(&bars.s_full[s], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc(&tmem_base_s, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const int tpc = p.P < kBN ? p.P : kBN;           // tokens per bulk copy
      const int n_copies = kBN / tpc;
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j & 1;
        const uint32_t par = (uint32_t)(((j >> 1) & 1) ^ 1);     // parity of the phase that freed the stage
        if (j >= 2) ptx::mbar_wait(&bars.k_empty[s], par);
        ptx::mbar_arrive_expect_tx(&bars.k_full[s], kKBytes);
        for (int i = 0; i < n_copies; ++i) {
          const int64_t key0 = (int64_t)j * kBN + (int64_t)i * tpc;
          int page = (int)(key0 / p.P);
          const int tok0 = (int)(key0 % p.P);
          if (page >= p.n_pages) page = p.n_pages - 1;  // wholly masked keys: any finite rows will do
          const int64_t base = p.kv_layer_off + (int64_t)kvh * p.kv_head_stride + (int64_t)p.kv_table[page] * p.kv_page_stride +
                               (int64_t)tok0 * 64;
#pragma unroll
          for (int b = 0; b < kQBlocks; ++b)
            bulk_g2s(ptx::smem_u32(sK + s * kKBytes + b * kBlkBytes + i * tpc * 128), p.k_pages + base + (int64_t)b * p.P * 64,
                     (uint32_t)tpc * 128u, &bars.k_full[s]);
        }
        if (j >= 2) ptx::mbar_wait(&bars.v_empty[s], par);
        ptx::mbar_arrive_expect_tx(&bars.v_full[s], kKBytes + kLrBytes);
        for (int i = 0; i < n_copies; ++i) {
          const int64_t key0 = (int64_t)j * kBN + (int64_t)i * tpc;
          int page = (int)(key0 / p.P);
          const int tok0 = (int)(key0 % p.P);
          if (page >= p.n_pages) page = p.n_pages - 1;
          const int64_t base = p.kv_layer_off + (int64_t)kvh * p.kv_head_stride + (int64_t)p.kv_table[page] * p.kv_page_stride +
                               (int64_t)tok0 * 64;
#pragma unroll
          for (int b = 0; b < kQBlocks; ++b)
            bulk_g2s(ptx::smem_u32(sV + s * kKBytes + b * kBlkBytes + i * tpc * 128), p.v_pages + base + (int64_t)b * p.P * 64,
                     (uint32_t)tpc * 128u, &bars.v_full[s]);
          if (RP > 0) {
            const int64_t lr_base = p.lr_layer_off + (int64_t)p.lr_table[page] * p.lr_page_stride + (int64_t)tok0 * RP;
            bulk_g2s(ptx::smem_u32(sLR + s * kLrBytes + i * tpc * kLrRow), p.lr_pages + lr_base, (uint32_t)tpc * kLrRow,
                     &bars.v_full[s]);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc_s = ptx::instr_desc_bf16(kBM, kBN, ptx::kMajorK, ptx::kMajorK);
      const uint32_t idesc_o = ptx::instr_desc_bf16(kBM, D, ptx::kMajorK, ptx::kMajorMN);
      const uint32_t idesc_lr = ptx::instr_desc_bf16(kBM, RP > 0 ? RP : 16, ptx::kMajorK, ptx::kMajorMN);
      const uint32_t lr_mode = RP == 64 ? ptx::kSw128 : RP == 32 ? ptx::kSw64 : ptx::kSw32;
      const uint32_t q_addr = ptx::smem_u32(sQ), p_addr = ptx::smem_u32(sP);
      auto issue_s = [&](int j) {
        const int s = j & 1;
        ptx::mbar_wait(&bars.k_full[s], (uint32_t)((j >> 1) & 1));
        ptx::tc_fence_after();
        const uint32_t k_addr = ptx::smem_u32(sK + s * kKBytes);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (uint32_t)(ks / 4) * kBlkBytes + (uint32_t)(ks % 4) * 32u;
          ptx::umma_bf16_ss(tmem + kTmemS + (uint32_t)s * kBN, ptx::smem_desc(q_addr + off, 16u, 1024u, ptx::kSw128),
                            ptx::smem_desc(k_addr + off, 16u, 1024u, ptx::kSw128), idesc_s, ks > 0 ? 1u : 0u);
        }
        ptx::umma_commit(&bars.k_empty[s]);
        ptx::umma_commit(&bars.s_full[s]);
      };
      ptx::mbar_wait(&bars.q_full, 0);
      ptx::tc_fence_after();
      issue_s(0);
      if (n_tiles > 1) issue_s(1);
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j & 1;
        ptx::mbar_wait(&bars.p_full, (uint32_t)(j & 1));
        ptx::mbar_wait(&bars.v_full[s], (uint32_t)((j >> 1) & 1));
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(sV + s * kKBytes), lr_addr = ptx::smem_u32(sLR + s * kLrBytes);
#pragma unroll
        for (int ks = 0; ks < kBN / 16; ++ks) {
          const uint64_t pd = ptx::smem_desc(p_addr + (uint32_t)(ks / 4) * kBlkBytes + (uint32_t)(ks % 4) * 32u, 16u, 1024u, ptx::kSw128);
          ptx::umma_bf16_ss(tmem + kTmemO, pd, ptx::smem_desc(v_addr + (uint32_t)ks * 2048u, kBlkBytes, 1024u, ptx::kSw128), idesc_o,
                            (j > 0 || ks > 0) ? 1u : 0u);
          if (RP > 0)
            ptx::umma_bf16_ss(tmem + kTmemLr, pd, ptx::smem_desc(lr_addr + (uint32_t)ks * 16u * kLrRow, kBN * kLrRow, 8u * kLrRow, lr_mode),
                              idesc_lr, (j > 0 || ks > 0) ? 1u : 0u);
        }
        ptx::umma_commit(&bars.v_empty[s]);
        ptx::umma_commit(&bars.pv_done);
        if (j + 2 < n_tiles) issue_s(j + 2);
      }
    }
  } else {
    // ===================== softmax / correction / epilogue: thread t == row t =====================
    const int row = tid;
    const int hg = row / PB;                                // q head within the group
    int64_t pos_local = row % PB;
    if (pos_local >= rows_here) pos_local = rows_here - 1;   // padding rows shadow the last real one
    const bool real_row = (row % PB) < rows_here;
    const int64_t pos = q0 + pos_local;
    const int64_t last_visible = p.query_offset + pos;
    const float ninf = -std::numeric_limits<float>::infinity();

    // ---- Q tile: coalesced fp32 rows -> bf16, K-major SWIZZLE_128B blocks ----
    for (int rr = warp * 32; rr < warp * 32 + 32; ++rr) {
      int64_t pl = rr % PB;
      if (pl >= rows_here) pl = rows_here - 1;
      const float* src = p.q + (q0 + pl) * (p.n_q_local * D) + ((int64_t)kvh * p.group + rr / PB) * D;
      if (4 * lane < D) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src) + lane);
        const int col = 4 * lane;
        const uint32_t off = (uint32_t)(col / 64) * kBlkBytes + ptx::sw128_offset((uint32_t)rr, (uint32_t)(col % 64));
        *reinterpret_cast<uint2*>(sQ + off) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
      }
    }
    ptx::fence_proxy_async_smem();
    ptx::mbar_arrive(&bars.q_full);

    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    float m_used = ninf, l_run = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j & 1;
      ptx::mbar_wait(&bars.s_full[sb], (uint32_t)((j >> 1) & 1));
      ptx::tc_fence_after();
      float sc[kBN];
      {
        uint32_t raw[kBN];
        ptx::tmem_ld128_wait(tmem + lane_base + kTmemS + (uint32_t)sb * kBN, raw);
#pragma unroll
        for (int c = 0; c < kBN; ++c) sc[c] = __uint_as_float(raw[c]);
      }

      const int64_t key0 = (int64_t)j * kBN;
      const bool tile_needs_mask = key0 + kBN - 1 > p.query_offset + q0;   // CTA-uniform
      float mx = ninf;
      if (tile_needs_mask) {
#pragma unroll
        for (int c = 0; c < kBN; ++c) {
          sc[c] = (key0 + c <= last_visible) ? sc[c] * p.scale_log2 : ninf;
          mx = fmaxf(mx, sc[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < kBN; ++c) {
          sc[c] *= p.scale_log2;
          mx = fmaxf(mx, sc[c]);
        }
      }
      const float m_cand = fmaxf(m_used, mx);
      const bool grow = m_cand > m_used + kRescaleThreshold;
      if (j == 0) {
        m_used = m_cand;          // key 0 is visible to every row, so this is finite
      } else if (__any_sync(0xffffffffu, grow)) {
        // correction: O and O_lr of this row are final for tile j-1 once pv_done(j-1) has fired
        ptx::mbar_wait(&bars.pv_done, (uint32_t)((j - 1) & 1));
        ptx::tc_fence_after();
        const float alpha = grow ? ex2(m_used - m_cand) : 1.f;
        if (grow) { m_used = m_cand; l_run *= alpha; }
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 16) {
          uint32_t r16[16];
          ptx::tmem_ld16(tmem + lane_base + kTmemO + c0, r16);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) r16[i] = __float_as_uint(__uint_as_float(r16[i]) * alpha);
          ptx::tmem_st16(tmem + lane_base + kTmemO + c0, r16);
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
      // P = exp2(s - m); masked entries are exact zeros
      float lsum = 0.f;
#pragma unroll
      for (int c = 0; c < kBN; ++c) {
        const float e = ex2(sc[c] - m_used);     // ex2(-inf) == 0 for masked entries
        sc[c] = e;
        lsum += e;
      }
      l_run += lsum;
      // the P buffer (and O) is free once PV(j-1) has completed
      if (j > 0) ptx::mbar_wait(&bars.pv_done, (uint32_t)((j - 1) & 1));
#pragma unroll
      for (int ch = 0; ch < kBN / 8; ++ch) {
        uint4 v;
        v.x = pack_bf16(sc[8 * ch + 0], sc[8 * ch + 1]);
        v.y = pack_bf16(sc[8 * ch + 2], sc[8 * ch + 3]);
        v.z = pack_bf16(sc[8 * ch + 4], sc[8 * ch + 5]);
        v.w = pack_bf16(sc[8 * ch + 6], sc[8 * ch + 7]);
        const uint32_t off = (uint32_t)(ch / 8) * kBlkBytes + (uint32_t)row * 128u + (uint32_t)(((ch % 8) ^ (row & 7)) << 4);
        *reinterpret_cast<uint4*>(sP + off) = v;
      }
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars.p_full);
    }

    // ---- epilogue: o += (lr_scale * o_lr[p]) * B[p,:], out = o / l ----
    ptx::mbar_wait(&bars.pv_done, (uint32_t)((n_tiles - 1) & 1));
    ptx::tc_fence_after();
    float* b_s = reinterpret_cast<float*>(sK);            // K stages are idle now: stage B[r][D] of this kv head
    for (int idx = tid; idx < p.r * D; idx += 128)
      b_s[idx] = p.b[(int64_t)(idx / D) * ((int64_t)p.n_kv_local * D) + (int64_t)kvh * D + idx % D];
    named_bar_sync(1, 128);
    float w[RP > 0 ? RP : 1];
#pragma unroll
    for (int c0 = 0; c0 < RP; c0 += 16) {
      uint32_t r16[16];
      ptx::tmem_ld16(tmem + lane_base + kTmemLr + c0, r16);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) w[c0 + i] = p.lr_scale * __uint_as_float(r16[i]);
    }
    const float inv_l = 1.0f / l_run;
    float* dst = p.out + pos * (p.n_q_local * D) + ((int64_t)kvh * p.group + hg) * D;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 16) {
      uint32_t r16[16];
      ptx::tmem_ld16(tmem + lane_base + kTmemO + c0, r16);
      ptx::tmem_wait_ld();
      float acc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = __uint_as_float(r16[i]);
#pragma unroll
      for (int k = 0; k < RP; ++k) {
        if (k < p.r) {
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = fmaf(w[k], b_s[k * D + c0 + i], acc[i]);
        }
      }
      if (real_row) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(dst + c0 + i) = make_float4(acc[i] * inv_l, acc[i + 1] * inv_l, acc[i + 2] * inv_l, acc[i + 3] * inv_l);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int D, int RP>
int launch_t(lorakv_ctx* ctx, const PrefillParams& pp, unsigned grid) {
  const size_t blk = (size_t)kBN * 128;
  const size_t smem = (D / 64) * blk * 5 + 2 * blk + 2 * (size_t)kBN * 2 * RP + 1024;
  auto kern = fla_prefill_umma_kernel<D, RP>;
  LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prof_mark(ctx, 0);
  kern<<<grid, kThreads, smem, ctx->stream>>>(pp);
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

template <int D>
int launch_rp(lorakv_ctx* ctx, const PrefillParams& pp, unsigned grid, int rp) {
  switch (rp) {
    case 0: return launch_t<D, 0>(ctx, pp, grid);
    case 16: return launch_t<D, 16>(ctx, pp, grid);
    case 32: return launch_t<D, 32>(ctx, pp, grid);
    default: return launch_t<D, 64>(ctx, pp, grid);
  }
}

}  // namespace

bool prefill_umma_supported(const PagedAttnCall& c) {
  const lorakv_pool* pool = c.pool;
  const int64_t d = pool->dims.d_head, rp = pool->r_pad, P = pool->P;
  if (pool->dims.dtype != LORAKV_BF16) return false;
  if (c.n_batch != 1 || c.rows_per_entry < 2 || c.layer_end - c.layer_begin != 1) return false;
  if (d != 64 && d != 128) return false;
  if (!(rp == 0 || rp == 16 || rp == 32 || rp == 64)) return false;
  const int64_t group = c.n_q_local / pool->n_kv_local;
  if (group < 1 || group > kBM || kBM % group != 0) return false;
  if (P < 16 || (P & (P - 1)) != 0) return false;           // power-of-two pages: tiles are made of whole runs
  if (c.L < 1) return false;
  return true;
}

int launch_prefill_umma(const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const int d = (int)pool->dims.d_head, r = (int)pool->dims.rank, rp = (int)pool->r_pad;
  if (r > 0 && !c.adapters) return fail("paged attention: rank %lld cache needs adapter tables", (long long)r);
  const int group = (int)(c.n_q_local / pool->n_kv_local);
  const int PB = kBM / group;
  const int64_t layer = c.layer_begin;
  // the single batch entry's agent id is on the host side of the call (api.cu stages it); B / scale are per agent
  PrefillParams pp;
  pp.k_pages = static_cast<const __nv_bfloat16*>(pool->k_pages);
  pp.v_pages = static_cast<const __nv_bfloat16*>(pool->v_pages);
  pp.lr_pages = static_cast<const __nv_bfloat16*>(pool->lr_pages);
  pp.kv_table = pool->kv_space.dev_table + c.kv_set * pool->kv_space.max_pages;
  pp.lr_table = rp > 0 ? pool->lr_space.dev_table + c.lr_set * pool->lr_space.max_pages : nullptr;
  pp.kv_layer_off = layer * pool->kv_layer_stride(); pp.kv_head_stride = pool->kv_head_stride();
  pp.kv_page_stride = pool->kv_page_stride();
  pp.lr_layer_off = layer * pool->lr_layer_stride(); pp.lr_page_stride = pool->lr_page_stride();
  pp.P = (int)pool->P; pp.group = group; pp.n_kv_local = (int)pool->n_kv_local;
  pp.n_pages = (int)((c.L + pool->P - 1) / pool->P); pp.r = r;
  pp.L = c.L; pp.L_c = c.rows_per_entry; pp.query_offset = c.query_offset; pp.n_q_local = c.n_q_local;
  pp.n_qblocks = (int)((c.rows_per_entry + PB - 1) / PB);
  pp.scale_log2 = (float)((1.0 / sqrt((double)d)) * 1.4426950408889634);
  const int64_t agent = c.agent_host;
  pp.lr_scale = (r > 0) ? c.adapters->scale_host[(size_t)(layer * c.adapters->n_agents + agent)] : 0.f;
  pp.b = (r > 0) ? c.adapters->b + ((layer * c.adapters->n_agents + agent) * r) * (pool->n_kv_local * (int64_t)d) : nullptr;
  pp.q = c.q_dev; pp.out = c.out_dev;
  const unsigned grid = (unsigned)((int64_t)pp.n_qblocks * pool->n_kv_local);
  if (d == 128) LK_TRY(launch_rp<128>(ctx, pp, grid, rp));
  else LK_TRY(launch_rp<64>(ctx, pp, grid, rp));
  ctx->last_kernel = "fla_prefill_umma";
  return LORAKV_OK;
}

}  // namespace lk
