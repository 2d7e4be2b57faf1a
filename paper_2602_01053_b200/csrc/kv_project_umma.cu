// kv_project_umma.cu -- the step that feeds the cache: K / V_base projection of new context rows, RoPE on the
// keys and the append into the paged cache, in one pass.
//
// Reference (proj/include/lorakv/engine.hpp:376-403): for the rows of the plan's kv range
//     k_rows = x_norm * Wk ; apply_rope(k_rows, n_kv_heads, d_head, kv_range.begin)   (:380-383, :225-243)
//     v_rows = x_norm * Wv                                                             (:384)
//     store.append_key / append_value(layer, agent, kv_range.begin, ...)               (:402-403)
// i.e. two triple-loop matmuls (matrix.hpp:101-111), a rotation pass and two row-by-row copies.
//
// Here, for bf16 pools with d_head 128:
//   pack_x        X (fp32, caller's layout) -> bf16 A-operand tiles [row tile 128][k block 64][128][64], SWIZZLE_128B,
//                 so that one plain cp.async.bulk of 16 KB lands as a canonical K-major tcgen05 operand
//   pack_w        (once per upload) [Wk | Wv] of the pool's kv heads -> bf16 [n block 64][d_model][64], SWIZZLE_128B:
//                 a 64-row slice of a block is a canonical MN-major B operand (the layout V pages use)
//   rope_table    cos / sin of pos * 10000^(-2c/d) in double, stored as float2 (the reference casts the double
//                 cos / sin to T, engine.hpp:235-236)
//   kv_project    one CTA per 128 rows x 256 output columns (two heads): warp 0 streams operand stages with the TMA
//                 engine, warp 1 issues tcgen05.mma (M 128, N 256, accumulators in TMEM), warps 2-5 read the
//                 accumulators, rotate key heads (pairs c, c + 64 sit in the same thread), round to bf16 and store
//                 16-byte chunks straight into the swizzled pages of the right head -- no K / V round trip through HBM.
// fp32 pools (tolerance 1e-4 rules out bf16 operands) and other head sizes take proj_matmul (the reference's
// summation order, bit for bit) + rope + the scatter kernel of cache_kernels.cu.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr int kStages = 4;
constexpr uint32_t kABytes = kBM * kBK * 2;            // 16 KB
constexpr uint32_t kBBlk = kBK * 128;                  // one 64-column n block of a k block: 8 KB
constexpr uint32_t kBBytes = (kBN / 64) * kBBlk;       // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// X[n_rows][d_model] fp32 (row stride ld) -> packed bf16 A tiles; one thread per 16-byte chunk (8 columns)
__global__ void pack_x_kernel(const float* __restrict__ x, int64_t n_rows, int64_t ld, int d_model, __nv_bfloat16* __restrict__ out) {
  const int kb_n = d_model / kBK;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = ((n_rows + kBM - 1) / kBM) * kBM * (int64_t)(d_model / 8);
  if (idx >= total) return;
  const int chunk = (int)(idx % (d_model / 8));
  const int64_t row = idx / (d_model / 8);
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (row < n_rows) {
    const float* src = x + row * ld + (int64_t)chunk * 8;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(src)), b = __ldcs(reinterpret_cast<const float4*>(src + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[u];
    }
  }
  const int64_t tile = row / kBM;
  const int r = (int)(row % kBM), kb = chunk / 8, c = (chunk % 8) * 8;
  unsigned char* dst = reinterpret_cast<unsigned char*>(out) + ((tile * kb_n + kb) * (int64_t)kABytes) + ptx::sw128_offset((uint32_t)r, (uint32_t)c);
  uint4 pk;
  pk.x = pack_bf16(v[0], v[1]); pk.y = pack_bf16(v[2], v[3]); pk.z = pack_bf16(v[4], v[5]); pk.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(dst) = pk;
}

// W[d_model][n_src] fp32 row-major (device), columns [col0, col0 + n_cols) -> packed bf16 n blocks starting at block nb0
__global__ void pack_w_kernel(const float* __restrict__ w, int64_t ldw, int64_t col0, int n_cols, int d_model, int nb0,
                              __nv_bfloat16* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;       // (k row, 8-column chunk)
  const int chunks = n_cols / 8;
  if (idx >= (int64_t)d_model * chunks) return;
  const int k = (int)(idx / chunks), ch = (int)(idx % chunks);
  const float* src = w + (int64_t)k * ldw + col0 + (int64_t)ch * 8;
  float v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = src[u];
  const int nb = nb0 + ch / 8, c = (ch % 8) * 8;
  unsigned char* dst = reinterpret_cast<unsigned char*>(out) + (int64_t)nb * d_model * 128 + ptx::sw128_offset((uint32_t)k, (uint32_t)c);
  uint4 pk;
  pk.x = pack_bf16(v[0], v[1]); pk.y = pack_bf16(v[2], v[3]); pk.z = pack_bf16(v[4], v[5]); pk.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(dst) = pk;
}

// ---- fp32 accuracy on the bf16 tensor pipe (fp32 pools; see fla_prefill_split.cu) --------------------------------------
// x = x0 + x1 + x2 and w = w0 + w1 + w2 (bf16 planes, exact to 2^-27): x w = sum of the six plane products above 2^-25.  The
// products are laid out along the reduction dimension, K' = 6 K, smallest terms first (the accumulator truncates: the large
// x0 w0 terms go last), so that the bf16 GEMM kernel below runs unchanged over the extended operands:
//   A' = [x1 | x0 | x2 | x0 | x1 | x0],  B' = [w1 ; w2 ; w0 ; w1 ; w0 ; w0]
__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }
__device__ __forceinline__ void planes3(const float (&v)[8], uint4 (&o)[3]) {
  float r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = v[i];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[i] = pack_bf16(r[2 * i], r[2 * i + 1]);
      r[2 * i] -= bf16_lo(w[i]);
      r[2 * i + 1] -= bf16_hi(w[i]);
    }
    o[p] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void pack_x_planes_kernel(const float* __restrict__ x, int64_t n_rows, int64_t ld, int d_model, __nv_bfloat16* __restrict__ out) {
  const int kb_n = d_model / kBK;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = ((n_rows + kBM - 1) / kBM) * kBM * (int64_t)(d_model / 8);
  if (idx >= total) return;
  const int chunk = (int)(idx % (d_model / 8));
  const int64_t row = idx / (d_model / 8);
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (row < n_rows) {
    const float* src = x + row * ld + (int64_t)chunk * 8;
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = src[u];
  }
  uint4 o[3];
  planes3(v, o);
  const int64_t tile = row / kBM;
  const int r = (int)(row % kBM), kb = chunk / 8, c = (chunk % 8) * 8;
#pragma unroll
  for (int seg = 0; seg < 6; ++seg) {
    unsigned char* dst = reinterpret_cast<unsigned char*>(out) + ((tile * (6 * kb_n) + seg * kb_n + kb) * (int64_t)kABytes) +
                         ptx::sw128_offset((uint32_t)r, (uint32_t)c);
    *reinterpret_cast<uint4*>(dst) = o[seg == 0 || seg == 4 ? 1 : seg == 2 ? 2 : 0];
  }
}

__global__ void pack_w_planes_kernel(const float* __restrict__ w, int64_t ldw, int64_t col0, int n_cols, int d_model,
                                     __nv_bfloat16* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;       // (k row, 8-column chunk)
  const int chunks = n_cols / 8;
  if (idx >= (int64_t)d_model * chunks) return;
  const int k = (int)(idx / chunks), ch = (int)(idx % chunks);
  const float* src = w + (int64_t)k * ldw + col0 + (int64_t)ch * 8;
  float v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = src[u];
  uint4 o[3];
  planes3(v, o);
  const int nb = ch / 8, c = (ch % 8) * 8;
#pragma unroll
  for (int seg = 0; seg < 6; ++seg) {
    unsigned char* dst = reinterpret_cast<unsigned char*>(out) + (int64_t)nb * (6 * d_model) * 128 +
                         ptx::sw128_offset((uint32_t)(seg * d_model + k), (uint32_t)c);
    *reinterpret_cast<uint4*>(dst) = o[seg == 0 || seg == 3 ? 1 : seg == 1 ? 2 : 0];
  }
}

// the LoRA k block, A side: [hi(s d) | lo(s d) | 0] per row, d = x A (float32 [n_rows][rank]), as one packed A tile per row tile
__global__ void pack_down_kernel(const float* __restrict__ down, int64_t n_rows, int rank, float scale, __nv_bfloat16* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;       // (row, 8-column chunk)
  const int64_t total = ((n_rows + kBM - 1) / kBM) * kBM * 8;
  if (idx >= total) return;
  const int64_t row = idx / 8;
  const int c = (int)(idx % 8) * 8;
  __nv_bfloat16 v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int col = c + u;
    float x = 0.f;
    if (row < n_rows && col < 2 * rank) {
      const float d = scale * down[row * rank + col % rank];
      const float hi = __bfloat162float(__float2bfloat16_rn(d));
      x = col < rank ? hi : d - hi;
    }
    v[u] = __float2bfloat16_rn(x);
  }
  unsigned char* dst = reinterpret_cast<unsigned char*>(out) + (row / kBM) * (int64_t)kABytes + ptx::sw128_offset((uint32_t)(row % kBM), (uint32_t)c);
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
}

// the LoRA k block, B side: rows [0, r) and [r, 2r) both hold B[k][col0 + n] (bf16), the rest is zero
__global__ void pack_lora_b_kernel(const float* __restrict__ b, int64_t ldb, int64_t col0, int n_cols, int rank, __nv_bfloat16* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;       // (k row of 64, 8-column chunk)
  const int chunks = n_cols / 8;
  if (idx >= (int64_t)64 * chunks) return;
  const int k = (int)(idx / chunks), ch = (int)(idx % chunks);
  __nv_bfloat16 v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = __float2bfloat16_rn(k < 2 * rank ? b[(int64_t)(k % rank) * ldb + col0 + (int64_t)ch * 8 + u] : 0.f);
  const int nb = ch / 8, c = (ch % 8) * 8;
  unsigned char* dst = reinterpret_cast<unsigned char*>(out) + (int64_t)nb * kBBlk + ptx::sw128_offset((uint32_t)k, (uint32_t)c);
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
}

// cos / sin table of engine.hpp:233-236 for positions [pos0, pos0 + n): tab[(i * half + c)] = (cos, sin)
__global__ void rope_table_kernel(int64_t pos0, int64_t n, int d_head, float2* __restrict__ tab) {
  const int half = d_head / 2;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * half) return;
  const int c = (int)(idx % half);
  const double pos = (double)(pos0 + idx / half);
  const double freq = pow(10000.0, -2.0 * (double)c / (double)d_head);
  double s, co;
  sincos(pos * freq, &s, &co);
  tab[idx] = make_float2((float)co, (float)s);
}

struct ProjParams {
  const __nv_bfloat16* xa;     // packed X tiles
  const __nv_bfloat16* wb;     // packed [Wk | Wv] of this layer
  const float2* rope;          // [n_rows][64] or null
  __nv_bfloat16 *k_pages, *v_pages;   // page arrays of this layer
  const int32_t* table;        // logical -> physical page of the kv set
  int64_t head_stride, page_stride;
  int P, d_model, n_kv_local;
  int64_t row0, n_rows;        // first logical row of the call's rows; rows computed
  int64_t k_from, v_from;      // logical rows below these already exist in the K / V cache (first writer wins)
  int n_col_blocks, n_row_tiles;      // the persistent CTAs walk tiles t = blockIdx.x + i * gridDim.x, column block fastest
  // LoRA up-projection folded into the GEMM as ONE more k block (query mode, rank <= 32): A = [hi(s d) | lo(s d) | 0],
  // B = [B_q ; B_q ; 0] with d = x A_q -- the tensor pipe adds (s d) B_q for 1.5 % more MMA work instead of 2 r FMAs per
  // output element in the epilogue
  const __nv_bfloat16* xa_extra;      // [row tile][128][64] or null
  const __nv_bfloat16* wb_extra;      // [64-column block][64][64] of this (layer, agent) or null
  // query mode (kQuery): q = rope(x * Wq + q_scale * (x * A_q) * B_q[agent]) as float32 rows (engine.hpp:362-373, :422)
  float* q_out;                // [n_rows][ldq]
  int64_t ldq;
  const float* down;           // x * A_q, [n_rows][r] float32, or null without adapters
  const float* bq;             // B_q[agent] restricted to this shard's heads: [r][ldb]
  int64_t ldb;
  int r;
  float q_scale;
};

struct ProjBarriers {
  uint64_t full[kStages], empty[kStages], acc_full[2], acc_empty[2];
};
constexpr int kLoraSmemRank = 32;                                   // B slice [r][256] float32 fits beside the stages up to this rank
constexpr uint32_t kLoraSmemBytes = kLoraSmemRank * kBN * 4;        // 32 KB

template <bool kQuery>
__global__ void __launch_bounds__(kThreads, 1) kv_project_umma_kernel(const ProjParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ ProjBarriers bars;
  __shared__ uint32_t tmem_base_s;
  unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Persistent: CTA b walks tiles t = b, b + gridDim.x, ...; t -> (column block t % n_col_blocks, row tile t / n_col_blocks), column
  // block fastest so that the CTAs sharing an X tile run together and X is read from HBM once (with the row tile fastest it
  // was re-read per column block: 982 MB of DRAM reads for 151 MB of operands).  Two accumulators in TMEM (2 x 256 columns):
  // the epilogue warps drain tile i while the MMA thread already accumulates tile i + 1.
  const int kb_w = p.d_model / kBK;                               // k blocks of the weight matrix
  const int kb_n = kb_w + (p.xa_extra != nullptr ? 1 : 0);         // + the LoRA block
  const int total_tiles = p.n_col_blocks * p.n_row_tiles;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) { ptx::mbar_init(&bars.full[s], 1); ptx::mbar_init(&bars.empty[s], 1); }
    for (int a = 0; a < 2; ++a) { ptx::mbar_init(&bars.acc_full[a], 1); ptx::mbar_init(&bars.acc_empty[a], 128); }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(&tmem_base_s, 2 * kBN);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (ptx::elect_one()) {
      int kbg = 0;                                   // k blocks issued so far: the ring runs on across tiles
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const int nblk = t % p.n_col_blocks, tile = t / p.n_col_blocks;
        const unsigned char* a_src = reinterpret_cast<const unsigned char*>(p.xa) + (int64_t)tile * kb_w * kABytes;
        const unsigned char* b_src = reinterpret_cast<const unsigned char*>(p.wb) + (int64_t)nblk * (kBN / 64) * p.d_model * 128;
        for (int kb = 0; kb < kb_n; ++kb, ++kbg) {
          const int s = kbg % kStages;
          if (kbg >= kStages) ptx::mbar_wait(&bars.empty[s], (uint32_t)(((kbg / kStages) & 1) ^ 1));
          ptx::mbar_arrive_expect_tx(&bars.full[s], kStageBytes);
          const uint32_t dst = ptx::smem_u32(smem + s * kStageBytes);
          if (kb < kb_w) {
            bulk_g2s(dst, a_src + (int64_t)kb * kABytes, kABytes, &bars.full[s]);
#pragma unroll
            for (int nb = 0; nb < kBN / 64; ++nb)
              bulk_g2s(dst + kABytes + nb * kBBlk, b_src + (int64_t)nb * p.d_model * 128 + (int64_t)kb * kBBlk, kBBlk, &bars.full[s]);
          } else {                                   // the LoRA block
            bulk_g2s(dst, reinterpret_cast<const unsigned char*>(p.xa_extra) + (int64_t)tile * kABytes, kABytes, &bars.full[s]);
            bulk_g2s(dst + kABytes, reinterpret_cast<const unsigned char*>(p.wb_extra) + (int64_t)nblk * kBBytes, kBBytes, &bars.full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (ptx::elect_one()) {
      const uint32_t idesc = ptx::instr_desc_bf16(kBM, kBN, ptx::kMajorK, ptx::kMajorMN);
      const uint64_t ad = ptx::smem_desc(ptx::smem_u32(smem), 16u, 1024u, ptx::kSw128);
      const uint64_t bd = ptx::smem_desc(ptx::smem_u32(smem) + kABytes, kBBlk, 1024u, ptx::kSw128);
      const uint32_t ad_hi = (uint32_t)(ad >> 32), bd_hi = (uint32_t)(bd >> 32);
      int kbg = 0, li = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++li) {
        const int ab = li & 1;                       // accumulator of this tile
        if (li >= 2) {                               // the epilogue warps have drained its previous tile
          ptx::mbar_wait(&bars.acc_empty[ab], (uint32_t)(((li >> 1) & 1) ^ 1));
          ptx::tc_fence_after();
        }
        for (int kb = 0; kb < kb_n; ++kb, ++kbg) {
          const int s = kbg % kStages;
          ptx::mbar_wait(&bars.full[s], (uint32_t)((kbg / kStages) & 1));
          ptx::tc_fence_after();
          const uint32_t a_lo = (uint32_t)ad + (uint32_t)s * (kStageBytes >> 4), b_lo = (uint32_t)bd + (uint32_t)s * (kStageBytes >> 4);
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks)
            ptx::umma_bf16_ss(tmem + (uint32_t)ab * kBN, ((uint64_t)ad_hi << 32) | (a_lo + (uint32_t)ks * 2u),
                              ((uint64_t)bd_hi << 32) | (b_lo + (uint32_t)ks * (2048u >> 4)), idesc, (kb > 0 || ks > 0) ? 1u : 0u);
          ptx::umma_commit(&bars.empty[s]);
        }
        ptx::umma_commit(&bars.acc_full[ab]);
      }
    }
  } else {
    // ===================== epilogue: TMEM -> (RoPE) -> bf16 -> swizzled pages =====================
    const int q4 = warp & 3;                                    // TMEM lane quarter this warp may read
    const int r = q4 * 32 + lane;
    float* bq_s = reinterpret_cast<float*>(smem + kStages * kStageBytes);      // LoRA slice of the current tile
    const bool lora_smem = p.down != nullptr && p.r <= kLoraSmemRank;
    int li = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++li) {
    const int nblk = t % p.n_col_blocks, tile = t / p.n_col_blocks, ab = li & 1;
    const int64_t i_row = (int64_t)tile * kBM + r;              // row of the call
    const int64_t row = p.row0 + i_row;                         // logical row of the trajectory = position
    const bool live = i_row < p.n_rows;
    const uint32_t lane_base = ((uint32_t)(q4 * 32) << 16) + (uint32_t)ab * kBN;
    if constexpr (kQuery) {
      // every 128-column block is one q head: add the LoRA up-projection, rotate, store float32 rows
      const float* dn = (p.down != nullptr) ? p.down + (live ? i_row : 0) * p.r : nullptr;    // this row's x * A_q
      // B_q[agent][:, the 256 columns of this tile] -> shared memory beside the stages (rank <= 32): the up-projection
      // then reads broadcast float4s instead of 2 * r global loads per element; wider ranks read B through L1
      if (lora_smem) {
        asm volatile("bar.sync 1, 128;" ::: "memory");             // the previous tile's readers are done
        const int et = tid - 64;                                   // 0..127 over the four epilogue warps
        for (int idx = et; idx < p.r * (kBN / 4); idx += 128) {
          const int k = idx / (kBN / 4), c4 = idx % (kBN / 4);
          reinterpret_cast<float4*>(bq_s)[idx] = __ldg(reinterpret_cast<const float4*>(p.bq + (int64_t)k * p.ldb + (int64_t)nblk * kBN) + c4);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      ptx::mbar_wait(&bars.acc_full[ab], (uint32_t)((li >> 1) & 1));
      ptx::tc_fence_after();
#pragma unroll 1
      for (int hb = 0; hb < kBN / 128; ++hb) {
        const int64_t col0 = (int64_t)(nblk * (kBN / 128) + hb) * 128;
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t lo_u[32], hi_u[32];
          ptx::tmem_ld32(tmem + lane_base + (uint32_t)(hb * 128 + c0), lo_u);
          ptx::tmem_ld32(tmem + lane_base + (uint32_t)(hb * 128 + 64 + c0), hi_u);
          ptx::tmem_wait_ld();
          float lo[32], hi[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) { lo[i] = __uint_as_float(lo_u[i]); hi[i] = __uint_as_float(hi_u[i]); }
          if (p.down != nullptr) {
            for (int k = 0; k < p.r; ++k) {
              const float4* brow = lora_smem ? reinterpret_cast<const float4*>(bq_s + k * kBN + hb * 128 + c0)   // same address in every lane
                                             : reinterpret_cast<const float4*>(p.bq + (int64_t)k * p.ldb + col0 + c0);
              const float dk = p.q_scale * __ldg(dn + k);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 bl = brow[i], bh = brow[16 + i];
                lo[4 * i] = fmaf(dk, bl.x, lo[4 * i]); lo[4 * i + 1] = fmaf(dk, bl.y, lo[4 * i + 1]);
                lo[4 * i + 2] = fmaf(dk, bl.z, lo[4 * i + 2]); lo[4 * i + 3] = fmaf(dk, bl.w, lo[4 * i + 3]);
                hi[4 * i] = fmaf(dk, bh.x, hi[4 * i]); hi[4 * i + 1] = fmaf(dk, bh.y, hi[4 * i + 1]);
                hi[4 * i + 2] = fmaf(dk, bh.z, hi[4 * i + 2]); hi[4 * i + 3] = fmaf(dk, bh.w, hi[4 * i + 3]);
              }
            }
          }
          if (p.rope != nullptr && live) {
            const float2* tab = p.rope + i_row * 64 + c0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float2 cs = __ldg(tab + i);
              const float x0 = lo[i], x1 = hi[i];
              lo[i] = x0 * cs.x - x1 * cs.y;
              hi[i] = x0 * cs.y + x1 * cs.x;
            }
          }
          if (live) {
            float* dst = p.q_out + i_row * p.ldq + col0 + c0;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              *reinterpret_cast<float4*>(dst + i) = make_float4(lo[i], lo[i + 1], lo[i + 2], lo[i + 3]);
              *reinterpret_cast<float4*>(dst + 64 + i) = make_float4(hi[i], hi[i + 1], hi[i + 2], hi[i + 3]);
            }
          }
        }
      }
    } else {
    const int64_t phys = live ? p.table[row / p.P] : 0;
    const int tok = (int)(row % p.P);
    // "full values" schemes (NonShared, FullShared) store v_base + (alpha/r) (x A_v) B_v[agent] (engine.hpp:385-393):
    // the B_v columns of this tile's value heads are staged beside the operand stages, as in query mode
    const float* dn = (p.down != nullptr) ? p.down + (live ? i_row : 0) * p.r : nullptr;
    if (lora_smem) {
      asm volatile("bar.sync 1, 128;" ::: "memory");             // the previous tile's readers are done
      const int et = tid - 64;
      for (int idx = et; idx < p.r * (kBN / 4); idx += 128) {
        const int k = idx / (kBN / 4), c4 = idx % (kBN / 4);
        const int gbv = nblk * (kBN / 128) + c4 / 32;            // head block of this float4
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gbv >= p.n_kv_local)
          v = __ldg(reinterpret_cast<const float4*>(p.bq + (int64_t)k * p.ldb + (int64_t)(gbv - p.n_kv_local) * 128) + c4 % 32);
        reinterpret_cast<float4*>(bq_s)[idx] = v;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    ptx::mbar_wait(&bars.acc_full[ab], (uint32_t)((li >> 1) & 1));
    ptx::tc_fence_after();
#pragma unroll 1
    for (int hb = 0; hb < kBN / 128; ++hb) {
      const int gb = nblk * (kBN / 128) + hb;                   // head block among [K heads | V heads]
      const bool is_k = gb < p.n_kv_local;
      const int head = is_k ? gb : gb - p.n_kv_local;
      const bool write = live && row >= (is_k ? p.k_from : p.v_from);
      __nv_bfloat16* page = (is_k ? p.k_pages : p.v_pages) + (int64_t)head * p.head_stride + phys * p.page_stride;
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t lo_u[32], hi_u[32];
        ptx::tmem_ld32(tmem + lane_base + (uint32_t)(hb * 128 + c0), lo_u);
        ptx::tmem_ld32(tmem + lane_base + (uint32_t)(hb * 128 + 64 + c0), hi_u);
        ptx::tmem_wait_ld();
        float lo[32], hi[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) { lo[i] = __uint_as_float(lo_u[i]); hi[i] = __uint_as_float(hi_u[i]); }
        if (is_k && p.rope != nullptr && live) {
          const float2* tab = p.rope + i_row * 64 + c0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 cs = __ldg(tab + i);
            const float x0 = lo[i], x1 = hi[i];
            lo[i] = x0 * cs.x - x1 * cs.y;                      // engine.hpp:239-240
            hi[i] = x0 * cs.y + x1 * cs.x;
          }
        }
        if (!is_k && p.down != nullptr) {
          for (int k = 0; k < p.r; ++k) {
            const float4* brow = lora_smem ? reinterpret_cast<const float4*>(bq_s + k * kBN + hb * 128 + c0)
                                           : reinterpret_cast<const float4*>(p.bq + (int64_t)k * p.ldb + (int64_t)head * 128 + c0);
            const float dk = p.q_scale * __ldg(dn + k);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 bl = brow[i], bh = brow[16 + i];
              lo[4 * i] = fmaf(dk, bl.x, lo[4 * i]); lo[4 * i + 1] = fmaf(dk, bl.y, lo[4 * i + 1]);
              lo[4 * i + 2] = fmaf(dk, bl.z, lo[4 * i + 2]); lo[4 * i + 3] = fmaf(dk, bl.w, lo[4 * i + 3]);
              hi[4 * i] = fmaf(dk, bh.x, hi[4 * i]); hi[4 * i + 1] = fmaf(dk, bh.y, hi[4 * i + 1]);
              hi[4 * i + 2] = fmaf(dk, bh.z, hi[4 * i + 2]); hi[4 * i + 3] = fmaf(dk, bh.w, hi[4 * i + 3]);
            }
          }
        }
        if (write) {
          // page = [2 column blocks][P tokens][64] with the 16-byte chunks of a token's 128-byte row XOR-swizzled by token % 8
          unsigned char* b0 = reinterpret_cast<unsigned char*>(page) + (int64_t)tok * 128;
          unsigned char* b1 = b0 + (int64_t)p.P * 128;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const int chunk = ((c0 / 8 + ch) ^ (tok & 7)) * 16;
            uint4 a, b;
            a.x = pack_bf16(lo[8 * ch + 0], lo[8 * ch + 1]); a.y = pack_bf16(lo[8 * ch + 2], lo[8 * ch + 3]);
            a.z = pack_bf16(lo[8 * ch + 4], lo[8 * ch + 5]); a.w = pack_bf16(lo[8 * ch + 6], lo[8 * ch + 7]);
            b.x = pack_bf16(hi[8 * ch + 0], hi[8 * ch + 1]); b.y = pack_bf16(hi[8 * ch + 2], hi[8 * ch + 3]);
            b.z = pack_bf16(hi[8 * ch + 4], hi[8 * ch + 5]); b.w = pack_bf16(hi[8 * ch + 6], hi[8 * ch + 7]);
            *reinterpret_cast<uint4*>(b0 + chunk) = a;
            *reinterpret_cast<uint4*>(b1 + chunk) = b;
          }
        }
      }
    }
    }
    // this thread's TMEM reads of the tile are complete (every tcgen05.ld above was waited for): hand the accumulator back
    ptx::tc_fence_before();
    ptx::mbar_arrive(&bars.acc_empty[ab]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 2 * kBN);
}

// ---- exact fp32 path: the reference's matmul order (matrix.hpp:101-111) and rotation ------------------------
__global__ void proj_matmul_kernel(const float* __restrict__ x, int64_t ld, const float* __restrict__ w, int64_t ldw, int64_t col0,
                                   int64_t M, int K, int N, float* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  const int64_t i = idx / N, j = idx % N;
  float acc = 0.f;
  for (int k = 0; k < K; ++k) acc = __fadd_rn(acc, __fmul_rn(x[i * ld + k], w[(int64_t)k * ldw + col0 + j]));
  out[idx] = acc;
}
__global__ void axpy_rn_kernel(float* __restrict__ y, const float* __restrict__ x, float a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __fadd_rn(y[i], __fmul_rn(a, x[i]));       // q.data[i] += q_scale * q_up.data[i], engine.hpp:372
}
__global__ void rope_rows_kernel(float* __restrict__ m, int64_t n_rows, int n_heads, int d_head, const float2* __restrict__ tab) {
  const int half = d_head / 2;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * n_heads * half) return;
  const int c = (int)(idx % half), h = (int)((idx / half) % n_heads);
  const int64_t i = idx / ((int64_t)half * n_heads);
  float* base = m + i * ((int64_t)n_heads * d_head) + (int64_t)h * d_head;
  const float2 cs = tab[i * half + c];
  const float x0 = base[c], x1 = base[c + half];
  base[c] = __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
  base[c + half] = __fadd_rn(__fmul_rn(x0, cs.y), __fmul_rn(x1, cs.x));
}

}  // namespace

bool kv_project_fused_shape(int dtype, int64_t d_head, int64_t d_model) {
  return dtype == LORAKV_BF16 && d_head == 128 && d_model % kBK == 0 && d_model >= kBK;
}

int64_t kv_project_packed_elems(int64_t d_model, int64_t n_kv_local, int64_t d_head) { return 2 * n_kv_local * d_head * d_model; }

int launch_pack_w(lorakv_ctx* ctx, const float* w_dev, int64_t ldw, int64_t col0, int64_t n_cols, int64_t d_model, int64_t nb0, void* packed) {
  const int64_t n = d_model * (n_cols / 8);
  pack_w_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(w_dev, ldw, col0, (int)n_cols, (int)d_model, (int)nb0,
                                                                        static_cast<__nv_bfloat16*>(packed));
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

int launch_pack_lora_b(lorakv_ctx* ctx, const float* b_dev, int64_t ldb, int64_t col0, int64_t n_cols, int64_t rank, void* packed) {
  const int64_t n = 64 * (n_cols / 8);
  pack_lora_b_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(b_dev, ldb, col0, (int)n_cols, (int)rank,
                                                                             static_cast<__nv_bfloat16*>(packed));
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

namespace {
// out[n_rows][n_cols] (float32, row stride n_cols) = rope?(x W[:, col0 : col0 + n_cols] + scale * down B) on the tensor cores to
// fp32 accuracy: operands as six bf16 plane products along K (see pack_x_planes_kernel), the bf16 GEMM kernel in query mode.
// xa_planes: packed X planes of these rows (packed here when *xa_ready is false, so that K, V and q can share one pass over x).
bool planes_shape_ok(const lorakv_ctx* ctx, int dtype, int64_t d_head, int64_t d_model, int64_t n_cols, int64_t n_rows, int64_t ld,
                     const float* x_dev) {
  return ctx->policy == 0 && dtype == LORAKV_F32 && d_head == 128 && d_model % kBK == 0 && d_model >= kBK && n_cols % kBN == 0 &&
         n_rows >= 256 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(x_dev) & 15) == 0;
}
size_t planes_x_bytes(int64_t n_rows, int64_t d_model) { return (size_t)((n_rows + kBM - 1) / kBM) * kBM * d_model * 2 * 6; }
size_t planes_w_bytes(int64_t n_cols, int64_t d_model) { return (size_t)n_cols * d_model * 2 * 6; }

int launch_planes_gemm(lorakv_ctx* ctx, const float* x_dev, int64_t ld, int64_t n_rows, int64_t d_model, __nv_bfloat16* xa, bool pack_x,
                       const float* w_dev, int64_t ldw, int64_t col0, int64_t n_cols, __nv_bfloat16* wb, const float2* rope_tab,
                       int64_t pos0, const float* down, const float* b_up, int64_t ldb, int64_t rank, float scale, float* out) {
  const int64_t tiles = (n_rows + kBM - 1) / kBM;
  if (pack_x) {
    const int64_t nx = tiles * kBM * (d_model / 8);
    pack_x_planes_kernel<<<(unsigned)((nx + 255) / 256), 256, 0, ctx->stream>>>(x_dev, n_rows, ld, (int)d_model, xa);
    ctx->launches++;
  }
  const int64_t nw = d_model * (n_cols / 8);
  pack_w_planes_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, ctx->stream>>>(w_dev, ldw, col0, (int)n_cols, (int)d_model, wb);
  ctx->launches++;
  ProjParams pp{};
  pp.xa = xa; pp.wb = wb; pp.rope = rope_tab;
  pp.d_model = (int)(6 * d_model); pp.row0 = pos0; pp.n_rows = n_rows; pp.P = 1; pp.n_kv_local = 0;
  pp.q_out = out; pp.ldq = n_cols; pp.down = rank > 0 ? down : nullptr; pp.bq = b_up; pp.ldb = ldb; pp.r = (int)rank; pp.q_scale = scale;
  pp.xa_extra = nullptr; pp.wb_extra = nullptr;
  pp.n_col_blocks = (int)(n_cols / kBN); pp.n_row_tiles = (int)tiles;
  const size_t smem = (size_t)kStages * kStageBytes + kLoraSmemBytes + 1024;
  LK_CUDA(cudaFuncSetAttribute(kv_project_umma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)std::min<int64_t>((int64_t)pp.n_col_blocks * pp.n_row_tiles, ctx->sm_count);
  prof_mark(ctx, 0);
  kv_project_umma_kernel<true><<<grid, kThreads, smem, ctx->stream>>>(pp);
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}
}  // namespace

// rows [row0, row0 + n_rows) of the trajectory from x_dev (row i of x_dev is logical row row0 + i); K rows below k_from and V
// rows below v_from are already cached and are not written
int launch_kv_project(lorakv_pool* pool, const void* w_packed, const float* wk_dev, const float* wv_dev, int64_t layer, int64_t set,
                      int64_t row0, int64_t k_from, int64_t v_from, const float* x_dev, int64_t n_rows, int64_t ld, bool rope,
                      const float* down_dev, const float* av_dev, const float* bv_dev, int64_t rank, float v_scale) {
  if (n_rows == 0) return LORAKV_OK;
  lorakv_ctx* ctx = pool->ctx;
  const int64_t d = pool->dims.d_head, d_model = pool->dims.d_model, n_kv = pool->n_kv_local;
  const int64_t half = d / 2;
  auto up = [](size_t x) { return (x + 1023) / 1024 * 1024; };
  const size_t tab_bytes = rope ? up((size_t)(n_rows * half) * sizeof(float2)) : 0;
  if (w_packed) {
    const int64_t tiles = (n_rows + kBM - 1) / kBM;
    const size_t xa_bytes = (size_t)tiles * kBM * d_model * 2;
    LK_TRY(scratch_reserve(ctx, ctx->work, tab_bytes + xa_bytes));
    float2* tab = rope ? static_cast<float2*>(ctx->work.ptr) : nullptr;
    __nv_bfloat16* xa = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(ctx->work.ptr) + tab_bytes);
    if (rope) {
      const int64_t n = n_rows * half;
      rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(row0, n_rows, (int)d, tab);
      ctx->launches++;
    }
    const int64_t nx = tiles * kBM * (d_model / 8);
    pack_x_kernel<<<(unsigned)((nx + 255) / 256), 256, 0, ctx->stream>>>(x_dev, n_rows, ld, (int)d_model, xa);
    ctx->launches++;
    ProjParams pp;
    pp.xa = xa; pp.wb = static_cast<const __nv_bfloat16*>(w_packed); pp.rope = tab;
    pp.k_pages = static_cast<__nv_bfloat16*>(pool->k_pages) + layer * pool->kv_layer_stride();
    pp.v_pages = static_cast<__nv_bfloat16*>(pool->v_pages) + layer * pool->kv_layer_stride();
    pp.table = pool->kv_space.dev_table + set * pool->kv_space.max_pages;
    pp.head_stride = pool->kv_head_stride(); pp.page_stride = pool->kv_page_stride();
    pp.P = (int)pool->P; pp.d_model = (int)d_model; pp.n_kv_local = (int)n_kv;
    pp.row0 = row0; pp.n_rows = n_rows; pp.k_from = k_from; pp.v_from = v_from;
    pp.q_out = nullptr; pp.ldq = 0; pp.down = down_dev; pp.bq = bv_dev; pp.ldb = n_kv * d; pp.r = (int)rank; pp.q_scale = v_scale;
    pp.xa_extra = nullptr; pp.wb_extra = nullptr;
    pp.n_col_blocks = (int)(2 * n_kv * d / kBN); pp.n_row_tiles = (int)tiles;
    const size_t smem = (size_t)kStages * kStageBytes + kLoraSmemBytes + 1024;
    LK_CUDA(cudaFuncSetAttribute(kv_project_umma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)pp.n_col_blocks * pp.n_row_tiles, ctx->sm_count);
    prof_mark(ctx, 0);
    kv_project_umma_kernel<false><<<grid, kThreads, smem, ctx->stream>>>(pp);
    prof_mark(ctx, 1);
    ctx->launches++;
    LK_CUDA(cudaGetLastError());
    ctx->last_kernel = "kv_project_umma";
    return LORAKV_OK;
  }
  // exact fp32 path
  const int64_t dkv = n_kv * d;
  const size_t mat_bytes = up((size_t)(n_rows * dkv) * sizeof(float));
  LK_TRY(scratch_reserve(ctx, ctx->work, tab_bytes + 2 * mat_bytes));
  char* base = static_cast<char*>(ctx->work.ptr);
  float2* tab = rope ? reinterpret_cast<float2*>(base) : nullptr;
  float* kbuf = reinterpret_cast<float*>(base + tab_bytes);
  float* vbuf = reinterpret_cast<float*>(base + tab_bytes + mat_bytes);
  const int64_t col0 = pool->dims.kv_head_begin * d, ldw = pool->dims.n_kv_heads * d;
  const int64_t n = n_rows * dkv;
  // many rows of an fp32 pool: the tensor cores over bf16 planes (fp32-accurate, not the reference's summation order; policy 2
  // keeps the exact path).  The full-values merge rides in the V epilogue as fp32 FMAs.
  const bool planes = planes_shape_ok(ctx, pool->dims.dtype, d, d_model, dkv, n_rows, ld, x_dev) && (av_dev == nullptr || rank <= 64);
  if (planes) {
    float* vdown = nullptr;
    if (av_dev != nullptr && rank > 0) {
      LK_TRY(scratch_reserve(ctx, ctx->proj, (size_t)(n_rows * rank) * sizeof(float)));
      vdown = static_cast<float*>(ctx->proj.ptr);
      const int64_t nd = n_rows * rank;
      proj_matmul_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, ctx->stream>>>(x_dev, ld, av_dev, rank, 0, n_rows, (int)d_model, (int)rank, vdown);
      ctx->launches++;
    }
    const size_t xb = up(planes_x_bytes(n_rows, d_model)), wbytes = up(planes_w_bytes(dkv, d_model));
    LK_TRY(scratch_reserve(ctx, ctx->planes, xb + wbytes));
    __nv_bfloat16* xa = static_cast<__nv_bfloat16*>(ctx->planes.ptr);
    __nv_bfloat16* wb = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(ctx->planes.ptr) + xb);
    if (rope) {
      const int64_t nt = n_rows * half;
      rope_table_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, ctx->stream>>>(row0, n_rows, (int)d, tab);
      ctx->launches++;
    }
    LK_TRY(launch_planes_gemm(ctx, x_dev, ld, n_rows, d_model, xa, true, wk_dev, ldw, col0, dkv, wb, rope ? tab : nullptr, row0, nullptr,
                              nullptr, 0, 0, 0.f, kbuf));
    LK_TRY(launch_planes_gemm(ctx, x_dev, ld, n_rows, d_model, xa, false, wv_dev, ldw, col0, dkv, wb, nullptr, row0, vdown, bv_dev, dkv,
                              vdown ? rank : 0, v_scale, vbuf));
  } else {
  proj_matmul_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(x_dev, ld, wk_dev, ldw, col0, n_rows, (int)d_model, (int)dkv, kbuf);
  proj_matmul_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(x_dev, ld, wv_dev, ldw, col0, n_rows, (int)d_model, (int)dkv, vbuf);
  ctx->launches += 2;
  if (rope) {
    const int64_t nt = n_rows * half, nr = n_rows * n_kv * half;
    rope_table_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, ctx->stream>>>(row0, n_rows, (int)d, tab);
    rope_rows_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, ctx->stream>>>(kbuf, n_rows, (int)n_kv, (int)d, tab);
    ctx->launches += 2;
  }
  }
  if (!planes && av_dev != nullptr && rank > 0) {        // v_store = v_base + v_scale * ((x A_v) B_v), engine.hpp:385-393, in the reference's order
    LK_TRY(scratch_reserve(ctx, ctx->proj, (size_t)(n_rows * rank + n) * sizeof(float)));
    float* vdown = static_cast<float*>(ctx->proj.ptr);
    float* vup = vdown + n_rows * rank;
    const int64_t nd = n_rows * rank;
    proj_matmul_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, ctx->stream>>>(x_dev, ld, av_dev, rank, 0, n_rows, (int)d_model, (int)rank, vdown);
    proj_matmul_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(vdown, rank, bv_dev, dkv, 0, n_rows, (int)rank, (int)dkv, vup);
    axpy_rn_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(vbuf, vup, v_scale, n);
    ctx->launches += 3;
  }
  LK_CUDA(cudaGetLastError());
  if (k_from < row0 + n_rows) {
    const int64_t skip = k_from > row0 ? k_from - row0 : 0;
    LK_TRY(launch_append_scatter(pool, LORAKV_KEY, layer, set, row0 + skip, kbuf + skip * dkv, n_rows - skip, dkv));
  }
  if (v_from < row0 + n_rows) {
    const int64_t skip = v_from > row0 ? v_from - row0 : 0;
    LK_TRY(launch_append_scatter(pool, LORAKV_VALUE, layer, set, row0 + skip, vbuf + skip * dkv, n_rows - skip, dkv));
  }
  ctx->last_kernel = planes ? "kv_project_planes" : "kv_project_f32";
  return LORAKV_OK;
}

// ---- query projection: q = rope(x * Wq + scale * (x * A_q) * B_q[agent]) (engine.hpp:362-373, :422) -------------------

int launch_q_project(lorakv_ctx* ctx, bool fused, const void* wq_packed, const float* wq_dev, int64_t ldw, int64_t col0,
                     int64_t d_model, int64_t n_cols, int64_t d_head, const float* down_dev, const float* aq_dev, const float* bq_dev,
                     int64_t ldb, int64_t rank, float q_scale, int64_t pos0, const float* x_dev, int64_t n_rows, int64_t ld, bool rope,
                     float* q_dev, const void* bq_extra) {
  if (n_rows == 0 || n_cols == 0) return LORAKV_OK;
  const int64_t half = d_head / 2;
  auto up = [](size_t x) { return (x + 1023) / 1024 * 1024; };
  const size_t tab_bytes = rope ? up((size_t)(n_rows * half) * sizeof(float2)) : 0;
  if (fused) {
    const int64_t tiles = (n_rows + kBM - 1) / kBM;
    const size_t xa_bytes = (size_t)tiles * kBM * d_model * 2;
    const bool fold = rank > 0 && bq_extra != nullptr && down_dev != nullptr;      // LoRA as one more k block
    LK_TRY(scratch_reserve(ctx, ctx->work, tab_bytes + xa_bytes + (fold ? (size_t)tiles * kABytes : 0)));
    float2* tab = rope ? static_cast<float2*>(ctx->work.ptr) : nullptr;
    __nv_bfloat16* xa = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(ctx->work.ptr) + tab_bytes);
    __nv_bfloat16* xe = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(ctx->work.ptr) + tab_bytes + xa_bytes);
    if (rope) {
      const int64_t n = n_rows * half;
      rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(pos0, n_rows, (int)d_head, tab);
      ctx->launches++;
    }
    const int64_t nx = tiles * kBM * (d_model / 8);
    pack_x_kernel<<<(unsigned)((nx + 255) / 256), 256, 0, ctx->stream>>>(x_dev, n_rows, ld, (int)d_model, xa);
    ctx->launches++;
    if (fold) {
      const int64_t nd = tiles * kBM * 8;
      pack_down_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, ctx->stream>>>(down_dev, n_rows, (int)rank, q_scale, xe);
      ctx->launches++;
    }
    ProjParams pp{};
    pp.xa = xa; pp.wb = static_cast<const __nv_bfloat16*>(wq_packed); pp.rope = tab;
    pp.d_model = (int)d_model; pp.row0 = pos0; pp.n_rows = n_rows; pp.P = 1; pp.n_kv_local = 0;
    pp.q_out = q_dev; pp.ldq = n_cols; pp.down = (rank > 0 && !fold) ? down_dev : nullptr; pp.bq = bq_dev ? bq_dev + col0 : nullptr; pp.ldb = ldb;
    pp.r = (int)rank; pp.q_scale = q_scale;
    pp.xa_extra = fold ? xe : nullptr; pp.wb_extra = fold ? static_cast<const __nv_bfloat16*>(bq_extra) : nullptr;
    pp.n_col_blocks = (int)(n_cols / kBN); pp.n_row_tiles = (int)tiles;
    const size_t smem = (size_t)kStages * kStageBytes + kLoraSmemBytes + 1024;
    LK_CUDA(cudaFuncSetAttribute(kv_project_umma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)pp.n_col_blocks * pp.n_row_tiles, ctx->sm_count);
    prof_mark(ctx, 0);
    kv_project_umma_kernel<true><<<grid, kThreads, smem, ctx->stream>>>(pp);
    prof_mark(ctx, 1);
    ctx->launches++;
    LK_CUDA(cudaGetLastError());
    ctx->last_kernel = "q_project_umma";
    return LORAKV_OK;
  }
  // exact fp32 path in the reference's order: q = x Wq; q_down = x A; q_up = q_down B; q += s * q_up; rope
  const int64_t n = n_rows * n_cols;
  const size_t up_bytes = rank > 0 ? up((size_t)n * sizeof(float)) + up((size_t)(n_rows * rank) * sizeof(float)) : 0;
  LK_TRY(scratch_reserve(ctx, ctx->work, tab_bytes + up_bytes));
  char* base = static_cast<char*>(ctx->work.ptr);
  float2* tab = rope ? reinterpret_cast<float2*>(base) : nullptr;
  if (planes_shape_ok(ctx, LORAKV_F32, d_head, d_model, n_cols, n_rows, ld, x_dev) && rank <= 64) {
    // many rows in fp32 mode: the tensor cores over bf16 planes; q-LoRA = x A_q on the CUDA cores (d_model x rank), its
    // up-projection as fp32 FMAs in the GEMM epilogue
    float* qdown = nullptr;
    if (rank > 0) {
      qdown = reinterpret_cast<float*>(base + tab_bytes);
      const int64_t nd = n_rows * rank;
      proj_matmul_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, ctx->stream>>>(x_dev, ld, aq_dev, rank, 0, n_rows, (int)d_model, (int)rank, qdown);
      ctx->launches++;
    }
    if (rope) {
      const int64_t nt = n_rows * half;
      rope_table_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, ctx->stream>>>(pos0, n_rows, (int)d_head, tab);
      ctx->launches++;
    }
    const size_t xb = up(planes_x_bytes(n_rows, d_model)), wbytes = up(planes_w_bytes(n_cols, d_model));
    LK_TRY(scratch_reserve(ctx, ctx->planes, xb + wbytes));
    __nv_bfloat16* xa = static_cast<__nv_bfloat16*>(ctx->planes.ptr);
    __nv_bfloat16* wb = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(ctx->planes.ptr) + xb);
    LK_TRY(launch_planes_gemm(ctx, x_dev, ld, n_rows, d_model, xa, true, wq_dev, ldw, col0, n_cols, wb, rope ? tab : nullptr, pos0, qdown,
                              bq_dev ? bq_dev + col0 : nullptr, ldb, rank, q_scale, q_dev));
    ctx->last_kernel = "q_project_planes";
    return LORAKV_OK;
  }
  proj_matmul_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(x_dev, ld, wq_dev, ldw, col0, n_rows, (int)d_model, (int)n_cols, q_dev);
  ctx->launches++;
  if (rank > 0) {
    float* qup = reinterpret_cast<float*>(base + tab_bytes);
    float* qdown = reinterpret_cast<float*>(base + tab_bytes + up((size_t)n * sizeof(float)));
    const int64_t nd = n_rows * rank;
    proj_matmul_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, ctx->stream>>>(x_dev, ld, aq_dev, rank, 0, n_rows, (int)d_model, (int)rank, qdown);
    proj_matmul_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(qdown, rank, bq_dev, ldb, col0, n_rows, (int)rank, (int)n_cols, qup);
    axpy_rn_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(q_dev, qup, q_scale, n);
    ctx->launches += 3;
  }
  if (rope) {
    const int64_t nt = n_rows * half, nr = n_rows * (n_cols / d_head) * half;
    rope_table_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, ctx->stream>>>(pos0, n_rows, (int)d_head, tab);
    rope_rows_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, ctx->stream>>>(q_dev, n_rows, (int)(n_cols / d_head), (int)d_head, tab);
    ctx->launches += 2;
  }
  LK_CUDA(cudaGetLastError());
  ctx->last_kernel = "q_project_f32";
  return LORAKV_OK;
}

}  // namespace lk
