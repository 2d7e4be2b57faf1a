// fla_paged_simt.cu -- Flash-LoRA-Attention over the PAGED cache on CUDA cores.
//
// The shape-general device-resident path: any d_head that is a multiple of 4 up to 256, any rank
// up to 128, fp32 or bf16 pages, decode batches and prefill blocks.  It is what the fp32 storage
// mode runs on (TF32 tensor cores would break the 1e-4 contract) and what the
// tcgen05 kernels are validated against.  One CTA owns one (layer, kv head, key split, row block);
// the g query heads of the kv head and all batch entries are rows of the same block, so a K/V/LR
// tile is read from HBM once for all of them -- the reuse the reference's per-head loop
// (attention.hpp:347-361) does not have.
//
// Per 32-key tile (detail::flash_tile_update, attention.hpp:140-200):
//   warp w owns rows w, w+8, ...; lane = key for the scores, lane = column quad for P*V.
// The epilogue (attention.hpp:244-259) runs in the merge kernel after the split reduction:
//   o += (lr_scale * o_lr[p]) * B[agent][p, :], then out = o / l.
#include <cuda_bf16.h>

#include <limits>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kTile = 32;       // keys per tile
constexpr int kThreads = 256;   // 8 warps
constexpr int kRowBlock = 64;   // max rows per CTA

struct SimtParams {
  const void *k_pages, *v_pages, *lr_pages;
  const int32_t *kv_table, *lr_table;      // logical -> physical page of the selected sets
  int64_t kv_layer_stride, kv_head_stride, kv_page_stride, lr_layer_stride, lr_page_stride;
  int P, d, r_pad, group, n_kv_local;
  PageLayout kv_lay, lr_lay;                // element placement inside a page (page_layout.cuh)
  int64_t L;                                // cached rows
  int64_t layer_begin;
  int64_t n_batch, rows_per_entry, query_offset;
  int64_t rows_total;                       // n_batch * rows_per_entry * group  (per kv head)
  int splits;
  int64_t chunk;                            // keys per split, multiple of kTile
  const float* q;                           // [layers][n_batch][rows_per_entry][n_q_local*d]
  float* part;                              // [layers][kv heads][rows_total][splits][2 + d + r_pad]
  int64_t part_stride;
  // key-side low-rank term: the head dimension is extended by rk_pad columns -- q' = [q | qk], K' tile = [K_base | L_k]
  const void* lk_pages; const int32_t* lk_table; int64_t lk_layer_stride, lk_page_stride; int rk_pad; PageLayout lk_lay;
  const float* qk;                          // [layers][n_batch][rows_per_entry][n_q_local][rk_pad]
};

template <class S> struct Elem;
template <> struct Elem<float> {
  static constexpr int kPerChunk = 4;       // elements per 16 bytes
  static __device__ __forceinline__ void load_chunk(const float* p, float* dst) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
  }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kPerChunk = 8;
  static __device__ __forceinline__ void load_chunk(const __nv_bfloat16* p, float* dst) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dst[2 * i] = __uint_as_float(w[i] << 16);
      dst[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};

__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// RW = rows per warp (rows in the block = 8 * RW), QD = column quads per lane (d <= 128 * QD)
template <class S, int RW, int QD>
__global__ void __launch_bounds__(kThreads) fla_paged_simt_kernel(SimtParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = p.d, rp = p.r_pad, rk = p.rk_pad;
  const int dx = d + rk;                         // extended head dimension of the score product
  const int kd = d + 4, kr = rp + 4, kx = dx + 4;   // padded pitches (floats): conflict-free LDS.128
  float* q_s = reinterpret_cast<float*>(smem_raw);          // [8*RW][dx]
  float* k_s = q_s + 8 * RW * dx;                           // [kTile][kx]
  float* v_s = k_s + kTile * kx;                            // [kTile][kd]
  float* lr_s = v_s + kTile * kd;                           // [kTile][kr]
  float* p_s = lr_s + kTile * kr;                           // [8*RW][kTile]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row_block = blockIdx.x;
  const int kvh = blockIdx.y % p.n_kv_local;
  const int64_t layer_rel = blockIdx.y / p.n_kv_local;
  const int split = blockIdx.z;
  const int64_t layer = p.layer_begin + layer_rel;
  const float ninf = -std::numeric_limits<float>::infinity();
  const float inv_sqrt_d = 1.0f / sqrtf(static_cast<float>(d));
  const int64_t n_q_local = (int64_t)p.n_kv_local * p.group;

  // rows of this block: rho = row_block*8*RW + local; rho -> (entry, token, group index)
  const int64_t rho0 = (int64_t)row_block * 8 * RW;
  int64_t row_pos[RW];      // last visible key of each owned row, -1 for padding rows
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int64_t rho = rho0 + warp + 8 * t;
    row_pos[t] = -1;
    if (rho < p.rows_total) {
      const int64_t tok = (rho / p.group) % p.rows_per_entry;
      row_pos[t] = p.query_offset + tok;
    }
  }
  // stage q rows (float) once
  for (int idx = tid; idx < 8 * RW * (d / 4); idx += kThreads) {
    const int lr_ = idx / (d / 4), c4 = idx % (d / 4);
    const int64_t rho = rho0 + lr_;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rho < p.rows_total) {
      const int64_t gi = rho % p.group, et = rho / p.group;   // et = entry*rows_per_entry + token
      const float* src = p.q + ((layer_rel * p.n_batch * p.rows_per_entry + et) * n_q_local +
                                (int64_t)kvh * p.group + gi) * d;
      v = *reinterpret_cast<const float4*>(src + 4 * c4);
    }
    *reinterpret_cast<float4*>(q_s + lr_ * dx + 4 * c4) = v;
  }
  for (int idx = tid; idx < 8 * RW * (rk / 4); idx += kThreads) {      // qk = k_scale * (q B_k^T), columns [d, d + rk)
    const int lr_ = idx / (rk / 4), c4 = idx % (rk / 4);
    const int64_t rho = rho0 + lr_;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rho < p.rows_total) {
      const int64_t gi = rho % p.group, et = rho / p.group;
      v = *reinterpret_cast<const float4*>(p.qk + ((layer_rel * p.n_batch * p.rows_per_entry + et) * n_q_local + (int64_t)kvh * p.group + gi) * rk + 4 * c4);
    }
    *reinterpret_cast<float4*>(q_s + lr_ * dx + d + 4 * c4) = v;
  }

  float o[RW][QD][4], olr[RW][4], m_run[RW], l_run[RW];
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    m_run[t] = ninf; l_run[t] = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      olr[t][u] = 0.f;
#pragma unroll
      for (int qd = 0; qd < QD; ++qd) o[t][qd][u] = 0.f;
    }
  }

  // key range of this split, clipped to the last position any row of the block can see
  int64_t block_last = -1;
  {
    const int64_t rho_last = min(rho0 + 8 * RW, p.rows_total) - 1;
    const int64_t tok_hi = (p.rows_per_entry == 1) ? 0 : ((rho_last / p.group) % p.rows_per_entry);
    // rows of one block may wrap over entries when rows_per_entry > 1 and n_batch > 1; take the
    // safe bound (last token of an entry) in that case
    const int64_t tok_lo = (rho0 / p.group) % p.rows_per_entry;
    block_last = p.query_offset + ((tok_hi >= tok_lo) ? tok_hi : p.rows_per_entry - 1);
  }
  const int64_t j_begin = (int64_t)split * p.chunk;
  int64_t j_end = min(j_begin + p.chunk, p.L);
  j_end = min(j_end, block_last + 1);

  const S* kp = static_cast<const S*>(p.k_pages) + layer * p.kv_layer_stride + (int64_t)kvh * p.kv_head_stride;
  const S* vp = static_cast<const S*>(p.v_pages) + layer * p.kv_layer_stride + (int64_t)kvh * p.kv_head_stride;
  const S* lp = rp > 0 ? static_cast<const S*>(p.lr_pages) + layer * p.lr_layer_stride : nullptr;
  const S* lkp = rk > 0 ? static_cast<const S*>(p.lk_pages) + layer * p.lk_layer_stride : nullptr;
  constexpr int EPC = Elem<S>::kPerChunk;
  const int kv_chunks = d / EPC, lr_chunks = rp / EPC, lk_chunks = rk / EPC;

  for (int64_t j0 = j_begin; j0 < j_end; j0 += kTile) {
    __syncthreads();   // previous tile fully consumed (also orders the q_s staging on iteration 0)
    // ---- stage the K / V / LR tile, converting to float ------------------------------------
    for (int idx = tid; idx < kTile * kv_chunks; idx += kThreads) {
      const int jj = idx / kv_chunks, c = idx % kv_chunks;
      const int64_t j = j0 + jj;
      float tmp_k[EPC], tmp_v[EPC];
      if (j < j_end) {
        const int64_t phys = p.kv_table[j / p.P];
        const int64_t off = phys * p.kv_page_stride + page_offset(p.kv_lay, (int)(j % p.P), c * EPC);
        Elem<S>::load_chunk(kp + off, tmp_k);
        Elem<S>::load_chunk(vp + off, tmp_v);
      } else {
#pragma unroll
        for (int u = 0; u < EPC; ++u) { tmp_k[u] = 0.f; tmp_v[u] = 0.f; }
      }
#pragma unroll
      for (int u = 0; u < EPC; u += 4) {
        *reinterpret_cast<float4*>(k_s + jj * kx + c * EPC + u) = make_float4(tmp_k[u], tmp_k[u + 1], tmp_k[u + 2], tmp_k[u + 3]);
        *reinterpret_cast<float4*>(v_s + jj * kd + c * EPC + u) = make_float4(tmp_v[u], tmp_v[u + 1], tmp_v[u + 2], tmp_v[u + 3]);
      }
    }
    for (int idx = tid; idx < kTile * lr_chunks; idx += kThreads) {
      const int jj = idx / lr_chunks, c = idx % lr_chunks;
      const int64_t j = j0 + jj;
      float tmp[EPC];
      if (j < j_end) {
        const int64_t phys = p.lr_table[j / p.P];
        Elem<S>::load_chunk(lp + phys * p.lr_page_stride + page_offset(p.lr_lay, (int)(j % p.P), c * EPC), tmp);
      } else {
#pragma unroll
        for (int u = 0; u < EPC; ++u) tmp[u] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < EPC; u += 4)
        *reinterpret_cast<float4*>(lr_s + jj * kr + c * EPC + u) = make_float4(tmp[u], tmp[u + 1], tmp[u + 2], tmp[u + 3]);
    }
    for (int idx = tid; idx < kTile * lk_chunks; idx += kThreads) {       // L_k tile into columns [d, d + rk) of the key tile
      const int jj = idx / lk_chunks, c = idx % lk_chunks;
      const int64_t j = j0 + jj;
      float tmp[EPC];
      if (j < j_end) {
        const int64_t phys = p.lk_table[j / p.P];
        Elem<S>::load_chunk(lkp + phys * p.lk_page_stride + page_offset(p.lk_lay, (int)(j % p.P), c * EPC), tmp);
      } else {
#pragma unroll
        for (int u = 0; u < EPC; ++u) tmp[u] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < EPC; u += 4)
        *reinterpret_cast<float4*>(k_s + jj * kx + d + c * EPC + u) = make_float4(tmp[u], tmp[u + 1], tmp[u + 2], tmp[u + 3]);
    }
    __syncthreads();

    // ---- scores: lane = key --------------------------------------------------------------
    float dot[RW];
#pragma unroll
    for (int t = 0; t < RW; ++t) dot[t] = 0.f;
    const float* k_row = k_s + lane * kx;
    for (int c = 0; c < dx; c += 4) {             // q . K_base[j] + qk . L_k[j]: one product over the extended dimension
      const float4 kv = *reinterpret_cast<const float4*>(k_row + c);
#pragma unroll
      for (int t = 0; t < RW; ++t) {
        const float4 qv = *reinterpret_cast<const float4*>(q_s + (warp + 8 * t) * dx + c);
        dot[t] = fmaf(qv.x, kv.x, dot[t]);
        dot[t] = fmaf(qv.y, kv.y, dot[t]);
        dot[t] = fmaf(qv.z, kv.z, dot[t]);
        dot[t] = fmaf(qv.w, kv.w, dot[t]);
      }
    }
    const int64_t j = j0 + lane;
    float alpha[RW];
#pragma unroll
    for (int t = 0; t < RW; ++t) {
      const bool valid = j < j_end && j <= row_pos[t];
      const float s = valid ? dot[t] * inv_sqrt_d : ninf;
      const float tile_max = wmax(s);
      float pj = 0.f;
      alpha[t] = 1.f;
      if (tile_max != ninf) {                 // row sees at least one key of this tile (:165)
        const float m_new = fmaxf(m_run[t], tile_max);
        alpha[t] = (m_run[t] == ninf) ? 0.f : expf(m_run[t] - m_new);
        pj = valid ? expf(s - m_new) : 0.f;
        l_run[t] = alpha[t] * l_run[t] + wsum(pj);
        m_run[t] = m_new;
      }
      p_s[(warp + 8 * t) * kTile + lane] = pj;
    }
    __syncwarp();

    // ---- accumulate: lane = column quad -------------------------------------------------
#pragma unroll
    for (int t = 0; t < RW; ++t) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        olr[t][u] *= alpha[t];
#pragma unroll
        for (int qd = 0; qd < QD; ++qd) o[t][qd][u] *= alpha[t];
      }
    }
    const int n_valid = (int)min((int64_t)kTile, j_end - j0);
    const bool lr_lane = 4 * lane < rp;
    for (int jj = 0; jj < n_valid; ++jj) {
      float4 vv[QD];
#pragma unroll
      for (int qd = 0; qd < QD; ++qd) {
        const int c = 4 * (lane + 32 * qd);
        vv[qd] = c < d ? *reinterpret_cast<const float4*>(v_s + jj * kd + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float4 lv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lr_lane) lv = *reinterpret_cast<const float4*>(lr_s + jj * kr + 4 * lane);
#pragma unroll
      for (int t = 0; t < RW; ++t) {
        const float pj = p_s[(warp + 8 * t) * kTile + jj];
#pragma unroll
        for (int qd = 0; qd < QD; ++qd) {
          o[t][qd][0] = fmaf(pj, vv[qd].x, o[t][qd][0]);
          o[t][qd][1] = fmaf(pj, vv[qd].y, o[t][qd][1]);
          o[t][qd][2] = fmaf(pj, vv[qd].z, o[t][qd][2]);
          o[t][qd][3] = fmaf(pj, vv[qd].w, o[t][qd][3]);
        }
        olr[t][0] = fmaf(pj, lv.x, olr[t][0]);
        olr[t][1] = fmaf(pj, lv.y, olr[t][1]);
        olr[t][2] = fmaf(pj, lv.z, olr[t][2]);
        olr[t][3] = fmaf(pj, lv.w, olr[t][3]);
      }
    }
    __syncwarp();
  }

  // ---- write the partial state of every real row ------------------------------------------
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int64_t rho = rho0 + warp + 8 * t;
    if (rho >= p.rows_total) continue;
    float* dst = p.part + ((((layer_rel * p.n_kv_local + kvh) * p.rows_total + rho) * p.splits) + split) * p.part_stride;
    if (lane == 0) { dst[0] = m_run[t]; dst[1] = l_run[t]; }
#pragma unroll
    for (int qd = 0; qd < QD; ++qd) {
      const int c = 4 * (lane + 32 * qd);
      if (c < d) *reinterpret_cast<float4*>(dst + 4 + c) = make_float4(o[t][qd][0], o[t][qd][1], o[t][qd][2], o[t][qd][3]);
    }
    if (4 * lane < rp)
      *reinterpret_cast<float4*>(dst + 4 + d + 4 * lane) = make_float4(olr[t][0], olr[t][1], olr[t][2], olr[t][3]);
  }
}

// qk[row][head][p] = scale_k[agent] * sum_c q[row][head d + c] * B_k[agent][p][kvh d + c], zero-padded to rk_pad columns.
// One CTA of four warps per (row, head): the query row sits in shared memory, warp w takes p = w, w + 4, ..., its lanes the
// columns (coalesced B_k rows), a shuffle tree finishes each dot product.
__global__ void __launch_bounds__(128) qk_project_kernel(const float* __restrict__ q, const float* __restrict__ bk,
                                                         const float* __restrict__ scale_k, const int32_t* __restrict__ agent_ids,
                                                         int64_t layer_begin, int64_t n_agents, int64_t n_batch, int64_t rows_per_entry,
                                                         int n_q_local, int group, int d, int r_k, int rk_pad, int n_kv_local,
                                                         float* __restrict__ qk) {
  extern __shared__ float q_s[];                     // [d]
  const int64_t hrow = blockIdx.x;                   // (layer, entry, token, head)
  const int h = (int)(hrow % n_q_local);
  const int64_t et = hrow / n_q_local;               // layer_rel * n_batch * rows_per_entry + entry * rows_per_entry + token
  const int64_t layer_rel = et / (n_batch * rows_per_entry);
  const int64_t entry = (et / rows_per_entry) % n_batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ptx::pdl_wait();                                   // q comes from the previous kernel of the stream
  ptx::pdl_launch_dependents();
  for (int c = threadIdx.x; c < d; c += 128) q_s[c] = q[hrow * d + c];
  __syncthreads();
  const int agent = agent_ids ? agent_ids[entry] : 0;
  const int64_t layer = layer_begin + layer_rel;
  const float sc = scale_k[layer * n_agents + agent];
  for (int p = warp; p < rk_pad; p += 4) {
    float acc = 0.f;
    if (p < r_k) {
      const float* b_row = bk + (((layer * n_agents + agent) * r_k) + p) * ((int64_t)n_kv_local * d) + (int64_t)(h / group) * d;
      for (int c = lane; c < d; c += 32) acc = fmaf(q_s[c], __ldg(b_row + c), acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    }
    if (lane == 0) qk[hrow * rk_pad + p] = sc * acc;
  }
}

}  // namespace

int launch_qk_project(const PagedAttnCall& c, float* qk_out) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const lorakv_adapters* ad = c.adapters;
  const int64_t n_layers = c.layer_end - c.layer_begin;
  const int64_t rows = n_layers * c.n_batch * c.rows_per_entry * c.n_q_local;
  if (rows == 0) return LORAKV_OK;
  const int group = (int)(c.n_q_local / pool->n_kv_local);
  const int d = (int)pool->dims.d_head;
  LK_CUDA(launch_kernel(ctx, qk_project_kernel, dim3((unsigned)rows), dim3(128), (size_t)d * sizeof(float), true, c.q_dev,
                        (const float*)ad->b_k, (const float*)ad->scale_k, c.agent_ids_dev, c.layer_begin, ad->n_agents, c.n_batch,
                        c.rows_per_entry, (int)c.n_q_local, group, d, (int)pool->dims.rank_k, (int)pool->rk_pad, (int)pool->n_kv_local,
                        qk_out));
  ctx->launches++;
  return LORAKV_OK;
}

// ---- split merge + up-projection epilogue, shared by every paged path --------------------------
// part: [layers][kv heads][rows_total][splits][4 + d + r_pad]  (slot 0 = m, 1 = l; 2,3 unused so
// that the vectors stay 16-byte aligned)
struct MergeParams {
  const float* part;
  int64_t part_stride;
  int splits, d, r, r_pad, group, n_kv_local;
  int64_t rows_total, n_batch, rows_per_entry;
  int64_t layer_begin;
  const int32_t* agent_ids;    // [n_batch]
  const float* b;              // [n_layers][n_agents][r][n_kv_local*d]
  const float* scale;          // [n_layers][n_agents]
  int64_t n_agents;
  float* out;                  // [layers][n_batch][rows_per_entry][n_q_local*d]
};

__global__ void __launch_bounds__(128) fla_paged_merge_kernel(MergeParams p) {
  extern __shared__ float sm[];
  float* w_s = sm;                 // [splits]
  float* olr_s = sm + p.splits;    // [r]
  __shared__ float l_total;
  const int64_t rho = blockIdx.x;
  const int kvh = blockIdx.y % p.n_kv_local;
  const int64_t layer_rel = blockIdx.y / p.n_kv_local;
  const float ninf = -std::numeric_limits<float>::infinity();
  const float* base = p.part + ((layer_rel * p.n_kv_local + kvh) * p.rows_total + rho) * p.splits * p.part_stride;
  if (threadIdx.x < 32) {
    float mx = ninf;
    for (int s = threadIdx.x; s < p.splits; s += 32) mx = fmaxf(mx, base[s * p.part_stride]);
    mx = wmax(mx);
    float l = 0.f;
    for (int s = threadIdx.x; s < p.splits; s += 32) {
      const float ms = base[s * p.part_stride];
      const float w = (ms == ninf) ? 0.f : expf(ms - mx);
      w_s[s] = w;
      l += w * base[s * p.part_stride + 1];
    }
    l = wsum(l);
    if (threadIdx.x == 0) l_total = l;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < p.r; t += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < p.splits; ++s)
      if (w_s[s] != 0.f) acc = fmaf(w_s[s], base[s * p.part_stride + 4 + p.d + t], acc);
    olr_s[t] = acc;
  }
  __syncthreads();
  const int64_t gi = rho % p.group, et = rho / p.group;
  const int64_t entry = et / p.rows_per_entry;
  const int64_t layer = p.layer_begin + layer_rel;
  const int64_t n_q_local = (int64_t)p.n_kv_local * p.group;
  const int64_t dkv = (int64_t)p.n_kv_local * p.d;
  const int agent = p.agent_ids ? p.agent_ids[entry] : 0;
  const float* b = p.r > 0 ? p.b + ((layer * p.n_agents + agent) * p.r) * dkv + (int64_t)kvh * p.d : nullptr;
  const float scale = p.r > 0 ? p.scale[layer * p.n_agents + agent] : 0.f;
  float* dst = p.out + ((layer_rel * p.n_batch * p.rows_per_entry + et) * n_q_local + (int64_t)kvh * p.group + gi) * p.d;
  const float inv_l = 1.0f / l_total;
  for (int c = threadIdx.x; c < p.d; c += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < p.splits; ++s)
      if (w_s[s] != 0.f) acc = fmaf(w_s[s], base[s * p.part_stride + 4 + c], acc);
    for (int t = 0; t < p.r; ++t) acc = fmaf(scale * olr_s[t], b[t * dkv + c], acc);
    dst[c] = acc * inv_l;
  }
}

int launch_paged_merge(lorakv_ctx* ctx, const MergeParams& mp, int64_t n_layers) {
  dim3 grid((unsigned)mp.rows_total, (unsigned)(n_layers * mp.n_kv_local));
  fla_paged_merge_kernel<<<grid, 128, (mp.splits + mp.r + 1) * sizeof(float), ctx->stream>>>(mp);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

template <class S, int RW, int QD>
static int launch_simt_t(lorakv_ctx* ctx, const SimtParams& sp, dim3 grid) {
  const int d = sp.d, rp = sp.r_pad;
  const int rk = sp.rk_pad;
  const size_t smem = sizeof(float) * ((size_t)8 * RW * (d + rk) + kTile * (d + rk + 4) + kTile * (d + 4) + kTile * (rp + 4) + (size_t)8 * RW * kTile);
  auto kern = fla_paged_simt_kernel<S, RW, QD>;
  LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prof_mark(ctx, 0);
  kern<<<grid, kThreads, smem, ctx->stream>>>(sp);
  prof_mark(ctx, 1);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

template <class S>
static int launch_simt_s(lorakv_ctx* ctx, const SimtParams& sp, dim3 grid, int rw) {
  const bool wide = sp.d > 128;
  switch (rw) {
    case 1: return wide ? launch_simt_t<S, 1, 2>(ctx, sp, grid) : launch_simt_t<S, 1, 1>(ctx, sp, grid);
    case 2: return wide ? launch_simt_t<S, 2, 2>(ctx, sp, grid) : launch_simt_t<S, 2, 1>(ctx, sp, grid);
    case 4: return wide ? launch_simt_t<S, 4, 2>(ctx, sp, grid) : launch_simt_t<S, 4, 1>(ctx, sp, grid);
    default: return wide ? launch_simt_t<S, 8, 2>(ctx, sp, grid) : launch_simt_t<S, 8, 1>(ctx, sp, grid);
  }
}

int launch_paged_simt(const PagedAttnCall& c) {
  lorakv_pool* pool = c.pool;
  lorakv_ctx* ctx = pool->ctx;
  const int64_t d = pool->dims.d_head, r = pool->dims.rank, rp = pool->r_pad;
  if (d % 4 != 0 || d > 256) return fail("paged attention: d_head %lld must be a multiple of 4 and <= 256", (long long)d);
  if (rp > 128) return fail("paged attention: rank %lld > 128 is not supported", (long long)r);
  if (pool->dims.dtype == LORAKV_BF16 && d % 8 != 0) return fail("paged attention: bf16 pages need d_head %% 8 == 0");
  const int64_t n_layers = c.layer_end - c.layer_begin;
  const int group = (int)(c.n_q_local / pool->n_kv_local);
  const int64_t rows_total = c.n_batch * c.rows_per_entry * group;
  if (rows_total == 0 || n_layers == 0) return LORAKV_OK;

  int rw = 1;
  while (8 * rw < rows_total && rw < 8) rw *= 2;
  const int64_t row_blocks = (rows_total + 8 * rw - 1) / (8 * rw);
  const int64_t visible = c.query_offset + c.rows_per_entry;   // keys any row can see
  const int64_t ctas = row_blocks * n_layers * pool->n_kv_local;
  int splits = (int)((ctx->sm_count * 2 + ctas - 1) / ctas);
  const int max_splits = (int)((visible + 4 * kTile - 1) / (4 * kTile));
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  int64_t chunk = (visible + splits - 1) / splits;
  chunk = (chunk + kTile - 1) / kTile * kTile;
  splits = (int)((visible + chunk - 1) / chunk);
  if (splits < 1) splits = 1;

  const int64_t part_stride = 4 + d + rp;
  const size_t part_bytes = (size_t)(n_layers * pool->n_kv_local * rows_total * splits * part_stride) * sizeof(float);
  LK_TRY(scratch_reserve(ctx, ctx->work, part_bytes));

  SimtParams sp;
  sp.k_pages = pool->k_pages; sp.v_pages = pool->v_pages; sp.lr_pages = pool->lr_pages;
  sp.kv_table = pool->kv_space.dev_table + c.kv_set * pool->kv_space.max_pages;
  sp.lr_table = rp > 0 ? pool->lr_space.dev_table + c.lr_set * pool->lr_space.max_pages : nullptr;
  sp.kv_layer_stride = pool->kv_layer_stride(); sp.kv_head_stride = pool->kv_head_stride();
  sp.kv_page_stride = pool->kv_page_stride();
  sp.lr_layer_stride = pool->lr_layer_stride(); sp.lr_page_stride = pool->lr_page_stride();
  sp.P = (int)pool->P; sp.d = (int)d; sp.r_pad = (int)rp; sp.group = group; sp.n_kv_local = (int)pool->n_kv_local;
  sp.kv_lay = make_page_layout((int)pool->P, (int)d, (int)pool->elem);
  sp.lr_lay = make_page_layout((int)pool->P, (int)rp, (int)pool->elem);
  sp.L = c.L; sp.layer_begin = c.layer_begin;
  sp.n_batch = c.n_batch; sp.rows_per_entry = c.rows_per_entry; sp.query_offset = c.query_offset;
  sp.rows_total = rows_total; sp.splits = splits; sp.chunk = chunk;
  sp.q = c.q_dev; sp.part = static_cast<float*>(ctx->work.ptr); sp.part_stride = part_stride;
  sp.lk_pages = pool->lk_pages; sp.lk_table = pool->lk_space.dev_table; sp.lk_layer_stride = pool->lk_layer_stride();
  sp.lk_page_stride = pool->lk_page_stride(); sp.rk_pad = (int)pool->rk_pad;
  sp.lk_lay = make_page_layout((int)pool->P, (int)std::max<int64_t>(pool->rk_pad, 8), (int)pool->elem);
  sp.qk = c.qk_dev;
  if (pool->rk_pad > 0 && !c.qk_dev) return fail("paged attention: the key-side low-rank term needs the projected queries (launch_qk_project)");
  dim3 grid((unsigned)row_blocks, (unsigned)(n_layers * pool->n_kv_local), (unsigned)splits);
  if (pool->dims.dtype == LORAKV_BF16) LK_TRY(launch_simt_s<__nv_bfloat16>(ctx, sp, grid, rw));
  else LK_TRY(launch_simt_s<float>(ctx, sp, grid, rw));

  MergeParams mp;
  mp.part = sp.part; mp.part_stride = part_stride; mp.splits = splits; mp.d = (int)d; mp.r = (int)r;
  mp.r_pad = (int)rp; mp.group = group; mp.n_kv_local = (int)pool->n_kv_local;
  mp.rows_total = rows_total; mp.n_batch = c.n_batch; mp.rows_per_entry = c.rows_per_entry;
  mp.layer_begin = c.layer_begin; mp.agent_ids = c.agent_ids_dev;
  mp.b = c.adapters ? c.adapters->b : nullptr; mp.scale = c.adapters ? c.adapters->scale : nullptr;
  mp.n_agents = c.adapters ? c.adapters->n_agents : 1;
  if (r > 0 && !c.adapters) return fail("paged attention: rank %lld cache needs adapter tables", (long long)r);
  mp.out = c.out_dev;
  LK_TRY(launch_paged_merge(ctx, mp, n_layers));
  ctx->last_kernel = "fla_paged_simt";
  return LORAKV_OK;
}

}  // namespace lk
