// step_layer.cu -- the projections of ONE decode layer-step in two launches.
//
// The reference's step() (proj/include/lorakv/engine.hpp:331-443) does, per layer and for the new token rows x:
//     q  = x Wq + s_q (x A_q) B_q[agent]; apply_rope(q)                       (:352-373, :422-427)
//     k  = apply_rope(x Wk); v = x Wv [+ s_v (x A_v) B_v[agent]]              (:376-393)
//     append_key / append_value                                              (:395-403)
//     append_lr(x A_v)                                                       (:411-419, the schemes with an LR cache)
//     gqa_attention(q, key_view, value_view, lr_view, B_v[agent], ...)        (:429-443)
// Through the separate entry points that was ~9 launches per layer-step for one row (x A_q, Wq partial sums + finish,
// Wk|Wv partial sums + finish, x A_v, attention, merge) and the decode phase was bound by launch latency
// (profiles/r1_trace_replay.md: ~160 us wall for ~60 us of kernels).  Here:
//
//   step_partial_kernel   ONE pass over [Wq | Wk | Wv] (the packed bf16 weights the tcgen05 GEMMs use) and over A_q, A_v
//                         (float32), every SM streaming a (64-column block, K slice) of them: float32 partial sums of
//                         all five products.  A row or two is a GEMV, bound by one read of the weights (48 MB per
//                         Llama-3.1-8B layer); eight independent 16-byte loads per lane are in flight at a time.
//   step_finish_kernel    sums the K slices, adds the q / v adapter terms, rotates q and k (angles in double, as the
//                         reference casts them), stores float32 q rows, bf16 K / V rows into their swizzled pages and the
//                         V_lr row (x A_v, unscaled, lora.hpp:9-11) into its LR page.
//
// Both are programmatic dependent launches (umma.cuh: pdl_wait), and so are the attention kernel and its merge epilogue
// that follow (fla_decode_tma.cu): four launches per layer-step whose launch latencies hide under their predecessors.
// Same arithmetic as rows_project.cu / the GEMM path (bf16 products of bf16-rounded x, fp32 accumulation), another summation
// order; parity in tests/test_gpu_step_layer.py.
#include <cuda_bf16.h>

#include <algorithm>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

constexpr int kMaxRows = 8;
constexpr int kThreads = 256;
constexpr int kLoadBatch = 8;       // 16-byte weight loads of a lane in flight together

__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

struct StepPartial {
  const float* x; int64_t ld; int M;
  const __nv_bfloat16* wq;    // [nb_q][d_model][64] packed, swizzled by k % 8
  const __nv_bfloat16* wkv;   // [nb_kv][d_model][64]
  int nb_q, nb_kv, d_model, kc, n_cols;
  const float* a_q; int r_q;  // [d_model][r_q] or null
  const float* a_v; int r_v;  // [d_model][r_v] or null
  float* part;                // [splits][M][n_cols]
  float* down_part;           // [2][splits][M][64]  (0: x A_q, 1: x A_v)
};

template <int M_>
__device__ __forceinline__ void weight_block(const StepPartial& p, const float* xs, const unsigned char* wb, int k0, int nb_out, int split,
                                             float* red) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = lane & 7, rr = lane >> 3;          // logical 16-byte chunk (8 columns), row within a group of 4
  float acc[M_][8];
#pragma unroll
  for (int m = 0; m < M_; ++m)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[m][u] = 0.f;
  // warp w, row group rr: k = 4 w + rr, + 32, + 64, ... ; kLoadBatch of them loaded before any is used
  for (int kk0 = warp * 4 + rr; kk0 < p.kc; kk0 += 32 * kLoadBatch) {
    uint4 raw[kLoadBatch];
#pragma unroll
    for (int b = 0; b < kLoadBatch; ++b) {
      const int kk = kk0 + 32 * b, k = k0 + kk;
      raw[b] = kk < p.kc ? __ldg(reinterpret_cast<const uint4*>(wb + (int64_t)k * 128 + ((c ^ (k & 7)) << 4))) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int b = 0; b < kLoadBatch; ++b) {
      const int kk = kk0 + 32 * b;
      if (kk >= p.kc) break;
      float wv[8];
      const uint32_t r4[4] = {raw[b].x, raw[b].y, raw[b].z, raw[b].w};
#pragma unroll
      for (int u = 0; u < 4; ++u) { wv[2 * u] = __uint_as_float(r4[u] << 16); wv[2 * u + 1] = __uint_as_float(r4[u] & 0xFFFF0000u); }
#pragma unroll
      for (int m = 0; m < M_; ++m) {
        const float xv = xs[m * p.kc + kk];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[m][u] = fmaf(xv, wv[u], acc[m][u]);
      }
    }
  }
  // the 4 row groups of a warp, then the 8 warps
#pragma unroll
  for (int m = 0; m < M_; ++m)
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[m][u] += __shfl_xor_sync(0xffffffffu, acc[m][u], 8);
      acc[m][u] += __shfl_xor_sync(0xffffffffu, acc[m][u], 16);
    }
  if (rr == 0) {
#pragma unroll
    for (int m = 0; m < M_; ++m)
#pragma unroll
      for (int u = 0; u < 8; ++u) red[(warp * M_ + m) * 64 + c * 8 + u] = acc[m][u];
  }
  __syncthreads();
  for (int i = tid; i < M_ * 64; i += kThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) s += red[w * M_ * 64 + i];
    p.part[((int64_t)split * M_ + i / 64) * p.n_cols + (int64_t)nb_out * 64 + i % 64] = s;
  }
}

// grid (nb_q + nb_kv + 2, splits): weight blocks first, then the two down-projections
template <int M_>
__global__ void __launch_bounds__(kThreads) step_partial_kernel(const StepPartial p) {
  extern __shared__ __align__(16) float sm[];    // xs [M][kc] | red [8 warps][M][64] (at least 1024 floats)
  float* xs = sm;
  float* red = sm + M_ * p.kc;
  const int tid = threadIdx.x, split = blockIdx.y, k0 = split * p.kc;
  const int nb = blockIdx.x, nb_w = p.nb_q + p.nb_kv;
  if (nb >= nb_w) {                              // the adapter of this CTA may be absent: nothing to do
    const bool which_v = nb - nb_w == 1;
    if ((which_v ? p.a_v : p.a_q) == nullptr) return;
  }
  ptx::pdl_wait();                               // x comes from the previous kernel of the stream
  ptx::pdl_launch_dependents();
  for (int i = tid; i < M_ * p.kc; i += kThreads) xs[i] = bf16_round(p.x[(int64_t)(i / p.kc) * p.ld + k0 + i % p.kc]);
  __syncthreads();
  if (nb < nb_w) {
    const bool is_q = nb < p.nb_q;
    const unsigned char* wb = reinterpret_cast<const unsigned char*>(is_q ? p.wq : p.wkv) + (int64_t)(is_q ? nb : nb - p.nb_q) * p.d_model * 128;
    weight_block<M_>(p, xs, wb, k0, nb, split, red);
    return;
  }
  // x A over this K slice; A is float32 (the adapters stay in full precision).  Ranks that are multiples of 4: thread ->
  // (column quad, k group), float4 loads, all of a thread's loads issued before the first use (a loop with one load per
  // iteration took 20 us for a 32 KB slice and was the tail of the whole launch); other ranks keep the scalar loop.
  const int which = nb - nb_w;
  const float* A = which == 1 ? p.a_v : p.a_q;
  const int r = which == 1 ? p.r_v : p.r_q;
  float* down = p.down_part + (((int64_t)which * gridDim.y + split) * M_) * 64;
  if (r % 4 == 0) {
    const int quads = r / 4, groups = kThreads / quads;          // k groups of the CTA (>= 16 for r <= 64)
    const int cq = tid % quads, g = tid / quads;
    float acc[M_][4];
#pragma unroll
    for (int m = 0; m < M_; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
    if (g < groups)
      for (int kk0 = g; kk0 < p.kc; kk0 += groups * kLoadBatch) {
        float4 av[kLoadBatch];
#pragma unroll
        for (int b = 0; b < kLoadBatch; ++b) {
          const int kk = kk0 + groups * b;
          av[b] = kk < p.kc ? __ldg(reinterpret_cast<const float4*>(A + (int64_t)(k0 + kk) * r) + cq) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int b = 0; b < kLoadBatch; ++b) {
          const int kk = kk0 + groups * b;
          if (kk >= p.kc) break;
#pragma unroll
          for (int m = 0; m < M_; ++m) {
            const float xv = xs[m * p.kc + kk];
            acc[m][0] = fmaf(xv, av[b].x, acc[m][0]); acc[m][1] = fmaf(xv, av[b].y, acc[m][1]);
            acc[m][2] = fmaf(xv, av[b].z, acc[m][2]); acc[m][3] = fmaf(xv, av[b].w, acc[m][3]);
          }
        }
      }
    // k groups -> one sum per (row, column): through shared memory, M_ rows at a time to stay inside `red` (8 x M x 64 floats)
    __syncthreads();
    for (int m = 0; m < M_; ++m) {
      if (g < groups) *reinterpret_cast<float4*>(red + (size_t)g * r + 4 * cq) = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
      __syncthreads();
      if (tid < r) {
        float s = 0.f;
        for (int gg = 0; gg < groups; ++gg) s += red[(size_t)gg * r + tid];
        down[m * 64 + tid] = s;
      }
      __syncthreads();
    }
    return;
  }
  const int G = min(kThreads / r, kThreads / 32), j = tid % r, g = tid / r;      // <= 8 groups: `red` holds 8 x M x 64 floats
  float acc[M_];
#pragma unroll
  for (int m = 0; m < M_; ++m) acc[m] = 0.f;
  if (g < G)
    for (int kk = g; kk < p.kc; kk += G) {
      const float a = __ldg(A + (int64_t)(k0 + kk) * r + j);
#pragma unroll
      for (int m = 0; m < M_; ++m) acc[m] = fmaf(xs[m * p.kc + kk], a, acc[m]);
    }
  __syncthreads();
  if (g < G) {
#pragma unroll
    for (int m = 0; m < M_; ++m) red[(g * M_ + m) * 64 + j] = acc[m];
  }
  __syncthreads();
  for (int i = tid; i < M_ * r; i += kThreads) {
    const int m = i / r, jj = i % r;
    float s = 0.f;
    for (int gg = 0; gg < G; ++gg) s += red[(gg * M_ + m) * 64 + jj];
    down[m * 64 + jj] = s;
  }
}

struct StepFinish {
  const float* part; const float* down_part; int splits, M, n_cols;
  int dq, dkv, d_head, n_kv_local;      // q columns, K (= V) columns of this shard
  bool rope; int64_t pos0;
  const float* b_q; int64_t ldb_q; int r_q; float s_q;       // q adapter (null: none)
  const float* b_v; int64_t ldb_v; int r_v; float s_v;       // value adapter merged into the stored rows (full-values schemes; null: none)
  float* q_out; int64_t ldq;
  __nv_bfloat16 *k_pages, *v_pages; const int32_t* kv_table; int64_t head_stride, kv_page_stride; PageLayout kv_lay;
  __nv_bfloat16* lr_pages; const int32_t* lr_table; int64_t lr_page_stride; int r_pad; PageLayout lr_lay;   // V_lr append (null: none)
};

__device__ __forceinline__ float2 rope_cs(const StepFinish& f, int m, int c) {
  const double freq = pow(10000.0, -2.0 * (double)c / (double)f.d_head);
  double s, co;
  sincos((double)(f.pos0 + m) * freq, &s, &co);
  return make_float2((float)co, (float)s);
}

// one thread per (row, head, c < d/2) over the q heads, the key heads and the value heads: the rotation pair (c, c + d/2)
__global__ void __launch_bounds__(kThreads) step_finish_kernel(const StepFinish f) {
  __shared__ float down_s[2][kMaxRows][64];
  const int tid = threadIdx.x;
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  // down-projections: sum of the K slices (every CTA needs them for its adapter terms)
  for (int i = tid; i < 2 * f.M * 64; i += kThreads) {
    const int which = i / (f.M * 64), m = (i / 64) % f.M, j = i % 64;
    const int r = which == 1 ? f.r_v : f.r_q;
    float s = 0.f;
    if (j < r)
      for (int sp = 0; sp < f.splits; ++sp) s += f.down_part[(((int64_t)which * f.splits + sp) * f.M + m) * 64 + j];
    down_s[which][m][j] = s;
  }
  __syncthreads();
  const int half = f.d_head / 2;
  const int per_row = f.n_cols / 2;
  const int idx = blockIdx.x * kThreads + tid;
  // V_lr append: the first CTA also stores x A_v (unscaled) into the LR pages, zero-padded to the page's rank
  if (blockIdx.x == 0 && f.lr_pages != nullptr)
    for (int i = tid; i < f.M * f.r_pad; i += kThreads) {
      const int m = i / f.r_pad, j = i % f.r_pad;
      const int64_t row = f.pos0 + m;
      __nv_bfloat16* page = f.lr_pages + (int64_t)f.lr_table[row / f.lr_lay.P] * f.lr_page_stride;
      page[page_offset(f.lr_lay, (int)(row % f.lr_lay.P), j)] = __float2bfloat16_rn(j < f.r_v ? down_s[1][m][j] : 0.f);
    }
  if (idx >= f.M * per_row) return;
  const int m = idx / per_row, hb = (idx % per_row) / half, c = idx % half;
  const int col0 = hb * f.d_head + c, col1 = col0 + half;       // columns of the partial-sum matrix [q | k | v]
  float x0 = 0.f, x1 = 0.f;
  for (int sp = 0; sp < f.splits; ++sp) {
    const float* row = f.part + ((int64_t)sp * f.M + m) * f.n_cols;
    x0 += row[col0]; x1 += row[col1];
  }
  const int n_q_heads = f.dq / f.d_head;
  if (hb < n_q_heads) {                          // ---- query head ----
    if (f.b_q != nullptr)
      for (int k = 0; k < f.r_q; ++k) {
        const float dk = f.s_q * down_s[0][m][k];
        x0 = fmaf(dk, __ldg(f.b_q + (int64_t)k * f.ldb_q + col0), x0);
        x1 = fmaf(dk, __ldg(f.b_q + (int64_t)k * f.ldb_q + col1), x1);
      }
    if (f.rope) {
      const float2 cs = rope_cs(f, m, c);
      const float a = x0 * cs.x - x1 * cs.y, b = x0 * cs.y + x1 * cs.x;
      x0 = a; x1 = b;
    }
    f.q_out[(int64_t)m * f.ldq + col0] = x0;
    f.q_out[(int64_t)m * f.ldq + col1] = x1;
    return;
  }
  const int hk = hb - n_q_heads;                 // ---- key head (< n_kv_local) or value head ----
  const bool is_k = hk < f.n_kv_local;
  const int head = is_k ? hk : hk - f.n_kv_local;
  if (is_k && f.rope) {
    const float2 cs = rope_cs(f, m, c);
    const float a = x0 * cs.x - x1 * cs.y, b = x0 * cs.y + x1 * cs.x;
    x0 = a; x1 = b;
  }
  if (!is_k && f.b_v != nullptr)
    for (int k = 0; k < f.r_v; ++k) {
      const float dk = f.s_v * down_s[1][m][k];
      x0 = fmaf(dk, __ldg(f.b_v + (int64_t)k * f.ldb_v + head * f.d_head + c), x0);
      x1 = fmaf(dk, __ldg(f.b_v + (int64_t)k * f.ldb_v + head * f.d_head + c + half), x1);
    }
  const int64_t row = f.pos0 + m;
  __nv_bfloat16* page = (is_k ? f.k_pages : f.v_pages) + (int64_t)head * f.head_stride + (int64_t)f.kv_table[row / f.kv_lay.P] * f.kv_page_stride;
  const int t = (int)(row % f.kv_lay.P);
  page[page_offset(f.kv_lay, t, c)] = __float2bfloat16_rn(x0);
  page[page_offset(f.kv_lay, t, c + half)] = __float2bfloat16_rn(x1);
}

template <int M_>
int launch_partial(lorakv_ctx* ctx, const StepPartial& p, dim3 grid, size_t smem) {
  static int attr_device = -1;
  if (attr_device != ctx->device) {
    LK_CUDA(cudaFuncSetAttribute(step_partial_kernel<M_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    attr_device = ctx->device;
  }
  LK_CUDA(launch_kernel(ctx, step_partial_kernel<M_>, grid, dim3(kThreads), smem, true, p));
  return LORAKV_OK;
}

}  // namespace

bool step_layer_supported(int64_t n_rows, int64_t d_model, int64_t d_head, int64_t r_q, int64_t r_v) {
  return n_rows >= 1 && n_rows <= kMaxRows && d_model % 64 == 0 && d_model <= 65536 && d_head % 2 == 0 && r_q <= 64 && r_v <= 64;
}

int launch_step_layer(lorakv_pool* pool, const StepLayerCall& c) {
  lorakv_ctx* ctx = pool->ctx;
  const int64_t d = pool->dims.d_head, n_kv = pool->n_kv_local, dkv = n_kv * d, d_model = pool->dims.d_model;
  const int M = (int)c.n_rows;
  const int nb_q = (int)(c.dq / 64), nb_kv = (int)(2 * dkv / 64);
  const int n_cols = (int)(c.dq + 2 * dkv);
  // K slices: every CTA streams >= 64 reduction rows, and there are enough CTAs for two waves of 256-thread blocks
  int splits = 1;
  auto can_double = [&]() { return d_model % (2 * splits) == 0 && d_model / (2 * splits) >= 128 && splits < 64; };
  while (d_model / splits > 1024 && can_double()) splits *= 2;
  while ((nb_q + nb_kv) * splits < 4 * ctx->sm_count && can_double()) splits *= 2;
  const int kc = (int)(d_model / splits);
  const size_t part_bytes = (size_t)splits * M * n_cols * sizeof(float);
  const size_t down_bytes = (size_t)2 * splits * M * 64 * sizeof(float);
  // ctx->proj (not ctx->work: the attention kernel that follows keeps its partials there)
  LK_TRY(scratch_reserve(ctx, ctx->proj, part_bytes + down_bytes));
  float* part = static_cast<float*>(ctx->proj.ptr);
  float* down_part = reinterpret_cast<float*>(static_cast<char*>(ctx->proj.ptr) + part_bytes);

  StepPartial p;
  p.x = c.x_dev; p.ld = c.ld; p.M = M;
  p.wq = static_cast<const __nv_bfloat16*>(c.wq_packed); p.wkv = static_cast<const __nv_bfloat16*>(c.wkv_packed);
  p.nb_q = nb_q; p.nb_kv = nb_kv; p.d_model = (int)d_model; p.kc = kc; p.n_cols = n_cols;
  p.a_q = c.a_q; p.r_q = (int)c.r_q; p.a_v = c.a_v; p.r_v = (int)c.r_v;
  p.part = part; p.down_part = down_part;
  const dim3 grid((unsigned)(nb_q + nb_kv + 2), (unsigned)splits);
  // xs [M][kc] | red: 8 warps x M x 64 partial sums of a weight block, or 256 / (r/4) k groups x r of a down-projection (1024)
  const size_t smem = (size_t)(M * kc + std::max((kThreads / 32) * M * 64, 1024)) * sizeof(float);
  switch (M) {
    case 1: LK_TRY(launch_partial<1>(ctx, p, grid, smem)); break;
    case 2: LK_TRY(launch_partial<2>(ctx, p, grid, smem)); break;
    case 3: LK_TRY(launch_partial<3>(ctx, p, grid, smem)); break;
    case 4: LK_TRY(launch_partial<4>(ctx, p, grid, smem)); break;
    case 5: LK_TRY(launch_partial<5>(ctx, p, grid, smem)); break;
    case 6: LK_TRY(launch_partial<6>(ctx, p, grid, smem)); break;
    case 7: LK_TRY(launch_partial<7>(ctx, p, grid, smem)); break;
    default: LK_TRY(launch_partial<8>(ctx, p, grid, smem)); break;
  }
  ctx->launches++;

  StepFinish f;
  f.part = part; f.down_part = down_part; f.splits = splits; f.M = M; f.n_cols = n_cols;
  f.dq = (int)c.dq; f.dkv = (int)dkv; f.d_head = (int)d; f.n_kv_local = (int)n_kv;
  f.rope = c.rope; f.pos0 = c.row0;
  f.b_q = c.a_q ? c.b_q : nullptr; f.ldb_q = c.ldb_q; f.r_q = (int)c.r_q; f.s_q = c.s_q;
  f.b_v = c.merge_v ? c.b_v : nullptr; f.ldb_v = dkv; f.r_v = (int)c.r_v; f.s_v = c.s_v;
  f.q_out = c.q_dev; f.ldq = c.dq;
  f.k_pages = static_cast<__nv_bfloat16*>(pool->k_pages) + c.layer * pool->kv_layer_stride();
  f.v_pages = static_cast<__nv_bfloat16*>(pool->v_pages) + c.layer * pool->kv_layer_stride();
  f.kv_table = pool->kv_space.dev_table + c.kv_set * pool->kv_space.max_pages;
  f.head_stride = pool->kv_head_stride(); f.kv_page_stride = pool->kv_page_stride();
  f.kv_lay = make_page_layout((int)pool->P, (int)d, 2);
  f.lr_pages = nullptr; f.lr_table = nullptr; f.lr_page_stride = 0; f.r_pad = 0; f.lr_lay = make_page_layout((int)pool->P, 8, 2);
  if (c.append_lr) {
    f.lr_pages = static_cast<__nv_bfloat16*>(pool->lr_pages) + c.layer * pool->lr_layer_stride();
    f.lr_table = pool->lr_space.dev_table + c.lr_set * pool->lr_space.max_pages;
    f.lr_page_stride = pool->lr_page_stride(); f.r_pad = (int)pool->r_pad;
    f.lr_lay = make_page_layout((int)pool->P, (int)pool->r_pad, 2);
  }
  const int n = M * n_cols / 2;
  LK_CUDA(launch_kernel(ctx, step_finish_kernel, dim3((unsigned)((n + kThreads - 1) / kThreads)), dim3(kThreads), 0, true, f));
  ctx->launches++;
  ctx->last_kernel = "step_layer_project";
  return LORAKV_OK;
}

}  // namespace lk
