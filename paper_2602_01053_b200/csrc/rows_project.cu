// rows_project.cu -- the projections of a decode step: a handful of new rows (<= 8) through Wq / Wk / Wv and the
// LoRA down-projections (engine.hpp:362-419 with one token per call).  The tcgen05 GEMM of kv_project_umma.cu needs
// a 128-row tile per CTA: with one row it runs 8-16 CTAs that each walk the whole reduction dimension (36-41 us,
// latency-bound; the tensor-core X*A kernel 58 us on one CTA -- profiles/r1_trace_replay.md).  A row or two is a
// GEMV: bound by ONE pass over the bf16 weights, so here every SM streams a slice of them.
//
//   rows_xa            x A (A float32, x rounded to bf16 as the cache dtype implies): dense float32 [M][r]
//   rows_partial       grid (64-column weight block, K split): each CTA streams its slice of the PACKED bf16 weights
//                      (the layout the tcgen05 kernel consumes: [block][d_model][64], 16-byte chunks swizzled by k % 8;
//                      a lane reads the chunk of its LOGICAL columns, so a row is still one 128-byte line per 8 lanes)
//                      and writes float32 partial sums [split][M][columns]
//                      and, for the V_lr append, the same row rounded to bf16 straight into the LR pages
//   rows_kv_finish     sums the splits, adds the value adapter (full-values schemes), rotates the keys (angles in double,
//   rows_q_finish      inline), rounds to bf16 and stores into the swizzled pages / the float32 query rows
// Same arithmetic as the GEMM path (bf16 products, fp32 accumulation), a different summation order.
#include <cuda_bf16.h>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"

namespace lk {

namespace {

constexpr int kMaxRows = 8;
constexpr int kPartThreads = 128;

__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// down[m][j] = sum_k bf16(x[m][k]) * A[k][j]; one CTA per row, thread (g, j): k = g, g + G, ...
struct LrPages {             // when given, the row is also rounded to bf16 and stored into the LR pages (V_lr append)
  __nv_bfloat16* pages; const int32_t* table; int64_t page_stride, row0; int r_pad; PageLayout lay;
};

__global__ void __launch_bounds__(256) rows_xa_kernel(const float* __restrict__ x, int64_t ld, const float* __restrict__ A, int d_model,
                                                      int rank, float* __restrict__ down, LrPages lp) {
  __shared__ float red[256];
  const int m = blockIdx.x, tid = threadIdx.x;
  const int G = 256 / rank;                      // rank <= 64 -> at least 4 groups
  const int j = tid % rank, g = tid / rank;
  float acc = 0.f;
  if (g < G)
    for (int k = g; k < d_model; k += G) acc = fmaf(bf16_round(x[(int64_t)m * ld + k]), A[(int64_t)k * rank + j], acc);
  red[tid] = (g < G) ? acc : 0.f;
  __syncthreads();
  if (tid < rank) {
    float s = 0.f;
    for (int gg = 0; gg < G; ++gg) s += red[gg * rank + tid];
    if (down != nullptr) down[m * rank + tid] = s;
    red[tid] = s;
  }
  if (lp.pages != nullptr) {
    __syncthreads();
    if (tid < lp.r_pad) {
      const int64_t row = lp.row0 + m;
      __nv_bfloat16* page = lp.pages + (int64_t)lp.table[row / lp.lay.P] * lp.page_stride;
      page[page_offset(lp.lay, (int)(row % lp.lay.P), tid)] = __float2bfloat16_rn(tid < rank ? red[tid] : 0.f);
    }
  }
}

// partial[split][m][nb * 64 + c] over k in [split * kc, (split + 1) * kc)
__global__ void __launch_bounds__(kPartThreads) rows_partial_kernel(const float* __restrict__ x, int64_t ld, int M, const __nv_bfloat16* __restrict__ w,
                                                                    int d_model, int n_cols, int kc, float* __restrict__ part) {
  extern __shared__ float xs[];                  // [M][kc] bf16-rounded rows of this K slice, then the cross-warp reduction
  const int nb = blockIdx.x, split = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k0 = split * kc;
  for (int i = tid; i < M * kc; i += kPartThreads) xs[i] = bf16_round(x[(int64_t)(i / kc) * ld + k0 + i % kc]);
  __syncthreads();
  const int c = lane & 7, rr = lane >> 3;        // logical 16-byte chunk (8 columns), row within a group of 4
  float acc[kMaxRows][8];
#pragma unroll
  for (int m = 0; m < kMaxRows; ++m)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[m][u] = 0.f;
  const unsigned char* wb = reinterpret_cast<const unsigned char*>(w) + (int64_t)nb * d_model * 128;
  for (int kk = warp * 4 + rr; kk < kc; kk += 16) {
    const int k = k0 + kk;
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(wb + (int64_t)k * 128 + ((c ^ (k & 7)) << 4)));
    float wv[8];
    const uint32_t r4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) { wv[2 * u] = __uint_as_float(r4[u] << 16); wv[2 * u + 1] = __uint_as_float(r4[u] & 0xFFFF0000u); }
#pragma unroll
    for (int m = 0; m < kMaxRows; ++m) {
      if (m < M) {
        const float xv = xs[m * kc + kk];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[m][u] = fmaf(xv, wv[u], acc[m][u]);
      }
    }
  }
  // the 4 row groups of a warp, then the 4 warps
#pragma unroll
  for (int m = 0; m < kMaxRows; ++m)
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[m][u] += __shfl_xor_sync(0xffffffffu, acc[m][u], 8);
      acc[m][u] += __shfl_xor_sync(0xffffffffu, acc[m][u], 16);
    }
  __syncthreads();                               // xs is reused
  float* red = xs;                               // [4 warps][M][64]
  if (rr == 0) {
#pragma unroll
    for (int m = 0; m < kMaxRows; ++m)
      if (m < M) {
#pragma unroll
        for (int u = 0; u < 8; ++u) red[(warp * M + m) * 64 + c * 8 + u] = acc[m][u];
      }
  }
  __syncthreads();
  for (int i = tid; i < M * 64; i += kPartThreads) {
    const float s = (red[i] + red[M * 64 + i]) + (red[2 * M * 64 + i] + red[3 * M * 64 + i]);
    part[((int64_t)split * M + i / 64) * n_cols + (int64_t)nb * 64 + i % 64] = s;
  }
}

struct RowsFinish {
  const float* part; int splits, M, n_cols;
  bool rope; int64_t pos0;     // rotate with positions pos0 + m (engine.hpp:225-243: angles in double, cos / sin cast to float)
  const float* down; const float* b; int64_t ldb; int r; float scale;   // LoRA up-projection (null = none)
  int d_head;
};

__device__ __forceinline__ float2 rope_cs(const RowsFinish& f, int m, int c) {
  const double freq = pow(10000.0, -2.0 * (double)c / (double)f.d_head);
  double s, co;
  sincos((double)(f.pos0 + m) * freq, &s, &co);
  return make_float2((float)co, (float)s);
}

__device__ __forceinline__ float rows_sum(const RowsFinish& f, int m, int col) {
  float s = 0.f;
  for (int sp = 0; sp < f.splits; ++sp) s += f.part[((int64_t)sp * f.M + m) * f.n_cols + col];
  return s;
}

// q rows: one thread per (row, head, c < d/2): the rotation pair (c, c + d/2)
__global__ void rows_q_finish_kernel(RowsFinish f, float* __restrict__ q_out, int64_t ldq) {
  const int half = f.d_head / 2;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = f.n_cols / 2;
  if (idx >= f.M * per_row) return;
  const int m = idx / per_row, h = (idx % per_row) / half, c = idx % half;
  const int c0 = h * f.d_head + c, c1 = c0 + half;
  float x0 = rows_sum(f, m, c0), x1 = rows_sum(f, m, c1);
  if (f.down != nullptr)
    for (int k = 0; k < f.r; ++k) {
      const float dk = f.scale * f.down[m * f.r + k];
      x0 = fmaf(dk, f.b[(int64_t)k * f.ldb + c0], x0);
      x1 = fmaf(dk, f.b[(int64_t)k * f.ldb + c1], x1);
    }
  if (f.rope) {
    const float2 cs = rope_cs(f, m, c);
    const float a = x0 * cs.x - x1 * cs.y, b = x0 * cs.y + x1 * cs.x;
    x0 = a; x1 = b;
  }
  q_out[(int64_t)m * ldq + c0] = x0;
  q_out[(int64_t)m * ldq + c1] = x1;
}

struct RowsPages {
  __nv_bfloat16 *k_pages, *v_pages;
  const int32_t* table;
  int64_t head_stride, page_stride, row0, k_from, v_from;
  int n_kv_local;
  PageLayout lay;
};

// K and V rows: columns [0, n_kv * d) are key heads, the rest value heads (the packed [Wk | Wv] order)
__global__ void rows_kv_finish_kernel(RowsFinish f, RowsPages pg) {
  const int half = f.d_head / 2;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = f.n_cols / 2;
  if (idx >= f.M * per_row) return;
  const int m = idx / per_row, hb = (idx % per_row) / half, c = idx % half;
  const bool is_k = hb < pg.n_kv_local;
  const int head = is_k ? hb : hb - pg.n_kv_local;
  const int c0 = hb * f.d_head + c, c1 = c0 + half;
  float x0 = rows_sum(f, m, c0), x1 = rows_sum(f, m, c1);
  if (is_k && f.rope) {
    const float2 cs = rope_cs(f, m, c);
    const float a = x0 * cs.x - x1 * cs.y, b = x0 * cs.y + x1 * cs.x;
    x0 = a; x1 = b;
  }
  if (!is_k && f.down != nullptr)
    for (int k = 0; k < f.r; ++k) {
      const float dk = f.scale * f.down[m * f.r + k];
      x0 = fmaf(dk, f.b[(int64_t)k * f.ldb + head * f.d_head + c], x0);
      x1 = fmaf(dk, f.b[(int64_t)k * f.ldb + head * f.d_head + c + half], x1);
    }
  const int64_t row = pg.row0 + m;
  if (row < (is_k ? pg.k_from : pg.v_from)) return;          // first writer wins: already cached
  __nv_bfloat16* page = (is_k ? pg.k_pages : pg.v_pages) + (int64_t)head * pg.head_stride + (int64_t)pg.table[row / pg.lay.P] * pg.page_stride;
  const int t = (int)(row % pg.lay.P);
  page[page_offset(pg.lay, t, c)] = __float2bfloat16_rn(x0);
  page[page_offset(pg.lay, t, c + half)] = __float2bfloat16_rn(x1);
}

// K splits: enough CTAs for ~3 per SM, a slice of at least 64 and at most 1024 reduction rows (the rows of x live in
// shared memory)
int pick_splits(int d_model, int n_blocks, int sm_count) {
  int splits = 1;
  auto can_double = [&]() { return d_model % (2 * splits) == 0 && d_model / (2 * splits) >= 64 && splits < 64; };
  while (d_model / splits > 1024 && can_double()) splits *= 2;
  while (n_blocks * splits < 3 * sm_count && can_double()) splits *= 2;
  return splits;
}

}  // namespace

bool rows_project_supported(int64_t n_rows, int64_t d_model, int64_t rank) {
  return n_rows >= 1 && n_rows <= kMaxRows && d_model % 64 == 0 && d_model <= 65536 && rank <= 64;
}

int launch_rows_xa(lorakv_ctx* ctx, const float* a_dev, int64_t d_model, int64_t rank, const float* x_dev, int64_t n_rows, int64_t ld,
                   float* down_dev) {
  if (n_rows == 0 || rank == 0) return LORAKV_OK;
  rows_xa_kernel<<<(unsigned)n_rows, 256, 0, ctx->stream>>>(x_dev, ld, a_dev, (int)d_model, (int)rank, down_dev, LrPages{});
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

// partial sums of x * W over the packed weights into ctx->work; returns the split count and the buffer
static int rows_partial(lorakv_ctx* ctx, const void* w_packed, int64_t d_model, int64_t n_cols, const float* x_dev, int64_t n_rows,
                        int64_t ld, size_t head_bytes, int* splits_out, float** part_out) {
  const int n_blocks = (int)(n_cols / 64);
  const int splits = pick_splits((int)d_model, n_blocks, ctx->sm_count);
  const int kc = (int)(d_model / splits);
  LK_TRY(scratch_reserve(ctx, ctx->work, head_bytes + (size_t)splits * n_rows * n_cols * sizeof(float)));
  float* part = reinterpret_cast<float*>(static_cast<char*>(ctx->work.ptr) + head_bytes);
  const size_t smem = (size_t)std::max<int64_t>(n_rows * kc, 4 * n_rows * 64) * sizeof(float);
  rows_partial_kernel<<<dim3((unsigned)n_blocks, (unsigned)splits), kPartThreads, smem, ctx->stream>>>(
      x_dev, ld, (int)n_rows, static_cast<const __nv_bfloat16*>(w_packed), (int)d_model, (int)n_cols, kc, part);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  *splits_out = splits; *part_out = part;
  return LORAKV_OK;
}

int launch_rows_kv_project(lorakv_pool* pool, const void* w_packed, int64_t layer, int64_t set, int64_t row0, int64_t k_from,
                           int64_t v_from, const float* x_dev, int64_t n_rows, int64_t ld, bool rope, const float* down_dev,
                           const float* bv_dev, int64_t rank, float v_scale) {
  lorakv_ctx* ctx = pool->ctx;
  const int64_t d = pool->dims.d_head, n_kv = pool->n_kv_local, n_cols = 2 * n_kv * d;
  int splits; float* part;
  LK_TRY(rows_partial(ctx, w_packed, pool->dims.d_model, n_cols, x_dev, n_rows, ld, 0, &splits, &part));
  RowsFinish f{part, splits, (int)n_rows, (int)n_cols, rope, row0, down_dev, bv_dev, n_kv * d, (int)rank, v_scale, (int)d};
  RowsPages pg;
  pg.k_pages = static_cast<__nv_bfloat16*>(pool->k_pages) + layer * pool->kv_layer_stride();
  pg.v_pages = static_cast<__nv_bfloat16*>(pool->v_pages) + layer * pool->kv_layer_stride();
  pg.table = pool->kv_space.dev_table + set * pool->kv_space.max_pages;
  pg.head_stride = pool->kv_head_stride(); pg.page_stride = pool->kv_page_stride();
  pg.row0 = row0; pg.k_from = k_from; pg.v_from = v_from; pg.n_kv_local = (int)n_kv;
  pg.lay = make_page_layout((int)pool->P, (int)d, 2);
  const int n = (int)(n_rows * n_cols / 2);
  rows_kv_finish_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(f, pg);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  ctx->last_kernel = "rows_kv_project";
  return LORAKV_OK;
}

int launch_rows_q_project(lorakv_ctx* ctx, const void* wq_packed, int64_t d_model, int64_t n_cols, int64_t d_head, const float* down_dev,
                          const float* bq_dev, int64_t ldb, int64_t rank, float q_scale, int64_t pos0, const float* x_dev, int64_t n_rows,
                          int64_t ld, bool rope, float* q_dev) {
  int splits; float* part;
  LK_TRY(rows_partial(ctx, wq_packed, d_model, n_cols, x_dev, n_rows, ld, 0, &splits, &part));
  RowsFinish f{part, splits, (int)n_rows, (int)n_cols, rope, pos0, rank > 0 ? down_dev : nullptr, bq_dev, ldb, (int)rank, q_scale, (int)d_head};
  const int n = (int)(n_rows * n_cols / 2);
  rows_q_finish_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(f, q_dev, n_cols);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  ctx->last_kernel = "rows_q_project";
  return LORAKV_OK;
}

int launch_rows_lr_project(lorakv_pool* pool, const float* a_dev, int64_t d_model, int64_t rank, int64_t layer, int64_t set, int64_t row0,
                           const float* x_dev, int64_t n_rows, int64_t ld) {
  lorakv_ctx* ctx = pool->ctx;
  LrPages lp;
  lp.pages = static_cast<__nv_bfloat16*>(pool->lr_pages) + layer * pool->lr_layer_stride();
  lp.table = pool->lr_space.dev_table + set * pool->lr_space.max_pages;
  lp.page_stride = pool->lr_page_stride(); lp.row0 = row0; lp.r_pad = (int)pool->r_pad;
  lp.lay = make_page_layout((int)pool->P, (int)pool->r_pad, 2);
  rows_xa_kernel<<<(unsigned)n_rows, 256, 0, ctx->stream>>>(x_dev, ld, a_dev, (int)d_model, (int)rank, nullptr, lp);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

}  // namespace lk
