// cache_kernels.cu -- append / read-back kernels of the paged cache.
//
//   kv_append_scatter : GrowMat::append (proj/include/lorakv/kvcache.hpp:171-182) -- new K / V_base /
//                       V_lr rows copied into pages, 16-byte vectorised, converting to the pool dtype
//   lr_append_project : engine.hpp:414-418 -- V_lr rows = X * A (unscaled, matrix.hpp:101-111) computed
//                       once for all agents and written straight into the LR pages
//   gather_rows       : key_view / value_view / lr_view (kvcache.hpp:307-324) -- pages back to a
//                       dense row-major float32 matrix
// First-writer-wins (kvcache.hpp:400-407) and page allocation are resolved on the host before
// launch, so no kernel here needs atomics.
#include <cuda_bf16.h>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"

namespace lk {

namespace {

struct PageAddr {
  void* base;               // page array of the buffer (layer offset applied)
  const int32_t* table;     // logical -> physical page of the set
  int64_t head_stride;      // elements between kv heads (0 for LR)
  int64_t page_stride;      // elements per page
  int P, width;             // tokens per page; elements per row within one head (d or r_pad)
  int n_heads;              // heads in a source row (1 for LR)
  int src_cols;             // valid source columns per head (d or rank); the rest is zero padding
  PageLayout lay;           // element placement inside one page (page_layout.cuh)
};

template <class S> __device__ __forceinline__ S to_store(float x);
template <> __device__ __forceinline__ float to_store<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 to_store<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <class S> __device__ __forceinline__ float from_store(S x);
template <> __device__ __forceinline__ float from_store<float>(float x) { return x; }
template <> __device__ __forceinline__ float from_store<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

// one thread per 8 consecutive elements of a row (one 16-byte bf16 store / two fp32 stores)
template <class S>
__global__ void kv_append_scatter_kernel(PageAddr a, int64_t row0, const float* __restrict__ src,
                                         int64_t n_rows, int64_t ld) {
  const int vec_per_head = a.width / 8;
  const int64_t vec_per_row = (int64_t)vec_per_head * a.n_heads;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * vec_per_row) return;
  const int64_t i = idx / vec_per_row;
  const int v = (int)(idx % vec_per_row);
  const int head = v / vec_per_head, c = (v % vec_per_head) * 8;
  const float* s = src + i * ld + (int64_t)head * a.src_cols + c;
  float x[8];
  const bool full = c + 8 <= a.src_cols;
  if (full && ((reinterpret_cast<uintptr_t>(s) & 15) == 0)) {
    const float4 lo = *reinterpret_cast<const float4*>(s), hi = *reinterpret_cast<const float4*>(s + 4);
    x[0] = lo.x; x[1] = lo.y; x[2] = lo.z; x[3] = lo.w; x[4] = hi.x; x[5] = hi.y; x[6] = hi.z; x[7] = hi.w;
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = (c + u < a.src_cols) ? s[u] : 0.f;   // zero padding is exact
  }
  const int64_t row = row0 + i;
  const int64_t phys = a.table[row / a.P];
  S* dst = static_cast<S*>(a.base) + (int64_t)head * a.head_stride + phys * a.page_stride +
           page_offset(a.lay, (int)(row % a.P), c);
  if (sizeof(S) == 2) {
    __nv_bfloat162 p0 = __floats2bfloat162_rn(x[0], x[1]), p1 = __floats2bfloat162_rn(x[2], x[3]);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(x[4], x[5]), p3 = __floats2bfloat162_rn(x[6], x[7]);
    uint4 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&p0); pk.y = *reinterpret_cast<uint32_t*>(&p1);
    pk.z = *reinterpret_cast<uint32_t*>(&p2); pk.w = *reinterpret_cast<uint32_t*>(&p3);
    *reinterpret_cast<uint4*>(dst) = pk;
  } else {
    float* df = reinterpret_cast<float*>(dst);
    *reinterpret_cast<float4*>(df) = make_float4(x[0], x[1], x[2], x[3]);
    *reinterpret_cast<float4*>(df + 4) = make_float4(x[4], x[5], x[6], x[7]);
  }
}

// scalar variant for head dims that are not a multiple of 8
template <class S>
__global__ void kv_append_scatter_scalar_kernel(PageAddr a, int64_t row0, const float* __restrict__ src,
                                                int64_t n_rows, int64_t ld) {
  const int64_t per_row = (int64_t)a.width * a.n_heads;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * per_row) return;
  const int64_t i = idx / per_row;
  const int v = (int)(idx % per_row);
  const int head = v / a.width, c = v % a.width;
  const float x = c < a.src_cols ? src[i * ld + (int64_t)head * a.src_cols + c] : 0.f;
  const int64_t row = row0 + i;
  const int64_t phys = a.table[row / a.P];
  static_cast<S*>(a.base)[(int64_t)head * a.head_stride + phys * a.page_stride + page_offset(a.lay, (int)(row % a.P), c)] = to_store<S>(x);
}

template <class S>
__global__ void gather_rows_kernel(PageAddr a, int64_t row0, int64_t n_rows, float* __restrict__ dst) {
  const int64_t per_row = (int64_t)a.src_cols * a.n_heads;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * per_row) return;
  const int64_t i = idx / per_row;
  const int v = (int)(idx % per_row);
  const int head = v / a.src_cols, c = v % a.src_cols;
  const int64_t row = row0 + i;
  const int64_t phys = a.table[row / a.P];
  dst[idx] = from_store<S>(static_cast<const S*>(a.base)[(int64_t)head * a.head_stride + phys * a.page_stride +
                                                        page_offset(a.lay, (int)(row % a.P), c)]);
}

// V_lr = X * A on CUDA cores: a 64-row x r_pad tile per CTA, K staged through shared memory in
// slices of 32.  X is streamed once from HBM (the bound: d_model*4 bytes per row against 2*r flops
// per element); A (d_model x r) stays L2 resident.  Accumulation order over k is ascending, like
// matmul_accumulate (matrix.hpp:101-111).
constexpr int kProjRows = 64, kProjK = 32, kProjThreads = 256;
template <class S>
__global__ void __launch_bounds__(kProjThreads) lr_append_project_kernel(
    PageAddr a, int64_t row0, const float* __restrict__ x, int64_t n_rows, int64_t ld,
    const float* __restrict__ A, int d_model, int rank, bool round_inputs) {
  __shared__ float x_s[kProjRows][kProjK + 1];
  extern __shared__ float a_s[];                 // [kProjK][r_pad]
  const int rp = a.width;
  const int tid = threadIdx.x;
  const int r_local = tid / 4;                   // row within the tile
  const int cg = tid % 4;                        // column group: columns cg, cg+4, ... (<= 32 per thread)
  const int64_t tile0 = (int64_t)blockIdx.x * kProjRows;
  float acc[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) acc[u] = 0.f;
  for (int k0 = 0; k0 < d_model; k0 += kProjK) {
    for (int idx = tid; idx < kProjRows * kProjK; idx += kProjThreads) {
      const int rr = idx / kProjK, kk = idx % kProjK;
      const int64_t row = tile0 + rr;
      float v = (row < n_rows && k0 + kk < d_model) ? x[row * ld + k0 + kk] : 0.f;
      if (round_inputs) v = __bfloat162float(__float2bfloat16_rn(v));
      x_s[rr][kk] = v;
    }
    for (int idx = tid; idx < kProjK * rp; idx += kProjThreads) {
      const int kk = idx / rp, c = idx % rp;
      a_s[idx] = (k0 + kk < d_model && c < rank) ? A[(int64_t)(k0 + kk) * rank + c] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kProjK; ++kk) {
      const float xv = x_s[r_local][kk];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int c = cg + 4 * u;
        if (c < rp) acc[u] = fmaf(xv, a_s[kk * rp + c], acc[u]);
      }
    }
    __syncthreads();
  }
  const int64_t i = tile0 + r_local;
  if (i >= n_rows) return;
  const int64_t row = row0 + i;
  const int64_t phys = a.table[row / a.P];
  S* dst = static_cast<S*>(a.base) + phys * a.page_stride;
  const int t = (int)(row % a.P);
#pragma unroll
  for (int u = 0; u < 32; ++u) {
    const int c = cg + 4 * u;
    if (c < rp) dst[page_offset(a.lay, t, c)] = to_store<S>(c < rank ? acc[u] : 0.f);
  }
}

PageAddr make_addr(const lorakv_pool* pool, int which, int64_t layer, int64_t set) {
  PageAddr a;
  const int64_t elem = pool->elem;
  if (which == LORAKV_LR) {
    a.base = static_cast<char*>(pool->lr_pages) + layer * pool->lr_layer_stride() * elem;
    a.table = pool->lr_space.dev_table + set * pool->lr_space.max_pages;
    a.head_stride = 0;
    a.page_stride = pool->lr_page_stride();
    a.width = (int)pool->r_pad;
    a.n_heads = 1;
    a.src_cols = (int)pool->dims.rank;
  } else {
    void* pages = which == LORAKV_KEY ? pool->k_pages : pool->v_pages;
    a.base = static_cast<char*>(pages) + layer * pool->kv_layer_stride() * elem;
    a.table = pool->kv_space.dev_table + set * pool->kv_space.max_pages;
    a.head_stride = pool->kv_head_stride();
    a.page_stride = pool->kv_page_stride();
    a.width = (int)pool->dims.d_head;
    a.n_heads = (int)pool->n_kv_local;
    a.src_cols = (int)pool->dims.d_head;
  }
  a.P = (int)pool->P;
  a.lay = make_page_layout(a.P, a.width, (int)elem);
  return a;
}

}  // namespace

int launch_append_scatter(lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                          const float* src_dev, int64_t n_rows, int64_t ld) {
  if (n_rows == 0) return LORAKV_OK;
  lorakv_ctx* ctx = pool->ctx;
  const PageAddr a = make_addr(pool, which, layer, set);
  if (a.width == 0) return LORAKV_OK;   // rank-0 cache tracks row counts only (kvcache.hpp:173-176)
  const bool bf16 = pool->dims.dtype == LORAKV_BF16;
  if (a.width % 8 == 0) {
    const int64_t n = n_rows * (a.width / 8) * a.n_heads;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (bf16) kv_append_scatter_kernel<__nv_bfloat16><<<blocks, 256, 0, ctx->stream>>>(a, row0, src_dev, n_rows, ld);
    else kv_append_scatter_kernel<float><<<blocks, 256, 0, ctx->stream>>>(a, row0, src_dev, n_rows, ld);
  } else {
    const int64_t n = n_rows * a.width * a.n_heads;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (bf16) kv_append_scatter_scalar_kernel<__nv_bfloat16><<<blocks, 256, 0, ctx->stream>>>(a, row0, src_dev, n_rows, ld);
    else kv_append_scatter_scalar_kernel<float><<<blocks, 256, 0, ctx->stream>>>(a, row0, src_dev, n_rows, ld);
  }
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

int launch_gather_rows(const lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                       int64_t n_rows, float* dst_dev) {
  if (n_rows == 0) return LORAKV_OK;
  lorakv_ctx* ctx = pool->ctx;
  const PageAddr a = make_addr(pool, which, layer, set);
  if (a.src_cols == 0) return LORAKV_OK;
  const int64_t n = n_rows * a.src_cols * a.n_heads;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (pool->dims.dtype == LORAKV_BF16) gather_rows_kernel<__nv_bfloat16><<<blocks, 256, 0, ctx->stream>>>(a, row0, n_rows, dst_dev);
  else gather_rows_kernel<float><<<blocks, 256, 0, ctx->stream>>>(a, row0, n_rows, dst_dev);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

int launch_lr_project(lorakv_pool* pool, const lorakv_adapters* ad, int64_t layer, int64_t set,
                      int64_t row0, const float* x_dev, int64_t n_rows, int64_t ld) {
  if (n_rows == 0) return LORAKV_OK;
  lorakv_ctx* ctx = pool->ctx;
  const PageAddr a = make_addr(pool, LORAKV_LR, layer, set);
  if (a.width == 0) return LORAKV_OK;
  if (a.width > 128) return fail("lr_append_project: rank %lld > 128 is not supported", (long long)pool->dims.rank);
  const float* A = ad->a + layer * ad->d_model * ad->rank;
  const unsigned blocks = (unsigned)((n_rows + kProjRows - 1) / kProjRows);
  const size_t smem = sizeof(float) * kProjK * a.width;
  const bool bf16 = pool->dims.dtype == LORAKV_BF16;
  if (bf16)
    lr_append_project_kernel<__nv_bfloat16><<<blocks, kProjThreads, smem, ctx->stream>>>(
        a, row0, x_dev, n_rows, ld, A, (int)ad->d_model, (int)ad->rank, true);
  else
    lr_append_project_kernel<float><<<blocks, kProjThreads, smem, ctx->stream>>>(
        a, row0, x_dev, n_rows, ld, A, (int)ad->d_model, (int)ad->rank, false);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

}  // namespace lk
