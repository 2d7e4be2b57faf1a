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
template <class S> __device__ __forceinline__ S to_store(double x);
template <> __device__ __forceinline__ double to_store<double>(double x) { return x; }       // fp64 pages: exact
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
    // fp32 pages swizzle 16-byte chunks (page_layout.cuh): the two halves are placed separately
    float* df = reinterpret_cast<float*>(dst);
    float* df2 = df - page_offset(a.lay, (int)(row % a.P), c) + page_offset(a.lay, (int)(row % a.P), c + 4);
    *reinterpret_cast<float4*>(df) = make_float4(x[0], x[1], x[2], x[3]);
    *reinterpret_cast<float4*>(df2) = make_float4(x[4], x[5], x[6], x[7]);
  }
}

// scalar variant for head dims that are not a multiple of 8
template <class S, class Src = float>
__global__ void kv_append_scatter_scalar_kernel(PageAddr a, int64_t row0, const Src* __restrict__ src,
                                                int64_t n_rows, int64_t ld) {
  const int64_t per_row = (int64_t)a.width * a.n_heads;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * per_row) return;
  const int64_t i = idx / per_row;
  const int v = (int)(idx % per_row);
  const int head = v / a.width, c = v % a.width;
  const Src x = c < a.src_cols ? src[i * ld + (int64_t)head * a.src_cols + c] : Src(0);
  const int64_t row = row0 + i;
  const int64_t phys = a.table[row / a.P];
  static_cast<S*>(a.base)[(int64_t)head * a.head_stride + phys * a.page_stride + page_offset(a.lay, (int)(row % a.P), c)] = to_store<S>(x);
}

__global__ void gather_rows_f64_kernel(PageAddr a, int64_t row0, int64_t n_rows, double* __restrict__ dst) {
  const int64_t per_row = (int64_t)a.src_cols * a.n_heads;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * per_row) return;
  const int64_t i = idx / per_row;
  const int v = (int)(idx % per_row);
  const int head = v / a.src_cols, c = v % a.src_cols;
  const int64_t row = row0 + i;
  const int64_t phys = a.table[row / a.P];
  dst[idx] = static_cast<const double*>(a.base)[(int64_t)head * a.head_stride + phys * a.page_stride + page_offset(a.lay, (int)(row % a.P), c)];
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

// V_lr = X * A (engine.hpp:414-418 through matmul_accumulate, matrix.hpp:101-111), bound by the one
// pass over X in HBM (d_model * 4 bytes per row against 2 * r flops per element).
//
// A warp owns R rows (R * RP = 128 accumulators per lane) and its lanes split the reduction
// dimension: per 128-wide k chunk lane l takes k = 4l .. 4l+3, so every X row is read as one fully
// coalesced 512-byte line per chunk and never revisited.  The matching A chunk (128 x RP) is staged
// once per CTA in shared memory in a [k % 4][column quad][lane] order that makes the per-lane float4
// reads conflict-free.  The 32 partial sums per output are combined by a halving butterfly
// (124 shuffles for 128 outputs, not 640) that leaves four consecutive columns of one row per lane.
constexpr int kProjWarps = 4, kProjChunk = 128;

template <class S, int RP>
__global__ void __launch_bounds__(kProjWarps * 32) lr_append_project_kernel(
    PageAddr a, int64_t row0, const float* __restrict__ x, int64_t n_rows, int64_t ld,
    const float* __restrict__ A, int d_model, int rank, bool round_inputs, bool vec_ok) {
  constexpr int R = 128 / RP;                      // rows per warp
  constexpr int Q4 = RP / 4;                       // column quads
  extern __shared__ float4 a_dyn[];                // [buffer][i][quad][lane]
  float4 (*a_s)[4 * Q4 * 32] = reinterpret_cast<float4 (*)[4 * Q4 * 32]>(a_dyn);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t r_first = ((int64_t)blockIdx.x * kProjWarps + warp) * R;

  float acc[R * RP];
#pragma unroll
  for (int i = 0; i < R * RP; ++i) acc[i] = 0.f;

  auto stage_a = [&](int buf, int k0) {            // A[k0 .. k0+127][0 .. RP) -> a_s[buf]
    for (int idx = tid; idx < 4 * Q4 * 32; idx += kProjWarps * 32) {
      const int l = idx % 32, qd = (idx / 32) % Q4, i = idx / (32 * Q4);
      const int k = k0 + 4 * l + i;
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = 4 * qd + u;
        v[u] = (k < d_model && c < rank) ? A[(int64_t)k * rank + c] : 0.f;
      }
      a_s[buf][idx] = make_float4(v[0], v[1], v[2], v[3]);
    }
  };

  const int n_chunks = (d_model + kProjChunk - 1) / kProjChunk;
  stage_a(0, 0);
  __syncthreads();
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int buf = ch & 1, k0 = ch * kProjChunk;
    if (ch + 1 < n_chunks) stage_a(buf ^ 1, k0 + kProjChunk);
    float xv[R][4];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int64_t row = r_first + rr;
      const int k = k0 + 4 * lane;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < n_rows) {
        const float* src = x + row * ld + k;
        if (vec_ok && k + 3 < d_model) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          if (k < d_model) v.x = src[0];
          if (k + 1 < d_model) v.y = src[1];
          if (k + 2 < d_model) v.z = src[2];
          if (k + 3 < d_model) v.w = src[3];
        }
      }
      if (round_inputs) {
        v.x = __bfloat162float(__float2bfloat16_rn(v.x)); v.y = __bfloat162float(__float2bfloat16_rn(v.y));
        v.z = __bfloat162float(__float2bfloat16_rn(v.z)); v.w = __bfloat162float(__float2bfloat16_rn(v.w));
      }
      xv[rr][0] = v.x; xv[rr][1] = v.y; xv[rr][2] = v.z; xv[rr][3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int qd = 0; qd < Q4; ++qd) {
        const float4 av = a_s[buf][(i * Q4 + qd) * 32 + lane];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          acc[rr * RP + 4 * qd + 0] = fmaf(xv[rr][i], av.x, acc[rr * RP + 4 * qd + 0]);
          acc[rr * RP + 4 * qd + 1] = fmaf(xv[rr][i], av.y, acc[rr * RP + 4 * qd + 1]);
          acc[rr * RP + 4 * qd + 2] = fmaf(xv[rr][i], av.z, acc[rr * RP + 4 * qd + 2]);
          acc[rr * RP + 4 * qd + 3] = fmaf(xv[rr][i], av.w, acc[rr * RP + 4 * qd + 3]);
        }
      }
    }
    __syncthreads();     // the next chunk of A is staged; the current one may be overwritten after this
  }

  // halving butterfly: after the step with stride s a lane keeps the half of its values selected by
  // its bit s; at the end lane l holds outputs [4 * bitrev-weighted(l), +4) fully reduced
  int first = 0;
#pragma unroll
  for (int s = 16, n = (R * RP) / 2; s >= 1; s >>= 1, n >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const float send = upper ? acc[i] : acc[i + n];
      const float keep = upper ? acc[i + n] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
    if (upper) first += n;
  }
  const int rr = first / RP, c0 = first % RP;       // four consecutive columns of one row
  const int64_t i_row = r_first + rr;
  if (i_row >= n_rows) return;
  const int64_t row = row0 + i_row;
  const int64_t phys = a.table[row / a.P];
  S* dst = static_cast<S*>(a.base) + phys * a.page_stride + page_offset(a.lay, (int)(row % a.P), c0);
#pragma unroll
  for (int u = 0; u < 4; ++u) dst[u] = to_store<S>(c0 + u < rank ? acc[u] : 0.f);
}

// ---- tensor-core X * A for bf16 pools -------------------------------------------------------------
// The CUDA-core kernel above issues 2 * r FFMA per element of X and tops out near 560 GB/s of X; the
// product is HBM-bound (one pass over X, d_model * 4 bytes per row) once the MACs run on the tensor
// pipe.  bf16 pools round X to bf16 anyway (the cache stores bf16), so X tiles are converted in
// registers and fed to mma.sync.m16n8k16 (bf16 x bf16 -> fp32); A is split into bf16 hi + lo parts
// (two MMAs), which keeps its fp32 value to 2^-17 whatever the caller uploaded.
//
// Layout of the work: a warp owns 16 * MT rows and one quarter of the reduction dimension (split-K
// across the 4 warps of a CTA, combined through shared memory), so 4x as many warps stream X
// concurrently.  A lane reads X as float4 (a quad covers 64 contiguous bytes of a row); the k order
// inside a 16-wide step is permuted accordingly (slots 2t, 2t+1, 2t+8, 2t+9 <-> k0 + 4t .. 4t+3) and
// the B fragments are pre-packed in that order by lr_project_pack_a, one 16-byte load per lane.
constexpr int kMmaProjWarps = 4;

__global__ void lr_project_pack_a_kernel(const float* __restrict__ A, int d_model, int rank, int n_tiles, uint4* __restrict__ frag) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;          // (k16 block, n8 tile, lane)
  const int total = (d_model / 16) * n_tiles * 32;
  if (idx >= total) return;
  const int lane = idx % 32, nt = (idx / 32) % n_tiles, kb = idx / (32 * n_tiles);
  const int g = lane >> 2, t = lane & 3, n = nt * 8 + g;
  float v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) v[u] = n < rank ? A[(int64_t)(kb * 16 + 4 * t + u) * rank + n] : 0.f;
  __nv_bfloat16 hi[4], lo[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) { hi[u] = __float2bfloat16_rn(v[u]); lo[u] = __float2bfloat16_rn(v[u] - __bfloat162float(hi[u])); }
  auto pack = [](__nv_bfloat16 a, __nv_bfloat16 b) { return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16); };
  frag[idx] = make_uint4(pack(hi[0], hi[1]), pack(hi[2], hi[3]), pack(lo[0], lo[1]), pack(lo[2], lo[3]));
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int RP, int MT>
__global__ void __launch_bounds__(kMmaProjWarps * 32) lr_append_project_mma_kernel(
    PageAddr a, int64_t row0, const float* __restrict__ x, int64_t n_rows, int64_t ld, const uint4* __restrict__ frag,
    int d_model, int rank, float* __restrict__ dense) {
  constexpr int NT = RP / 8, ROWS = 16 * MT;
  __shared__ float red[kMmaProjWarps][ROWS][RP + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int64_t r_first = (int64_t)blockIdx.x * ROWS;
  const int kb_total = d_model / 16;
  const int kb0 = (int)((int64_t)kb_total * warp / kMmaProjWarps), kb1 = (int)((int64_t)kb_total * (warp + 1) / kMmaProjWarps);

  float acc[MT][NT][4];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[m][n][u] = 0.f;

  const float* xr[MT][2];
  bool ok[MT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = r_first + 16 * m + g + 8 * h;
      ok[m][h] = row < n_rows;
      xr[m][h] = x + (ok[m][h] ? row : 0) * ld + 4 * t;
    }
  auto pack2 = [](float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
  };
#pragma unroll 2
  for (int kb = kb0; kb < kb1; ++kb) {
    float4 xv[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        xv[m][h] = ok[m][h] ? __ldcs(reinterpret_cast<const float4*>(xr[m][h] + kb * 16)) : make_float4(0.f, 0.f, 0.f, 0.f);
    uint4 bf[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) bf[n] = __ldg(frag + ((int64_t)kb * NT + n) * 32 + lane);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      uint32_t af[4];
      af[0] = pack2(xv[m][0].x, xv[m][0].y); af[1] = pack2(xv[m][1].x, xv[m][1].y);
      af[2] = pack2(xv[m][0].z, xv[m][0].w); af[3] = pack2(xv[m][1].z, xv[m][1].w);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        mma_bf16_16816(acc[m][n], af, bf[n].x, bf[n].y);
        mma_bf16_16816(acc[m][n], af, bf[n].z, bf[n].w);
      }
    }
  }
  // split-K partials -> shared memory, then 8 consecutive columns of a row (one 16-byte chunk of the
  // swizzled page) per thread
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      red[warp][16 * m + g][8 * n + 2 * t] = acc[m][n][0]; red[warp][16 * m + g][8 * n + 2 * t + 1] = acc[m][n][1];
      red[warp][16 * m + g + 8][8 * n + 2 * t] = acc[m][n][2]; red[warp][16 * m + g + 8][8 * n + 2 * t + 1] = acc[m][n][3];
    }
  __syncthreads();
  for (int item = tid; item < ROWS * NT; item += kMmaProjWarps * 32) {
    const int rr = item / NT, c0 = (item % NT) * 8;
    const int64_t i_row = r_first + rr;
    if (i_row >= n_rows) continue;
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float sum = 0.f;
#pragma unroll
      for (int w = 0; w < kMmaProjWarps; ++w) sum += red[w][rr][c0 + u];
      v[u] = c0 + u < rank ? sum : 0.f;
    }
    if (dense != nullptr) {               // float32 rows [n_rows][rank] instead of pages (the q-LoRA down-projection)
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + u < rank) dense[i_row * rank + c0 + u] = v[u];
      continue;
    }
    const int64_t row = row0 + i_row;
    const int64_t phys = a.table[row / a.P];
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(a.base) + phys * a.page_stride + page_offset(a.lay, (int)(row % a.P), c0);
    uint4 pk;
    pk.x = pack2(v[0], v[1]); pk.y = pack2(v[2], v[3]); pk.z = pack2(v[4], v[5]); pk.w = pack2(v[6], v[7]);
    *reinterpret_cast<uint4*>(dst) = pk;
  }
}

PageAddr make_addr(const lorakv_pool* pool, int which, int64_t layer, int64_t set) {
  PageAddr a;
  const int64_t elem = pool->elem;
  if (which == LORAKV_HIDDEN) {          // one cache for the trajectory, paged through the K / V table
    a.base = pool->hidden_pages;
    a.table = pool->kv_space.dev_table;
    a.head_stride = 0;
    a.page_stride = pool->P * pool->dims.d_model;
    a.width = (int)pool->dims.d_model;
    a.n_heads = 1;
    a.src_cols = (int)pool->dims.d_model;
  } else if (which == LORAKV_LK) {       // key-side low-rank cache: layer-wide like the shared V_lr cache
    a.base = static_cast<char*>(pool->lk_pages) + layer * pool->lk_layer_stride() * elem;
    a.table = pool->lk_space.dev_table;
    a.head_stride = 0;
    a.page_stride = pool->lk_page_stride();
    a.width = (int)pool->rk_pad;
    a.n_heads = 1;
    a.src_cols = (int)pool->dims.rank_k;
  } else if (which == LORAKV_LR) {
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
                          const double* src_dev, int64_t n_rows, int64_t ld) {
  if (n_rows == 0) return LORAKV_OK;
  if (pool->dims.dtype != LORAKV_F64) return fail("append: float64 rows need an fp64 pool");
  lorakv_ctx* ctx = pool->ctx;
  const PageAddr a = make_addr(pool, which, layer, set);
  if (a.width == 0) return LORAKV_OK;
  const int64_t n = n_rows * a.width * a.n_heads;
  kv_append_scatter_scalar_kernel<double, double><<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(a, row0, src_dev, n_rows, ld);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

int launch_gather_rows(const lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                       int64_t n_rows, double* dst_dev) {
  if (n_rows == 0) return LORAKV_OK;
  if (pool->dims.dtype != LORAKV_F64) return fail("read: float64 rows need an fp64 pool");
  lorakv_ctx* ctx = pool->ctx;
  const PageAddr a = make_addr(pool, which, layer, set);
  if (a.src_cols == 0) return LORAKV_OK;
  const int64_t n = n_rows * a.src_cols * a.n_heads;
  gather_rows_f64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(a, row0, n_rows, dst_dev);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

int launch_append_scatter(lorakv_pool* pool, int which, int64_t layer, int64_t set, int64_t row0,
                          const float* src_dev, int64_t n_rows, int64_t ld) {
  if (n_rows == 0) return LORAKV_OK;
  if (pool->dims.dtype == LORAKV_F64) return fail("append: an fp64 pool takes float64 rows (lorakv_pool_append_f64)");
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
  if (pool->dims.dtype == LORAKV_F64) return fail("read: an fp64 pool returns float64 rows (lorakv_pool_read_f64)");
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

int launch_lr_project(lorakv_pool* pool, const float* a_dev, int64_t d_model, int64_t rank, int64_t layer, int64_t set,
                      int64_t row0, const float* x_dev, int64_t n_rows, int64_t ld, int which) {
  if (n_rows == 0) return LORAKV_OK;
  lorakv_ctx* ctx = pool->ctx;
  const PageAddr a = make_addr(pool, which, layer, set);
  if (a.width == 0) return LORAKV_OK;
  if (a.width > 128) return fail("lr_append_project: rank %lld > 128 is not supported", (long long)pool->dims.rank);
  const float* A = a_dev;
  const bool bf16 = pool->dims.dtype == LORAKV_BF16;
  const bool vec_ok = (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(x_dev) & 15) == 0);
  // a decode step's handful of rows: one CTA per row streams A (rows_project.cu) instead of a latency-bound MMA tile
  if (which == LORAKV_LR && bf16 && ctx->policy != 1 && rows_project_supported(n_rows, d_model, rank) && a.width <= 64 && a.lay.bw == a.width && a.width % 8 == 0) {
    LK_TRY(launch_rows_lr_project(pool, A, d_model, rank, layer, set, row0, x_dev, n_rows, ld));
    return LORAKV_OK;
  }
  // bf16 pools: tensor-core kernel (policy 1 keeps the CUDA-core kernel for cross-checks)
  if (bf16 && ctx->policy != 1 && vec_ok && d_model % 16 == 0 && d_model >= 64 && a.width <= 64 && a.lay.bw == a.width && a.width % 8 == 0) {
    const int nt = a.width / 8;
    const size_t frag_bytes = (size_t)(d_model / 16) * nt * 32 * sizeof(uint4);
    LK_TRY(scratch_reserve(ctx, ctx->work, frag_bytes));
    uint4* frag = static_cast<uint4*>(ctx->work.ptr);
    const int total = (int)(d_model / 16) * nt * 32;
    lr_project_pack_a_kernel<<<(total + 255) / 256, 256, 0, ctx->stream>>>(A, (int)d_model, (int)rank, nt, frag);
    auto go = [&](auto kern, int rows) {
      kern<<<(unsigned)((n_rows + rows - 1) / rows), kMmaProjWarps * 32, 0, ctx->stream>>>(a, row0, x_dev, n_rows, ld, frag, (int)d_model, (int)rank, nullptr);
    };
    switch (a.width) {
      case 8: go(lr_append_project_mma_kernel<8, 2>, 32); break;
      case 16: go(lr_append_project_mma_kernel<16, 2>, 32); break;
      case 32: go(lr_append_project_mma_kernel<32, 2>, 32); break;
      default: go(lr_append_project_mma_kernel<64, 1>, 16); break;
    }
    ctx->launches += 2;
    LK_CUDA(cudaGetLastError());
    return LORAKV_OK;
  }
  auto launch = [&](auto kern, int rp) {
    const int rows_per_cta = kProjWarps * (128 / rp);
    const unsigned blocks = (unsigned)((n_rows + rows_per_cta - 1) / rows_per_cta);
    const size_t smem = (size_t)2 * rp * 512;       // two [4][rp/4][32] float4 buffers
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<blocks, kProjWarps * 32, smem, ctx->stream>>>(a, row0, x_dev, n_rows, ld, A, (int)d_model, (int)rank, bf16, vec_ok);
  };
  switch (a.width) {
    case 16: bf16 ? launch(lr_append_project_kernel<__nv_bfloat16, 16>, 16) : launch(lr_append_project_kernel<float, 16>, 16); break;
    case 32: bf16 ? launch(lr_append_project_kernel<__nv_bfloat16, 32>, 32) : launch(lr_append_project_kernel<float, 32>, 32); break;
    case 64: bf16 ? launch(lr_append_project_kernel<__nv_bfloat16, 64>, 64) : launch(lr_append_project_kernel<float, 64>, 64); break;
    case 128: bf16 ? launch(lr_append_project_kernel<__nv_bfloat16, 128>, 128) : launch(lr_append_project_kernel<float, 128>, 128); break;
    default: return fail("lr_append_project: padded rank %d is not one of 16/32/64/128", a.width);
  }
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

// x * A as dense float32 rows [n_rows][rank] (tensor-core kernel above; bf16 X, A kept to fp32 accuracy): the q-LoRA
// down-projection of engine.hpp:366-367
int launch_xa_dense(lorakv_ctx* ctx, const float* a_dev, int64_t d_model, int64_t rank, const float* x_dev, int64_t n_rows, int64_t ld,
                    float* out_dev) {
  if (n_rows == 0 || rank == 0) return LORAKV_OK;
  if (rank > 64 || d_model % 16 != 0 || ld % 4 != 0 || (reinterpret_cast<uintptr_t>(x_dev) & 15) != 0)
    return fail("xa_dense: unsupported shape (rank %lld, d_model %lld)", (long long)rank, (long long)d_model);
  const int rp = rank <= 8 ? 8 : rank <= 16 ? 16 : rank <= 32 ? 32 : 64;
  const int nt = rp / 8;
  const size_t frag_bytes = (size_t)(d_model / 16) * nt * 32 * sizeof(uint4);
  LK_TRY(scratch_reserve(ctx, ctx->work, frag_bytes));
  uint4* frag = static_cast<uint4*>(ctx->work.ptr);
  const int total = (int)(d_model / 16) * nt * 32;
  lr_project_pack_a_kernel<<<(total + 255) / 256, 256, 0, ctx->stream>>>(a_dev, (int)d_model, (int)rank, nt, frag);
  PageAddr none{};
  auto go = [&](auto kern, int rows) {
    kern<<<(unsigned)((n_rows + rows - 1) / rows), kMmaProjWarps * 32, 0, ctx->stream>>>(none, 0, x_dev, n_rows, ld, frag, (int)d_model, (int)rank, out_dev);
  };
  switch (rp) {
    case 8: go(lr_append_project_mma_kernel<8, 2>, 32); break;
    case 16: go(lr_append_project_mma_kernel<16, 2>, 32); break;
    case 32: go(lr_append_project_mma_kernel<32, 2>, 32); break;
    default: go(lr_append_project_mma_kernel<64, 1>, 16); break;
  }
  ctx->launches += 2;
  LK_CUDA(cudaGetLastError());
  return LORAKV_OK;
}

}  // namespace lk
