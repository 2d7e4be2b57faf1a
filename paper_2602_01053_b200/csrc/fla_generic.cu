// fla_generic.cu -- shape-generic Flash-LoRA-Attention on CUDA cores (float / double).
//
// Stands behind the header-template operators of the reference for ANY (L_c, L, d <= 256, r <= 128,
// query_offset, strides): flash_lora_attention (proj/include/lorakv/attention.hpp:210-268),
// expand_first_attention (:274-326), naive_attention (:81-112) and gqa_attention (:332-363).
// It is the no-CPU-fallback safety net for shapes the tcgen05 fast paths do not cover and the
// fp64 instantiation; the bf16 / Llama-shaped hot path lives in fla_decode_* / fla_prefill_*.
//
// Numerics contract (SURVEY.md 8a'): score = dot * (1/sqrt(d)); key j is invisible to row i iff
// j > query_offset + i and is never loaded nor exponentiated; O and O_lr stay unnormalised until
// the epilogue o += (lr_scale * o_lr[p]) * b_up[p,:], then out = o / l.
#include <cmath>
#include <cstring>
#include <limits>

#include "kernels.hpp"
#include "state.hpp"

namespace lk {

template <class T> __device__ __forceinline__ T dev_exp(T x);
template <> __device__ __forceinline__ float dev_exp<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double dev_exp<double>(double x) { return exp(x); }
template <class T> __device__ __forceinline__ T neg_inf() { return -std::numeric_limits<T>::infinity(); }

template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kMaxTD = 8;   // d <= 256
constexpr int kMaxTR = 4;   // r <= 128
constexpr int kWarps = 4;

template <class T>
struct GenericArgs {
  const T *q, *k, *v, *vlr, *extra;      // compact device copies; extra: L x (heads_kv*d) or null
  int64_t ldq, ldk, ldv, ldlr, ldextra;
  int64_t Lc, L, d, r, query_offset;
  int n_heads, group;                    // q head h reads kv head h / group
  int splits;
  int64_t chunk;                         // keys per split (multiple of 32)
  T* part;                               // [heads][Lc][splits][2 + d + r + (extra ? d : 0)]
  int64_t part_stride;
  // key-side low-rank term (an extension the reference does not have, see KeyLowRank in kernels.hpp):
  // score = (q . k_base[j] + qk . l_k[j]) / sqrt(d), qk = k_scale * (q B_k^T) computed once per (row, head)
  const T *lk, *qk;                      // L x r_k; [Lc][heads][r_k]; null when r_k == 0
  int64_t r_k;
};

// Stage 1: one warp per (query row, q head, key split); lanes own keys for the scores and
// columns for the accumulators.  Mirrors detail::flash_tile_update (attention.hpp:140-200) with a
// 32-key tile.
template <class T, bool kExtra>
__global__ void __launch_bounds__(kWarps * 32) fla_generic_partial(GenericArgs<T> a) {
  extern __shared__ unsigned char smem_raw[];
  T* q_s = reinterpret_cast<T*>(smem_raw) + (threadIdx.x / 32) * (a.d + a.r_k);
  T* qk_s = q_s + a.d;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kWarps + threadIdx.x / 32;
  const int h = blockIdx.y, split = blockIdx.z;
  if (i >= a.Lc) return;
  const int kvh = h / a.group;
  const T* q_row = a.q + i * a.ldq + (int64_t)h * a.d;
  for (int64_t c = lane; c < a.d; c += 32) q_s[c] = q_row[c];
  for (int64_t c = lane; c < a.r_k; c += 32) qk_s[c] = a.qk[(i * a.n_heads + h) * a.r_k + c];
  __syncwarp();

  const T* k_base = a.k + (int64_t)kvh * a.d;
  const T* v_base = a.v + (int64_t)kvh * a.d;
  const T* e_base = kExtra ? a.extra + (int64_t)kvh * a.d : nullptr;
  const T inv_sqrt_d = T(1) / sqrt(static_cast<T>(a.d));
  const T ninf = neg_inf<T>();

  T o[kMaxTD], olr[kMaxTR], ex[kExtra ? kMaxTD : 1];
#pragma unroll
  for (int t = 0; t < kMaxTD; ++t) o[t] = T(0);
#pragma unroll
  for (int t = 0; t < kMaxTR; ++t) olr[t] = T(0);
  if (kExtra) {
#pragma unroll
    for (int t = 0; t < kMaxTD; ++t) ex[t] = T(0);
  }
  T m = ninf, l = T(0);

  const int64_t last_visible = a.query_offset + i;
  const int64_t j_begin = (int64_t)split * a.chunk;
  int64_t j_end = j_begin + a.chunk;
  if (j_end > a.L) j_end = a.L;
  if (j_end > last_visible + 1) j_end = last_visible + 1;

  for (int64_t j0 = j_begin; j0 < j_end; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool valid = j < j_end;
    T s = ninf;
    if (valid) {
      const T* k_row = k_base + j * a.ldk;
      T dot = T(0);
      for (int64_t c = 0; c < a.d; ++c) dot += q_s[c] * k_row[c];
      if (a.r_k > 0) {
        const T* lk_row = a.lk + j * a.r_k;
        for (int64_t c = 0; c < a.r_k; ++c) dot += qk_s[c] * lk_row[c];
      }
      s = dot * inv_sqrt_d;
    }
    const T tile_max = warp_max(s);
    const T m_new = max(m, tile_max);
    const T alpha = (m == ninf) ? T(0) : dev_exp<T>(m - m_new);
    const T p = valid ? dev_exp<T>(s - m_new) : T(0);
    l = alpha * l + warp_sum(p);
    m = m_new;
#pragma unroll
    for (int t = 0; t < kMaxTD; ++t) o[t] *= alpha;
#pragma unroll
    for (int t = 0; t < kMaxTR; ++t) olr[t] *= alpha;
    if (kExtra) {
#pragma unroll
      for (int t = 0; t < kMaxTD; ++t) ex[t] *= alpha;
    }
    const int n_valid = (int)min((int64_t)32, j_end - j0);
    for (int jj = 0; jj < n_valid; ++jj) {
      const T pj = __shfl_sync(0xffffffffu, p, jj);
      if (pj == T(0)) continue;
      const T* v_row = v_base + (j0 + jj) * a.ldv;
#pragma unroll
      for (int t = 0; t < kMaxTD; ++t) {
        const int64_t c = lane + 32 * t;
        if (c < a.d) o[t] += pj * v_row[c];
      }
      if (a.r > 0) {
        const T* lr_row = a.vlr + (j0 + jj) * a.ldlr;
#pragma unroll
        for (int t = 0; t < kMaxTR; ++t) {
          const int64_t c = lane + 32 * t;
          if (c < a.r) olr[t] += pj * lr_row[c];
        }
      }
      if (kExtra) {
        const T* e_row = e_base + (j0 + jj) * a.ldextra;
#pragma unroll
        for (int t = 0; t < kMaxTD; ++t) {
          const int64_t c = lane + 32 * t;
          if (c < a.d) ex[t] += pj * e_row[c];
        }
      }
    }
  }

  T* dst = a.part + (((int64_t)h * a.Lc + i) * a.splits + split) * a.part_stride;
  if (lane == 0) { dst[0] = m; dst[1] = l; }
#pragma unroll
  for (int t = 0; t < kMaxTD; ++t) {
    const int64_t c = lane + 32 * t;
    if (c < a.d) dst[2 + c] = o[t];
  }
#pragma unroll
  for (int t = 0; t < kMaxTR; ++t) {
    const int64_t c = lane + 32 * t;
    if (c < a.r) dst[2 + a.d + c] = olr[t];
  }
  if (kExtra) {
#pragma unroll
    for (int t = 0; t < kMaxTD; ++t) {
      const int64_t c = lane + 32 * t;
      if (c < a.d) dst[2 + a.d + a.r + c] = ex[t];
    }
  }
}

template <class T>
struct MergeArgs {
  const T* part;
  int64_t part_stride;
  int splits;
  int64_t Lc, d, r;
  int n_heads, group;
  const T* b_up;           // r x (heads_kv*d) compact device copy (null when r == 0 or expand-first)
  int64_t ldb;
  T lr_scale;
  bool extra;
  T* out;                  // Lc x (n_heads*d)
  T *row_max, *row_denom;  // [n_heads][Lc] or null
  int* bad_row;            // first row whose denominator is not > 0 (atomicMin), init INT_MAX
};

// Stage 2: combine the splits of one (row, head), then the epilogue of attention.hpp:244-259.
template <class T>
__global__ void __launch_bounds__(128) fla_generic_merge(MergeArgs<T> a) {
  extern __shared__ unsigned char smem_raw[];
  T* w_s = reinterpret_cast<T*>(smem_raw);   // [splits]
  T* olr_s = w_s + a.splits;                 // [r]
  __shared__ T l_total, m_total;
  const int64_t i = blockIdx.x;
  const int h = blockIdx.y;
  const T* base = a.part + ((int64_t)h * a.Lc + i) * a.splits * a.part_stride;
  const T ninf = neg_inf<T>();
  if (threadIdx.x == 0) {
    T mx = ninf;
    for (int s = 0; s < a.splits; ++s) mx = max(mx, base[s * a.part_stride]);
    T l = T(0);
    for (int s = 0; s < a.splits; ++s) {
      const T ms = base[s * a.part_stride];
      const T w = (ms == ninf) ? T(0) : dev_exp<T>(ms - mx);
      w_s[s] = w;
      l += w * base[s * a.part_stride + 1];
    }
    l_total = l; m_total = mx;
    if (!(l > T(0))) atomicMin(a.bad_row, (int)min(i, (int64_t)0x7ffffffe));
    if (a.row_max) a.row_max[(int64_t)h * a.Lc + i] = mx;
    if (a.row_denom) a.row_denom[(int64_t)h * a.Lc + i] = l;
  }
  __syncthreads();
  for (int64_t p = threadIdx.x; p < a.r; p += blockDim.x) {
    T acc = T(0);
    for (int s = 0; s < a.splits; ++s)
      if (w_s[s] != T(0)) acc += w_s[s] * base[s * a.part_stride + 2 + a.d + p];
    olr_s[p] = acc;
  }
  __syncthreads();
  const int kvh = h / a.group;
  for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x) {
    T acc = T(0);
    for (int s = 0; s < a.splits; ++s)
      if (w_s[s] != T(0)) acc += w_s[s] * base[s * a.part_stride + 2 + c];
    if (a.b_up) {
      for (int64_t p = 0; p < a.r; ++p) {
        const T w = a.lr_scale * olr_s[p];
        acc += w * a.b_up[p * a.ldb + (int64_t)kvh * a.d + c];
      }
    }
    if (a.extra) {
      T e = T(0);
      for (int s = 0; s < a.splits; ++s)
        if (w_s[s] != T(0)) e += w_s[s] * base[s * a.part_stride + 2 + a.d + a.r + c];
      acc += e;
    }
    a.out[i * ((int64_t)a.n_heads * a.d) + (int64_t)h * a.d + c] = acc / l_total;
  }
}

// expanded[j, c] = lr_scale * sum_p v_lr[j,p] * b_up[p,c]   (attention.hpp:281-285)
// qk[i][h][p] = k_scale * sum_c q[i][h d + c] * b_k[p][kvh d + c]: the query seen through the key adapter, r_k numbers per
// (row, head), so that the full-width adapter keys k_scale * L_k B_k are never formed
template <class T>
__global__ void qk_generic_kernel(const T* q, int64_t ldq, const T* bk, int64_t ldbk, T k_scale, int64_t Lc, int n_heads, int group,
                                  int64_t d, int64_t r_k, T* qk) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Lc * n_heads * r_k) return;
  const int64_t p = idx % r_k, h = (idx / r_k) % n_heads, i = idx / (r_k * n_heads);
  const T* q_row = q + i * ldq + h * d;
  const T* b_row = bk + p * ldbk + (h / group) * d;
  T acc = T(0);
  for (int64_t c = 0; c < d; ++c) acc += q_row[c] * b_row[c];
  qk[idx] = k_scale * acc;
}

template <class T>
__global__ void expand_lr_kernel(const T* vlr, int64_t ldlr, const T* b, int64_t ldb, T scale,
                                 int64_t L, int64_t width, int64_t r, T* out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L * width) return;
  const int64_t j = idx / width, c = idx % width;
  T acc = T(0);
  for (int64_t p = 0; p < r; ++p) acc += vlr[j * ldlr + p] * b[p * ldb + c];
  out[idx] = acc * scale;
}

// ---- materialising algorithm (naive_attention, attention.hpp:81-112) -------------------------
template <class T>
__global__ void naive_scores_kernel(const T* q, int64_t ldq, const T* k, int64_t ldk, int64_t Lc,
                                    int64_t L, int64_t d, int64_t off, T* scores) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Lc * L) return;
  const int64_t i = idx / L, j = idx % L;
  if (j > off + i) { scores[idx] = neg_inf<T>(); return; }
  T dot = T(0);
  for (int64_t c = 0; c < d; ++c) dot += q[i * ldq + c] * k[j * ldk + c];
  scores[idx] = dot * (T(1) / sqrt(static_cast<T>(d)));
}

template <class T>
__global__ void naive_softmax_kernel(T* scores, int64_t L) {   // one block per row (matrix.hpp:138-155)
  __shared__ T red[32];
  T* row = scores + (int64_t)blockIdx.x * L;
  T mx = neg_inf<T>();
  for (int64_t j = threadIdx.x; j < L; j += blockDim.x) mx = max(mx, row[j]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < (int)blockDim.x / 32; ++w) mx = max(mx, red[w]);
  __syncthreads();
  T sum = T(0);
  for (int64_t j = threadIdx.x; j < L; j += blockDim.x) {
    const T e = dev_exp<T>(row[j] - mx);
    row[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = sum;
  __syncthreads();
  T denom = T(0);
  for (int w = 0; w < (int)blockDim.x / 32; ++w) denom += red[w];
  for (int64_t j = threadIdx.x; j < L; j += blockDim.x) row[j] /= denom;
}

template <class T>
__global__ void naive_value_kernel(const T* v, int64_t ldv, const T* expanded, int64_t L, int64_t d,
                                   T* value) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L * d) return;
  const int64_t j = idx / d, c = idx % d;
  value[idx] = v[j * ldv + c] + (expanded ? expanded[idx] : T(0));
}

template <class T>
__global__ void naive_pv_kernel(const T* probs, const T* value, int64_t Lc, int64_t L, int64_t d,
                                T* out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Lc * d) return;
  const int64_t i = idx / d, c = idx % d;
  T acc = T(0);
  for (int64_t j = 0; j < L; ++j) acc += probs[i * L + j] * value[j * d + c];
  out[idx] = acc;
}

// ---- host drivers ------------------------------------------------------------------------------
static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

template <class T>
static int upload2d(lorakv_ctx* ctx, T* dst, const T* src, int64_t rows, int64_t cols, int64_t ld) {
  if (rows == 0 || cols == 0) return LORAKV_OK;
  LK_CUDA(cudaMemcpy2DAsync(dst, cols * sizeof(T), src, ld * sizeof(T), cols * sizeof(T), rows,
                            cudaMemcpyHostToDevice, ctx->stream));
  return LORAKV_OK;
}

template <class T>
static int check_shapes(const char* op, int64_t Lc, int64_t L, int64_t d, int64_t r, int64_t off) {
  if (Lc < 0 || L < 0 || d < 1 || r < 0) return fail("%s: invalid shape", op);
  if (off < 0 || off + Lc > L)
    return fail("attention: query_offset %lld with L_c %lld exceeds L %lld", (long long)off,
                (long long)Lc, (long long)L);
  if (d > 32 * kMaxTD) return fail("%s: head dim %lld > %d is not supported by the generic kernel",
                                   op, (long long)d, 32 * kMaxTD);
  if (r > 32 * kMaxTR) return fail("%s: rank %lld > %d is not supported by the generic kernel", op,
                                   (long long)r, 32 * kMaxTR);
  return LORAKV_OK;
}

template <class T>
static int finite_or_fail(const T* out, int64_t n, const char* op) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(static_cast<double>(out[i]))) return fail("%s produced a non-finite entry", op);
  return LORAKV_OK;
}

// mode: 0 = flash (reordered), 1 = expand-first
template <class T>
int generic_forward(lorakv_ctx* ctx, const char* op, int mode, const T* q, int64_t ldq, const T* k,
                    int64_t ldk, const T* v, int64_t ldv, const T* vlr, int64_t ldlr, const T* b,
                    int64_t ldb, T lr_scale, int64_t Lc, int64_t L, int n_q, int n_kv, int64_t d,
                    int64_t r, int64_t off, T* out, T* row_max, T* row_denom, const KeyLowRank<T>* key) {
  if (!ctx) return fail("%s: null context", op);
  LK_TRY(check_shapes<T>(op, Lc, L, d, r, off));
  const int64_t r_k = key ? key->r_k : 0;
  if (r_k < 0 || r_k > 128) return fail("%s: key rank %lld outside [0,128]", op, (long long)r_k);
  if (r_k > 0 && (!key->l_k || !key->b_k)) return fail("%s: key-side low-rank operands are null", op);
  if (r_k > 0 && mode == 1) return fail("expand_first_attention has no key-side low-rank variant");
  if (Lc == 0) return LORAKV_OK;
  LK_CUDA(cudaSetDevice(ctx->device));
  const int group = n_q / n_kv;
  const int64_t wq = (int64_t)n_q * d, wkv = (int64_t)n_kv * d;
  const bool extra = mode == 1 && r > 0;

  // device staging: q | k | v | vlr | b | expanded | out | stats | flag
  size_t off_q = 0, off_k = align_up(off_q + Lc * wq * sizeof(T), 256);
  size_t off_v = align_up(off_k + L * wkv * sizeof(T), 256);
  size_t off_lr = align_up(off_v + L * wkv * sizeof(T), 256);
  size_t off_b = align_up(off_lr + L * r * sizeof(T), 256);
  size_t off_ex = align_up(off_b + r * wkv * sizeof(T), 256);
  size_t off_out = align_up(off_ex + (extra ? L * wkv * sizeof(T) : 0), 256);
  size_t off_st = align_up(off_out + Lc * wq * sizeof(T), 256);
  size_t off_flag = align_up(off_st + 2 * n_q * Lc * sizeof(T), 256);
  size_t off_lk = align_up(off_flag + 256, 256);
  size_t off_bk = align_up(off_lk + L * r_k * sizeof(T), 256);
  size_t off_qk = align_up(off_bk + r_k * wkv * sizeof(T), 256);
  size_t total = off_qk + Lc * n_q * r_k * sizeof(T) + 256;
  LK_TRY(scratch_reserve(ctx, ctx->in, total));
  char* base = static_cast<char*>(ctx->in.ptr);
  T* dq = reinterpret_cast<T*>(base + off_q);
  T* dk = reinterpret_cast<T*>(base + off_k);
  T* dv = reinterpret_cast<T*>(base + off_v);
  T* dlr = reinterpret_cast<T*>(base + off_lr);
  T* db = reinterpret_cast<T*>(base + off_b);
  T* dex = reinterpret_cast<T*>(base + off_ex);
  T* dout = reinterpret_cast<T*>(base + off_out);
  T* dst = reinterpret_cast<T*>(base + off_st);
  int* dflag = reinterpret_cast<int*>(base + off_flag);
  LK_TRY(upload2d(ctx, dq, q, Lc, wq, ldq));
  LK_TRY(upload2d(ctx, dk, k, L, wkv, ldk));
  LK_TRY(upload2d(ctx, dv, v, L, wkv, ldv));
  if (r > 0) {
    LK_TRY(upload2d(ctx, dlr, vlr, L, r, ldlr));
    LK_TRY(upload2d(ctx, db, b, r, wkv, ldb));
  }
  const int init_flag = 0x7fffffff;
  LK_CUDA(cudaMemcpyAsync(dflag, &init_flag, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  T* dlk = reinterpret_cast<T*>(base + off_lk);
  T* dbk = reinterpret_cast<T*>(base + off_bk);
  T* dqk = reinterpret_cast<T*>(base + off_qk);
  if (r_k > 0) {
    LK_TRY(upload2d(ctx, dlk, key->l_k, L, r_k, key->ld_lk));
    LK_TRY(upload2d(ctx, dbk, key->b_k, r_k, wkv, key->ld_bk));
    const int64_t n = Lc * n_q * r_k;
    qk_generic_kernel<T><<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(dq, wq, dbk, wkv, key->k_scale, Lc, n_q, group, d, r_k, dqk);
    ctx->launches++;
  }

  if (extra) {
    const int64_t n = L * wkv;
    expand_lr_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(dlr, r, db, wkv,
                                                                              lr_scale, L, wkv, r, dex);
    ctx->launches++;
  }

  // split the key range so that short query blocks still fill the machine
  // (the decomposition depends only on the keys some row can see, so rows hidden behind the
  // causal boundary never change a single rounding: test_attention.cpp:144-175)
  const int64_t warps = Lc * n_q;
  const int64_t visible = off + Lc;
  int splits = (int)((ctx->sm_count * 16 + warps - 1) / warps);
  const int max_splits = (int)((visible + 255) / 256);
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  int64_t chunk = (visible + splits - 1) / splits;
  chunk = (chunk + 31) / 32 * 32;
  splits = (int)((visible + chunk - 1) / chunk);
  if (splits < 1) splits = 1;

  const int64_t r_part = mode == 1 ? 0 : r;
  const int64_t part_stride = 2 + d + r_part + (extra ? d : 0);
  LK_TRY(scratch_reserve(ctx, ctx->work, (size_t)(warps * splits * part_stride) * sizeof(T)));

  GenericArgs<T> ga;
  ga.q = dq; ga.k = dk; ga.v = dv; ga.vlr = mode == 1 ? nullptr : dlr; ga.extra = extra ? dex : nullptr;
  ga.ldq = wq; ga.ldk = wkv; ga.ldv = wkv; ga.ldlr = r; ga.ldextra = wkv;
  ga.Lc = Lc; ga.L = L; ga.d = d; ga.r = r_part; ga.query_offset = off;
  ga.n_heads = n_q; ga.group = group; ga.splits = splits; ga.chunk = chunk;
  ga.part = static_cast<T*>(ctx->work.ptr); ga.part_stride = part_stride;
  ga.lk = r_k > 0 ? dlk : nullptr; ga.qk = r_k > 0 ? dqk : nullptr; ga.r_k = r_k;
  dim3 grid((unsigned)((Lc + kWarps - 1) / kWarps), (unsigned)n_q, (unsigned)splits);
  const size_t smem = kWarps * (d + r_k) * sizeof(T);
  if (extra) fla_generic_partial<T, true><<<grid, kWarps * 32, smem, ctx->stream>>>(ga);
  else fla_generic_partial<T, false><<<grid, kWarps * 32, smem, ctx->stream>>>(ga);
  ctx->launches++;

  MergeArgs<T> ma;
  ma.part = ga.part; ma.part_stride = part_stride; ma.splits = splits;
  ma.Lc = Lc; ma.d = d; ma.r = r_part; ma.n_heads = n_q; ma.group = group;
  ma.b_up = (mode == 0 && r > 0) ? db : nullptr; ma.ldb = wkv; ma.lr_scale = lr_scale;
  ma.extra = extra; ma.out = dout;
  ma.row_max = (row_max || row_denom) ? dst : nullptr;
  ma.row_denom = (row_max || row_denom) ? dst + n_q * Lc : nullptr;
  ma.bad_row = dflag;
  fla_generic_merge<T><<<dim3((unsigned)Lc, (unsigned)n_q), 128, (splits + r_part + 1) * sizeof(T),
                         ctx->stream>>>(ma);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());

  int flag = 0;
  LK_CUDA(cudaMemcpyAsync(out, dout, Lc * wq * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  if (row_max)
    LK_CUDA(cudaMemcpyAsync(row_max, dst, n_q * Lc * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  if (row_denom)
    LK_CUDA(cudaMemcpyAsync(row_denom, dst + n_q * Lc, n_q * Lc * sizeof(T), cudaMemcpyDeviceToHost,
                            ctx->stream));
  LK_CUDA(cudaMemcpyAsync(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->last_kernel = "fla_generic";
  if (flag != 0x7fffffff) return fail("%s: zero softmax denominator at row %d", op, flag);
  return finite_or_fail(out, Lc * wq, op);
}

template <class T>
int naive_forward(lorakv_ctx* ctx, const T* q, int64_t ldq, const T* k, int64_t ldk, const T* v,
                  int64_t ldv, const T* vlr, int64_t ldlr, const T* b, int64_t ldb, T lr_scale,
                  int64_t Lc, int64_t L, int64_t d, int64_t r, int64_t off, T* out) {
  if (!ctx) return fail("naive_attention: null context");
  if (Lc < 0 || L < 0 || d < 1 || r < 0) return fail("naive_attention: invalid shape");
  if (off < 0 || off + Lc > L)
    return fail("attention: query_offset %lld with L_c %lld exceeds L %lld", (long long)off,
                (long long)Lc, (long long)L);
  if (Lc == 0) return LORAKV_OK;
  LK_CUDA(cudaSetDevice(ctx->device));
  size_t o_q = 0, o_k = align_up(Lc * d * sizeof(T), 256);
  size_t o_v = align_up(o_k + L * d * sizeof(T), 256);
  size_t o_lr = align_up(o_v + L * d * sizeof(T), 256);
  size_t o_b = align_up(o_lr + L * r * sizeof(T), 256);
  size_t o_ex = align_up(o_b + r * d * sizeof(T), 256);
  size_t o_val = align_up(o_ex + L * d * sizeof(T), 256);
  size_t o_s = align_up(o_val + L * d * sizeof(T), 256);
  size_t o_out = align_up(o_s + Lc * L * sizeof(T), 256);
  LK_TRY(scratch_reserve(ctx, ctx->in, o_out + Lc * d * sizeof(T)));
  char* base = static_cast<char*>(ctx->in.ptr);
  T *dq = (T*)(base + o_q), *dk = (T*)(base + o_k), *dv = (T*)(base + o_v), *dlr = (T*)(base + o_lr),
    *db = (T*)(base + o_b), *dex = (T*)(base + o_ex), *dval = (T*)(base + o_val), *ds = (T*)(base + o_s),
    *dout = (T*)(base + o_out);
  LK_TRY(upload2d(ctx, dq, q, Lc, d, ldq));
  LK_TRY(upload2d(ctx, dk, k, L, d, ldk));
  LK_TRY(upload2d(ctx, dv, v, L, d, ldv));
  if (r > 0) {
    LK_TRY(upload2d(ctx, dlr, vlr, L, r, ldlr));
    LK_TRY(upload2d(ctx, db, b, r, d, ldb));
    expand_lr_kernel<T><<<(unsigned)((L * d + 255) / 256), 256, 0, ctx->stream>>>(dlr, r, db, d, lr_scale,
                                                                                  L, d, r, dex);
    ctx->launches++;
  }
  naive_scores_kernel<T><<<(unsigned)((Lc * L + 255) / 256), 256, 0, ctx->stream>>>(dq, d, dk, d, Lc, L, d,
                                                                                    off, ds);
  naive_softmax_kernel<T><<<(unsigned)Lc, 256, 0, ctx->stream>>>(ds, L);
  naive_value_kernel<T><<<(unsigned)((L * d + 255) / 256), 256, 0, ctx->stream>>>(dv, d, r > 0 ? dex : nullptr,
                                                                                  L, d, dval);
  naive_pv_kernel<T><<<(unsigned)((Lc * d + 255) / 256), 256, 0, ctx->stream>>>(ds, dval, Lc, L, d, dout);
  ctx->launches += 4;
  LK_CUDA(cudaGetLastError());
  LK_CUDA(cudaMemcpyAsync(out, dout, Lc * d * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->last_kernel = "naive_materialising";
  return finite_or_fail(out, Lc * d, "naive_attention");
}

template int generic_forward<float>(lorakv_ctx*, const char*, int, const float*, int64_t, const float*,
                                    int64_t, const float*, int64_t, const float*, int64_t, const float*,
                                    int64_t, float, int64_t, int64_t, int, int, int64_t, int64_t, int64_t,
                                    float*, float*, float*, const KeyLowRank<float>*);
template int generic_forward<double>(lorakv_ctx*, const char*, int, const double*, int64_t, const double*,
                                     int64_t, const double*, int64_t, const double*, int64_t,
                                     const double*, int64_t, double, int64_t, int64_t, int, int, int64_t,
                                     int64_t, int64_t, double*, double*, double*, const KeyLowRank<double>*);
template int naive_forward<float>(lorakv_ctx*, const float*, int64_t, const float*, int64_t, const float*,
                                  int64_t, const float*, int64_t, const float*, int64_t, float, int64_t,
                                  int64_t, int64_t, int64_t, int64_t, float*);
template int naive_forward<double>(lorakv_ctx*, const double*, int64_t, const double*, int64_t,
                                   const double*, int64_t, const double*, int64_t, const double*, int64_t,
                                   double, int64_t, int64_t, int64_t, int64_t, int64_t, double*);

}  // namespace lk
