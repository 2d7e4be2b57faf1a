// linalg_kernels.cu -- device matmul behind lorakv::matmul (proj/include/lorakv/matrix.hpp:101-135),
// the triple loop the adapters use: expand_lr (lora.hpp:39-47) and forward_decomposed (lora.hpp:97-108,
// whose y_lr = x * A is the down-projection of engine.hpp:414-418).
//
// out(i,j) = sum_p a(i,p) * b(p,j) accumulated in ascending p with a separately rounded multiply and
// add -- the reference is built with -ffp-contract=off (proj/CMakeLists.txt:12-14), so this order and
// these roundings reproduce its result bit for bit (tests/test_matrix.cpp:43-50 pins 0 ULP).
#include <cmath>

#include "kernels.hpp"
#include "state.hpp"

namespace lk {

namespace {

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <class T>
__global__ void matmul_rowmajor_kernel(const T* __restrict__ a, const T* __restrict__ b, int64_t M, int64_t K,
                                       int64_t N, T* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  const int64_t i = idx / N, j = idx % N;
  T acc = T(0);
  for (int64_t p = 0; p < K; ++p) acc = add_rn(acc, mul_rn(a[i * K + p], b[p * N + j]));
  out[idx] = acc;
}

}  // namespace

template <class T>
int matmul_forward(lorakv_ctx* ctx, const T* a, int64_t lda, const T* b, int64_t ldb, int64_t M, int64_t K,
                   int64_t N, T* out) {
  if (!ctx) return fail("matmul: null context");
  if (M < 0 || K < 0 || N < 0) return fail("matmul: invalid shape");
  if (M == 0 || N == 0) return LORAKV_OK;
  LK_CUDA(cudaSetDevice(ctx->device));
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t off_b = up((size_t)(M * K) * sizeof(T)), off_o = off_b + up((size_t)(K * N) * sizeof(T));
  LK_TRY(scratch_reserve(ctx, ctx->in, off_o + (size_t)(M * N) * sizeof(T)));
  char* base = static_cast<char*>(ctx->in.ptr);
  T* da = reinterpret_cast<T*>(base);
  T* db = reinterpret_cast<T*>(base + off_b);
  T* dout = reinterpret_cast<T*>(base + off_o);
  if (K > 0) {
    LK_CUDA(cudaMemcpy2DAsync(da, K * sizeof(T), a, lda * sizeof(T), K * sizeof(T), M, cudaMemcpyHostToDevice, ctx->stream));
    LK_CUDA(cudaMemcpy2DAsync(db, N * sizeof(T), b, ldb * sizeof(T), N * sizeof(T), K, cudaMemcpyHostToDevice, ctx->stream));
  }
  const int64_t n = M * N;
  matmul_rowmajor_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(da, db, M, K, N, dout);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  LK_CUDA(cudaMemcpyAsync(out, dout, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(static_cast<double>(out[i]))) return fail("matmul produced a non-finite entry");
  return LORAKV_OK;
}

template int matmul_forward<float>(lorakv_ctx*, const float*, int64_t, const float*, int64_t, int64_t, int64_t, int64_t, float*);
template int matmul_forward<double>(lorakv_ctx*, const double*, int64_t, const double*, int64_t, int64_t, int64_t, int64_t, double*);

}  // namespace lk
