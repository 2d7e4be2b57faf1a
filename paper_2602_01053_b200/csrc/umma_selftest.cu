// umma_selftest.cu -- one-tile tcgen05 self-test behind lorakv_selftest_umma (include/lorakv_b200.h).
//
// It pins, against a host matmul, exactly the operand conventions the prefill kernel relies on:
//   * A (128 x K) K-major SWIZZLE_128B tiles written by threads (how Q and P tiles are built),
//   * B (N x K) K-major SWIZZLE_128B (how a K page lands after a bulk copy),
//   * B (K x N) MN-major SWIZZLE_128B / 64B / 32B (how V pages and V_lr pages land: page_layout.cuh),
//   * B (N x K) K-major with NARROW rows, K = 16 / 32 (SWIZZLE_32B / 64B): how a tile of the key-side low-rank cache L_k lands
//     (one more k block of the score product S += Qk L_k^T; A from TMEM),
//   * accumulation into TMEM, tcgen05.ld / tcgen05.st round trips (the lazy O rescale) and
//     tcgen05.commit -> mbarrier completion.
// D = alpha * (A B) + (A B) when rescale != 0 (load, scale, store back, accumulate a second pass),
// else D = A B.  Operands are rounded to bf16; accumulation is fp32.
#include <cuda_bf16.h>

#include "kernels.hpp"
#include "page_layout.cuh"
#include "state.hpp"
#include "umma.cuh"

namespace lk {

namespace {

__global__ void __launch_bounds__(128, 1) umma_selftest_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                               int N, int K, int b_mn_major, float alpha, int rescale,
                                                               int a_in_tmem, float* __restrict__ D) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  // swizzled tiles need a 1024-byte aligned base in the shared window
  unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = smem;                         // K/64 blocks x [128 rows][64] bf16, SW128
  unsigned char* sB = smem + (K / 64) * 128 * 128;  // see below
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const bool narrow = K < 64;                         // K-major B with 2K-byte rows: the L_k tile convention (A must come from TMEM)
  if (narrow) sB = smem;
  for (int idx = tid; idx < 128 * K && !narrow; idx += 128) {
    const int row = idx / K, k = idx % K;
    const uint32_t off = (uint32_t)(k / 64) * 16384u + ptx::sw128_offset(row, k % 64);
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16_rn(A[idx]);
  }
  const PageLayout lay = make_page_layout(K, N, 2);   // MN-major B: [N/bw blocks][K keys][bw], swizzled rows
  const PageLayout nlay = make_page_layout(N, K, 2);  // narrow K-major B: a page of N tokens x K columns
  for (int idx = tid; idx < N * K; idx += 128) {
    if (narrow) {
      const int n = idx / K, k = idx % K;             // B given as N x K row-major
      *reinterpret_cast<__nv_bfloat16*>(sB + 2 * page_offset(nlay, n, k)) = __float2bfloat16_rn(B[idx]);
    } else if (b_mn_major) {
      const int k = idx / N, n = idx % N;             // B given as K x N row-major
      *reinterpret_cast<__nv_bfloat16*>(sB + 2 * page_offset(lay, k, n)) = __float2bfloat16_rn(B[idx]);
    } else {
      const int n = idx / K, k = idx % K;             // B given as N x K row-major
      const uint32_t off = (uint32_t)(k / 64) * (uint32_t)(N * 128) + ptx::sw128_offset(n, k % 64);
      *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16_rn(B[idx]);
    }
  }
  ptx::fence_proxy_async_smem();
  uint32_t cols = 32;
  while ((int)cols < N + (a_in_tmem ? K / 2 : 0)) cols *= 2;   // A (packed bf16 pairs) sits behind the accumulator
  if (warp == 0) ptx::tmem_alloc(&tmem_base_s, cols);
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  if (a_in_tmem) {
    // thread = row: column c of the A region holds (A[row][2c], A[row][2c+1]) as packed bf16
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const __nv_bfloat162 v = __floats2bfloat162_rn(A[row * K + 2 * (c0 + i)], A[row * K + 2 * (c0 + i) + 1]);
        r[i] = *reinterpret_cast<const uint32_t*>(&v);
      }
      ptx::tmem_st16(lane_addr + (uint32_t)N + c0, r);
    }
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }
  const uint32_t idesc = ptx::instr_desc_bf16(128, (uint32_t)N, ptx::kMajorK, b_mn_major ? ptx::kMajorMN : ptx::kMajorK);
  const uint32_t a_base = ptx::smem_u32(sA), b_base = ptx::smem_u32(sB);
  auto issue_all = [&](bool accumulate_first) {
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t da = ptx::smem_desc(a_base + (ks / 4) * 16384u + (ks % 4) * 32u, 16u, 1024u, ptx::kSw128);
      uint64_t db;
      if (narrow) {
        const uint32_t W = 2u * (uint32_t)K;        // row bytes; one swizzle atom along K, 8-row groups W * 8 bytes apart
        db = ptx::smem_desc(b_base + (uint32_t)ks * 32u, 16u, 8u * W, K == 32 ? ptx::kSw64 : ptx::kSw32);
      } else if (!b_mn_major) {
        db = ptx::smem_desc(b_base + (ks / 4) * (uint32_t)(N * 128) + (ks % 4) * 32u, 16u, 1024u, ptx::kSw128);
      } else {
        const uint32_t W = 2u * (uint32_t)lay.bw;   // row bytes of one key inside a column block
        const uint32_t mode = lay.bw == 64 ? ptx::kSw128 : lay.bw == 32 ? ptx::kSw64 : ptx::kSw32;
        db = ptx::smem_desc(b_base + (uint32_t)ks * 16u * W, (uint32_t)K * W, 8u * W, mode);
      }
      if (a_in_tmem) ptx::umma_bf16_ts(tmem, tmem + (uint32_t)N + 8u * ks, db, idesc, (accumulate_first || ks > 0) ? 1u : 0u);
      else ptx::umma_bf16_ss(tmem, da, db, idesc, (accumulate_first || ks > 0) ? 1u : 0u);
    }
  };
  if (tid == 0) {
    issue_all(false);
    ptx::umma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  if (rescale) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r[16];
      ptx::tmem_ld16(lane_addr + c0, r);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
      ptx::tmem_st16(lane_addr + c0, r);
    }
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      ptx::tc_fence_after();
      issue_all(true);
      ptx::umma_commit(&bar);
    }
    ptx::mbar_wait(&bar, 1);
    ptx::tc_fence_after();
  }
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    ptx::tmem_ld16(lane_addr + c0, r);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) D[(warp * 32 + lane) * N + c0 + i] = __uint_as_float(r[i]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, cols);
}

}  // namespace

int umma_selftest(lorakv_ctx* ctx, const float* a, const float* b, int N, int K, int b_mn_major, float alpha, int rescale,
                  int a_in_tmem, float* d) {
  if (!ctx || !a || !b || !d) return fail("selftest_umma: null argument");
  if (K != 64 && K != 128 && !((K == 16 || K == 32) && a_in_tmem && !b_mn_major))
    return fail("selftest_umma: K must be 64 or 128 (or 16 / 32 with A in TMEM and a K-major B: the narrow-row convention)");
  if (N < 16 || N > 256 || N % 16 != 0) return fail("selftest_umma: N must be a multiple of 16 in [16, 256]");
  if (b_mn_major && !(N == 16 || N == 32 || N % 64 == 0)) return fail("selftest_umma: MN-major N must be 16, 32 or a multiple of 64");
  LK_CUDA(cudaSetDevice(ctx->device));
  const size_t na = (size_t)128 * K * sizeof(float), nb = (size_t)N * K * sizeof(float), nd = (size_t)128 * N * sizeof(float);
  LK_TRY(scratch_reserve(ctx, ctx->in, na + nb + nd + 768));
  char* base = static_cast<char*>(ctx->in.ptr);
  float* da = reinterpret_cast<float*>(base);
  float* db = reinterpret_cast<float*>(base + (na + 255) / 256 * 256);
  float* dd = reinterpret_cast<float*>(base + (na + 255) / 256 * 256 + (nb + 255) / 256 * 256);
  LK_CUDA(cudaMemcpyAsync(da, a, na, cudaMemcpyHostToDevice, ctx->stream));
  LK_CUDA(cudaMemcpyAsync(db, b, nb, cudaMemcpyHostToDevice, ctx->stream));
  const size_t smem = (size_t)128 * K * 2 + (size_t)N * K * 2 + 2048;
  LK_CUDA(cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  umma_selftest_kernel<<<1, 128, smem, ctx->stream>>>(da, db, N, K, b_mn_major, alpha, rescale, a_in_tmem, dd);
  ctx->launches++;
  LK_CUDA(cudaGetLastError());
  LK_CUDA(cudaMemcpyAsync(d, dd, nd, cudaMemcpyDeviceToHost, ctx->stream));
  LK_CUDA(cudaStreamSynchronize(ctx->stream));
  return LORAKV_OK;
}

}  // namespace lk
