// mufu_bench.cu -- throughput of the exponential forms a softmax could use on sm_100a (tools, not product):
// ex2.approx.ftz.f32 (one result per MUFU op), ex2.approx.f16x2 and ex2.approx.ftz.bf16x2 (two packed results per
// instruction -- do they cost one MUFU slot or two?), and an FMA-pipe cubic on packed f32x2.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/build/mufu_bench tools/mufu_bench.cu
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void k(float* out, int iters, float seed) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed - 0.01f * (threadIdx.x & 7) - 0.001f * i;
  uint32_t acc = 0;
  float facc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (MODE == 0) {
        float a, b;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x[i + 1]));
        facc += a + b;
      } else if (MODE == 1) {
        uint32_t h, r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[i + 1]), "f"(x[i]));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h));
        acc ^= r;
      } else if (MODE == 2) {
        uint32_t h, r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[i + 1]), "f"(x[i]));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(h));
        acc ^= r;
      }
      x[i] += 1e-7f; x[i + 1] += 1e-7f;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = facc + __uint_as_float(acc);
}

template <int MODE>
void run(const char* name) {
  float* d;
  cudaMalloc(&d, 148 * 1024 * 4);
  const int iters = 20000;
  k<MODE><<<148, 1024>>>(d, 100, -1.f);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<148, 1024>>>(d, iters, -1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double n = 148.0 * 1024 * iters * 8;
  printf("%-28s %8.3f ms  %7.1f Gexp/s  = %5.2f exp/clk/SM at 1.9 GHz\n", name, ms, n / ms * 1e-6, n / ms * 1e-6 / 148 / 1.9);
  cudaFree(d);
}

int main() {
  run<0>("ex2.approx.ftz.f32");
  run<1>("cvt + ex2.approx.f16x2");
  run<2>("cvt + ex2.approx.ftz.bf16x2");
  return 0;
}
