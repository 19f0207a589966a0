// Microbenchmark: throughput of ex2.approx (MUFU), cvt.rn.bf16x2.f32 (F2FP pack) and an integer
// round-to-nearest bf16 pack (IADD + PRMT on the ALU pipe), alone and mixed, 148 CTAs x 512 threads.
// Question: do MUFU.EX2 and F2FP share one pipe (the softmax's real limit in K4/K5)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t cvt2(float a, float b) {
  uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a)); return r;
}
__device__ __forceinline__ uint32_t ipack2(float a, float b) {   // round-half-up on the magnitude, then take the top halves
  const uint32_t ua = __float_as_uint(a) + 0x8000u, ub = __float_as_uint(b) + 0x8000u;
  return __byte_perm(ua, ub, 0x7632);
}

__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }

template <int MODE>
__global__ void __launch_bounds__(512, 1) xu(int iters, float seed, uint32_t* sink, long long* cyc) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed * (threadIdx.x + k) * 1e-6f - 1.f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      if (MODE == 0) { x[k] = ex2(x[k]) - 1.f; x[k + 1] = ex2(x[k + 1]) - 1.f; }                 // 2 MUFU
      if (MODE == 1) { acc += cvt2(x[k], x[k + 1]); x[k] += 1e-7f; }                                // 1 F2FP
      if (MODE == 2) { x[k] = ex2(x[k]) - 1.f; x[k + 1] = ex2(x[k + 1]) - 1.f; acc += cvt2(x[k], x[k + 1]); }  // 2 MUFU + 1 F2FP
      if (MODE == 3) { x[k] = ex2(x[k]) - 1.f; x[k + 1] = ex2(x[k + 1]) - 1.f; acc += ipack2(x[k], x[k + 1]); } // 2 MUFU + int pack
      if (MODE == 5) { uint32_t h = __float_as_uint(x[k]); h = ex2h2(h); acc += h; x[k] = __uint_as_float(h ^ 0x00010001u); }  // 1 MUFU f16x2 (2 exps)
      if (MODE == 6) { uint32_t h = __float_as_uint(x[k]); h = ex2b2(h); acc += h; x[k] = __uint_as_float(h ^ 0x00010001u); }  // 1 MUFU bf16x2 (2 exps)
      if (MODE == 4) { acc += ipack2(x[k], x[k + 1]); x[k] += 1e-7f; }                              // int pack
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc + __float_as_uint(x[0] + x[3] + x[5] + x[7]);
}

template <int MODE>
void run(const char* name, int mufu_per_pair, int pack_per_pair) {
  uint32_t* sink; long long* cyc;
  cudaMalloc(&sink, 4096); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  xu<MODE><<<148, 512>>>(iters, 1.f, sink, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double pairs = 512.0 * 4 * iters;   // per SM
  printf("%-28s %8.2f pairs/clk/SM  (MUFU %.2f/clk, packs %.2f/clk)  cycles %lld  %s\n", name, pairs / h[0],
         mufu_per_pair * pairs / h[0], pack_per_pair * pairs / h[0], h[0], cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink); cudaFree(cyc);
}

int main() {
  run<0>("ex2 x2", 2, 0);
  run<1>("cvt.rn.bf16x2 (F2FP)", 0, 1);
  run<2>("ex2 x2 + F2FP", 2, 1);
  run<3>("ex2 x2 + int pack", 2, 1);
  run<4>("int pack (IADD x2 + PRMT)", 0, 1);
  run<5>("ex2.f16x2 (2 exps/op)", 1, 0);
  run<6>("ex2.bf16x2 (2 exps/op)", 1, 0);
  return 0;
}
