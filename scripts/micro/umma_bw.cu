// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1) issue rate for SS and TS operand modes at
// M=128, N in {64,128,256}, K=16 per instruction -- shows whether smem operand reads bound the MMA.
#include "tc_common.cuh"
#include <cstdio>

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) umma_rate(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 32) {
    constexpr uint32_t id = tc::idesc_bf16_f32(128, N, 0, 0);
    const uint32_t a = smem_u32(smem), bb = smem_u32(smem + 16384);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          tc::umma_f16_ts(tmem, tmem + 256 + kk * 8, tc::sdesc_sw128(bb + kk * 32, 16, 1024), id, 1u);
        else
          tc::umma_f16_ss(tmem, tc::sdesc_sw128(a + kk * 32, 16, 1024), tc::sdesc_sw128(bb + kk * 32, 16, 1024), id, 1u);
      }
    }
    tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 512); }
}

template <int N, bool TS>
void run(long long* cyc) {
  const int iters = 2048;
  cudaFuncSetAttribute(umma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  umma_rate<N, TS><<<148, 128, 65536>>>(iters, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 16 * 4 * iters;
  printf("M128 N%3d %s: %.1f cyc/instr, %.0f flops/clk/SM, smem operand B/clk %.0f  (%s)\n", N, TS ? "TS" : "SS",
         (double)h / (4 * iters), flops / h, (TS ? 0 : 128 * 16 * 2.0) / ((double)h / (4 * iters)) + N * 16 * 2.0 / ((double)h / (4 * iters)),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<64, false>(cyc); run<128, false>(cyc); run<256, false>(cyc);
  run<64, true>(cyc); run<128, true>(cyc); run<256, true>(cyc);
  return 0;
}
