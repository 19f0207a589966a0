// Microbenchmark: tcgen05.mma cta_group::2 (CTA pair, M=256) issue rate, N in {128, 256}, SS operands.
#include "tc_common.cuh"
#include <cstdio>

__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) umma2_rate(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = crank();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  csync();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32 && rank == 0) {
    constexpr uint32_t id = tc::idesc_bf16_f32(256, N, 0, 0);
    const uint32_t a = smem_u32(smem), bb = smem_u32(smem + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(tc::sdesc_sw128(a + kk * 32, 16, 1024)), "l"(tc::sdesc_sw128(bb + kk * 32, 16, 1024)), "r"(id), "r"(1u)
                     : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    tc::mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  if (threadIdx.x == 32 && rank == 1) tc::mbar_wait(&bar, 0);
  tc::tc_fence_before();
  csync();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
  }
}

template <int N>
void run(long long* cyc) {
  const int iters = 2048;
  cudaFuncSetAttribute(umma2_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  umma2_rate<N><<<148, 128, 65536>>>(iters, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 256 * N * 16 * 4 * iters;  // per pair
  printf("2CTA M256 N%3d SS: %.1f cyc/instr, %.0f flops/clk per SM  (%s)\n", N, (double)h / (4 * iters),
         flops / h / 2, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<128>(cyc); run<256>(cyc);
  return 0;
}
