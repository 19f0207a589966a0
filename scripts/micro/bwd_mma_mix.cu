// Microbenchmark: the attention-backward per-tile MMA sequence in isolation (no compute warps):
//   dV (TS, N=64) x8, S (TS, N=128) x4, dK (TS, N=64) x8, dP (TS, N=128) x4, dQ (SS, N=64, A MN-major) x8
#include "tc_common.cuh"
#include <cstdio>

template <int VAR>
__global__ void __launch_bounds__(128, 1) mix(int iters, long long* cyc, int random_data) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[5];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) { tc::mbar_init(&bar, 1); for (int i = 0; i < 5; ++i) tc::mbar_init(&bar2[i], 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (random_data) {
    // bf16 values ~N(0,1)-ish in every operand (smem tiles and the TMEM A regions)
    uint32_t st = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
    auto rnd = [&]() { st ^= st << 13; st ^= st >> 17; st ^= st << 5; return st; };
    uint32_t* sm = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) sm[i] = (rnd() & 0x807F807Fu) | 0x3F003F00u;
    tc::fence_proxy_async();
    uint32_t r[32];
    for (int col = 0; col < 512; col += 32) {
#pragma unroll
      for (int e = 0; e < 32; ++e) r[e] = (rnd() & 0x807F807Fu) | 0x3F003F00u;
      tc::tmem_st_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + col, r);
    }
    tc::tmem_st_wait();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
  }
  if (threadIdx.x == 32) {
    const uint32_t tST = tmem, tDPT = tmem + 128, tDV = tmem + 256, tDK = tmem + 320, tDQ = tmem + 384, tK = tmem + 448,
                   tV = tmem + 480;
    constexpr uint32_t idSS = tc::idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t idG = tc::idesc_bf16_f32(128, 64, 0, 1);
    constexpr uint32_t idQ = tc::idesc_bf16_f32(128, 64, 1, 1);
    const uint32_t aQ = smem_u32(smem), aDO = aQ + 16384, aDS = aQ + 32768, aK = aQ + 65536;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (VAR == 0 || VAR == 1) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::umma_f16_ts(tDV, tST + 32 * (kk >> 1) + 8 * (kk & 1), tc::sdesc_sw128(aDO + kk * 2048, 8192, 1024), idG, 1u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::umma_f16_ts(tST, tK + 8 * kk, tc::sdesc_sw128(aQ + kk * 32, 16, 1024), idSS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::umma_f16_ts(tDK, tDPT + 32 * (kk >> 1) + 8 * (kk & 1), tc::sdesc_sw128(aQ + kk * 2048, 8192, 1024), idG, 1u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::umma_f16_ts(tDPT, tV + 8 * kk, tc::sdesc_sw128(aDO + kk * 32, 16, 1024), idSS, kk > 0);
      }
      if (VAR == 3) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::umma_f16_ts(tDV, tST + 32 * (kk >> 1) + 8 * (kk & 1), tc::sdesc_sw128(aDO + kk * 2048, 8192, 1024), idG, 1u);
        tc::umma_commit(&bar2[0]);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::umma_f16_ts(tST, tK + 8 * kk, tc::sdesc_sw128(aQ + kk * 32, 16, 1024), idSS, kk > 0);
        tc::umma_commit(&bar2[1]);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::umma_f16_ts(tDK, tDPT + 32 * (kk >> 1) + 8 * (kk & 1), tc::sdesc_sw128(aQ + kk * 2048, 8192, 1024), idG, 1u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::umma_f16_ts(tDPT, tV + 8 * kk, tc::sdesc_sw128(aDO + kk * 32, 16, 1024), idSS, kk > 0);
        tc::umma_commit(&bar2[2]);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::umma_f16_ss(tDQ, tc::sdesc_sw128(aDS + kk * 2048, 16384, 1024), tc::sdesc_sw128(aK + kk * 2048, 8192, 1024), idQ, kk > 0);
        tc::umma_commit(&bar2[3]);
        tc::umma_commit(&bar2[4]);
        tc::tc_fence_after();
      }
      if (VAR == 0 || VAR == 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::umma_f16_ss(tDQ, tc::sdesc_sw128(aDS + kk * 2048, 16384, 1024), tc::sdesc_sw128(aK + kk * 2048, 8192, 1024), idQ, kk > 0);
      }
    }
    tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 512); }
}

template <int VAR>
void run(long long* cyc, const char* name, int rnd = 0) {
  const int iters = 1024;
  cudaFuncSetAttribute(mix<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  mix<VAR><<<148, 128, 131072>>>(iters, cyc, rnd);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %.0f cycles per tile step (%s)\n", name, (double)h / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<0>(cyc, "full mix (dV,S,dK,dP TS + dQ SS MN-major)");
  run<1>(cyc, "dV,S,dK,dP (TS) only");
  run<2>(cyc, "dQ (SS, A MN-major) only");
  run<0>(cyc, "full mix, random bf16 operands", 1);
  run<3>(cyc, "full mix + 5 commits + fences per step");
  run<1>(cyc, "dV,S,dK,dP (TS), random operands", 1);
  return 0;
}
