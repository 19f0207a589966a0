// Microbenchmark: TMEM read (tcgen05.ld) and write (tcgen05.st) bandwidth per SM on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2309_16669_b200/csrc tmem_bw.cu -lcuda
#include "tc_common.cuh"
#include <cstdio>

__global__ void __launch_bounds__(512, 1) tmem_rd(int iters, int nwarps_active, uint32_t* sink, long long* cyc, int mode) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < nwarps_active) {
    const uint32_t col = (warp >> 2) * 32 % 512;
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      if (mode == 0) {
        tc::tmem_ld_32x32b_x32(tmem + lane_off + col, r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= r[e];
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = acc + e + it;
        tc::tmem_st_32x32b_x32(tmem + lane_off + col, r);
        tc::tmem_st_wait();
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678) sink[threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 512); }
}

int main() {
  uint32_t* sink; long long* cyc;
  cudaMalloc(&sink, 4096); cudaMalloc(&cyc, 148 * 8);
  for (int mode = 0; mode < 2; ++mode)
  for (int nw : {4, 8, 16}) {
    const int iters = 4096;
    tmem_rd<<<148, 512>>>(iters, nw, sink, cyc, mode);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = (double)nw * 32 * 32 * 4 * iters;  // per CTA (= per SM)
    printf("%s warps=%2d: %.1f B/clk/SM (cycles %lld) err=%s\n", mode ? "tcgen05.st" : "tcgen05.ld", nw, bytes / h[0], h[0],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
