// K6: LayerNorm forward/backward over [M, D] bf16 rows (HBM-bound), fp32 statistics.
// Pre-LN ViT blocks (no reference code).
//
// One warp per row; each lane owns columns {lane*8 + k*256 + 0..7} so every load is a
// 16-byte vector.  Backward fuses the residual-stream accumulation (dx += LN'(dy)) and
// reduces dgamma/dbeta per block in shared memory before one atomic per column per block.
#include "common.cuh"

#include <algorithm>

namespace {

constexpr int kMaxChunks = 4;  // D <= 1024

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 v = __bfloat1622float2(h[e]);
    f[2 * e] = v.x;
    f[2 * e + 1] = v.y;
  }
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 q;
  q.x = pack_bf16x2(f[0], f[1]);
  q.y = pack_bf16x2(f[2], f[3]);
  q.z = pack_bf16x2(f[4], f[5]);
  q.w = pack_bf16x2(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = q;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

__global__ void __launch_bounds__(256) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                                     __nv_bfloat16* __restrict__ y, int64_t ldy, float* __restrict__ mean,
                                                     float* __restrict__ rstd, int M, int D, float eps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunk = D / 256 + ((D % 256) > lane * 8 ? 1 : 0);
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < M; row += (int64_t)gridDim.x * 8) {
    float v[kMaxChunks][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k) {
      if (k < nchunk) {
        ld8(x + row * ldx + k * 256 + lane * 8, v[k]);
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[k][e];
      }
    }
    const float mu = warp_sum(s) / D;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k)
      if (k < nchunk) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = v[k][e] - mu;
          q += d * d;
        }
      }
    const float rs = rsqrtf(warp_sum(q) / D + eps);
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k)
      if (k < nchunk) {
        const int c = k * 256 + lane * 8;
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (v[k][e] - mu) * rs * __ldg(gamma + c + e) + __ldg(beta + c + e);
        st8(y + row * ldy + c, o);
      }
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
  }
}

__global__ void __launch_bounds__(256) ln_bwd_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy,
                                                     const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ gamma, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, __nv_bfloat16* dx, int64_t lddx,
                                                     float* __restrict__ dgamma, float* __restrict__ dbeta, int M, int D,
                                                     int accumulate) {
  extern __shared__ float red[];  // [2][D]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunk = D / 256 + ((D % 256) > lane * 8 ? 1 : 0);
  for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) red[i] = 0.f;
  __syncthreads();
  float dg[kMaxChunks][8], db[kMaxChunks][8];
#pragma unroll
  for (int k = 0; k < kMaxChunks; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) dg[k][e] = db[k][e] = 0.f;

  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < M; row += (int64_t)gridDim.x * 8) {
    const float mu = mean[row], rs = rstd[row];
    float xh[kMaxChunks][8], g[kMaxChunks][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k)
      if (k < nchunk) {
        const int c = k * 256 + lane * 8;
        float xv[8], dv[8];
        ld8(x + row * ldx + c, xv);
        ld8(dy + row * lddy + c, dv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[k][e] = (xv[e] - mu) * rs;
          g[k][e] = dv[e] * __ldg(gamma + c + e);
          s1 += g[k][e];
          s2 += g[k][e] * xh[k][e];
          dg[k][e] += dv[e] * xh[k][e];
          db[k][e] += dv[e];
        }
      }
    const float m1 = warp_sum(s1) / D, m2 = warp_sum(s2) / D;
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k)
      if (k < nchunk) {
        const int c = k * 256 + lane * 8;
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = rs * (g[k][e] - m1 - xh[k][e] * m2);
        if (accumulate) {
          float prev[8];
          ld8(dx + row * lddx + c, prev);
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] += prev[e];
        }
        st8(dx + row * lddx + c, o);
      }
  }
#pragma unroll
  for (int k = 0; k < kMaxChunks; ++k)
    if (k < nchunk) {
      const int c = k * 256 + lane * 8;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        atomicAdd(&red[c + e], dg[k][e]);
        atomicAdd(&red[D + c + e], db[k][e]);
      }
    }
  __syncthreads();
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    if (dgamma) atomicAdd(dgamma + i, red[i]);
    if (dbeta) atomicAdd(dbeta + i, red[D + i]);
  }
}

}  // namespace

extern "C" int avb_layernorm_fwd(const void* x, int64_t ldx, const float* gamma, const float* beta, void* y,
                                 int64_t ldy, float* mean, float* rstd, int M, int D, float eps, void* stream) {
  AVB_CHECK_ARG(M >= 0 && D >= 8 && D <= 256 * kMaxChunks && D % 8 == 0, "LayerNorm needs D % 8 == 0, D <= 1024");
  if (M == 0) return AVB_OK;
  AVB_CHECK_ARG(x && gamma && beta && y && mean && rstd, "null pointer");
  AVB_CHECK_ARG(ldx % 8 == 0 && ldy % 8 == 0, "row strides must be multiples of 8");
  const int blocks = (int)std::min<int64_t>((M + 7) / 8, (int64_t)avb::sm_count() * 16);
  ln_fwd_kernel<<<blocks, 256, 0, avb::as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), ldx, gamma, beta, reinterpret_cast<__nv_bfloat16*>(y), ldy, mean,
      rstd, M, D, eps);
  return avb::launch_status("avb_layernorm_fwd");
}

extern "C" int avb_layernorm_bwd(const void* dy, int64_t lddy, const void* x, int64_t ldx, const float* gamma,
                                 const float* mean, const float* rstd, void* dx, int64_t lddx, float* dgamma,
                                 float* dbeta, int M, int D, int accumulate, void* stream) {
  AVB_CHECK_ARG(M >= 0 && D >= 8 && D <= 256 * kMaxChunks && D % 8 == 0, "LayerNorm needs D % 8 == 0, D <= 1024");
  if (M == 0) return AVB_OK;
  AVB_CHECK_ARG(dy && x && gamma && mean && rstd && dx, "null pointer");
  AVB_CHECK_ARG(lddy % 8 == 0 && ldx % 8 == 0 && lddx % 8 == 0, "row strides must be multiples of 8");
  const int blocks = (int)std::min<int64_t>((M + 7) / 8, (int64_t)avb::sm_count() * 4);
  ln_bwd_kernel<<<blocks, 256, 2 * D * sizeof(float), avb::as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(dy), lddy, reinterpret_cast<const __nv_bfloat16*>(x), ldx, gamma, mean,
      rstd, reinterpret_cast<__nv_bfloat16*>(dx), lddx, dgamma, dbeta, M, D, accumulate);
  return avb::launch_status("avb_layernorm_bwd");
}
