// K6: LayerNorm forward/backward over [M, D] bf16 rows (HBM-bound), fp32 statistics.
// Pre-LN ViT blocks (no reference code).
//
// One warp per row; lane l owns columns {l*8 + k*256 + 0..7}, k < NC = ceil(D/256), so every
// access is a 16-byte vector.  Rows are kept as packed bf16 (4 registers per 8 columns) and
// re-expanded on use, so a warp keeps two rows in flight.  The backward fuses the residual-
// stream accumulation (dx += LN'(dy)) and reduces dgamma/dbeta per block in shared memory before
// one atomic per column per block.
#include "common.cuh"

#include <algorithm>

namespace {

__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 v = __bfloat1622float2(h[e]);
    f[2 * e] = v.x;
    f[2 * e + 1] = v.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 q;
  q.x = pack_bf16x2(f[0], f[1]);
  q.y = pack_bf16x2(f[2], f[3]);
  q.z = pack_bf16x2(f[4], f[5]);
  q.w = pack_bf16x2(f[6], f[7]);
  return q;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

template <int NC>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                                     __nv_bfloat16* __restrict__ y, int64_t ldy, float* __restrict__ mean,
                                                     float* __restrict__ rstd, int M, int D, float eps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < M; row += nwarps) {
    uint4 raw[NC];
    bool ok[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      ok[k] = k * 256 + lane * 8 < D;
      raw[k] = ok[k] ? *reinterpret_cast<const uint4*>(x + row * ldx + k * 256 + lane * 8) : make_uint4(0, 0, 0, 0);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      float f[8];
      unpack8(raw[k], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += f[e];
    }
    const float mu = warp_sum(s) / D;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      float f[8];
      unpack8(raw[k], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = f[e] - mu;
        q += d * d;
      }
    }
    const float rs = rsqrtf(warp_sum(q) / D + eps);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      const int c = k * 256 + lane * 8;
      float f[8];
      unpack8(raw[k], f);
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + c));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + c + 4));
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = (f[e] - mu) * rs * gg[e] + bb[e];
      *reinterpret_cast<uint4*>(y + row * ldy + c) = pack8(f);
    }
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
  }
}

template <int NC, bool SUM>
__global__ void __launch_bounds__(256, (NC <= 3 ? 2 : 1)) ln_bwd_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy,
                                                     const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ gamma, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, __nv_bfloat16* dx, int64_t lddx,
                                                     float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                     float* __restrict__ dsum, int M, int D, int accumulate) {
  extern __shared__ float red[];  // [3][D]: dgamma, dbeta, column sums of the output dx
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * D; i += blockDim.x) red[i] = 0.f;
  __syncthreads();
  float dg[NC][8], db[NC][8], cs[NC][8];
#pragma unroll
  for (int k = 0; k < NC; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) dg[k][e] = db[k][e] = cs[k][e] = 0.f;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < M; row += nwarps) {
    const float mu = mean[row], rs = rstd[row];
    // every load of the row (x, dy and the residual-stream gradient dx) issued up front: one
    // memory round trip per row instead of two (the dx read does not depend on the row sums)
    uint4 rx[NC], rd[NC], rp[NC];
    bool ok[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = k * 256 + lane * 8;
      ok[k] = c < D;
      rx[k] = ok[k] ? *reinterpret_cast<const uint4*>(x + row * ldx + c) : make_uint4(0, 0, 0, 0);
      rd[k] = ok[k] ? *reinterpret_cast<const uint4*>(dy + row * lddy + c) : make_uint4(0, 0, 0, 0);
      rp[k] = (ok[k] && accumulate) ? *reinterpret_cast<const uint4*>(dx + row * lddx + c) : make_uint4(0, 0, 0, 0);
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      const int c = k * 256 + lane * 8;
      float xv[8], dv[8];
      unpack8(rx[k], xv);
      unpack8(rd[k], dv);
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
      const float gm[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (xv[e] - mu) * rs;
        const float g = dv[e] * gm[e];
        s1 += g;
        s2 += g * xh;
        dg[k][e] += dv[e] * xh;
        db[k][e] += dv[e];
      }
    }
    const float m1 = warp_sum(s1) / D, m2 = warp_sum(s2) / D;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      const int c = k * 256 + lane * 8;
      float xv[8], dv[8], pv[8], o[8];
      unpack8(rx[k], xv);
      unpack8(rd[k], dv);
      unpack8(rp[k], pv);
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
      const float gm[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (xv[e] - mu) * rs;
        o[e] = rs * (dv[e] * gm[e] - m1 - xh * m2) + pv[e];
      }
      const uint4 q = pack8(o);
      *reinterpret_cast<uint4*>(dx + row * lddx + c) = q;
      if (SUM) {
        float ob[8];
        unpack8(q, ob);   // sum what was stored (bf16), like a separate column-sum pass would
#pragma unroll
        for (int e = 0; e < 8; ++e) cs[k][e] += ob[e];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = k * 256 + lane * 8;
    if (c < D) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        atomicAdd(&red[c + e], dg[k][e]);
        atomicAdd(&red[D + c + e], db[k][e]);
        if (SUM) atomicAdd(&red[2 * D + c + e], cs[k][e]);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    if (dgamma) atomicAdd(dgamma + i, red[i]);
    if (dbeta) atomicAdd(dbeta + i, red[D + i]);
    if (SUM) atomicAdd(dsum + i, red[2 * D + i]);
  }
}

template <typename F>
int dispatch_nc(int D, F&& f) {
  const int nc = (D + 255) / 256;
  switch (nc) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    default: return f(std::integral_constant<int, 4>{});
  }
}

}  // namespace

extern "C" int avb_layernorm_fwd(const void* x, int64_t ldx, const float* gamma, const float* beta, void* y,
                                 int64_t ldy, float* mean, float* rstd, int M, int D, float eps, void* stream) {
  AVB_CHECK_ARG(M >= 0 && D >= 8 && D <= 1024 && D % 8 == 0, "LayerNorm needs D % 8 == 0, D <= 1024");
  if (M == 0) return AVB_OK;
  AVB_CHECK_ARG(x && gamma && beta && y && mean && rstd, "null pointer");
  AVB_CHECK_ARG(ldx % 8 == 0 && ldy % 8 == 0, "row strides must be multiples of 8");
  const int blocks = (int)std::min<int64_t>((M + 7) / 8, (int64_t)avb::sm_count() * 8);
  return dispatch_nc(D, [&](auto nc) {
    ln_fwd_kernel<decltype(nc)::value><<<blocks, 256, 0, avb::as_stream(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), ldx, gamma, beta, reinterpret_cast<__nv_bfloat16*>(y), ldy, mean,
        rstd, M, D, eps);
    return avb::launch_status("avb_layernorm_fwd");
  });
}

extern "C" int avb_layernorm_bwd(const void* dy, int64_t lddy, const void* x, int64_t ldx, const float* gamma,
                                 const float* mean, const float* rstd, void* dx, int64_t lddx, float* dgamma,
                                 float* dbeta, float* dx_colsum, int M, int D, int accumulate, void* stream) {
  AVB_CHECK_ARG(M >= 0 && D >= 8 && D <= 1024 && D % 8 == 0, "LayerNorm needs D % 8 == 0, D <= 1024");
  if (M == 0) return AVB_OK;
  AVB_CHECK_ARG(dy && x && gamma && mean && rstd && dx, "null pointer");
  AVB_CHECK_ARG(lddy % 8 == 0 && ldx % 8 == 0 && lddx % 8 == 0, "row strides must be multiples of 8");
  const int blocks = (int)std::min<int64_t>((M + 7) / 8, (int64_t)avb::sm_count() * 2);
  return dispatch_nc(D, [&](auto nc) {
    constexpr int NCv = decltype(nc)::value;
    if (dx_colsum)
      ln_bwd_kernel<NCv, true><<<blocks, 256, 3 * D * sizeof(float), avb::as_stream(stream)>>>(
          reinterpret_cast<const __nv_bfloat16*>(dy), lddy, reinterpret_cast<const __nv_bfloat16*>(x), ldx, gamma,
          mean, rstd, reinterpret_cast<__nv_bfloat16*>(dx), lddx, dgamma, dbeta, dx_colsum, M, D, accumulate);
    else
      ln_bwd_kernel<NCv, false><<<blocks, 256, 3 * D * sizeof(float), avb::as_stream(stream)>>>(
          reinterpret_cast<const __nv_bfloat16*>(dy), lddy, reinterpret_cast<const __nv_bfloat16*>(x), ldx, gamma,
          mean, rstd, reinterpret_cast<__nv_bfloat16*>(dx), lddx, dgamma, dbeta, nullptr, M, D, accumulate);
    return avb::launch_status("avb_layernorm_bwd");
  });
}
