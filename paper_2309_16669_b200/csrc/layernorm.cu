// K6: LayerNorm forward/backward over [M, D] bf16 rows (HBM-bound), fp32 statistics.
// Pre-LN ViT blocks (no reference code).
//
// One warp per row; lane l owns columns {l*8 + k*256 + 0..7}, k < NC = ceil(D/256), so every
// access is a 16-byte vector.  Inputs stream through a per-lane cp.async ring (rows prefetched
// S-1 ahead, see below); gamma/beta live in registers as fp32 pairs and the math runs on packed
// f32x2 instructions.  The backward fuses the residual-stream accumulation (dx += LN'(dy)); its
// dgamma/dbeta (and the optional dx column sums) are reduced in a fixed order -- warp partials,
// block partials, then the blocks in order -- so they are bit-reproducible.
#include "common.cuh"

#include <algorithm>

namespace {

// packed fp32 pairs (FFMA2 / FADD2 / FMUL2): half the FP instructions of the scalar forms
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return r;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return r;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return r;
}
__device__ __forceinline__ void unpack8x2(const uint4& q, float2 (&f)[4]) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) f[e] = make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
}
__device__ __forceinline__ uint4 pack8x2(const float2 (&f)[4]) {
  uint4 q;
  q.x = pack_bf16x2(f[0].x, f[0].y);
  q.y = pack_bf16x2(f[1].x, f[1].y);
  q.z = pack_bf16x2(f[2].x, f[2].y);
  q.w = pack_bf16x2(f[3].x, f[3].y);
  return q;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

// Per-lane software pipeline: every lane cp.async-copies its own 16-byte pieces of the rows S-1
// rows ahead into a warp-private smem ring and later reads back exactly those bytes, so a
// cp.async.wait_group is the only synchronisation (no barriers) and each warp keeps S-1 rows of
// every input in flight without spending registers on them.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

#ifndef AVB_LN_FWD_STAGES
#define AVB_LN_FWD_STAGES 4
#endif
#ifndef AVB_LN_FWD_BLOCKS
#define AVB_LN_FWD_BLOCKS 2   // 98 registers (gamma/beta pairs in registers): 2 blocks/SM, no spills
#endif
// same-box sweep at config 4 (bwd warps x stages): 8x4 0.122 ms, 12x3 0.112, 16x2 0.112, 6x5 0.155;
// fwd (stages x blocks/SM, before the f32x2 rewrite): 4x4 0.0647, 6x4 0.0651, 3x6 0.0669, 8x3 0.0725;
// with f32x2 math (blocks/SM bound): 2: 0.0606, 3 (80 regs + spills): 0.0657, 4 (64 regs + spills): 0.0799
#ifndef AVB_LN_BWD_WARPS
#define AVB_LN_BWD_WARPS 12
#endif
#ifndef AVB_LN_BWD_STAGES
#define AVB_LN_BWD_STAGES 3
#endif
constexpr int kLnFwdWarps = 8, kLnFwdStages = AVB_LN_FWD_STAGES;   // AVB_LN_FWD_BLOCKS blocks / SM (launch bound)
constexpr int kLnBwdWarps = AVB_LN_BWD_WARPS, kLnBwdStages = AVB_LN_BWD_STAGES;   // 1 block / SM

template <int NC>
constexpr int ln_fwd_smem() { return kLnFwdWarps * kLnFwdStages * NC * 512; }
template <int NC>
constexpr int ln_bwd_smem() { return kLnBwdWarps * kLnBwdStages * (3 * NC * 512 + 256); }
static_assert(kLnBwdWarps * kLnBwdStages * (3 * 512 + 256) >= kLnBwdWarps * 3 * 256 * 4, "per-warp partials fit the ring");

template <int NC>
__global__ void __launch_bounds__(32 * kLnFwdWarps, AVB_LN_FWD_BLOCKS) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                                     __nv_bfloat16* __restrict__ y, int64_t ldy, float* __restrict__ mean,
                                                     float* __restrict__ rstd, int M, int D, float eps) {
  constexpr int S = kLnFwdStages;
  extern __shared__ uint4 ln_ring[];   // [warp][stage][NC][32 lanes]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* ring = ln_ring + warp * S * NC * 32 + lane;
  const int64_t nw = (int64_t)gridDim.x * kLnFwdWarps;
  bool ok[NC];
  float2 gg[NC][4], bb[NC][4];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = k * 256 + lane * 8;
    ok[k] = c < D;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      gg[k][e] = ok[k] ? make_float2(__ldg(gamma + c + 2 * e), __ldg(gamma + c + 2 * e + 1)) : make_float2(0.f, 0.f);
      bb[k][e] = ok[k] ? make_float2(__ldg(beta + c + 2 * e), __ldg(beta + c + 2 * e + 1)) : make_float2(0.f, 0.f);
    }
  }
  auto issue = [&](int64_t row, int s) {
    if (row < M) {
#pragma unroll
      for (int k = 0; k < NC; ++k)
        cp_async16(ring + (s * NC + k) * 32, ok[k] ? x + row * ldx + k * 256 + lane * 8 : x, ok[k]);
    }
    cp_async_commit();   // one group per row slot, empty or not, so wait_group<S-1> counts rows
  };
  int64_t row = (int64_t)blockIdx.x * kLnFwdWarps + warp;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(row + s * nw, s);
  for (int s = 0; row < M; row += nw, s = (s + 1 == S) ? 0 : s + 1) {
    issue(row + (S - 1) * nw, s == 0 ? S - 1 : s - 1);
    cp_async_wait<S - 1>();
    uint4 raw[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) raw[k] = ok[k] ? ring[(s * NC + k) * 32] : make_uint4(0, 0, 0, 0);
    float2 sum = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      float2 f[4];
      unpack8x2(raw[k], f);
#pragma unroll
      for (int e = 0; e < 4; ++e) sum = f2add(sum, f[e]);
    }
    const float mu = warp_sum(sum.x + sum.y) / D;
    const float2 nmu = make_float2(-mu, -mu);
    float2 q = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      float2 f[4];
      unpack8x2(raw[k], f);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 d = f2add(f[e], nmu);
        q = f2fma(d, d, q);
      }
    }
    const float rs = rsqrtf(warp_sum(q.x + q.y) / D + eps);
    const float2 rs2 = make_float2(rs, rs), nmr2 = make_float2(-mu * rs, -mu * rs);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      float2 f[4];
      unpack8x2(raw[k], f);
#pragma unroll
      for (int e = 0; e < 4; ++e) f[e] = f2fma(f2fma(f[e], rs2, nmr2), gg[k][e], bb[k][e]);   // (x - mu) rs g + b
      *reinterpret_cast<uint4*>(y + row * ldy + k * 256 + lane * 8) = pack8x2(f);
    }
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
  }
  cp_async_wait<0>();
}

template <int NC, bool SUM>
__global__ void __launch_bounds__(32 * kLnBwdWarps, 1) ln_bwd_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy,
                                                     const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ gamma, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, __nv_bfloat16* dx, int64_t lddx,
                                                     float* __restrict__ part, int M, int D, int accumulate) {
  constexpr int S = kLnBwdStages;
  constexpr int SLOT = 3 * NC * 32 + 16;   // uint4 per (warp, stage): x, dy, dx pieces + mean/rstd per lane
  extern __shared__ uint4 ln_ring[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* ring = ln_ring + warp * S * SLOT;
  bool ok[NC];
  float2 gm[NC][4], dg[NC][4], db[NC][4], cs[NC][4];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = k * 256 + lane * 8;
    ok[k] = c < D;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      gm[k][e] = ok[k] ? make_float2(__ldg(gamma + c + 2 * e), __ldg(gamma + c + 2 * e + 1)) : make_float2(0.f, 0.f);
      dg[k][e] = db[k][e] = cs[k][e] = make_float2(0.f, 0.f);
    }
  }
  const int64_t nw = (int64_t)gridDim.x * kLnBwdWarps;
  auto issue = [&](int64_t row, int s) {
    if (row < M) {
      uint4* slot = ring + s * SLOT;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int c = k * 256 + lane * 8;
        cp_async16(slot + k * 32 + lane, ok[k] ? x + row * ldx + c : x, ok[k]);
        cp_async16(slot + (NC + k) * 32 + lane, ok[k] ? dy + row * lddy + c : dy, ok[k]);
        cp_async16(slot + (2 * NC + k) * 32 + lane, (ok[k] && accumulate) ? dx + row * lddx + c : dx,
                   ok[k] && accumulate);
      }
      float* st = reinterpret_cast<float*>(slot + 3 * NC * 32) + 2 * lane;   // this lane's private copy
      cp_async4(st, mean + row);
      cp_async4(st + 1, rstd + row);
    }
    cp_async_commit();
  };
  int64_t row = (int64_t)blockIdx.x * kLnBwdWarps + warp;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(row + s * nw, s);
  for (int s = 0; row < M; row += nw, s = (s + 1 == S) ? 0 : s + 1) {
    issue(row + (S - 1) * nw, s == 0 ? S - 1 : s - 1);
    cp_async_wait<S - 1>();
    const uint4* slot = ring + s * SLOT;
    const float2 st = reinterpret_cast<const float2*>(slot + 3 * NC * 32)[lane];
    const float2 rs2 = make_float2(st.y, st.y), nmr2 = make_float2(-st.x * st.y, -st.x * st.y);   // xh = x rs - mu rs
    float2 s1 = make_float2(0.f, 0.f), s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      float2 xv[4], dv[4];
      unpack8x2(slot[k * 32 + lane], xv);
      unpack8x2(slot[(NC + k) * 32 + lane], dv);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xh = f2fma(xv[e], rs2, nmr2);
        const float2 g = f2mul(dv[e], gm[k][e]);
        s1 = f2add(s1, g);
        s2 = f2fma(g, xh, s2);
        dg[k][e] = f2fma(dv[e], xh, dg[k][e]);
        db[k][e] = f2add(db[k][e], dv[e]);
      }
    }
    const float m1 = warp_sum(s1.x + s1.y) / D, m2 = warp_sum(s2.x + s2.y) / D;
    const float2 nm1 = make_float2(-m1, -m1), nm2 = make_float2(-m2, -m2);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!ok[k]) continue;
      float2 xv[4], dv[4], pv[4], o[4];
      unpack8x2(slot[k * 32 + lane], xv);
      unpack8x2(slot[(NC + k) * 32 + lane], dv);
      unpack8x2(slot[(2 * NC + k) * 32 + lane], pv);   // zero-filled when !accumulate
#pragma unroll
      for (int e = 0; e < 4; ++e) {   // rs (dy gamma - m1 - xh m2) + dx_prev
        const float2 xh = f2fma(xv[e], rs2, nmr2);
        const float2 t = f2fma(xh, nm2, f2fma(dv[e], gm[k][e], nm1));
        o[e] = f2fma(t, rs2, pv[e]);
      }
      const uint4 q = pack8x2(o);
      *reinterpret_cast<uint4*>(dx + row * lddx + k * 256 + lane * 8) = q;
      if (SUM) {
        float2 ob[4];
        unpack8x2(q, ob);   // sum what was stored (bf16), like a separate column-sum pass would
#pragma unroll
        for (int e = 0; e < 4; ++e) cs[k][e] = f2add(cs[k][e], ob[e]);
      }
    }
  }
  // fixed-order reductions (bit-reproducible): each warp's column partials -> smem (over the drained
  // ring), the block sums them warp by warp -> part[block][3][D]; ln_bwd_reduce sums the blocks in order
  cp_async_wait<0>();
  __syncthreads();
  float* wpart = reinterpret_cast<float*>(ln_ring);   // [warp][3][D]
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = k * 256 + lane * 8;
    if (c < D) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        *reinterpret_cast<float2*>(&wpart[(warp * 3 + 0) * D + c + 2 * e]) = dg[k][e];
        *reinterpret_cast<float2*>(&wpart[(warp * 3 + 1) * D + c + 2 * e]) = db[k][e];
        *reinterpret_cast<float2*>(&wpart[(warp * 3 + 2) * D + c + 2 * e]) = SUM ? cs[k][e] : make_float2(0.f, 0.f);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * D; i += blockDim.x) {
    const int j = i / D, col = i - j * D;
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < kLnBwdWarps; ++w) acc += wpart[(w * 3 + j) * D + col];
    part[(int64_t)blockIdx.x * 3 * D + i] = acc;
  }
}

// One warp per (column, quantity): lane l sums block partials l, l+32, ... in order, then a fixed
// xor-shuffle tree -> deterministic.  part is [nblocks][3][D]; dst = dgamma / dbeta / dsum.
__global__ void ln_bwd_reduce_kernel(const float* __restrict__ part, int nblocks, int D, float* __restrict__ dgamma,
                                     float* __restrict__ dbeta, float* __restrict__ dsum) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= 3 * D) return;
  const int j = w / D, i = w - j * D;
  float* dst = j == 0 ? dgamma : (j == 1 ? dbeta : dsum);
  if (!dst) return;
  float acc = 0.f;
  for (int k = lane; k < nblocks; k += 32) acc += part[((int64_t)k * 3 + j) * D + i];
  acc = warp_sum(acc);
  if (lane == 0) dst[i] += acc;
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
  const int blocks = (int)std::min<int64_t>((M + kLnFwdWarps - 1) / kLnFwdWarps, (int64_t)avb::sm_count() * AVB_LN_FWD_BLOCKS);
  return dispatch_nc(D, [&](auto nc) {
    constexpr int NCv = decltype(nc)::value;
    constexpr int smem = ln_fwd_smem<NCv>();
    if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(ln_fwd_kernel<NCv>), smem, "ln_fwd smem attr"))
      return e;
    ln_fwd_kernel<NCv><<<blocks, 32 * kLnFwdWarps, smem, avb::as_stream(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), ldx, gamma, beta, reinterpret_cast<__nv_bfloat16*>(y), ldy, mean,
        rstd, M, D, eps);
    return avb::launch_status("avb_layernorm_fwd");
  });
}

extern "C" int avb_layernorm_bwd(const void* dy, int64_t lddy, const void* x, int64_t ldx, const float* gamma,
                                 const float* mean, const float* rstd, void* dx, int64_t lddx, float* dgamma,
                                 float* dbeta, float* dx_colsum, float* work, int M, int D, int accumulate,
                                 void* stream) {
  AVB_CHECK_ARG(M >= 0 && D >= 8 && D <= 1024 && D % 8 == 0, "LayerNorm needs D % 8 == 0, D <= 1024");
  if (M == 0) return AVB_OK;
  AVB_CHECK_ARG(dy && x && gamma && mean && rstd && dx && work, "null pointer");
  AVB_CHECK_ARG(lddy % 8 == 0 && ldx % 8 == 0 && lddx % 8 == 0, "row strides must be multiples of 8");
  const int blocks = (int)std::min<int64_t>((M + kLnBwdWarps - 1) / kLnBwdWarps, (int64_t)avb::sm_count());
  return dispatch_nc(D, [&](auto nc) {
    constexpr int NCv = decltype(nc)::value;
    constexpr int smem = ln_bwd_smem<NCv>();
    auto launch = [&](auto kern) {
      if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(kern), smem, "ln_bwd smem attr")) return e;
      kern<<<blocks, 32 * kLnBwdWarps, smem, avb::as_stream(stream)>>>(
          reinterpret_cast<const __nv_bfloat16*>(dy), lddy, reinterpret_cast<const __nv_bfloat16*>(x), ldx, gamma,
          mean, rstd, reinterpret_cast<__nv_bfloat16*>(dx), lddx, work, M, D, accumulate);
      if (int e = avb::launch_status("avb_layernorm_bwd")) return e;
      if (!dgamma && !dbeta && !dx_colsum) return AVB_OK;
      ln_bwd_reduce_kernel<<<(3 * D * 32 + 255) / 256, 256, 0, avb::as_stream(stream)>>>(work, blocks, D, dgamma,
                                                                                          dbeta, dx_colsum);
      return avb::launch_status("avb_layernorm_bwd (reduce)");
    };
    return dx_colsum ? launch(ln_bwd_kernel<NCv, true>) : launch(ln_bwd_kernel<NCv, false>);
  });
}

extern "C" int avb_layernorm_bwd_workspace(int D) { return avb::sm_count() * 3 * D; }
