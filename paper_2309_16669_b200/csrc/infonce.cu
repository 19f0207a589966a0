// K7: fused CLIP InfoNCE over a global contrastive batch (latency-bound).
//
// PAPER.md:291, :857, :1196 (projection dim 256):  with v^ = v/|v|, t^ = t/|t|,
//   S = s * v^ t^T  (Bg x Bg),  L = 1/(2Bg) * [ sum_i (lse_r[i] - S_ii) + sum_j (lse_c[j] - S_jj) ]
// No reference code exists.
//
// avb_infonce_fwd: (1) row norms, (2) one CTA per 8 rows + the same 8 columns computes its
//   S rows and S columns into shared memory, the row/column log-sum-exp, the loss terms and
//   dL/ds = 1/(2Bg s) * [ sum_i (E_r[i] - S_ii) + sum_j (E_c[j] - S_jj) ], E = softmax-weighted S.
// avb_infonce_bwd: one CTA per 8 local rows (video side) or 8 local columns (text side)
//   recomputes its S slice, forms dS = 1/(2Bg) [softmax_r - I + softmax_c - I] and
//   d v^_i = s * sum_j dS_ij t^_j, then back through the L2 normalisation:
//   d v_i = (d v^_i - v^_i (v^_i . d v^_i)) / |v_i|, scaled by grad_scale (DP: world size,
//   because each rank back-propagates only its local rows of a loss replicated on every rank).
#include "common.cuh"

namespace {

constexpr int RB = 8;        // rows (or columns) per CTA
constexpr int kThr = 256;

__global__ void rownorm_kernel(const float* __restrict__ x, int n, int E, float* __restrict__ nrm) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  float s = 0.f;
  for (int e = lane; e < E; e += 32) {
    const float v = x[(int64_t)row * E + e];
    s += v * v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  if (lane == 0) nrm[row] = fmaxf(sqrtf(s), 1e-12f);
}

// S values of RB fixed (normalised) vectors `fix` [RB][E] (smem) against all Bg rows of `other`,
// scaled by scale / |other_j|; out[r][j]
__device__ void dots_vs_all(const float* __restrict__ fix, const float* __restrict__ other,
                            const float* __restrict__ nother, int Bg, int E, float scale, float* out) {
  for (int j = threadIdx.x; j < Bg; j += blockDim.x) {
    float acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = 0.f;
    const float4* o4 = reinterpret_cast<const float4*>(other + (int64_t)j * E);
    for (int k = 0; k < E / 4; ++k) {
      const float4 b = __ldg(o4 + k);
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const float4 a = *reinterpret_cast<const float4*>(fix + r * E + 4 * k);
        acc[r] = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, acc[r]))));
      }
    }
    const float sc = scale / nother[j];
#pragma unroll
    for (int r = 0; r < RB; ++r) out[r * Bg + j] = acc[r] * sc;
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

// CLIP parameterisation: s = exp(min(log_scale, ln 100)); the clamp blocks the gradient
__device__ __forceinline__ float clip_scale(const float* log_scale) { return __expf(fminf(*log_scale, 4.6051702f)); }

__global__ void __launch_bounds__(kThr) infonce_stats_kernel(const float* __restrict__ v, const float* __restrict__ t,
                                                             const float* __restrict__ nv, const float* __restrict__ nt,
                                                             int Bg, int E, const float* __restrict__ log_scale,
                                                             float* __restrict__ lse_r, float* __restrict__ lse_c,
                                                             float* __restrict__ loss, float* __restrict__ dlog_scale) {
  extern __shared__ float sm[];
  const float scale = clip_scale(log_scale);
  const float dpar = (*log_scale < 4.6051702f) ? scale : 0.f;   // ds / d log_scale
  float* vrow = sm;                 // [RB][E]  normalised v rows i0..
  float* tcol = vrow + RB * E;      // [RB][E]  normalised t rows j0..
  float* Sr = tcol + RB * E;        // [RB][Bg] S[i0+r][j]
  float* Sc = Sr + RB * Bg;         // [RB][Bg] S[i][j0+c]
  const int i0 = blockIdx.x * RB;
  for (int idx = threadIdx.x; idx < RB * E; idx += blockDim.x) {
    const int r = idx / E, e = idx - r * E;
    vrow[idx] = (i0 + r < Bg) ? v[(int64_t)(i0 + r) * E + e] / nv[i0 + r] : 0.f;
    tcol[idx] = (i0 + r < Bg) ? t[(int64_t)(i0 + r) * E + e] / nt[i0 + r] : 0.f;
  }
  __syncthreads();
  dots_vs_all(vrow, t, nt, Bg, E, scale, Sr);   // rows of S
  dots_vs_all(tcol, v, nv, Bg, E, scale, Sc);   // columns of S (S_ij = S_ji of the transposed pairing)
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float inv2b = 0.5f / Bg;
  // warps 0-7: row r = warp (row stats); then column c = warp
  for (int pass = 0; pass < 2; ++pass) {
    const int r = warp;
    if (r < RB && i0 + r < Bg) {
      const float* S = (pass == 0 ? Sr : Sc) + r * Bg;
      float mx = -INFINITY;
      for (int j = lane; j < Bg; j += 32) mx = fmaxf(mx, S[j]);
      mx = warp_max(mx);
      float se = 0.f, sx = 0.f;
      for (int j = lane; j < Bg; j += 32) {
        const float p = __expf(S[j] - mx);
        se += p;
        sx += p * S[j];
      }
      se = warp_sum(se);
      sx = warp_sum(sx);
      if (lane == 0) {
        const float lse = mx + __logf(se);
        const float diag = S[i0 + r];
        (pass == 0 ? lse_r : lse_c)[i0 + r] = lse;
        atomicAdd(loss, inv2b * (lse - diag));
        if (dlog_scale) atomicAdd(dlog_scale, dpar * inv2b / scale * (sx / se - diag));
      }
    }
  }
}

// which = 0: d v for rows [r0, r0+n); which = 1: d t for columns [r0, r0+n)
__global__ void __launch_bounds__(kThr) infonce_grad_kernel(const float* __restrict__ v, const float* __restrict__ t,
                                                            const float* __restrict__ nv, const float* __restrict__ nt,
                                                            int Bg, int E, const float* __restrict__ log_scale,
                                                            const float* __restrict__ lse_r,
                                                            const float* __restrict__ lse_c, int r0, int n,
                                                            float grad_scale, float* __restrict__ dv,
                                                            float* __restrict__ dt) {
  extern __shared__ float sm[];
  const int which = blockIdx.y;
  const float* fixsrc = which ? t : v;
  const float* nfix = which ? nt : nv;
  const float* oth = which ? v : t;
  const float* noth = which ? nv : nt;
  const float* lse_fix = which ? lse_c : lse_r;   // softmax along the fixed index's own direction
  const float* lse_oth = which ? lse_r : lse_c;
  float* out = which ? dt : dv;
  const float scale = clip_scale(log_scale);
  float* fix = sm;                 // [RB][E] normalised
  float* S = fix + RB * E;         // [RB][Bg]
  float* red = S + RB * Bg;        // [RB]
  const int k0 = blockIdx.x * RB;  // local index
  for (int idx = threadIdx.x; idx < RB * E; idx += blockDim.x) {
    const int r = idx / E, e = idx - r * E;
    const int gi = r0 + k0 + r;
    fix[idx] = (k0 + r < n) ? fixsrc[(int64_t)gi * E + e] / nfix[gi] : 0.f;
  }
  if (threadIdx.x < RB) red[threadIdx.x] = 0.f;
  __syncthreads();
  dots_vs_all(fix, oth, noth, Bg, E, scale, S);
  __syncthreads();
  const float inv2b = 0.5f / Bg;
  for (int idx = threadIdx.x; idx < RB * Bg; idx += blockDim.x) {
    const int r = idx / Bg, j = idx - r * Bg;
    const int gi = r0 + k0 + r;
    float d = 0.f;
    if (k0 + r < n) {
      const float s = S[idx];
      const float diag = (j == gi) ? 1.f : 0.f;
      d = inv2b * (__expf(s - lse_fix[gi]) - diag + __expf(s - lse_oth[j]) - diag);
    }
    S[idx] = d;   // dS in place
  }
  __syncthreads();
  // d fix^_r[e] = scale * sum_j dS[r][j] * oth^_j[e]   (kept in dfix, then projected)
  float* dfix = red + RB;  // [RB][E]
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = 0.f;
    for (int j = 0; j < Bg; ++j) {
      const float o = __ldg(oth + (int64_t)j * E + e) / noth[j];
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = fmaf(S[r * Bg + j], o, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      acc[r] *= scale;
      dfix[r * E + e] = acc[r];
      atomicAdd(&red[r], acc[r] * fix[r * E + e]);
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < RB * E; idx += blockDim.x) {
    const int r = idx / E, e = idx - r * E;
    const int gi = r0 + k0 + r;
    if (k0 + r < n) out[(int64_t)(k0 + r) * E + e] = grad_scale * (dfix[idx] - fix[idx] * red[r]) / nfix[gi];
  }
}

}  // namespace

extern "C" int avb_infonce_fwd(const float* v, const float* t, int Bg, int E, const float* log_scale, float* norms_v,
                               float* norms_t, float* lse_r, float* lse_c, float* loss, float* dlog_scale,
                               void* stream) {
  AVB_CHECK_ARG(Bg >= 1 && E >= 4 && E % 4 == 0 && E <= 1024, "InfoNCE needs E % 4 == 0, E <= 1024");
  AVB_CHECK_ARG(v && t && norms_v && norms_t && lse_r && lse_c && loss && log_scale, "null pointer");
  cudaStream_t st = avb::as_stream(stream);
  rownorm_kernel<<<(Bg + 7) / 8, 256, 0, st>>>(v, Bg, E, norms_v);
  rownorm_kernel<<<(Bg + 7) / 8, 256, 0, st>>>(t, Bg, E, norms_t);
  const size_t smem = sizeof(float) * (2 * RB * E + 2 * (size_t)RB * Bg);
  AVB_CHECK_ARG(smem <= 200 * 1024, "global batch too large for one InfoNCE pass (Bg=%d)", Bg);
  if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(infonce_stats_kernel), 200 * 1024, "infonce attr"))
    return e;
  infonce_stats_kernel<<<(Bg + RB - 1) / RB, kThr, smem, st>>>(v, t, norms_v, norms_t, Bg, E, log_scale, lse_r,
                                                               lse_c, loss, dlog_scale);
  return avb::launch_status("avb_infonce_fwd");
}

extern "C" int avb_infonce_bwd(const float* v, const float* t, int Bg, int E, const float* log_scale, const float* norms_v,
                               const float* norms_t, const float* lse_r, const float* lse_c, int r0, int n,
                               float grad_scale, float* dv, float* dt, void* stream) {
  AVB_CHECK_ARG(Bg >= 1 && E >= 4 && E % 4 == 0 && E <= 1024, "InfoNCE needs E % 4 == 0, E <= 1024");
  AVB_CHECK_ARG(r0 >= 0 && n >= 0 && r0 + n <= Bg, "local rows out of range");
  if (n == 0) return AVB_OK;
  AVB_CHECK_ARG(v && t && log_scale && norms_v && norms_t && lse_r && lse_c && dv && dt, "null pointer");
  const size_t smem = sizeof(float) * (2 * RB * E + (size_t)RB * Bg + RB);
  AVB_CHECK_ARG(smem <= 200 * 1024, "global batch too large for one InfoNCE pass (Bg=%d)", Bg);
  if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(infonce_grad_kernel), 200 * 1024, "infonce attr"))
    return e;
  dim3 grid((n + RB - 1) / RB, 2);
  infonce_grad_kernel<<<grid, kThr, smem, avb::as_stream(stream)>>>(v, t, norms_v, norms_t, Bg, E, log_scale, lse_r,
                                                                    lse_c, r0, n, grad_scale, dv, dt);
  return avb::launch_status("avb_infonce_bwd");
}
