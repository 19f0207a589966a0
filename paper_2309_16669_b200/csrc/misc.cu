// Supporting kernels of the training step (all HBM/latency-bound, no reference code):
//   bias-gradient column sums, token assembly (cls + pos-embed),
//   softmax cross-entropy head loss (fine-tune), fused AdamW (K8).
#include "common.cuh"

#include <algorithm>

namespace {

__device__ __forceinline__ void ld8f(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 v = __bfloat1622float2(h[e]);
    f[2 * e] = v.x;
    f[2 * e + 1] = v.y;
  }
}
__device__ __forceinline__ void st8f(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 q;
  q.x = pack_bf16x2(f[0], f[1]);
  q.y = pack_bf16x2(f[2], f[3]);
  q.z = pack_bf16x2(f[4], f[5]);
  q.w = pack_bf16x2(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = q;
}

// out[n] += sum_m X[m, n]; block (64, 4): 64 column-octets x 4 row lanes, 4 rows in flight per thread
__global__ void colsum_kernel(const __nv_bfloat16* __restrict__ X, int64_t ldx, int M, int N, float* __restrict__ out) {
  __shared__ float red[4][64 * 8 + 4];
  const int c8 = blockIdx.x * 64 + threadIdx.x;
  const int col = c8 * 8;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (col < N) {
    const int64_t step = (int64_t)gridDim.y * 4;
    int64_t r = (int64_t)blockIdx.y * 4 + threadIdx.y;
    for (; r + 3 * step < M; r += 4 * step) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = *reinterpret_cast<const uint4*>(X + (r + u * step) * ldx + col);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      }
    }
    for (; r < M; r += step) {
      float f[8];
      ld8f(X + r * ldx + col, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += f[e];
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[threadIdx.y][threadIdx.x * 8 + e] = acc[e];
  __syncthreads();
  if (threadIdx.y == 0 && col < N) {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      atomicAdd(out + col + e, red[0][threadIdx.x * 8 + e] + red[1][threadIdx.x * 8 + e] + red[2][threadIdx.x * 8 + e] +
                                   red[3][threadIdx.x * 8 + e]);
  }
}

// x[b, 0] = cls + pos[0];  x[b, 1+n] = pe[b*Np + n] + pos[1+n]
// Separable space-time position embedding: PE[t*S + s] = PE_t[t] + PE_s[1 + s];
// the cls token takes PE_s[0] (CLIP's spatial table keeps a cls slot).
__global__ void tokens_fwd_kernel(const __nv_bfloat16* __restrict__ pe, const float* __restrict__ cls,
                                  const float* __restrict__ pos_s, const float* __restrict__ pos_t,
                                  __nv_bfloat16* __restrict__ x, int B, int Np, int S, int D) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = D / 8;
  const int64_t total = (int64_t)B * (Np + 1) * per_row;
  if (gid >= total) return;
  const int c = (gid % per_row) * 8;
  const int64_t tok = gid / per_row;
  const int n = tok % (Np + 1);
  const int b = tok / (Np + 1);
  float f[8];
  if (n == 0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = cls[c + e] + pos_s[c + e];
  } else {
    const int t = (n - 1) / S, sp = (n - 1) - t * S;
    ld8f(pe + ((int64_t)b * Np + n - 1) * D + c, f);
    const float4* ps = reinterpret_cast<const float4*>(pos_s + (int64_t)(1 + sp) * D + c);
    const float4* pt = reinterpret_cast<const float4*>(pos_t + (int64_t)t * D + c);
    const float4 s0 = ps[0], s1 = ps[1], t0 = pt[0], t1 = pt[1];
    f[0] += s0.x + t0.x; f[1] += s0.y + t0.y; f[2] += s0.z + t0.z; f[3] += s0.w + t0.w;
    f[4] += s1.x + t1.x; f[5] += s1.y + t1.y; f[6] += s1.z + t1.z; f[7] += s1.w + t1.w;
  }
  st8f(x + tok * D + c, f);
}

// One thread per (token n, 8 columns): acc = sum_b dx[b, n]; dpe = dx[:, 1:];
// dcls, dpos_s[0] += acc(n = 0); dpos_s[1+s] += acc; dpos_t[t] += acc (fp32 atomics: T' resp. S
// contributions per element, so these two small gradients are not bit-reproducible run to run).
// Token-embedding backward in two deterministic passes (no float atomics: bit-reproducible).
// Pass 1, one thread per (token n, 8 columns): tok[n] = sum_b dx[b, n] in clip order (and dpe = dx[:, 1:]).
__global__ void tokens_bwd_kernel(const __nv_bfloat16* __restrict__ dx, __nv_bfloat16* __restrict__ dpe,
                                  float* __restrict__ tok, int B, int Np, int D) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = D / 8;
  const int64_t total = (int64_t)(Np + 1) * per_row;
  if (gid >= total) return;
  const int c = (gid % per_row) * 8;
  const int n = gid / per_row;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = 0; b < B; ++b) {
    float f[8];
    const int64_t t = (int64_t)b * (Np + 1) + n;
    ld8f(dx + t * D + c, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += f[e];
    if (n > 0 && dpe) st8f(dpe + ((int64_t)b * Np + n - 1) * D + c, f);
  }
  float4* o = reinterpret_cast<float4*>(tok + (int64_t)n * D + c);
  o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

// Pass 2, one warp per (table row, 4 columns), rows = [cls/pos_s[0]] + pos_s[1..S] + pos_t[0..T'): lane l
// sums the row's tokens l, l+32, ... in order, then a fixed xor-shuffle tree (deterministic).
__global__ void tokens_bwd_tables_kernel(const float* __restrict__ tok, float* __restrict__ dcls,
                                         float* __restrict__ dpos_s, float* __restrict__ dpos_t, int Np, int S, int D) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int per_row = D / 4;
  const int Tn = Np / S;
  if (w >= (int64_t)(1 + S + Tn) * per_row) return;
  const int c = (int)(w % per_row) * 4;
  const int r = (int)(w / per_row);
  // the row's tokens: r = 0 -> {0}; r in [1, S] -> {1 + t*S + (r-1)}, t < Tn; else {1 + t*S + sp}, sp < S
  const int cnt = r == 0 ? 1 : (r <= S ? Tn : S);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int m = lane; m < cnt; m += 32) {
    const int n = r == 0 ? 0 : (r <= S ? 1 + m * S + (r - 1) : 1 + (r - 1 - S) * S + m);
    const float4 v = *reinterpret_cast<const float4*>(tok + (int64_t)n * D + c);
    acc = make_float4(acc.x + v.x, acc.y + v.y, acc.z + v.z, acc.w + v.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if (lane != 0) return;
  auto upd = [&](float* dst) {
    if (!dst) return;
    float4* d = reinterpret_cast<float4*>(dst + c);
    const float4 o = *d;
    *d = make_float4(o.x + acc.x, o.y + acc.y, o.z + acc.z, o.w + acc.w);
  };
  if (r == 0) {   // the cls token: its own parameter and slot 0 of the spatial table
    upd(dcls);
    upd(dpos_s);
  } else if (r <= S) {
    upd(dpos_s ? dpos_s + (int64_t)r * D : nullptr);
  } else {
    upd(dpos_t ? dpos_t + (int64_t)(r - 1 - S) * D : nullptr);
  }
}

// Tubelet patchify of normalised clips: x bf16 [B,3,T,H,W] (contiguous) -> rows [B*Np, 3*tt*th*tw] in
// Conv3d-weight feature order ((c*tt + dt)*th + dy)*tw + dx, row n = (t/tt * H/th + y/th) * W/tw + x/tw.
// One thread per (row, c, dt, dy) segment of tw elements (tw even: bf16 pairs).
__global__ void patchify_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ dst, int B, int T,
                                int H, int W, int tt, int th, int tw) {
  const int nT = T / tt, nH = H / th, nW = W / tw;
  const int64_t segs_per_row = 3LL * tt * th;
  const int64_t total = (int64_t)B * nT * nH * nW * segs_per_row;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const int64_t row = gid / segs_per_row;
  int seg = (int)(gid - row * segs_per_row);
  const int dy = seg % th;
  seg /= th;
  const int dt = seg % tt;
  const int c = seg / tt;
  int64_t r = row;
  const int px = r % nW; r /= nW;
  const int py = r % nH; r /= nH;
  const int pt = r % nT;
  const int b = (int)(r / nT);
  const int64_t src = ((((int64_t)b * 3 + c) * T + pt * tt + dt) * H + py * th + dy) * W + (int64_t)px * tw;
  const int64_t dof = row * (3LL * tt * th * tw) + ((int64_t)(c * tt + dt) * th + dy) * tw;
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(x + src);
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + dof);
  for (int k = 0; k < tw / 2; ++k) d32[k] = s32[k];
}

// one block per row: loss += scale * (lse - z[y]);  dlogits = scale * (softmax - onehot)
__global__ void xent_kernel(const float* __restrict__ logits, int64_t ld, const int32_t* __restrict__ labels, int C,
                            float scale, float* __restrict__ loss, __nv_bfloat16* __restrict__ dlogits, int64_t ldd) {
  __shared__ float sh[32];
  const int row = blockIdx.x;
  const float* z = logits + (int64_t)row * ld;
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < C; j += blockDim.x) mx = fmaxf(mx, z[j]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffff, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, sh[w]);
  __syncthreads();
  float s = 0.f;
  for (int j = threadIdx.x; j < C; j += blockDim.x) s += __expf(z[j] - mx);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  s = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
  const float lse = mx + __logf(s);
  const int y = labels[row];
  // a label outside [0, C) never reads out of bounds: the row is ignored (no loss, zero gradient),
  // like an ignore_index target
  const bool valid = y >= 0 && y < C;
  if (threadIdx.x == 0 && valid) atomicAdd(loss, scale * (lse - z[y]));
  if (dlogits) {
    for (int j = threadIdx.x; j < C; j += blockDim.x) {
      const float p = valid ? __expf(z[j] - lse) - (j == y ? 1.f : 0.f) : 0.f;
      dlogits[(int64_t)row * ldd + j] = __float2bfloat16_rn(scale * p);
    }
  }
}

// bias corrections 1 - beta^step, from the host value or (step_dev != null) from a device counter,
// so a captured CUDA graph replays the optimizer with the right step
__device__ __forceinline__ void adamw_bc(const int* step_dev, float b1, float b2, float& bc1, float& bc2) {
  if (step_dev) {
    const float st = (float)*step_dev;
    bc1 = 1.f - powf(b1, st);
    bc2 = 1.f - powf(b2, st);
  }
}

__global__ void adamw_tick_kernel(int* step_dev) { *step_dev += 1; }

// AdamW (decoupled weight decay), bias-corrected; optional bf16 shadow of the updated weights
__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, __nv_bfloat16* __restrict__ pb, const uint8_t* __restrict__ mask,
                             int64_t n, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                             float gscale, const int* __restrict__ step_dev) {
  adamw_bc(step_dev, b1, b2, bc1, bc2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i] * gscale;
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float wdi = (mask == nullptr || mask[i]) ? wd : 0.f;
    float pi = p[i] * (1.f - lr * wdi);
    pi -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
    p[i] = pi;
    if (pb) pb[i] = __float2bfloat16_rn(pi);
  }
}

// Same update, four parameters per thread (16-byte p/g/m/v, 4-byte mask, 8-byte bf16 shadow):
// the optimizer step is a pure HBM stream (31 B/param), so every access is vectorised.
__global__ void adamw_vec4_kernel(float4* __restrict__ p, const float4* __restrict__ g, float4* __restrict__ m,
                                  float4* __restrict__ v, uint2* __restrict__ pb, const uchar4* __restrict__ mask,
                                  int64_t n4, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                                  float gscale, const int* __restrict__ step_dev) {
  adamw_bc(step_dev, b1, b2, bc1, bc2);
  const float ib1 = 1.f / bc1, ib2 = 1.f / bc2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 g4 = g[i], m4 = m[i], v4 = v[i], p4 = p[i];
    const uchar4 k4 = mask ? mask[i] : make_uchar4(1, 1, 1, 1);
    const float gi[4] = {g4.x, g4.y, g4.z, g4.w}, mi0[4] = {m4.x, m4.y, m4.z, m4.w};
    const float vi0[4] = {v4.x, v4.y, v4.z, v4.w}, pi0[4] = {p4.x, p4.y, p4.z, p4.w};
    const uint8_t ki[4] = {k4.x, k4.y, k4.z, k4.w};
    float mo[4], vo[4], po[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gg = gi[e] * gscale;
      mo[e] = b1 * mi0[e] + (1.f - b1) * gg;
      vo[e] = b2 * vi0[e] + (1.f - b2) * gg * gg;
      const float wdi = ki[e] ? wd : 0.f;
      po[e] = pi0[e] * (1.f - lr * wdi) - lr * (mo[e] * ib1) / (sqrtf(vo[e] * ib2) + eps);
    }
    m[i] = make_float4(mo[0], mo[1], mo[2], mo[3]);
    v[i] = make_float4(vo[0], vo[1], vo[2], vo[3]);
    p[i] = make_float4(po[0], po[1], po[2], po[3]);
    if (pb) pb[i] = make_uint2(pack_bf16x2(po[0], po[1]), pack_bf16x2(po[2], po[3]));
  }
}

__global__ void cast_bf16_kernel(const float* __restrict__ s, __nv_bfloat16* __restrict__ d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

// x[b*L + l] = table[tok[b*L + l]] + pos[l]  (fp32 table -> bf16 rows)
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const float* __restrict__ table,
                                 const float* __restrict__ pos, __nv_bfloat16* __restrict__ x, int B, int L, int D,
                                 int V) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = D / 8;
  if (gid >= (int64_t)B * L * per) return;
  const int c = (gid % per) * 8;
  const int64_t r = gid / per;
  const int l = r % L;
  int id = tok[r];
  id = id < 0 ? 0 : (id >= V ? V - 1 : id);
  float f[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) f[e] = table[(int64_t)id * D + c + e] + pos[(int64_t)l * D + c + e];
  st8f(x + r * D + c, f);
}

// dtable[tok] += dx (atomics; repeated ids accumulate); dpos[l] += sum_b dx[b, l]
__global__ void embed_bwd_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ dx,
                                 float* __restrict__ dtable, float* __restrict__ dpos, int B, int L, int D, int V) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = D / 8;
  if (gid >= (int64_t)L * per) return;
  const int c = (gid % per) * 8;
  const int l = gid / per;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = 0; b < B; ++b) {
    const int64_t r = (int64_t)b * L + l;
    float f[8];
    ld8f(dx + r * D + c, f);
    int id = tok[r];
    id = id < 0 ? 0 : (id >= V ? V - 1 : id);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc[e] += f[e];
      if (dtable) atomicAdd(dtable + (int64_t)id * D + c + e, f[e]);
    }
  }
  if (dpos) {
#pragma unroll
    for (int e = 0; e < 8; ++e) dpos[(int64_t)l * D + c + e] += acc[e];
  }
}

// dst[dst_idx ? dst_idx[i] : i] = src[src_idx ? src_idx[i] : i]  (bf16 rows of D)
__global__ void rows_copy_kernel(const __nv_bfloat16* __restrict__ src, int64_t lds, const int32_t* __restrict__ sidx,
                                 __nv_bfloat16* __restrict__ dst, int64_t ldd, const int32_t* __restrict__ didx, int n,
                                 int D) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = D / 8;
  if (gid >= (int64_t)n * per) return;
  const int c = (gid % per) * 8;
  const int i = gid / per;
  const int64_t rs = sidx ? sidx[i] : i, rd = didx ? didx[i] : i;
  *reinterpret_cast<uint4*>(dst + rd * ldd + c) = *reinterpret_cast<const uint4*>(src + rs * lds + c);
}

}  // namespace

extern "C" int avb_embed_fwd(const int32_t* tokens, const float* table, const float* pos, void* x, int B, int L, int D,
                             int V, void* stream) {
  AVB_CHECK_ARG(B >= 0 && L >= 1 && D % 8 == 0 && V >= 1, "embed: D % 8 == 0");
  if (B == 0) return AVB_OK;
  AVB_CHECK_ARG(tokens && table && pos && x, "null pointer");
  const int64_t total = (int64_t)B * L * (D / 8);
  embed_fwd_kernel<<<(unsigned)((total + 255) / 256), 256, 0, avb::as_stream(stream)>>>(
      tokens, table, pos, reinterpret_cast<__nv_bfloat16*>(x), B, L, D, V);
  return avb::launch_status("avb_embed_fwd");
}

extern "C" int avb_embed_bwd(const int32_t* tokens, const void* dx, float* dtable, float* dpos, int B, int L, int D,
                             int V, void* stream) {
  AVB_CHECK_ARG(B >= 0 && L >= 1 && D % 8 == 0 && V >= 1, "embed: D % 8 == 0");
  if (B == 0) return AVB_OK;
  AVB_CHECK_ARG(tokens && dx, "null pointer");
  const int64_t total = (int64_t)L * (D / 8);
  embed_bwd_kernel<<<(unsigned)((total + 255) / 256), 256, 0, avb::as_stream(stream)>>>(
      tokens, reinterpret_cast<const __nv_bfloat16*>(dx), dtable, dpos, B, L, D, V);
  return avb::launch_status("avb_embed_bwd");
}

extern "C" int avb_rows_copy(const void* src, int64_t lds, const int32_t* src_idx, void* dst, int64_t ldd,
                             const int32_t* dst_idx, int n, int D, void* stream) {
  AVB_CHECK_ARG(n >= 0 && D % 8 == 0 && lds % 8 == 0 && ldd % 8 == 0, "rows_copy: D, lds, ldd multiples of 8");
  if (n == 0) return AVB_OK;
  AVB_CHECK_ARG(src && dst, "null pointer");
  const int64_t total = (int64_t)n * (D / 8);
  rows_copy_kernel<<<(unsigned)((total + 255) / 256), 256, 0, avb::as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(src), lds, src_idx, reinterpret_cast<__nv_bfloat16*>(dst), ldd, dst_idx,
      n, D);
  return avb::launch_status("avb_rows_copy");
}

extern "C" int avb_colsum_accum(const void* X, int64_t ldx, int M, int N, float* out, void* stream) {
  AVB_CHECK_ARG(M >= 0 && N >= 0 && N % 8 == 0 && ldx % 8 == 0, "colsum needs N and ldx multiples of 8");
  if (M == 0 || N == 0) return AVB_OK;
  AVB_CHECK_ARG(X && out, "null pointer");
  dim3 block(64, 4);
  const int gx = (N / 8 + 63) / 64;
  const int gy = std::max(1, std::min((M + 3) / 4, avb::sm_count() * 8 / gx));
  colsum_kernel<<<dim3(gx, gy), block, 0, avb::as_stream(stream)>>>(reinterpret_cast<const __nv_bfloat16*>(X), ldx, M,
                                                                      N, out);
  return avb::launch_status("avb_colsum_accum");
}

extern "C" int avb_tokens_fwd(const void* pe, const float* cls, const float* pos_s, const float* pos_t, void* x,
                              int B, int Np, int S, int D, void* stream) {
  AVB_CHECK_ARG(B >= 0 && Np >= 0 && D % 8 == 0, "tokens: D must be a multiple of 8");
  AVB_CHECK_ARG(S >= 1 && Np % S == 0, "tokens: Np=%d must be a multiple of the spatial count S=%d", Np, S);
  if (B == 0) return AVB_OK;
  AVB_CHECK_ARG(pe && cls && pos_s && pos_t && x, "null pointer");
  AVB_CHECK_ARG((reinterpret_cast<uintptr_t>(pos_s) & 15) == 0 && (reinterpret_cast<uintptr_t>(pos_t) & 15) == 0,
                "pos_s / pos_t must be 16-byte aligned");
  const int64_t total = (int64_t)B * (Np + 1) * (D / 8);
  tokens_fwd_kernel<<<(unsigned)((total + 255) / 256), 256, 0, avb::as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(pe), cls, pos_s, pos_t, reinterpret_cast<__nv_bfloat16*>(x), B, Np, S,
      D);
  return avb::launch_status("avb_tokens_fwd");
}

extern "C" int avb_tokens_bwd(const void* dx, void* dpe, float* dcls, float* dpos_s, float* dpos_t, float* work,
                              int B, int Np, int S, int D, void* stream) {
  AVB_CHECK_ARG(B >= 0 && Np >= 0 && D % 8 == 0, "tokens: D must be a multiple of 8");
  AVB_CHECK_ARG(S >= 1 && Np % S == 0, "tokens: Np=%d must be a multiple of the spatial count S=%d", Np, S);
  if (B == 0) return AVB_OK;
  AVB_CHECK_ARG(dx && work, "null pointer");
  AVB_CHECK_ARG((reinterpret_cast<uintptr_t>(work) & 15) == 0 && (!dcls || (reinterpret_cast<uintptr_t>(dcls) & 15) == 0) &&
                    (!dpos_s || (reinterpret_cast<uintptr_t>(dpos_s) & 15) == 0) &&
                    (!dpos_t || (reinterpret_cast<uintptr_t>(dpos_t) & 15) == 0),
                "tokens_bwd: work / dcls / dpos_s / dpos_t must be 16-byte aligned");
  const int64_t total = (int64_t)(Np + 1) * (D / 8);
  tokens_bwd_kernel<<<(unsigned)((total + 255) / 256), 256, 0, avb::as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(dx), reinterpret_cast<__nv_bfloat16*>(dpe), work, B, Np, D);
  if (int e = avb::launch_status("avb_tokens_bwd")) return e;
  const int64_t total2 = (int64_t)(1 + S + Np / S) * (D / 4) * 32;   // one warp per (row, 4 columns)
  tokens_bwd_tables_kernel<<<(unsigned)((total2 + 255) / 256), 256, 0, avb::as_stream(stream)>>>(work, dcls, dpos_s,
                                                                                               dpos_t, Np, S, D);
  return avb::launch_status("avb_tokens_bwd (tables)");
}

extern "C" int avb_patchify(const void* x, int B, int T, int H, int W, int tt, int th, int tw, void* dst,
                            void* stream) {
  AVB_CHECK_ARG(B >= 0 && T >= 1 && H >= 1 && W >= 1 && tt >= 1 && th >= 1 && tw >= 2 && tw % 2 == 0,
                "patchify: bad dims (tw must be even)");
  AVB_CHECK_ARG(T % tt == 0 && H % th == 0 && W % tw == 0, "patchify: tubelet %dx%dx%d must tile %dx%dx%d", tt, th,
                tw, T, H, W);
  if (B == 0) return AVB_OK;
  AVB_CHECK_ARG(x && dst, "null pointer");
  AVB_CHECK_ARG((reinterpret_cast<uintptr_t>(x) & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 3) == 0,
                "patchify: 4-byte aligned buffers");
  const int64_t total = (int64_t)B * (T / tt) * (H / th) * (W / tw) * 3 * tt * th;
  patchify_kernel<<<(unsigned)((total + 255) / 256), 256, 0, avb::as_stream(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<__nv_bfloat16*>(dst), B, T, H, W, tt, th, tw);
  return avb::launch_status("avb_patchify");
}

extern "C" int avb_xent(const float* logits, int64_t ld, const int32_t* labels, int B, int C, float scale, float* loss,
                        void* dlogits, int64_t ldd, void* stream) {
  AVB_CHECK_ARG(B >= 0 && C >= 1 && ld >= C, "bad xent dims");
  if (B == 0) return AVB_OK;
  AVB_CHECK_ARG(logits && labels && loss, "null pointer");
  xent_kernel<<<B, 256, 0, avb::as_stream(stream)>>>(logits, ld, labels, C, scale, loss,
                                                     reinterpret_cast<__nv_bfloat16*>(dlogits), ldd);
  return avb::launch_status("avb_xent");
}

static int adamw_launch(float* p, const float* g, float* m, float* v, void* p_bf16, const uint8_t* decay_mask,
                        int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay, int step,
                        const int* step_dev, float grad_scale, void* stream) {
  if (n == 0) return AVB_OK;
  AVB_CHECK_ARG(p && g && m && v, "null pointer");
  const float bc1 = step_dev ? 1.f : 1.f - powf(beta1, (float)step), bc2 = step_dev ? 1.f : 1.f - powf(beta2, (float)step);
  auto al = [](const void* q, uintptr_t b) { return (reinterpret_cast<uintptr_t>(q) & (b - 1)) == 0; };
  const bool vec = al(p, 16) && al(g, 16) && al(m, 16) && al(v, 16) && (!p_bf16 || al(p_bf16, 8)) &&
                   (!decay_mask || al(decay_mask, 4));
  int64_t done = 0;
  if (vec && n >= 4) {
    const int64_t n4 = n / 4;
    const int blocks = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)avb::sm_count() * 8);
    adamw_vec4_kernel<<<blocks, 256, 0, avb::as_stream(stream)>>>(
        reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g), reinterpret_cast<float4*>(m),
        reinterpret_cast<float4*>(v), reinterpret_cast<uint2*>(p_bf16), reinterpret_cast<const uchar4*>(decay_mask),
        n4, lr, beta1, beta2, eps, weight_decay, bc1, bc2, grad_scale, step_dev);
    int s = avb::launch_status("avb_adamw");
    if (s) return s;
    done = n4 * 4;
  }
  if (done == n) return AVB_OK;
  const int64_t r = n - done;   // unaligned buffers, or the < 4 element tail
  const int blocks = (int)std::min<int64_t>((r + 255) / 256, (int64_t)avb::sm_count() * 8);
  adamw_kernel<<<blocks, 256, 0, avb::as_stream(stream)>>>(
      p + done, g + done, m + done, v + done, p_bf16 ? reinterpret_cast<__nv_bfloat16*>(p_bf16) + done : nullptr,
      decay_mask ? decay_mask + done : nullptr, r, lr, beta1, beta2, eps, weight_decay, bc1, bc2, grad_scale, step_dev);
  return avb::launch_status("avb_adamw");
}

extern "C" int avb_adamw(float* p, const float* g, float* m, float* v, void* p_bf16, const uint8_t* decay_mask,
                         int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay, int step,
                         float grad_scale, void* stream) {
  AVB_CHECK_ARG(n >= 0 && step >= 1, "adamw: n >= 0, step >= 1");
  return adamw_launch(p, g, m, v, p_bf16, decay_mask, n, lr, beta1, beta2, eps, weight_decay, step, nullptr,
                      grad_scale, stream);
}

extern "C" int avb_adamw_dev(float* p, const float* g, float* m, float* v, void* p_bf16, const uint8_t* decay_mask,
                             int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay,
                             int* step_dev, float grad_scale, void* stream) {
  AVB_CHECK_ARG(n >= 0 && step_dev, "adamw_dev: n >= 0 and a device step counter");
  adamw_tick_kernel<<<1, 1, 0, avb::as_stream(stream)>>>(step_dev);
  if (int s = avb::launch_status("avb_adamw_dev (tick)")) return s;
  return adamw_launch(p, g, m, v, p_bf16, decay_mask, n, lr, beta1, beta2, eps, weight_decay, 0, step_dev, grad_scale,
                      stream);
}

extern "C" int avb_cast_bf16(const float* src, void* dst, int64_t n, void* stream) {
  AVB_CHECK_ARG(n >= 0, "n >= 0");
  if (n == 0) return AVB_OK;
  AVB_CHECK_ARG(src && dst, "null pointer");
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)avb::sm_count() * 8);
  cast_bf16_kernel<<<blocks, 256, 0, avb::as_stream(stream)>>>(src, reinterpret_cast<__nv_bfloat16*>(dst), n);
  return avb::launch_status("avb_cast_bf16");
}
