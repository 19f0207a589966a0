// K1: fused RandomResizedCrop (crop -> hflip -> antialiased bilinear) + normalize + cast.
//
// Replaces, per clip, the reference's per-frame CPU step
//   decoder.py:257-271 (crop_planes :282-292) -> _codec.yuv_to_rgb / current_rgb
//   -> convert_to_rgb + hflip_planes + sws_scale(SWS_BILINEAR|SWS_ACCURATE_RND)
//   (codec.cpp:187-275, :452-467)
// and appends the normalize+cast the reference defers to the GPU.
//
// Design (HBM-bound):
//   grid = (bands of R output rows, T, B); one CTA owns R output rows of one frame.
//   1. tap tables (exact-integer ranges, fp64 weights) for its R rows and all Wt columns;
//   2. the source rows those R rows touch, crop columns only, are staged to shared
//      memory with coalesced 16-byte loads (rows are re-aligned with byte funnel shifts
//      because the 568*3 = 1704 B row pitch is only 8-byte aligned);
//   3. vertical pass over interleaved byte columns (channel-agnostic) -> fp32 rows in smem;
//   4. horizontal pass per (row, channel, column pair) with the flip folded into the
//      column index (the tent filter is symmetric, so flip-then-scale == scale-then-
//      mirror), then y = v*inv_std/255 - mean*inv_std, packed bf16x2 / float2 stores,
//      coalesced along Wt.
#include "common.cuh"
#include "tc_common.cuh"

#include <algorithm>
#include <atomic>
#include <math.h>
#include <stdlib.h>

#include <type_traits>
#include <vector>

namespace {

constexpr int kThreads = 256;
constexpr int kMaxTaps = 24;

struct K1Params {
  const uint8_t* src;
  int64_t B;
  int T, H, W;
  int64_t s_clip, s_t, s_h, s_w, s_c;
  const int32_t* boxes;
  const uint8_t* flips;
  int Ht, Wt;
  float scale[3], bias[3];
  void* dst;
  int out_dtype, out_layout;
  int R;          // output rows per CTA
  int tx_cap;     // tap-table stride along x
  int ty_cap;     // tap-table stride along y
  int rows_cap;   // staged source rows capacity
  int rowb_cap;   // staged bytes per row (multiple of 16)
  int fast;       // interleaved RGB (s_c == 1, s_w == 3)
  int tt, tph, tpw;  // tubelet (AVB_LAYOUT_TUBELET)
  int only_upscale;  // 1: skip clips that are downscales in both axes (v4 did them)
};

// Exact-integer tap range + fp64 tent weights (torch/PIL antialias rule).
__device__ __forceinline__ int k1_taps(int crop, int tgt, int i, float* w, int& lo_out) {
  const long long c2 = 2LL * tgt;
  long long lo, hi;
  if (crop >= tgt) {
    lo = floordiv_i64((long long)crop * (2 * i - 1) + tgt, c2);
    hi = floordiv_i64((long long)crop * (2 * i + 3) + tgt, c2);
  } else {
    lo = floordiv_i64((long long)crop * (2 * i + 1) - tgt, c2);
    hi = floordiv_i64((long long)crop * (2 * i + 1) + 3LL * tgt, c2);
  }
  if (lo < 0) lo = 0;
  if (hi > crop) hi = crop;
  int n = static_cast<int>(hi - lo);
  if (n > kMaxTaps) n = kMaxTaps;  // host guarantees this never triggers
  const double s = static_cast<double>(crop) / tgt;
  const double inv = s >= 1.0 ? 1.0 / s : 1.0;
  const double c = s * (i + 0.5);
  double tot = 0.0;
  double wd[kMaxTaps];
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    double d = fabs((lo + k + 0.5 - c) * inv);
    wd[k] = d < 1.0 ? 1.0 - d : 0.0;
    tot += wd[k];
  }
  const double r = tot > 0.0 ? 1.0 / tot : 0.0;
#pragma unroll 1
  for (int k = 0; k < n; ++k) w[k] = static_cast<float>(wd[k] * r);
  lo_out = static_cast<int>(lo);
  return n;
}

__global__ void k1_taps_kernel(int crop, int tgt, int32_t* lo, int32_t* hi, float* w, int max_taps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tgt) return;
  float tw[kMaxTaps];
  int l = 0;
  int n = k1_taps(crop, tgt, i, tw, l);
  lo[i] = l;
  hi[i] = l + n;
  for (int k = 0; k < max_taps; ++k) w[(size_t)i * max_taps + k] = k < n ? tw[k] : 0.f;
}

// 16 bytes starting at an arbitrary byte address p (only the bytes < end are meaningful).
// Two aligned 16B loads + byte funnel shift; an aligned chunk is only touched when it
// contains at least one wanted byte, so no load crosses into an unmapped page.
__device__ __forceinline__ uint4 load16_unaligned(const uint8_t* p, const uint8_t* end) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t base = a & ~uintptr_t(15);
  const int mis = static_cast<int>(a - base);
  int4 c0 = ld_nc_v4(reinterpret_cast<const void*>(base));
  if (mis == 0) return make_uint4(c0.x, c0.y, c0.z, c0.w);
  int4 c1 = make_int4(0, 0, 0, 0);
  if (reinterpret_cast<const uint8_t*>(base + 16) < end) c1 = ld_nc_v4(reinterpret_cast<const void*>(base + 16));
  uint32_t w[8] = {(uint32_t)c0.x, (uint32_t)c0.y, (uint32_t)c0.z, (uint32_t)c0.w,
                   (uint32_t)c1.x, (uint32_t)c1.y, (uint32_t)c1.z, (uint32_t)c1.w};
  const int q = mis >> 2;
  const uint32_t sel = 0x3210u + 0x1111u * static_cast<uint32_t>(mis & 3);
  uint32_t s[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    uint32_t v = w[k];
    v = q == 1 ? w[k + 1] : v;
    v = q == 2 ? w[k + 2] : v;
    v = q == 3 ? w[k + 3] : v;
    s[k] = v;
  }
  uint4 r;
  r.x = __byte_perm(s[0], s[1], sel);
  r.y = __byte_perm(s[1], s[2], sel);
  r.z = __byte_perm(s[2], s[3], sel);
  r.w = __byte_perm(s[3], s[4], sel);
  return r;
}

__global__ void __launch_bounds__(kThreads) k1_rrc_normalize_kernel(const K1Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int band = blockIdx.x, t = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int tid = threadIdx.x;
  const int i0 = band * p.R;
  const int nR = min(p.R, p.Ht - i0);
  if (nR <= 0) return;

  const int4 box = *reinterpret_cast<const int4*>(p.boxes + 4 * b);
  const int x0 = box.x, y0 = box.y, cw = box.z, ch = box.w;
  // device-side containment re-check (CropRect.contained_in, rrc.py:81-85)
  if (x0 < 0 || y0 < 0 || cw < 1 || ch < 1 || x0 + cw > p.W || y0 + ch > p.H) return;
  if (p.only_upscale && cw >= p.Wt && ch >= p.Ht) return;
  const bool flip = p.flips ? (p.flips[b] != 0) : false;

  // ---- shared-memory carve-up ----
  float* wx = reinterpret_cast<float*>(smem);                    // [Wt][tx_cap]
  float* wy = wx + p.Wt * p.tx_cap;                              // [R][ty_cap]
  int* xlo = reinterpret_cast<int*>(wy + p.R * p.ty_cap);        // [Wt]
  int* ylo = xlo + p.Wt;                                         // [R]
  int* yn = ylo + p.R;                                           // [R]
  size_t off = (reinterpret_cast<uint8_t*>(yn + p.R) - smem + 15) & ~size_t(15);
  uint8_t* rows = smem + off;                                    // [rows_cap][rowb_cap] bytes
  float* vbuf = reinterpret_cast<float*>(rows + (size_t)p.rows_cap * p.rowb_cap);  // [R][rowb_cap]

  // ---- 1. tap tables ----
  for (int j = tid; j < p.Wt; j += kThreads) {
    int lo;
    int n = k1_taps(cw, p.Wt, j, wx + j * p.tx_cap, lo);
    for (int k = n; k < p.tx_cap; ++k) wx[j * p.tx_cap + k] = 0.f;  // padded taps weigh 0
    xlo[j] = lo;
  }
  for (int r = tid; r < nR; r += kThreads) {
    int lo;
    int n = k1_taps(ch, p.Ht, i0 + r, wy + r * p.ty_cap, lo);
    ylo[r] = lo;
    yn[r] = n;
  }
  __syncthreads();

  const int r0 = ylo[0];
  const int nrows = ylo[nR - 1] + yn[nR - 1] - r0;
  const int rowbytes = cw * 3;
  const int nchunk = (rowbytes + 15) >> 4;

  // ---- 2. stage source rows (crop columns only) ----
  const uint8_t* clip = p.src + b * p.s_clip + (int64_t)t * p.s_t;
  if (p.fast) {
    const uint8_t* fend = clip + (int64_t)(p.H - 1) * p.s_h + (int64_t)p.W * 3;  // end of this frame
    for (int idx = tid; idx < nrows * nchunk; idx += kThreads) {
      const int rr = idx / nchunk, q = idx - rr * nchunk;
      const uint8_t* g = clip + (int64_t)(y0 + r0 + rr) * p.s_h + (int64_t)x0 * 3 + 16 * q;
      const uint8_t* rend = clip + (int64_t)(y0 + r0 + rr) * p.s_h + (int64_t)(x0 + cw) * 3;
      uint4 v = load16_unaligned(g, rend < fend ? rend : fend);
      *reinterpret_cast<uint4*>(rows + (size_t)rr * p.rowb_cap + 16 * q) = v;
    }
  } else {
    for (int idx = tid; idx < nrows * rowbytes; idx += kThreads) {
      const int rr = idx / rowbytes, u = idx - rr * rowbytes;
      const int x = u / 3, c = u - 3 * x;
      rows[(size_t)rr * p.rowb_cap + u] =
          clip[(int64_t)(y0 + r0 + rr) * p.s_h + (int64_t)(x0 + x) * p.s_w + (int64_t)c * p.s_c];
    }
  }
  __syncthreads();

  // ---- 3. vertical pass (byte columns, channel-agnostic) ----
  const int nword = (rowbytes + 3) >> 2;
  for (int idx = tid; idx < nR * nword; idx += kThreads) {
    const int r = idx / nword, wq = idx - r * nword;
    const int base = ylo[r] - r0, n = yn[r];
    const float* w = wy + r * p.ty_cap;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    const uint8_t* sp = rows + (size_t)base * p.rowb_cap + 4 * wq;
    for (int k = 0; k < n; ++k) {
      const uint32_t u = *reinterpret_cast<const uint32_t*>(sp + (size_t)k * p.rowb_cap);
      const float wk = w[k];
      a0 = fmaf(wk, (float)(u & 0xff), a0);
      a1 = fmaf(wk, (float)((u >> 8) & 0xff), a1);
      a2 = fmaf(wk, (float)((u >> 16) & 0xff), a2);
      a3 = fmaf(wk, (float)(u >> 24), a3);
    }
    *reinterpret_cast<float4*>(vbuf + (size_t)r * p.rowb_cap + 4 * wq) = make_float4(a0, a1, a2, a3);
  }
  __syncthreads();

  // ---- 4. horizontal pass + normalize + cast + store ----
  const int P = (p.Wt + 1) >> 1;
  const int64_t plane = (int64_t)p.Ht * p.Wt;
  const bool pair_ok = (p.Wt & 1) == 0;
  for (int idx = tid; idx < nR * 3 * P; idx += kThreads) {
    const int r = idx / (3 * P);
    const int rem = idx - r * 3 * P;
    const int c = rem / P;
    const int j = 2 * (rem - c * P);
    const float* vr = vbuf + (size_t)r * p.rowb_cap + c;
    float y[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int jo = j + e;
      float acc = 0.f;
      if (jo < p.Wt) {
        const int jj = flip ? (p.Wt - 1 - jo) : jo;
        const float* w = wx + jj * p.tx_cap;
        const float* vv = vr + 3 * xlo[jj];
        const int lim = min(p.tx_cap, cw - xlo[jj]);
        for (int k = 0; k < lim; ++k) acc = fmaf(w[k], vv[3 * k], acc);
      }
      y[e] = fmaf(acc, p.scale[c], p.bias[c]);
    }
    int64_t o;
    if (p.out_layout == AVB_LAYOUT_CTHW) {
      o = ((b * 3 + c) * p.T + t) * plane + (int64_t)(i0 + r) * p.Wt + j;
    } else if (p.out_layout == AVB_LAYOUT_TCHW) {
      o = ((b * p.T + t) * 3 + c) * plane + (int64_t)(i0 + r) * p.Wt + j;
    } else {
      // tubelet rows: patch n' = ((t/tt)*(Ht/ph) + y/ph)*(Wt/pw) + x/pw, feature
      // f = ((c*tt + t%tt)*ph + y%ph)*pw + x%pw  (Conv3d weight [D,3,tt,ph,pw] flattening)
      const int y = i0 + r;
      const int npy = p.Ht / p.tph, npx = p.Wt / p.tpw;
      const int64_t Np = (int64_t)(p.T / p.tt) * npy * npx;
      const int F = 3 * p.tt * p.tph * p.tpw;
      const int64_t n = ((int64_t)(t / p.tt) * npy + y / p.tph) * npx + j / p.tpw;
      const int f = ((c * p.tt + t % p.tt) * p.tph + y % p.tph) * p.tpw + j % p.tpw;
      o = (b * Np + n) * F + f;
    }
    if (p.out_dtype == AVB_DTYPE_BF16) {
      __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(p.dst) + o;
      if (pair_ok) {
        *reinterpret_cast<uint32_t*>(d) = pack_bf16x2(y[0], y[1]);
      } else {
        d[0] = __float2bfloat16_rn(y[0]);
        if (j + 1 < p.Wt) d[1] = __float2bfloat16_rn(y[1]);
      }
    } else {
      float* d = reinterpret_cast<float*>(p.dst) + o;
      if (pair_ok) {
        *reinterpret_cast<float2*>(d) = make_float2(y[0], y[1]);
      } else {
        d[0] = y[0];
        if (j + 1 < p.Wt) d[1] = y[1];
      }
    }
  }
}


// ------------------------------------------------------------------------------------------------
// K1 v2 (fast path: interleaved RGB, 4-byte aligned rows).
//   grid = (column strips, T, B); a CTA owns one strip of output columns of one frame and walks
//   down the frame in bands of R output rows.  Per band, the strip's source bytes of the rows the
//   band touches are copied with 16-byte cp.async (aligned chunks, zero-filled past the row end)
//   into one of two staging buffers while the previous band is computed (double buffering).
//   Because every row pitch is a multiple of 4, all staged rows share the same sub-word shift m4,
//   so the vertical pass reads whole 32-bit words at a per-row word offset; bytes become floats
//   with one PRMT + one FADD2 (0x4B0000xx - 2^23) and accumulate with packed FFMA2.  The
//   horizontal pass then reads the fp32 band per (row, output column) for all three channels.
struct K1v2Params {
  const uint8_t* src;
  int64_t s_clip, s_t, s_h;
  int T, H, W, Ht, Wt;
  const int32_t* boxes;
  const uint8_t* flips;
  float scale[3], bias[3];
  void* dst;
  int out_dtype, out_layout, tt, tph, tpw;
  int R, strips, cps;           // rows per band, column strips, output columns per strip
  int tx_cap, ty_cap;           // tap-table strides
  int rows_cap, rowb_cap;       // staging rows per band, staged bytes per row (multiple of 16)
  int64_t total_bytes;          // bytes of the source tensor (cp.async zero-fill guard)
  int only_upscale;             // 1: skip clips that are downscales in both axes (v4 did them)
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return r;
}

__device__ __forceinline__ int64_t k1_out_index(const K1v2Params& p, int64_t b, int c, int t, int y, int j) {
  const int64_t plane = (int64_t)p.Ht * p.Wt;
  if (p.out_layout == AVB_LAYOUT_CTHW) return ((b * 3 + c) * p.T + t) * plane + (int64_t)y * p.Wt + j;
  if (p.out_layout == AVB_LAYOUT_TCHW) return ((b * p.T + t) * 3 + c) * plane + (int64_t)y * p.Wt + j;
  const int npy = p.Ht / p.tph, npx = p.Wt / p.tpw;
  const int64_t Np = (int64_t)(p.T / p.tt) * npy * npx;
  const int F = 3 * p.tt * p.tph * p.tpw;
  const int64_t n = ((int64_t)(t / p.tt) * npy + y / p.tph) * npx + j / p.tpw;
  const int f = ((c * p.tt + t % p.tt) * p.tph + y % p.tph) * p.tpw + j % p.tpw;
  return (b * Np + n) * F + f;
}

__global__ void __launch_bounds__(kThreads) k1v2_kernel(const K1v2Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int strip = blockIdx.x, t = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int tid = threadIdx.x;
  const int4 box = *reinterpret_cast<const int4*>(p.boxes + 4 * b);
  const int x0 = box.x, y0 = box.y, cw = box.z, ch = box.w;
  if (x0 < 0 || y0 < 0 || cw < 1 || ch < 1 || x0 + cw > p.W || y0 + ch > p.H) return;
  if (p.only_upscale && cw >= p.Wt && ch >= p.Ht) return;
  const bool flip = p.flips ? (p.flips[b] != 0) : false;
  // this strip, in unflipped column space jj; output column j = flip ? Wt-1-jj : jj
  const int jj0 = strip * p.cps;
  const int jj1 = min(p.Wt, jj0 + p.cps);
  const int nj = jj1 - jj0;
  if (nj <= 0) return;

  // ---- smem carve-up
  float* wx = reinterpret_cast<float*>(smem);                 // [cps][tx_cap]
  int* xlo = reinterpret_cast<int*>(wx + p.cps * p.tx_cap);   // [cps]
  int* xn = xlo + p.cps;                                      // [cps] taps per column
  float* wy = reinterpret_cast<float*>(xn + p.cps);           // [Ht][ty_cap]
  int* ylo = reinterpret_cast<int*>(wy + p.Ht * p.ty_cap);    // [Ht]
  int* yn = ylo + p.Ht;                                       // [Ht]
  int* rmis = yn + p.Ht;                                      // [2][rows_cap] per staged row: mis - m4
  size_t off = (reinterpret_cast<uint8_t*>(rmis + 2 * p.rows_cap) - smem + 15) & ~size_t(15);
  uint8_t* stage = smem + off;                                // [2][rows_cap][rowb_cap]
  float* vbuf = reinterpret_cast<float*>(stage + 2 * (size_t)p.rows_cap * p.rowb_cap);  // [R][rowb_cap]

  for (int k = tid; k < nj; k += kThreads) {
    int lo;
    const int n = k1_taps(cw, p.Wt, jj0 + k, wx + k * p.tx_cap, lo);
    for (int e = n; e < p.tx_cap; ++e) wx[k * p.tx_cap + e] = 0.f;
    xlo[k] = lo;
    xn[k] = n;
  }
  for (int r = tid; r < p.Ht; r += kThreads) {
    int lo;
    const int n = k1_taps(ch, p.Ht, r, wy + r * p.ty_cap, lo);
    ylo[r] = lo;
    yn[r] = n;
  }
  __syncthreads();
  // strip source columns (crop-local) [sx0, sx1)
  const int sx0 = xlo[0];
  const int sx1 = min(cw, xlo[nj - 1] + p.tx_cap);
  const int nbytes = (sx1 - sx0) * 3;
  const uint8_t* frame = p.src + b * p.s_clip + (int64_t)t * p.s_t;
  const uintptr_t first = reinterpret_cast<uintptr_t>(frame + (int64_t)y0 * p.s_h + (int64_t)(x0 + sx0) * 3);
  const int m4 = (int)(first & 3);
  const int nwords = (nbytes + m4 + 3) >> 2;
  const uint8_t* src_end = p.src + p.total_bytes;
  const int nbands = (p.Ht + p.R - 1) / p.R;

  auto issue_band = [&](int band, int buf) {
    const int i0 = band * p.R, i1 = min(p.Ht, i0 + p.R);
    const int r_lo = ylo[i0], r_hi = ylo[i1 - 1] + yn[i1 - 1];
    const int nrows = r_hi - r_lo;
    uint8_t* sb = stage + (size_t)buf * p.rows_cap * p.rowb_cap;
    const int chunks = (nbytes + m4 + 15 + 12) >> 4;   // mis <= 15
    for (int idx = tid; idx < nrows * chunks; idx += kThreads) {
      const int rr = idx / chunks, k = idx - rr * chunks;
      const uint8_t* a = frame + (int64_t)(y0 + r_lo + rr) * p.s_h + (int64_t)(x0 + sx0) * 3;
      const uintptr_t al = reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15);
      const uint8_t* g = reinterpret_cast<const uint8_t*>(al) + 16 * k;
      const int64_t left = src_end - g;
      const int nb = left >= 16 ? 16 : (left > 0 ? (int)left : 0);
      if (16 * k < (int)(reinterpret_cast<uintptr_t>(a) - al) + nbytes)
        cp_async16(sb + (size_t)rr * p.rowb_cap + 16 * k, nb ? g : p.src, nb);
      if (k == 0) rmis[buf * p.rows_cap + rr] = (int)(reinterpret_cast<uintptr_t>(a) - al) - m4;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  issue_band(0, 0);
  for (int band = 0; band < nbands; ++band) {
    const int buf = band & 1;
    if (band + 1 < nbands) {
      issue_band(band + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int i0 = band * p.R, nR = min(p.R, p.Ht - i0);
    const int r_lo = ylo[i0];
    const uint8_t* sb = stage + (size_t)buf * p.rows_cap * p.rowb_cap;
    const int* mis = rmis + buf * p.rows_cap;
    // vertical pass: shifted byte columns u' = 4q..4q+3 of the strip (u' = crop byte - sx0*3 + m4)
    for (int idx = tid; idx < nR * nwords; idx += kThreads) {
      const int r = idx / nwords, q = idx - r * nwords;
      const int base = ylo[i0 + r] - r_lo, n = yn[i0 + r];
      const float* w = wy + (i0 + r) * p.ty_cap;
      float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
      for (int k = 0; k < n; ++k) {
        const int rr = base + k;
        const uint32_t u = *reinterpret_cast<const uint32_t*>(sb + (size_t)rr * p.rowb_cap + mis[rr] + 4 * q);
        const float2 magic = make_float2(-8388608.f, -8388608.f);
        float2 f01 = make_float2(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7440)),
                                 __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7441)));
        float2 f23 = make_float2(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7442)),
                                 __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7443)));
        f01.x += magic.x; f01.y += magic.y;
        f23.x += magic.x; f23.y += magic.y;
        const float2 ww = make_float2(w[k], w[k]);
        a01 = ffma2(ww, f01, a01);
        a23 = ffma2(ww, f23, a23);
      }
      *reinterpret_cast<float4*>(vbuf + (size_t)r * p.rowb_cap + 4 * q) = make_float4(a01.x, a01.y, a23.x, a23.y);
    }
    __syncthreads();
    // horizontal pass + normalize + store: item = (row, strip column)
    for (int idx = tid; idx < nR * nj; idx += kThreads) {
      const int r = idx / nj, k = idx - r * nj;
      const int jj = jj0 + k;
      const int j = flip ? (p.Wt - 1 - jj) : jj;
      const float* w = wx + k * p.tx_cap;
      const int lim = xn[k];
      const float* v = vbuf + (size_t)r * p.rowb_cap + (xlo[k] - sx0) * 3 + m4;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f;
      for (int e = 0; e < lim; ++e) {
        const float we = w[e];
        a0 = fmaf(we, v[3 * e], a0);
        a1 = fmaf(we, v[3 * e + 1], a1);
        a2 = fmaf(we, v[3 * e + 2], a2);
      }
      const float ys[3] = {fmaf(a0, p.scale[0], p.bias[0]), fmaf(a1, p.scale[1], p.bias[1]),
                           fmaf(a2, p.scale[2], p.bias[2])};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t o = k1_out_index(p, b, c, t, i0 + r, j);
        if (p.out_dtype == AVB_DTYPE_BF16)
          reinterpret_cast<__nv_bfloat16*>(p.dst)[o] = __float2bfloat16_rn(ys[c]);
        else
          reinterpret_cast<float*>(p.dst)[o] = ys[c];
      }
    }
    __syncthreads();
  }
}


// ------------------------------------------------------------------------------------------------
// K1 v4 (default for downscales of interleaved RGB): horizontal-first streaming.
//
//   grid = (frame groups, B): a CTA owns FPC frames of one clip (they share every tap; Wt = 224
//   gives FPC = 2, whose 224 column pairs fill exactly 7 warps) and streams the crop's source
//   rows top to bottom exactly once:
//   * one producer thread (warp `ncomp/32`) keeps a V4_RS-deep ring of staged rows full with one
//     `cp.async.bulk` per (row, frame) from the 16-byte-aligned-down row start (rows past
//     `tail_y`, whose rounded copy could cross the tensor end, take zero-filled 16-byte
//     cp.async); completion on a per-slot `full` mbarrier, release by the 7 compute warps on an
//     `empty` mbarrier;
//   * every compute lane owns two adjacent OUTPUT columns (j, j+1) of one frame for the whole
//     frame, with its horizontal taps (NT, zero-padded) in registers.  Per source row it reads
//     its two tap windows (funnel-shifted words), converts bytes to floats (PRMT into
//     0x4B0000xx, FADD2 -2^23) and filters the three channels of both columns with FFMA2 -- no
//     shared-memory traffic for intermediate values;
//   * the vertical pass is a push: the (<= NOPEN) output rows whose windows contain the source
//     row accumulate w * h in registers; a row is normalised, cast and stored the moment its
//     window closes.  The per-source-row weights / emission counts are a per-clip table built in
//     the prologue in O(1) per row, identical for every lane, so control flow is block-uniform.
//   No __syncthreads in the main loop; each source byte is read from HBM once.
constexpr int V4_RS = 16;  // staged-row ring depth (one row of every frame of the CTA per stage)

struct K1v4Params {
  const uint8_t* src;
  int64_t s_clip, s_t, s_h;
  int T, H, W, Ht, Wt;
  const int32_t* boxes;
  const uint8_t* flips;
  float scale[3], bias[3];
  void* dst;
  int out_dtype, out_layout, tt, tph, tpw;
  int fpc;         // frames per CTA
  int tpf;         // column pairs (compute lanes) per frame = ceil(Wt / 2)
  int ncomp;       // compute threads (multiple of 32); the producer warp follows
  int slot_bytes;  // bytes per staged row (multiple of 16); planar: 3 channel sub-slots of cslot bytes
  int cslot;       // planar input ([B,T,3,H,W] rows): bytes per channel sub-slot (multiple of 16)
  int64_t s_c;     // planar input: channel-plane stride in bytes (a multiple of 16)
  int64_t total_bytes;
  int nband;       // output-row bands per frame group (grid.x = frame groups * nband): finer work units
                   // balance the waves (each band re-reads the <= 3 source rows its neighbour also needs)
};

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return r;
}

// NT-tap (zero-padded) register copy of the exact-integer taps of output column i (same fp64 math
// and summation order as k1_taps, so the weights are bit-identical).  Downscale only.
template <int NT>
__device__ __forceinline__ void k1_taps_reg(int crop, int tgt, int i, float (&w)[NT], int& lo_out) {
  const long long c2 = 2LL * tgt;
  long long lo = floordiv_i64((long long)crop * (2 * i - 1) + tgt, c2);
  long long hi = floordiv_i64((long long)crop * (2 * i + 3) + tgt, c2);
  if (lo < 0) lo = 0;
  if (hi > crop) hi = crop;
  const int n = static_cast<int>(hi - lo);
  const double s = static_cast<double>(crop) / tgt;
  const double inv = 1.0 / s;
  const double c = s * (i + 0.5);
  double wd[NT];
  double tot = 0.0;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const double d = fabs((lo + k + 0.5 - c) * inv);
    wd[k] = (k < n && d < 1.0) ? 1.0 - d : 0.0;
    tot += wd[k];
  }
  const double r = tot > 0.0 ? 1.0 / tot : 0.0;
#pragma unroll
  for (int k = 0; k < NT; ++k) w[k] = static_cast<float>(wd[k] * r);
  lo_out = static_cast<int>(lo);
}

// Weight of source row y in output row i (downscale rule; 0 outside the row's window).
__device__ __forceinline__ float k1_row_weight(int crop, int tgt, int i, int y) {
  const long long c2 = 2LL * tgt;
  long long lo = floordiv_i64((long long)crop * (2 * i - 1) + tgt, c2);
  long long hi = floordiv_i64((long long)crop * (2 * i + 3) + tgt, c2);
  if (lo < 0) lo = 0;
  if (hi > crop) hi = crop;
  if (y < lo || y >= hi) return 0.f;
  const double s = static_cast<double>(crop) / tgt;
  const double inv = 1.0 / s;
  const double c = s * (i + 0.5);
  double tot = 0.0, wy = 0.0;
  for (long long k = 0; k < hi - lo; ++k) {
    const double d = fabs((lo + k + 0.5 - c) * inv);
    const double w = d < 1.0 ? 1.0 - d : 0.0;
    tot += w;
    if (lo + k == y) wy = w;
  }
  return static_cast<float>(wy * (tot > 0.0 ? 1.0 / tot : 0.0));
}

// #{output rows i : hi_i <= y} for source row y < crop (rows whose window ended before y).
__device__ __forceinline__ int k1_rows_done(int crop, int tgt, int y) {
  // hi_i <= y  <=>  crop*(2i+3) + tgt < 2*tgt*(y+1)  <=>  i < N / (2 crop)
  const long long N = 2LL * tgt * (y + 1) - tgt - 3LL * crop;
  if (N <= 0) return 0;
  const long long n = (N + 2LL * crop - 1) / (2LL * crop);
  return n > tgt ? tgt : static_cast<int>(n);
}

// The 4*NW bytes starting at byte offset o of a staged row, as NW words (o may be unaligned).
template <int NW>
__device__ __forceinline__ void k1_window(const uint8_t* slot, int o, uint32_t (&s)[NW]) {
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(slot + (o & ~3));
  const uint32_t sh = (o & 3) * 8;
  uint32_t u[NW + 1];
#pragma unroll
  for (int k = 0; k <= NW; ++k) u[k] = wp[k];
#pragma unroll
  for (int k = 0; k < NW; ++k) s[k] = __funnelshift_r(u[k], u[k + 1], sh);
}

// byte q of a word stream -> 2^23 + byte as a float bit pattern (exact)
template <int Q, int NW>
__device__ __forceinline__ float k1_magic(const uint32_t (&s)[NW]) {
  return __uint_as_float(__byte_perm(s[Q >> 2], 0x4B000000u, 0x7440u | (Q & 3)));
}

template <int NT, int C, int K = 0>
struct K1HTap {
  template <int NW>
  __device__ __forceinline__ static void run(const uint32_t (&s0)[NW], const uint32_t (&s1)[NW], const float2 (&wp)[NT],
                                             float2& h) {
    if constexpr (K < NT) {
      const float2 f = fadd2(make_float2(k1_magic<3 * K + C>(s0), k1_magic<3 * K + C>(s1)),
                             make_float2(-8388608.f, -8388608.f));
      h = ffma2(wp[K], f, h);
      K1HTap<NT, C, K + 1>::run(s0, s1, wp, h);
    }
  }
};

// planar rows: tap K of a channel is byte K of that channel's window
template <int NT, int K = 0>
struct K1HTapPL {
  template <int NW>
  __device__ __forceinline__ static void run(const uint32_t (&s0)[NW], const uint32_t (&s1)[NW], const float2 (&wp)[NT],
                                             float2& h) {
    if constexpr (K < NT) {
      const float2 f = fadd2(make_float2(k1_magic<K>(s0), k1_magic<K>(s1)), make_float2(-8388608.f, -8388608.f));
      h = ffma2(wp[K], f, h);
      K1HTapPL<NT, K + 1>::run(s0, s1, wp, h);
    }
  }
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int NT, int NOPEN, bool PL = false>
__global__ void __launch_bounds__(256, 4) k1v4_kernel(const K1v4Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NW = PL ? (NT + 3) / 4 : (3 * NT + 3) / 4;   // window words per column (one channel if planar)
  constexpr int NCH = PL ? 3 : 1;                             // bulk copies per (row, frame)
  static_assert(NOPEN <= 3, "emission count lives in rowtab.w");
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.y;
  const int band = blockIdx.x % p.nband;
  const int t0 = (blockIdx.x / p.nband) * p.fpc;
  const int4 box = *reinterpret_cast<const int4*>(p.boxes + 4 * b);
  const int x0 = box.x, y0 = box.y, cw = box.z, ch = box.w;
  if (x0 < 0 || y0 < 0 || cw < p.Wt || ch < p.Ht || x0 + cw > p.W || y0 + ch > p.H) return;
  const bool flip = p.flips ? (p.flips[b] != 0) : false;
  // this CTA emits output rows [i_lo, i_hi) and streams the source rows [ys, ye) their windows span;
  // the first row it pushes into is r0 = #rows closed before ys (rows < i_lo are accumulated, not stored)
  const int i_lo = band * p.Ht / p.nband, i_hi = (band + 1) * p.Ht / p.nband;
  int ys, ye;
  {
    const long long c2 = 2LL * p.Ht;
    long long lo = floordiv_i64((long long)ch * (2 * i_lo - 1) + p.Ht, c2);
    long long hi = floordiv_i64((long long)ch * (2 * (i_hi - 1) + 3) + p.Ht, c2);
    ys = lo < 0 ? 0 : (int)lo;
    ye = hi > ch ? ch : (int)hi;
  }
  const int r0 = k1_rows_done(ch, p.Ht, ys);

  // ---- smem: full [RS] | empty [RS] | rowtab [H] | ring [RS][fpc][slot_bytes]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + V4_RS;
  float4* rowtab = reinterpret_cast<float4*>(empty + V4_RS);
  uint8_t* ring = reinterpret_cast<uint8_t*>(rowtab + p.H);
  const size_t stage_stride = (size_t)p.fpc * p.slot_bytes;

  // ---- per-source-row push table: weights of the NOPEN open output rows, rows completed after it.
  // Built per output row (one fp64 normalisation per row, the same math and summation order as
  // k1_row_weight, so the weights are bit-identical) and scattered into the source rows it spans.
  float* rowtab_f = reinterpret_cast<float*>(rowtab);
  for (int y = ys + tid; y < ye; y += blockDim.x) {
    const int base = k1_rows_done(ch, p.Ht, y);
    const int next = (y + 1 < ch) ? k1_rows_done(ch, p.Ht, y + 1) : p.Ht;
    rowtab[y] = make_float4(0.f, 0.f, 0.f, __int_as_float(next - base));
  }
  __syncthreads();
  for (int i = r0 + tid; i < i_hi; i += blockDim.x) {
    const long long c2 = 2LL * p.Ht;
    long long lo = floordiv_i64((long long)ch * (2 * i - 1) + p.Ht, c2);
    long long hi = floordiv_i64((long long)ch * (2 * i + 3) + p.Ht, c2);
    if (lo < 0) lo = 0;
    if (hi > ch) hi = ch;
    const double sc = static_cast<double>(ch) / p.Ht;
    const double inv = 1.0 / sc;
    const double cc = sc * (i + 0.5);
    double tot = 0.0;
    for (long long k = 0; k < hi - lo; ++k) {
      const double d = fabs((lo + k + 0.5 - cc) * inv);
      tot += d < 1.0 ? 1.0 - d : 0.0;
    }
    const double r = tot > 0.0 ? 1.0 / tot : 0.0;
    for (long long k = 0; k < hi - lo; ++k) {
      const int y = (int)(lo + k);
      if (y < ys || y >= ye) continue;
      const int q = i - k1_rows_done(ch, p.Ht, y);   // slot of row i among the rows open at y
      const double d = fabs((lo + k + 0.5 - cc) * inv);
      if (q >= 0 && q < NOPEN) rowtab_f[4 * y + q] = static_cast<float>((d < 1.0 ? 1.0 - d : 0.0) * r);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < V4_RS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], p.ncomp);   // every compute thread arrives (no elected-lane branch)
    }
    tc::fence_barrier_init();
  }
  __syncthreads();

  if (tid >= p.ncomp) {
    // ================= producer: one lane, one bulk copy per (source row, frame)
    if (tid != p.ncomp) return;
    const uint8_t* src_end = p.src + p.total_bytes;
    const uint8_t* row0 = p.src + b * p.s_clip + (int64_t)t0 * p.s_t + (int64_t)y0 * p.s_h + (int64_t)x0 * (PL ? 1 : 3);
    const int nf = min(p.fpc, p.T - t0);
    const uint32_t span = PL ? (uint32_t)cw : 3u * cw;
    // first row whose rounded-up copy (of the last frame / channel) could reach past the tensor end
    int tail_y = ye;
    {
      const uint8_t* last = row0 + (int64_t)(nf - 1) * p.s_t + (PL ? 2 * p.s_c : 0);
      for (int y = ye - 1; y >= ys && last + (int64_t)y * p.s_h + span + 15 > src_end; --y) tail_y = y;
    }
    int s = 0;
    uint32_t ph = 0;
    const uint8_t* a_row = row0 + (int64_t)ys * p.s_h;
    for (int y = ys; y < ye; ++y, a_row += p.s_h) {
      if (y - ys >= V4_RS) tc::mbar_wait(&empty[s], ph ^ 1);
      uint8_t* dst = ring + (size_t)s * stage_stride;
      if (y < tail_y) {
        uint32_t tx = 0;
        const uint8_t* a = a_row;
        for (int f = 0; f < nf; ++f, a += p.s_t) tx += NCH * ((((uint32_t)(uintptr_t)a & 15u) + span + 15u) & ~15u);
        tc::mbar_arrive_expect_tx(&full[s], tx);
        a = a_row;
        for (int f = 0; f < nf; ++f, a += p.s_t) {
          const uint32_t mis = (uint32_t)(uintptr_t)a & 15u;   // the same for every plane (s_c % 16 == 0)
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            bulk_g2s(dst + (size_t)f * p.slot_bytes + c * p.cslot, a + c * p.s_c - mis, (mis + span + 15u) & ~15u,
                     &full[s]);
        }
      } else {  // bytes past the tensor end would fault: zero-filled 16-byte cp.async instead
        const uint8_t* a = a_row;
        for (int f = 0; f < nf; ++f, a += p.s_t) {
          for (int c = 0; c < NCH; ++c) {
            const uint8_t* ac = a + c * p.s_c;
            const uint8_t* al = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(ac) & ~uintptr_t(15));
            const uint32_t nb = ((uint32_t)(ac - al) + span + 15u) & ~15u;
            for (uint32_t k = 0; k < nb; k += 16) {
              const int64_t left = src_end - (al + k);
              const int n = left >= 16 ? 16 : (left > 0 ? (int)left : 0);
              cp_async16(dst + (size_t)f * p.slot_bytes + c * p.cslot + k, n ? al + k : p.src, n);
            }
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      }
      if (++s == V4_RS) { s = 0; ph ^= 1; }
    }
    return;
  }

  // ================= compute lanes: output columns (j0, j0+1) of frame t
  const int f = tid / p.tpf;
  const int m = tid - f * p.tpf;
  const int t = t0 + f;
  const bool active = f < p.fpc && t < p.T;
  const int j0 = 2 * m;
  const bool has1 = active && j0 + 1 < p.Wt;
  float2 wp[NT];
  int o0 = 0, o1 = 0;
  {
    float w0[NT], w1[NT];
    int lo0 = 0, lo1 = 0;
#pragma unroll
    for (int k = 0; k < NT; ++k) w0[k] = w1[k] = 0.f;
    if (active) k1_taps_reg<NT>(cw, p.Wt, flip ? p.Wt - 1 - j0 : j0, w0, lo0);
    if (has1) k1_taps_reg<NT>(cw, p.Wt, flip ? p.Wt - 2 - j0 : j0 + 1, w1, lo1);
    else lo1 = lo0;
#pragma unroll
    for (int k = 0; k < NT; ++k) wp[k] = make_float2(w0[k], w1[k]);
    o0 = (PL ? 1 : 3) * lo0;
    o1 = (PL ? 1 : 3) * lo1;
  }
  // output: element offset obase + rowoff(row) + c * cstride (32-bit within a clip, all layouts)
  int64_t obase;
  int cstride, small_step, big_step, rph = 0, ph_rows;
  {
    const int tt = active ? t : t0;
    const int plane = p.Ht * p.Wt;
    if (p.out_layout == AVB_LAYOUT_CTHW) {
      obase = (b * 3 * p.T + tt) * (int64_t)plane + j0;
      cstride = p.T * plane;
      small_step = big_step = p.Wt;
      ph_rows = 1 << 30;
    } else if (p.out_layout == AVB_LAYOUT_TCHW) {
      obase = (b * p.T + tt) * 3 * (int64_t)plane + j0;
      cstride = plane;
      small_step = big_step = p.Wt;
      ph_rows = 1 << 30;
    } else {
      const int npy = p.Ht / p.tph, npx = p.Wt / p.tpw;
      const int64_t Np = (int64_t)(p.T / p.tt) * npy * npx;
      const int F = 3 * p.tt * p.tph * p.tpw;
      obase = b * Np * F + ((int64_t)(tt / p.tt) * npy * npx + j0 / p.tpw) * F + (tt % p.tt) * p.tph * p.tpw +
              j0 % p.tpw;
      cstride = p.tt * p.tph * p.tpw;
      small_step = p.tpw;
      big_step = npx * F - (p.tph - 1) * p.tpw;
      ph_rows = p.tph;
    }
  }
  const bool pair_store = has1 && (p.Wt & 1) == 0;
  const bool bf16 = p.out_dtype == AVB_DTYPE_BF16;
  uint8_t* dbase = reinterpret_cast<uint8_t*>(p.dst) + obase * (bf16 ? 2 : 4);
  // low bits of each row's global address (its misalignment inside the 16-byte-aligned copy)
  uint32_t alo = (uint32_t)reinterpret_cast<uintptr_t>(p.src + b * p.s_clip + (int64_t)(active ? t : t0) * p.s_t +
                                                       (int64_t)(y0 + ys) * p.s_h + (int64_t)x0 * (PL ? 1 : 3));
  const uint32_t sh_lo = (uint32_t)p.s_h;
  const uint8_t* slot = ring + (size_t)(active ? f : 0) * p.slot_bytes;
  const uint8_t* slot0 = slot;
  const int lane = tid & 31;

  const float2 sc2[3] = {make_float2(p.scale[0], p.scale[0]), make_float2(p.scale[1], p.scale[1]),
                         make_float2(p.scale[2], p.scale[2])};
  const float2 bi2[3] = {make_float2(p.bias[0], p.bias[0]), make_float2(p.bias[1], p.bias[1]),
                         make_float2(p.bias[2], p.bias[2])};
  // the row loop, instantiated per (output dtype, paired store): no per-emission dtype branches
  auto rows_loop = [&](auto bf16_tag, auto pair_tag) {
  constexpr bool BF16 = decltype(bf16_tag)::value, PAIR = decltype(pair_tag)::value;
  float2 acc[NOPEN][3];
#pragma unroll
  for (int q = 0; q < NOPEN; ++q)
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[q][c] = make_float2(0.f, 0.f);
  // output row r0's offset (rows advance small_step within a tubelet band of ph_rows, big_step across)
  int rowoff = (ph_rows >= (1 << 29)) ? r0 * small_step
                                      : (r0 / ph_rows) * (big_step + (ph_rows - 1) * small_step) + (r0 % ph_rows) * small_step;
  rph = (ph_rows >= (1 << 29)) ? 0 : r0 % ph_rows;
  int orow = r0;
  int s = 0;
  uint32_t ph = 0;
  for (int y = ys; y < ye; ++y) {
    tc::mbar_wait(&full[s], ph);
    const float4 rw = rowtab[y];
    float2 h[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    {
      const int mis = (int)(alo & 15u);
      if constexpr (PL) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          uint32_t s0[NW], s1[NW];
          k1_window<NW>(slot + c * p.cslot, mis + o0, s0);
          k1_window<NW>(slot + c * p.cslot, mis + o1, s1);
          K1HTapPL<NT>::run(s0, s1, wp, h[c]);
        }
      } else {
        uint32_t s0[NW], s1[NW];
        k1_window<NW>(slot, mis + o0, s0);
        k1_window<NW>(slot, mis + o1, s1);
        K1HTap<NT, 0>::run(s0, s1, wp, h[0]);
        K1HTap<NT, 1>::run(s0, s1, wp, h[1]);
        K1HTap<NT, 2>::run(s0, s1, wp, h[2]);
      }
    }
    tc::mbar_arrive(&empty[s]);
    alo += sh_lo;
    slot += stage_stride;
    if (++s == V4_RS) { s = 0; ph ^= 1; slot = slot0; }
    const float wq[3] = {rw.x, rw.y, rw.z};
#pragma unroll
    for (int q = 0; q < NOPEN; ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[q][c] = ffma2(make_float2(wq[q], wq[q]), h[c], acc[q][c]);
    const int ne = __float_as_int(rw.w);
    for (int e = 0; e < ne; ++e, ++orow) {
      if (active && orow >= i_lo && orow < i_hi) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float2 v = ffma2(acc[0][c], sc2[c], bi2[c]);
          const int oc = rowoff + c * cstride;
          if constexpr (BF16) {
            __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dbase) + oc;
            if constexpr (PAIR) {
              *reinterpret_cast<uint32_t*>(d) = pack_bf16x2(v.x, v.y);
            } else {
              d[0] = __float2bfloat16_rn(v.x);
              if (has1) d[1] = __float2bfloat16_rn(v.y);
            }
          } else {
            float* d = reinterpret_cast<float*>(dbase) + oc;
            if constexpr (PAIR) {
              *reinterpret_cast<float2*>(d) = v;
            } else {
              d[0] = v.x;
              if (has1) d[1] = v.y;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q + 1 < NOPEN; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[q][c] = acc[q + 1][c];
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[NOPEN - 1][c] = make_float2(0.f, 0.f);
      if (++rph == ph_rows) { rph = 0; rowoff += big_step; } else { rowoff += small_step; }
    }
  }
  };
  if (bf16) {
    if (pair_store) rows_loop(std::true_type{}, std::true_type{});
    else rows_loop(std::true_type{}, std::false_type{});
  } else {
    if (pair_store) rows_loop(std::false_type{}, std::true_type{});
    else rows_loop(std::false_type{}, std::false_type{});
  }
}

// K1 identity: the reference's fused-decode path (decoder.py:137-211,
// PAPER.md:666-668) hands over frames the CPU already cropped and scaled to the target -- the
// planar Batch.frames layout [B,T,3,Ht,Wt] (loader.py:99-116).  Full-frame boxes at identity scale
// reduce K1 to flip + normalize + cast + re-layout: one thread per 16 pixels of one channel row,
// one 16-byte load, two 16-byte bf16 stores (16 output columns are contiguous in every layout).
// Each thread moves kIdU chunks spaced one grid apart: all kIdU 16-byte loads are issued before the
// first store (HBM needs ~40 KB in flight per SM; one chunk per thread left it latency-bound at 65 %),
// and the chunk -> (clip, frame, channel, row, column) decode runs in 32-bit arithmetic (IDX = uint32_t)
// whenever the chunk count allows (the 64-bit divisions were most of the instructions).
#ifndef AVB_K1_ID_U
#define AVB_K1_ID_U 4
#endif
constexpr int kIdU = AVB_K1_ID_U;
template <typename IDX>
__global__ void __launch_bounds__(256) k1_identity_kernel(const K1Params p, int64_t nchunks) {
  const IDX n = (IDX)nchunks;
  const IDX stride = (IDX)gridDim.x * blockDim.x;
  const IDX cpr = (IDX)(p.Wt >> 4);                 // 16-pixel chunks per row
  const int64_t plane = (int64_t)p.Ht * p.Wt;
  for (IDX g0 = (IDX)blockIdx.x * blockDim.x + threadIdx.x; g0 < n; g0 += stride * kIdU) {
    uint4 v[kIdU];
    int64_t o[kIdU];
    int cf[kIdU];                                   // channel | flip << 2; -1: past the end
#pragma unroll
    for (int u = 0; u < kIdU; ++u) {
      const IDX gid = g0 + (IDX)u * stride;
      cf[u] = -1;
      if (gid >= n) continue;
      IDX r = gid / cpr;
      const int xc = (int)(gid - r * cpr);
      const IDX r2 = r / (IDX)p.Ht;                 // ((b*T + t)*3 + c)*Ht + y
      const int y = (int)(r - r2 * (IDX)p.Ht);
      const IDX r3 = r2 / 3u;
      const int c = (int)(r2 - r3 * 3u);
      const IDX bb = r3 / (IDX)p.T;
      const int t = (int)(r3 - bb * (IDX)p.T);
      const int64_t b = (int64_t)bb;
      const bool flip = p.flips ? (p.flips[b] != 0) : false;
      const int x0 = flip ? p.Wt - 16 * (xc + 1) : 16 * xc;   // source chunk (mirrored when flipped)
      const uint8_t* src = p.src + b * p.s_clip + (int64_t)t * p.s_t + (int64_t)c * p.s_c + (int64_t)y * p.s_h + x0;
      v[u] = __ldg(reinterpret_cast<const uint4*>(src));
      cf[u] = c | (flip ? 4 : 0);
      const int j = 16 * xc;
      if (p.out_layout == AVB_LAYOUT_CTHW) {
        o[u] = ((b * 3 + c) * p.T + t) * plane + (int64_t)y * p.Wt + j;
      } else if (p.out_layout == AVB_LAYOUT_TCHW) {
        o[u] = ((b * p.T + t) * 3 + c) * plane + (int64_t)y * p.Wt + j;
      } else {
        const int npy = p.Ht / p.tph, npx = p.Wt / p.tpw;
        const int64_t Np = (int64_t)(p.T / p.tt) * npy * npx;
        const int F = 3 * p.tt * p.tph * p.tpw;
        o[u] = (b * Np + ((int64_t)(t / p.tt) * npy + y / p.tph) * npx + j / p.tpw) * F +
               ((c * p.tt + t % p.tt) * p.tph + y % p.tph) * p.tpw + j % p.tpw;
      }
    }
#pragma unroll
    for (int u = 0; u < kIdU; ++u) {
      if (cf[u] < 0) continue;
      const int c = cf[u] & 3;
      uint4 w = v[u];
      if (cf[u] & 4) {  // reverse the 16 bytes
        w = make_uint4(__byte_perm(w.w, 0, 0x0123), __byte_perm(w.z, 0, 0x0123), __byte_perm(w.y, 0, 0x0123),
                       __byte_perm(w.x, 0, 0x0123));
      }
      const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
      const float sc = p.scale[c], bi = p.bias[c];
      float f[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) f[k] = fmaf((float)((wd[k >> 2] >> (8 * (k & 3))) & 0xffu), sc, bi);
      if (p.out_dtype == AVB_DTYPE_BF16) {
        uint4 lo, hi;
        lo.x = pack_bf16x2(f[0], f[1]); lo.y = pack_bf16x2(f[2], f[3]); lo.z = pack_bf16x2(f[4], f[5]); lo.w = pack_bf16x2(f[6], f[7]);
        hi.x = pack_bf16x2(f[8], f[9]); hi.y = pack_bf16x2(f[10], f[11]); hi.z = pack_bf16x2(f[12], f[13]); hi.w = pack_bf16x2(f[14], f[15]);
        uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.dst) + o[u]);
        d[0] = lo;
        d[1] = hi;
      } else {
        float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.dst) + o[u]);
#pragma unroll
        for (int k = 0; k < 4; ++k) d[k] = make_float4(f[4 * k], f[4 * k + 1], f[4 * k + 2], f[4 * k + 3]);
      }
    }
  }
}

// Host-side envelope for v4, in the exact-integer tap ranges of k1_taps: the most taps of any output
// column (nt) and the most output rows whose vertical windows share one source row (nopen).
static void k1_range(int crop, int tgt, int i, int& lo, int& hi) {
  const long long c2 = 2LL * tgt;
  auto fd = [](long long a, long long d) { long long q = a / d; if ((a % d != 0) && (a < 0)) --q; return q; };
  const long long l = fd((long long)crop * (2 * i - 1) + tgt, c2);
  const long long h = fd((long long)crop * (2 * i + 3) + tgt, c2);
  lo = (int)std::max(0LL, l);
  hi = (int)std::min((long long)crop, h);
}
static int k1_max_taps(int crop, int tgt) {
  int nt = 0;
  for (int j = 0; j < tgt; ++j) {
    int l, h;
    k1_range(crop, tgt, j, l, h);
    nt = std::max(nt, h - l);
  }
  return nt;
}
static int k1_max_open(int crop, int tgt) {
  std::vector<int> lo(tgt), hi(tgt);
  for (int i = 0; i < tgt; ++i) k1_range(crop, tgt, i, lo[i], hi[i]);
  int nlo = 0, base = 0, no = 0;  // open rows at source row y: base(y) .. #{lo <= y} - 1
  for (int y = 0; y < crop; ++y) {
    while (nlo < tgt && lo[nlo] <= y) ++nlo;
    while (base < tgt && hi[base] <= y) ++base;
    no = std::max(no, nlo - base);
  }
  return no;
}
// boxes given: exact over the batch; false if some box is not a downscale in both axes.
static bool k1v4_envelope(const int32_t* boxes, int64_t B, int Ht, int Wt, int& nt, int& nopen) {
  nt = 0;
  nopen = 0;
  for (int64_t bi = 0; bi < B; ++bi) {
    const int cw = boxes[4 * bi + 2], ch = boxes[4 * bi + 3];
    if (cw < Wt || ch < Ht) return false;
    nt = std::max(nt, k1_max_taps(cw, Wt));
    nopen = std::max(nopen, k1_max_open(ch, Ht));
  }
  return true;
}
// device-only boxes: worst case over every downscale crop that fits the frame (cached per geometry).
static void k1v4_envelope_all(int H, int W, int Ht, int Wt, int& nt, int& nopen) {
  struct Entry { int H, W, Ht, Wt, nt, nopen; };
  static thread_local std::vector<Entry> cache;
  for (const Entry& e : cache)
    if (e.H == H && e.W == W && e.Ht == Ht && e.Wt == Wt) { nt = e.nt; nopen = e.nopen; return; }
  nt = 0;
  nopen = 0;
  for (int cw = Wt; cw <= W; ++cw) nt = std::max(nt, k1_max_taps(cw, Wt));
  for (int ch = Ht; ch <= H; ++ch) nopen = std::max(nopen, k1_max_open(ch, Ht));
  cache.push_back({H, W, Ht, Wt, nt, nopen});
}

std::atomic<int> g_force_path{AVB_K1_PATH_AUTO};

}  // namespace

extern "C" int avb_k1_force_path(int path) {
  AVB_CHECK_ARG(path == AVB_K1_PATH_AUTO || path == AVB_K1_PATH_GENERIC || path == AVB_K1_PATH_STRIP,
                "bad K1 path %d", path);
  return g_force_path.exchange(path);
}

extern "C" int avb_rrc_taps(int crop, int tgt, int32_t* lo_dev, int32_t* hi_dev, float* w_dev,
                            int max_taps, void* stream) {
  AVB_CHECK_ARG(crop >= 1 && tgt >= 1, "crop/target must be >= 1");
  AVB_CHECK_ARG(lo_dev && hi_dev && w_dev, "null output pointer");
  AVB_CHECK_ARG(max_taps >= 1, "max_taps must be >= 1");
  k1_taps_kernel<<<(tgt + 127) / 128, 128, 0, avb::as_stream(stream)>>>(crop, tgt, lo_dev, hi_dev, w_dev,
                                                                          max_taps);
  return avb::launch_status("avb_rrc_taps");
}

static int rrc_normalize_impl(const uint8_t* src, int64_t B, int T, int H, int W, int64_t s_clip, int64_t s_t,
                              int64_t s_h, int64_t s_w, int64_t s_c, const int32_t* boxes_dev,
                              const uint8_t* hflip_dev, const int32_t* boxes_host, int Ht, int Wt,
                              const float* mean3, const float* inv_std3, int out_dtype, int out_layout, int tt,
                              int tph, int tpw, void* dst, void* stream) {
  AVB_CHECK_ARG(B >= 0 && T >= 1 && H >= 1 && W >= 1, "bad frame dims B=%lld T=%d H=%d W=%d",
                (long long)B, T, H, W);
  AVB_CHECK_ARG(Ht >= 1 && Wt >= 1, "target size must be >= 1 pixel");
  AVB_CHECK_ARG(out_dtype == AVB_DTYPE_BF16 || out_dtype == AVB_DTYPE_F32, "bad out_dtype %d", out_dtype);
  AVB_CHECK_ARG(out_layout == AVB_LAYOUT_CTHW || out_layout == AVB_LAYOUT_TCHW || out_layout == AVB_LAYOUT_TUBELET,
                "bad out_layout %d", out_layout);
  if (out_layout == AVB_LAYOUT_TUBELET)
    AVB_CHECK_ARG(tt >= 1 && tph >= 1 && tpw >= 2 && tpw % 2 == 0 && T % tt == 0 && Ht % tph == 0 && Wt % tpw == 0,
                  "tubelet %dx%dx%d must tile %dx%dx%d with an even width", tt, tph, tpw, T, Ht, Wt);
  AVB_CHECK_ARG(mean3 && inv_std3, "mean/inv_std must be given");
  if (B == 0) return AVB_OK;
  AVB_CHECK_ARG(src && boxes_dev && dst, "null device pointer");
  AVB_CHECK_ARG((reinterpret_cast<uintptr_t>(boxes_dev) & 15) == 0, "boxes must be 16-byte aligned");
  AVB_CHECK_ARG(s_c >= 0 && s_w >= 0 && s_h >= 0 && s_t >= 0 && s_clip >= 0, "negative strides");
  if (boxes_host) {
    for (int64_t i = 0; i < B; ++i) {
      const int32_t* bx = boxes_host + 4 * i;
      if (!(bx[0] >= 0 && bx[1] >= 0 && bx[2] >= 1 && bx[3] >= 1 && bx[0] + bx[2] <= W &&
            bx[1] + bx[3] <= H)) {
        avb::set_error("crop (%d, %d, %d, %d) of clip %lld outside frame geometry %dx%d", bx[0], bx[1],
                       bx[2], bx[3], (long long)i, W, H);
        return AVB_E_BOX;
      }
    }
  }
  // envelope: taps per output <= floor(2*crop/tgt) + 2 <= kMaxTaps for the largest possible crop
  const int tx_cap = (2 * W) / Wt + 2;
  const int ty_cap = (2 * H) / Ht + 2;
  if (tx_cap > kMaxTaps || ty_cap > kMaxTaps) {
    avb::set_error("downscale factor above %d taps (W/Wt=%d/%d, H/Ht=%d/%d)", kMaxTaps, W, Wt, H, Ht);
    return AVB_E_UNSUPPORTED;
  }
  K1Params p;
  p.src = src; p.B = B; p.T = T; p.H = H; p.W = W;
  p.s_clip = s_clip; p.s_t = s_t; p.s_h = s_h; p.s_w = s_w; p.s_c = s_c;
  p.boxes = boxes_dev; p.flips = hflip_dev; p.Ht = Ht; p.Wt = Wt;
  for (int c = 0; c < 3; ++c) {
    p.scale[c] = inv_std3[c] / 255.0f;
    p.bias[c] = -mean3[c] * inv_std3[c];
  }
  p.dst = dst; p.out_dtype = out_dtype; p.out_layout = out_layout;
  p.tt = tt; p.tph = tph; p.tpw = tpw;
  p.tx_cap = tx_cap; p.ty_cap = ty_cap;
  p.rowb_cap = ((3 * W + 15) / 16) * 16 + 16;
  p.fast = (s_c == 1 && s_w == 3) ? 1 : 0;
  const double sy = H > Ht ? (double)H / Ht : 1.0;
  size_t smem = 0;
  int R = 8;
  for (; R >= 1; R >>= 1) {
    p.R = R;
    p.rows_cap = (int)ceil(sy * (R + 1)) + 4;
    if (p.rows_cap > H) p.rows_cap = H;
    size_t head = sizeof(float) * ((size_t)Wt * tx_cap + (size_t)R * ty_cap) + sizeof(int) * (Wt + 2 * R);
    head = (head + 15) & ~size_t(15);
    smem = head + (size_t)p.rows_cap * p.rowb_cap + sizeof(float) * (size_t)R * p.rowb_cap;
    if (smem <= 200 * 1024) break;
  }
  if (R < 1) {
    avb::set_error("frame too wide for the shared-memory staging (W=%d)", W);
    return AVB_E_UNSUPPORTED;
  }
  if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(k1_rrc_normalize_kernel), 200 * 1024, "k1 attr"))
    return e;
  if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(k1v2_kernel), 200 * 1024, "k1 attr")) return e;
  const int force = g_force_path.load();
  // identity: full-frame boxes at the target size, planar rows (the fused-decode hand-off)
  if (boxes_host && H == Ht && W == Wt && s_w == 1 && Wt % 16 == 0 && force == AVB_K1_PATH_AUTO &&
      (out_layout != AVB_LAYOUT_TUBELET || tpw % 16 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
      s_h % 16 == 0 && s_c % 16 == 0 && s_t % 16 == 0 && s_clip % 16 == 0 &&
      ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
    bool ident = true;
    for (int64_t i = 0; i < B && ident; ++i)
      ident = boxes_host[4 * i] == 0 && boxes_host[4 * i + 1] == 0 && boxes_host[4 * i + 2] == W &&
              boxes_host[4 * i + 3] == H;
    if (ident) {
      const int64_t nchunks = B * (int64_t)T * 3 * Ht * (Wt / 16);
      const int64_t blocks = std::min<int64_t>((nchunks + 256 * kIdU - 1) / (256 * kIdU), 65535LL * 1024);
      if (nchunks < (1LL << 31) - 256LL * kIdU * 2)
        k1_identity_kernel<uint32_t><<<(unsigned)blocks, 256, 0, avb::as_stream(stream)>>>(p, nchunks);
      else
        k1_identity_kernel<uint64_t><<<(unsigned)blocks, 256, 0, avb::as_stream(stream)>>>(p, nchunks);
      return avb::launch_status("avb_rrc_normalize (identity)");
    }
  }
  // v4: streaming kernel for interleaved RGB downscales (every config-2 crop).  With host boxes
  //     the tap envelope is exact; with device-only boxes it is the worst case over every
  //     downscale crop and a complement launch of v2 covers any upscale clip.
  //     Planar rows ([B,T,3,H,W], the reference Batch layout) take the same kernel with one bulk copy
  //     per channel plane when the planes are 16-byte aligned and the boxes are on the host.
  bool v4_done = false, v4_partial = false;
  const bool pl = !p.fast && s_w == 1 && s_c % 16 == 0 && s_c >= W && boxes_host != nullptr;
  if ((p.fast || pl) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && force == AVB_K1_PATH_AUTO && Ht <= H &&
      Wt <= W && Wt <= 448 && T <= 65535 && B <= 65535 && 3LL * T * Ht * Wt < (1LL << 31)) {
    int nt = 0, nopen = 0, cw_max = W;
    bool ok = true;
    if (boxes_host) {
      ok = k1v4_envelope(boxes_host, B, Ht, Wt, nt, nopen);
      cw_max = 0;
      for (int64_t i = 0; i < B; ++i) cw_max = std::max(cw_max, (int)boxes_host[4 * i + 2]);
    } else {
      k1v4_envelope_all(H, W, Ht, Wt, nt, nopen);
      v4_partial = true;
    }
    if (ok && nt <= 8 && nopen <= 3) {
      const int NT = nt <= 4 ? 4 : nt <= 5 ? 5 : nt <= 6 ? 6 : 8;
      const int NOPEN = nopen <= 2 ? 2 : 3;
      const int NW = pl ? (NT + 3) / 4 : (3 * NT + 3) / 4;
      K1v4Params q;
      q.src = src; q.s_clip = s_clip; q.s_t = s_t; q.s_h = s_h;
      q.T = T; q.H = H; q.W = W; q.Ht = Ht; q.Wt = Wt;
      q.boxes = boxes_dev; q.flips = hflip_dev;
      for (int c = 0; c < 3; ++c) { q.scale[c] = p.scale[c]; q.bias[c] = p.bias[c]; }
      q.dst = dst; q.out_dtype = out_dtype; q.out_layout = out_layout; q.tt = tt; q.tph = tph; q.tpw = tpw;
      q.tpf = (Wt + 1) / 2;
      q.fpc = std::max(1, std::min(T, 224 / q.tpf));
#ifdef AVB_DEBUG_KNOBS
      if (const char* e = getenv("AVB_K1_FPC")) q.fpc = std::max(1, std::min(T, atoi(e)));
#endif
      q.ncomp = ((q.fpc * q.tpf + 31) / 32) * 32;
      // a window read ends <= 15 (misalignment) + 3*cw (planar: cw per channel) + 4*(NW+1) bytes into the slot
      q.s_c = s_c;
      q.cslot = pl ? ((cw_max + 4 * (NW + 1) + 15 + 15) / 16) * 16 : 0;
      q.slot_bytes = pl ? 3 * q.cslot : ((3 * cw_max + 4 * (NW + 1) + 15 + 15) / 16) * 16;
      q.total_bytes = (B - 1) * s_clip + (int64_t)(T - 1) * s_t + (int64_t)(H - 1) * s_h +
                      (pl ? 2 * s_c + (int64_t)W : (int64_t)W * 3);
      const size_t smem4 = sizeof(uint64_t) * 2 * V4_RS + sizeof(float4) * (size_t)H +
                           (size_t)V4_RS * q.fpc * q.slot_bytes;
      if (smem4 <= 200 * 1024) {
        // output-row bands per frame group: enough CTAs that the last wave is a small fraction
        // (config 2: 8 frame groups x 64 clips = 512 CTAs on 592 slots -> 2 bands, 1024 CTAs)
        const int64_t groups = (int64_t)((T + q.fpc - 1) / q.fpc) * B;
        const int64_t slots = (int64_t)avb::sm_count() * 4;
        q.nband = groups >= 2 * slots ? 1 : (groups * 2 >= slots ? 2 : 4);   // same-box sweep: 1/2/3/4/6 bands
                                                                          // = 0.280/0.243/0.252/0.245/0.252 ms
        q.nband = std::min(q.nband, std::max(1, Ht / 16));
#ifdef AVB_DEBUG_KNOBS
        if (const char* e = getenv("AVB_K1_NBAND")) q.nband = std::max(1, std::min(Ht, atoi(e)));
#endif
        dim3 g4((unsigned)(((T + q.fpc - 1) / q.fpc) * q.nband), (unsigned)B);
        int ast = AVB_OK;
        auto launch = [&](auto kern) {
          ast = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(kern), 200 * 1024, "k1 v4 attr");
          if (ast == AVB_OK) kern<<<g4, q.ncomp + 32, smem4, avb::as_stream(stream)>>>(q);
        };
        auto by_nt = [&](auto nopen_c) {
          constexpr int NO = decltype(nopen_c)::value;
          if (pl) {
            if (NT == 4) launch(k1v4_kernel<4, NO, true>);
            else if (NT == 5) launch(k1v4_kernel<5, NO, true>);
            else if (NT == 6) launch(k1v4_kernel<6, NO, true>);
            else launch(k1v4_kernel<8, NO, true>);
            return;
          }
          if (NT == 4) launch(k1v4_kernel<4, NO>);
          else if (NT == 5) launch(k1v4_kernel<5, NO>);
          else if (NT == 6) launch(k1v4_kernel<6, NO>);
          else launch(k1v4_kernel<8, NO>);
        };
        if (NOPEN == 2) by_nt(std::integral_constant<int, 2>{});
        else by_nt(std::integral_constant<int, 3>{});
        if (ast != AVB_OK) return ast;
        const int st = avb::launch_status("avb_rrc_normalize");
        if (st != AVB_OK || !v4_partial) return st;
        v4_done = true;
      }
    }
  }
  const bool v2ok = p.fast && (s_h % 4 == 0) && (s_t % 4 == 0) && (s_clip % 4 == 0) &&
                    ((reinterpret_cast<uintptr_t>(src) & 3) == 0) && force != AVB_K1_PATH_GENERIC;
  if (v2ok) {
    K1v2Params q;
    q.src = src; q.s_clip = s_clip; q.s_t = s_t; q.s_h = s_h;
    q.T = T; q.H = H; q.W = W; q.Ht = Ht; q.Wt = Wt;
    q.boxes = boxes_dev; q.flips = hflip_dev;
    for (int c = 0; c < 3; ++c) { q.scale[c] = p.scale[c]; q.bias[c] = p.bias[c]; }
    q.dst = dst; q.out_dtype = out_dtype; q.out_layout = out_layout; q.tt = tt; q.tph = tph; q.tpw = tpw;
    q.tx_cap = tx_cap; q.ty_cap = ty_cap;
    q.total_bytes = (B - 1) * s_clip + (int64_t)(T - 1) * s_t + (int64_t)(H - 1) * s_h + (int64_t)W * 3;
    q.only_upscale = v4_done ? 1 : 0;
    q.strips = Wt >= 160 ? 2 : 1;
    q.cps = (Wt + q.strips - 1) / q.strips;
    // worst-case strip source width: every column of a full-width crop
    const int strip_src = (int)std::min<int64_t>(W, (int64_t)((double)W / Wt * q.cps) + tx_cap + 2);
    q.rowb_cap = ((strip_src * 3 + 15 + 16 + 4) / 16) * 16;
    size_t smem = 0;
    for (q.R = 16; q.R >= 1; q.R >>= 1) {
      q.rows_cap = std::min(H, (int)ceil(sy * (q.R + 1)) + 4);
      size_t head = sizeof(float) * ((size_t)q.cps * tx_cap + (size_t)Ht * ty_cap) +
                    sizeof(int) * (2 * (size_t)q.cps + 2 * (size_t)Ht + 2 * (size_t)q.rows_cap);
      head = (head + 15) & ~size_t(15);
      smem = head + 2 * (size_t)q.rows_cap * q.rowb_cap + sizeof(float) * (size_t)q.R * q.rowb_cap;
      if (smem <= 100 * 1024) break;
    }
    if (q.R >= 1) {
      dim3 g2(q.strips, T, (unsigned)B);
      k1v2_kernel<<<g2, kThreads, smem, avb::as_stream(stream)>>>(q);
      return avb::launch_status("avb_rrc_normalize");
    }
  }
  p.only_upscale = v4_done ? 1 : 0;
  dim3 grid((Ht + R - 1) / R, T, (unsigned)B);
  AVB_CHECK_ARG(B <= 65535 && T <= 65535, "B and T must be <= 65535");
  k1_rrc_normalize_kernel<<<grid, kThreads, smem, avb::as_stream(stream)>>>(p);
  return avb::launch_status("avb_rrc_normalize");
}

extern "C" int avb_rrc_normalize(const uint8_t* src, int64_t B, int T, int H, int W, int64_t s_clip, int64_t s_t,
                                 int64_t s_h, int64_t s_w, int64_t s_c, const int32_t* boxes_dev,
                                 const uint8_t* hflip_dev, const int32_t* boxes_host, int Ht, int Wt,
                                 const float* mean3, const float* inv_std3, int out_dtype, int out_layout, void* dst,
                                 void* stream) {
  AVB_CHECK_ARG(out_layout != AVB_LAYOUT_TUBELET, "use avb_rrc_normalize_tubelet for the tubelet layout");
  return rrc_normalize_impl(src, B, T, H, W, s_clip, s_t, s_h, s_w, s_c, boxes_dev, hflip_dev, boxes_host, Ht, Wt,
                            mean3, inv_std3, out_dtype, out_layout, 1, 1, 2, dst, stream);
}

extern "C" int avb_rrc_normalize_tubelet(const uint8_t* src, int64_t B, int T, int H, int W, int64_t s_clip,
                                         int64_t s_t, int64_t s_h, int64_t s_w, int64_t s_c,
                                         const int32_t* boxes_dev, const uint8_t* hflip_dev,
                                         const int32_t* boxes_host, int Ht, int Wt, const float* mean3,
                                         const float* inv_std3, int out_dtype, int tub_t, int tub_h, int tub_w,
                                         void* dst, void* stream) {
  return rrc_normalize_impl(src, B, T, H, W, s_clip, s_t, s_h, s_w, s_c, boxes_dev, hflip_dev, boxes_host, Ht, Wt,
                            mean3, inv_std3, out_dtype, AVB_LAYOUT_TUBELET, tub_t, tub_h, tub_w, dst, stream);
}
