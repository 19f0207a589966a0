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

}  // namespace

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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k1_rrc_normalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
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
