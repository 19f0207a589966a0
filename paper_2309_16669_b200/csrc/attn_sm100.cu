// K4/K5: blockwise (Flash-style) attention forward/backward on tcgen05, head_dim 64.
//
// PAPER.md:265-272, :350-357 (O(N) memory: no N x N tensor is stored; the memory
// contract the reference models at models.py:137-140 -- O plus per-row statistics).
// No reference code exists for the kernels themselves.
//
// Layout: Q/K/V/O are [B, N, H, 64] bf16 views with row stride `ld` and batch stride `sb`
// (elements), e.g. the packed QKV GEMM output [B*N, 3*H*64] with q=qkv, k=qkv+D, v=qkv+2D.
// LSE is fp32 [B*H, Npad], Npad = roundup(N, 128); the backward's statistics travel as per-query-tile
// extension tiles of the S^T / dP^T MMAs (kExtTile, 32 bytes per row).
//
// Forward (K4), one CTA per (two 128-query tiles, head, clip), 2 CTAs per SM (~100 KB smem, 256 TMEM
// columns each), 320 threads:
//   warp 8  TMA: both Q tiles once, then K_j/V_j (64-key tiles) through a 4-stage ring
//   warp 9  MMA (all lanes run the loop, one elected lane issues): S_g = Q_g K_j^T (M128 N64 K64, SS)
//           into TMEM; O_g += P_g V_j (M128 N64 K64, A = P_g read from TMEM, V MN-major)
//   warps 0-7 two softmax groups (group g = warps 4g..4g+3, thread = query row): row max over S_g,
//           exp2 (2 of 8 pairs on the FMA pipe), bf16 P_g packed over the consumed S_g columns, lazy
//           (> 2^8) rescale of O_g in TMEM; O / LSE written at the end.
// Backward (K5), persistent, one CTA per SM walking (128-key tile, head, clip) items, 704 threads:
//   warp 21 MMA: dV += P^T dO, S^T = K Q^T - lse/scale (next step), dK += dS^T Q,
//           dP^T = V dO^T - delta (next step), dQ = dS K -- K and V live in TMEM as the A operands of
//           S^T / dP^T, the statistics enter as a fifth K step (see kExtTile);
//   warp 20 TMA: K/V per item, Q/dO/extension tile (-lse/scale, -delta) through a 3-stage ring;
//   warps 0-15 (quadrant = w & 3 -> key rows, chunk = w >> 2 -> 32 queries): P^T = exp2(...) over the
//           S^T chunk (TMEM), then dS^T = P^T (dP^T - delta) over the dP^T chunk (TMEM) and into a
//           128B-swizzled smem tile (dQ's A operand), P kept in registers between the two;
//   warps 16-19 drain: dQ TMEM -> bf16 smem staging -> TMA reduce-add into the bf16 dq rows (or fp32
//           staging into an fp32 accumulator + a convert kernel, fp32_dq); at an item's end dK / dV
//           TMEM -> bf16 -> TMA stores.
#include "tc_common.cuh"

#include <cstdlib>
#include <type_traits>

namespace {

constexpr int HD = 64;
constexpr int BT = 128;  // tile rows (queries or keys)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return r;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return r;
}
// 2^x for a pair on the FMA pipe (FA4-style MUFU offload): round-to-nearest split x = j + f with the
// 1.5*2^23 magic add, a degree-3 minimax polynomial for 2^f on [-0.5, 0.5] (max rel. error 7.5e-5,
// far below the bf16 rounding of P), and j added straight into the exponent bits.
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c);
__device__ __forceinline__ float2 f2add(float2 a, float2 b);
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = f2add(x, make_float2(12582912.f, 12582912.f));
  const float2 j = f2add(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = f2fma(j, make_float2(-1.f, -1.f), x);
  float2 p = f2fma(f, make_float2(0.055157460272312164f, 0.055157460272312164f),
                   make_float2(0.24261002242565155f, 0.24261002242565155f));
  p = f2fma(p, f, make_float2(0.693263590335846f, 0.693263590335846f));
  p = f2fma(p, f, make_float2(0.9999282360076904f, 0.9999282360076904f));
  return make_float2(__int_as_float(__float_as_int(t.x) * (1 << 23) + __float_as_int(p.x)),
                     __int_as_float(__float_as_int(t.y) * (1 << 23) + __float_as_int(p.y)));
}

__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return r;
}

// write 8 consecutive bf16 (one 16B unit) of row `row` into a K-major SW128 tile set
// (tiles of [128 rows][64 cols], 16 KB each); col8 = column / 8 (0..15)
__device__ __forceinline__ void st_sw128(uint8_t* base, int row, int col8, uint4 v) {
  const int tile = col8 >> 3, u = col8 & 7;
  *reinterpret_cast<uint4*>(base + tile * 16384 + row * 128 + ((u ^ (row & 7)) << 4)) = v;
}

struct FwdArgs {
  int B, H, N, Npad;
  float scale_log2;
  __nv_bfloat16* o;
  int64_t ld_o, sb_o;
  float* lse;
  int causal;
  long long* trace;   // debug: per-tile clock64 events of CTA (0,0,0) (AVB_ATTN_FTRACE), else null
};

constexpr int FKB = 64;
// Debug timelines (scripts/trace_attn_{fwd,bwd}.py) are compiled in only with
// -DAVB_ATTN_TRACE_HOOKS (AVB_NVCC_DEFS at build time): the checks cost ~6 % in the forward.
#ifdef AVB_ATTN_TRACE_HOOKS
#define FWD_TRACE(ev, j)                                                                              \
  do {                                                                                                \
    if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0 && (j) < 64)    \
      a.trace[(j) * 16 + (ev)] = clock64();                                                           \
  } while (0)
#else
#define FWD_TRACE(ev, j) \
  do {                   \
  } while (0)
#endif                               // key tile
constexpr int F_STAGES = 4;
constexpr int F_SQ = 0;                               // 2 Q tiles (A, B) x 16 KB
constexpr int F_SKV = 32768;                          // F_STAGES x (K 8 KB + V 8 KB)
constexpr int F_BAR = F_SKV + F_STAGES * 16384;
constexpr int F_SMEM = F_BAR + 256 + 1024;   // + alignment slack
static_assert(F_SMEM <= 115712, "attn fwd: two CTAs per SM");

// TMEM (256 columns per CTA, 2 CTAs/SM -> four softmax groups per SM), per query tile g in {0,1}:
//   S_g fp32 [64 key columns] at 64*g, overwritten in place by P_g (bf16 pairs, 32 columns) as the
//   same thread consumes it; O_g fp32 at 128 + 64*g
constexpr float kRescaleThresh = 8.0f;  // log2 units: rescale O only when the running max grows by > 2^8
#ifndef AVB_FWD_POLY_FROM
#define AVB_FWD_POLY_FROM 6
#endif
constexpr int kFwdPolyFrom = AVB_FWD_POLY_FROM;  // exp2 pairs (e2 & 7) >= this go to the FMA pipe (2 of 8: measured best of 0-4)

__global__ void __launch_bounds__(320, 2)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const FwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // two CTAs per SM: align the 128B-swizzled tiles to 1 KB inside the window ourselves
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + F_SQ;
  uint8_t* sKV = smem + F_SKV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + F_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;              // [F_STAGES]
  uint64_t* kv_empty = bars + 1 + F_STAGES;  // [F_STAGES]
  uint64_t* gb = bars + 1 + 2 * F_STAGES;    // per group g: s_full, s_free, p_full, o_full at gb + 4g
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gb + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = blockIdx.x * 2 * BT;
  const bool hasB = q0 + BT < a.N;
  const int ng = hasB ? 2 : 1;
  const int nkv_all = (a.N + FKB - 1) / FKB;
  const int nkv = a.causal ? min(nkv_all, (q0 + ng * BT - 1) / FKB + 1) : nkv_all;

  if (warp == 8 && lane == 0) {
    tc::tma_prefetch(&tmQ);
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < F_STAGES; ++s) {
      tc::mbar_init(&kv_full[s], 1);
      tc::mbar_init(&kv_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      tc::mbar_init(gb + 4 * g + 0, 1);  // s_full
      tc::mbar_init(gb + 4 * g + 1, 4);  // s_free
      tc::mbar_init(gb + 4 * g + 2, 4);  // p_full
      tc::mbar_init(gb + 4 * g + 3, 1);  // o_full
    }
    tc::fence_barrier_init();
  }
  if (warp == 9) tc::tmem_alloc(tmem_slot, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(q_full, 16384 * ng);
      tc::tma_load_3d(sQ, &tmQ, q_full, h * HD, q0, b);
      if (hasB) tc::tma_load_3d(sQ + 16384, &tmQ, q_full, h * HD, q0 + BT, b);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % F_STAGES;
        tc::mbar_wait(&kv_empty[st], ((j / F_STAGES) & 1) ^ 1);
        FWD_TRACE(9, j);
        tc::mbar_arrive_expect_tx(&kv_full[st], 16384);
        tc::tma_load_3d(sKV + st * 16384, &tmK, &kv_full[st], h * HD, j * FKB, b);
        tc::tma_load_3d(sKV + st * 16384 + 8192, &tmV, &kv_full[st], h * HD, j * FKB, b);
      }
    }
  } else if (warp == 9) {
    {   // all 32 lanes run the issue loop (warp-uniform values); one elected lane issues
      constexpr uint32_t idS = tc::idesc_bf16_f32(128, FKB, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16_f32(128, 64, 0, 1);   // A = P from TMEM, B = V MN-major
      const uint32_t aQ = smem_u32(sQ);
      auto issue_s = [&](int g, int j) {
        const uint32_t aK = smem_u32(sKV + (j % F_STAGES) * 16384);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc::umma_f16_ss_w(tmem + 64 * g, tc::sdesc_sw128(aQ + g * 16384 + kk * 32, 16, 1024),
                          tc::sdesc_sw128(aK + kk * 32, 16, 1024), idS, kk > 0);
        tc::umma_commit_w(gb + 4 * g + 0);
      };
      auto issue_pv = [&](int g, int j) {
        const uint32_t aV = smem_u32(sKV + (j % F_STAGES) * 16384 + 8192);
#pragma unroll
        for (int kk = 0; kk < FKB / 16; ++kk)
          tc::umma_f16_ts_w(tmem + 128 + 64 * g, tmem + 64 * g + kk * 8,
                          tc::sdesc_sw128(aV + kk * 2048, 8192, 1024), idO, (j > 0 || kk > 0) ? 1u : 0u);
        tc::umma_commit_w(gb + 4 * g + 3);
      };
      tc::mbar_wait(q_full, 0);
      tc::mbar_wait(&kv_full[0], 0);
      tc::tc_fence_after();
      for (int g = 0; g < ng; ++g) issue_s(g, 0);
      for (int j = 0; j < nkv; ++j) {
        const bool more = j + 1 < nkv;
        if (more) tc::mbar_wait(&kv_full[(j + 1) % F_STAGES], ((j + 1) / F_STAGES) & 1);
        for (int g = 0; g < ng; ++g) {
          FWD_TRACE(g == 0 ? 0 : 10, j);
          tc::mbar_wait(gb + 4 * g + 2, j & 1);    // P_g(j) in TMEM, S_g(j) consumed
          tc::tc_fence_after();
          issue_pv(g, j);
          if (more) issue_s(g, j + 1);
          FWD_TRACE(g == 0 ? 1 : 2, j);
        }
        tc::umma_commit_w(&kv_empty[j % F_STAGES]);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax groups (thread = query row)
    const int g = warp >> 2, quad = warp & 3;
    if (g < ng) {
      uint64_t* s_full = gb + 4 * g;
      uint64_t* p_full = s_full + 2;
      uint64_t* o_full = s_full + 3;
      const uint32_t tS = tmem + 64 * g, tP = tS, tO = tmem + 128 + 64 * g;
      const int row = quad * 32 + lane;
      const int qi = q0 + g * BT + row;
      const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
      float m_run = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        tc::mbar_wait(s_full, j & 1);
        if (quad == 0) FWD_TRACE(g == 0 ? 3 : 7, j);
        tc::tc_fence_after();
        const int kv0 = j * FKB;
        int lim = a.N - kv0;
        if (a.causal) lim = min(lim, qi - kv0 + 1);
        // pass 1: row max (one TMEM round trip of 64 columns), 8 independent max chains
        const bool full = lim >= FKB;  // warp-uniform in the non-causal case: no per-element masking
        float mxa[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mxa[k] = -INFINITY;
        {
          uint32_t r0[32], r1[32];
          tc::tmem_ld_32x32b_x32(tS + lane_off, r0);
          tc::tmem_ld_32x32b_x32(tS + lane_off + 32, r1);
          tc::tmem_ld_wait();
          if (full) {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              mxa[e & 7] = fmaxf(mxa[e & 7], __uint_as_float(r0[e]));
              mxa[e & 7] = fmaxf(mxa[e & 7], __uint_as_float(r1[e]));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              if (e < lim) mxa[e & 7] = fmaxf(mxa[e & 7], __uint_as_float(r0[e]));
              if (32 + e < lim) mxa[e & 7] = fmaxf(mxa[e & 7], __uint_as_float(r1[e]));
            }
          }
        }
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        const float m_new = fmaxf(m_run, mx * a.scale_log2);
        if (quad == 0 && g == 0) FWD_TRACE(4, j);
        if (j > 0) {
          tc::mbar_wait(o_full, (j - 1) & 1);  // PV(j-1) done: O stable, P buffer free
          if (quad == 0 && g == 0) FWD_TRACE(5, j);
          tc::tc_fence_after();
        }
        // warp-uniform lazy rescale of the TMEM accumulator (tcgen05.ld/st are warp-collective)
        const bool need = (m_run == -INFINITY) ? (m_new != -INFINITY) : (m_new > m_run + kRescaleThresh);
        if (j > 0 && __any_sync(0xffffffff, need)) {
          const float alpha = (m_run == -INFINITY) ? 0.f : ex2(m_run - m_new);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32(tO + lane_off + c * 32, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tc::tmem_st_32x32b_x32(tO + lane_off + c * 32, r);
          }
          l *= alpha;
          m_run = m_new;
        } else if (j == 0) {
          m_run = m_new;
        }
        const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
        // pass 2: p = exp2(s*scale - m) (3 of every 8 pairs on the FMA pipe, the rest on MUFU), row sum
        // (2 f32x2 chains), bf16 P packed over the consumed S columns (P chunk c -> columns [16c, 16c+16),
        // inside S chunk 0 which this thread has already read)
        float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sl2 = make_float2(a.scale_log2, a.scale_log2), nm2 = make_float2(-m_use, -m_use);
        auto pass2 = [&](auto full_tag) {
          constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
          for (int c = 0; c < FKB / 32; ++c) {
            uint32_t rb[1][32];
            tc::tmem_ld_32x32b_x32(tS + lane_off + c * 32, rb[0]);
            tc::tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int e2 = 0; e2 < 16; ++e2) {
              const int col = c * 32 + 2 * e2;
              const float2 x = f2fma(make_float2(__uint_as_float(rb[0][2 * e2]), __uint_as_float(rb[0][2 * e2 + 1])),
                                     sl2, nm2);
              float2 p = ((e2 & 7) >= kFwdPolyFrom) ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
              if (!FULL) {
                p.x = (col < lim) ? p.x : 0.f;
                p.y = (col + 1 < lim) ? p.y : 0.f;
              }
              sum2[e2 & 1] = f2add(sum2[e2 & 1], p);
              pk[e2] = pack_bf16x2(p.x, p.y);
            }
            tc::tmem_st_32x32b_x16(tP + lane_off + c * 16, pk);
          }
        };
        if (__all_sync(0xffffffffu, full))  // tcgen05.ld/st are warp-collective: branch warp-uniformly
          pass2(std::true_type{});
        else
          pass2(std::false_type{});
        const float2 sm2 = f2add(sum2[0], sum2[1]);
        const float sm4[4] = {sm2.x, sm2.y, 0.f, 0.f};
        l += (sm4[0] + sm4[1]) + (sm4[2] + sm4[3]);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full);   // also frees S_g for S_g(j+1)
        if (quad == 0) FWD_TRACE(g == 0 ? 6 : 8, j);
      }
      tc::mbar_wait(o_full, (nkv - 1) & 1);
      tc::tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* dst = a.o + (int64_t)b * a.sb_o + (int64_t)qi * a.ld_o + h * HD;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
        tc::tmem_ld_32x32b_x32(tO + lane_off + c * 32, r);
        tc::tmem_ld_wait();
        if (qi < a.N) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(r[u * 8 + 0]) * inv, __uint_as_float(r[u * 8 + 1]) * inv);
            v.y = pack_bf16x2(__uint_as_float(r[u * 8 + 2]) * inv, __uint_as_float(r[u * 8 + 3]) * inv);
            v.z = pack_bf16x2(__uint_as_float(r[u * 8 + 4]) * inv, __uint_as_float(r[u * 8 + 5]) * inv);
            v.w = pack_bf16x2(__uint_as_float(r[u * 8 + 6]) * inv, __uint_as_float(r[u * 8 + 7]) * inv);
            reinterpret_cast<uint4*>(dst + c * 32)[u] = v;
          }
        }
      }
      if (qi < a.N)
        a.lse[(int64_t)(b * a.H + h) * a.Npad + qi] = (l > 0.f) ? (m_run + __log2f(l)) * kLn2 : -INFINITY;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------------------------- backward
struct BwdArgs {
  int B, H, N, Npad;
  float scale, scale_log2;
  const uint8_t* ext;     // [B*H][Npad/128] 4 KB K-extension tiles (written by the pre kernel), see kExt*
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int64_t ld_g, sb_g;     // strides of dk/dv
  int causal;
  int nkt, items;         // key tiles per (clip, head); work items = B * H * nkt (persistent grid)
  long long* trace;       // debug: per-step clock64 events of CTA 0 (AVB_ATTN_TRACE), else null
  int dbg;                // trace-build experiment flags (AVB_ATTN_DBG): 1 skip the dQ drain, 2 skip the dS smem
                          // stores, 4 skip the dS-phase TMEM ld/st, 8 skip the exp-phase TMEM ld/st, 16 no exp2
  int dq_det;             // 1 (deterministic mode): dQ_g of key tile kt is stored (not added) into fp32 slice kt of
                          // dq_acc [nkt][B, N, H, 64]; the convert kernel sums the slices in key-tile order
  int dq_bf16;            // 1: dQ_g (scaled) reduce-added straight into the bf16 dq view; 0: into the fp32
                          // accumulator (+ a convert kernel)
};

// The per-query softmax statistics ride inside the MMAs instead of being loaded by every compute
// warp: each S^T / dP^T MMA gets a fifth K=16 step against a per-query-tile "extension" tile
//   ext[q][0..1]  = bf16 hi/lo of -lse_q/scale   (so S'^T = S^T - lse/scale, and the compute warps
//   ext[q][8..9]  = bf16 hi/lo of -delta_q        form P = exp2(S' * scale*log2e) with one FMUL2)
//   (all other columns 0)                         (dP'^T = dP^T - delta, dS = P * dP')
// whose A operand is a constant key-side tile with ones in columns 0-1 (S) or 8-9 (dP).  The hi/lo
// split keeps the folded terms to ~2^-17 relative.  Tiles use the canonical no-swizzle K-major layout
// (core matrices of 8 rows x 16 B; byte (q, k) at (q/8)*256 + (k/8)*128 + (q%8)*16 + (k%8)*2).
constexpr int kExtTile = 4096;     // one [128 queries x 16] bf16 extension tile
constexpr int kOnesBytes = 6144;   // 16 row groups x [zeros | (1,1,0..) | zeros] core matrices (384 B apart)

// smem (dynamic base must be 1 KB aligned; checked): all 128B-swizzled bf16 tiles first.
// dS^T is the only tile the compute warps stage in smem (A operand of dK and, seen MN-major, of
// dQ); once dK/dQ of a step have completed, its buffer doubles as the staging of that step's dQ
// drain.
constexpr int B_QD_STAGES = 3;
constexpr int B_SK = 0, B_SV = 16384;
constexpr int B_SQD = 32768;                               // 3 stages x (Q 16K + dO 16K)
constexpr int B_SDS = B_SQD + B_QD_STAGES * 32768;         // 2 buffers x dS^T 32K (then dQ staging)
constexpr int B_SEXT = B_SDS + 2 * 32768;                  // 3 stages x extension tile 4K
constexpr int B_SK2 = B_SEXT + B_QD_STAGES * kExtTile;     // second K buffer (next work item)
constexpr int B_SONE = B_SK2 + 16384;                      // constant ones tiles (A of the fifth K step)
constexpr int B_BAR = B_SONE + kOnesBytes;
constexpr int B_SMEM = B_BAR + 256;
static_assert(B_SK2 % 1024 == 0, "attn bwd K2 alignment");
static_assert(B_SMEM <= 232448, "attn bwd smem");
constexpr int kBwdCompute = 16;              // compute warps: 4 per TMEM lane quadrant (one 32-query chunk each)
constexpr int kBwdDrain = 4;                 // dQ drain warps: one per TMEM lane quadrant
#ifndef AVB_BWD_POLY8_FROM
#define AVB_BWD_POLY8_FROM 6
#endif
constexpr int kBwdPoly8From = AVB_BWD_POLY8_FROM; // pairs with (index & 7) >= this take the FMA-pipe exp2
                                                // (same-box sweep 4/5/6: 1.503 / 1.475 / 1.436 ms at config 4)
constexpr int kBwdWarps = kBwdCompute + kBwdDrain + 2;
#ifndef AVB_BWD_DS_BF16X2
#define AVB_BWD_DS_BF16X2 1
#endif

#ifdef AVB_ATTN_TRACE_HOOKS
#define BWD_TRACE(ev, ii)                                                                       \
  do {                                                                                          \
    if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0 && (ii) < 1024) \
      a.trace[(ii) * 32 + (ev)] = clock64();                                                        \
  } while (0)
#define BWD_TRACE_NS(ev, ii)                                                                    \
  do {                                                                                          \
    if (a.trace && blockIdx.x == 0 && lane == 0 && (ii) < 1024) {                               \
      uint64_t ns;                                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));                                    \
      a.trace[(ii) * 32 + (ev)] = (long long)ns;                                                \
    }                                                                                           \
  } while (0)
#define BWD_DBG(f) ((a.dbg & (f)) != 0)
#else
#define BWD_DBG(f) false
#define BWD_TRACE(ev, ii) \
  do {                    \
  } while (0)
#define BWD_TRACE_NS(ev, ii) \
  do {                       \
  } while (0)
#endif


__device__ __forceinline__ float2 unpack_bf16x2(uint32_t v) {
  return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
}

// Persistent: gridDim.x CTAs (one per SM, 22 warps) walk work items w = blockIdx.x, +gridDim.x, ...;
// item w = (128-key tile kt, head h, clip b).  One global step counter g runs over every (item,
// query tile) pair of the CTA, so every per-step barrier keeps its phase across item boundaries
// and the pipeline never drains between items: the next item's K/V are loaded (second K buffer)
// and copied into TMEM while the current item's last tiles run, its first S^T / dP^T MMAs are
// issued in the slot the current item's S_{i+1} would take, and the dK/dV epilogue is done by the
// drain warps while the compute warps already work on the next item.  Per step g (TMEM lanes = keys):
//   MMA warp:  dV += P_g^T dO_g (A = P^T from TMEM) | S_{g+1}^T = K Q_{g+1}^T (A = K from TMEM)
//              dK += dS_g^T Q_g (A = dS^T from TMEM) | dP_{g+1}^T = V dO_{g+1}^T (A = V from TMEM)
//              dQ_g = dS_g K (dS^T smem tile, MN-major; K from smem) -> mma_done
//   exp group (warps 0-7): P^T = exp2(S^T*scale*log2e - lse*log2e) -> bf16 over S^T (TMEM)
//   dS group (warps 8-15): dS^T = P^T (dP^T - delta) -> bf16 over dP^T (TMEM) and into smem
//   drain warps 16-19: dQ_g TMEM -> 128B-swizzled fp32 staging (the dS^T_g buffer) -> TMA reduce-add;
//                      after an item's last step, its dK / dV TMEM -> bf16 global
//   warp 20 TMA (K, V per item; Q/dO/extension 3-stage ring), warp 21 MMA.
struct BwdItem {
  int kt, h, b, i0, nq;
};

__device__ __forceinline__ BwdItem bwd_item(const BwdArgs& a, int w) {
  BwdItem t;
  t.kt = w % a.nkt;
  const int r = w / a.nkt;
  t.h = r % a.H;
  t.b = r / a.H;
  t.i0 = a.causal ? t.kt : 0;   // first query tile that sees this key tile
  t.nq = a.nkt - t.i0;
  return t;
}

__global__ void __launch_bounds__(32 * kBwdWarps, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ CUtensorMap tmDK,
                    const __grid_constant__ CUtensorMap tmDV, const BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((reinterpret_cast<uintptr_t>(smem) & 1023) != 0) __trap();
  auto sKb = [&](int it) { return smem + ((it & 1) ? B_SK2 : B_SK); };   // K double buffer (per work item)
  uint8_t* sV = smem + B_SV;
  uint8_t* sQD = smem + B_SQD;
  uint8_t* sDS = smem + B_SDS;
  uint8_t* sEXT = smem + B_SEXT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + B_BAR);
  uint64_t* kv_full = bars + 0;                  // per item: K_it, V_it in smem
  uint64_t* qd_full = bars + 1;                  // [3]
  uint64_t* qd_empty = bars + 1 + B_QD_STAGES;   // [3]
  uint64_t* s_full = bars + 1 + 2 * B_QD_STAGES;
  uint64_t* dp_full = s_full + 1;
  uint64_t* ds_ready = s_full + 2;
  uint64_t* mma_done = s_full + 3;
  uint64_t* dq_free = s_full + 4;
  uint64_t* stage_free = s_full + 5;             // [2]
  uint64_t* acc_free = s_full + 7;               // per item: dK / dV read out of TMEM by the drain warps
  uint64_t* p_ready = s_full + 8;                // P_g^T stored in TMEM by every compute warp
  uint64_t* kv_tmem = s_full + 9;                // per item: K and V copied into TMEM (A operands of S^T / dP^T)
  uint64_t* kst_free = s_full + 11;              // [2] per item: its K buffer is free (dQ MMAs done, dK/dV staged out)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 13);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stride = gridDim.x;
  constexpr int kDrain0 = kBwdCompute, kTMA = kBwdCompute + kBwdDrain, kMMA = kTMA + 1;
  for (int i = threadIdx.x; i < kOnesBytes / 16; i += blockDim.x) {   // 16-byte rows of core matrices
    const bool one = ((i >> 3) % 3) == 1;   // middle core matrix of each 8-row group: (1, 1, 0, ..., 0)
    *reinterpret_cast<uint4*>(smem + B_SONE + 16 * i) = make_uint4(one ? 0x3F803F80u : 0u, 0u, 0u, 0u);
  }
  tc::fence_proxy_async();   // generic-proxy writes -> read by tcgen05.mma (async proxy) after the sync below

  if (warp == kTMA && lane == 0) {
    BWD_TRACE(13, 0);
    tc::tma_prefetch(&tmQ);
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    tc::tma_prefetch(&tmdO);
    tc::tma_prefetch(&tmDQ);
    tc::tma_prefetch(&tmDK);
    tc::tma_prefetch(&tmDV);
    tc::mbar_init(kv_full, 1);
    for (int s = 0; s < B_QD_STAGES; ++s) {
      tc::mbar_init(&qd_full[s], 1);
      tc::mbar_init(&qd_empty[s], 1);
    }
    tc::mbar_init(s_full, 1);
    tc::mbar_init(dp_full, 1);
    tc::mbar_init(ds_ready, kBwdCompute);       // every compute warp
    tc::mbar_init(mma_done, 1);
    tc::mbar_init(dq_free, kBwdDrain);
    tc::mbar_init(&stage_free[0], kBwdDrain);
    tc::mbar_init(&stage_free[1], kBwdDrain);
    tc::mbar_init(acc_free, kBwdDrain);
    tc::mbar_init(p_ready, kBwdCompute);        // every compute warp
    tc::mbar_init(kv_tmem, kBwdCompute / 2);    // the chunk-0 (K) and chunk-1 (V) warps
    tc::mbar_init(&kst_free[0], kBwdDrain);
    tc::mbar_init(&kst_free[1], kBwdDrain);
    tc::fence_barrier_init();
  }
  if (warp == kMMA) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S^T (P^T packed over it) | dP^T (dS^T packed over it) | dV | dK | dQ | K | V (bf16 pairs)
  const uint32_t tST = tmem, tDPT = tmem + 128, tDV = tmem + 256, tDK = tmem + 320, tDQ = tmem + 384,
                 tK = tmem + 448, tV = tmem + 480;

  if (warp == kTMA) {
    if (lane == 0) {
      int g = 0, it = 0;
      for (int w = blockIdx.x; w < a.items; w += stride, ++it) {
        const BwdItem t = bwd_item(a, w);
        const int64_t bh = (int64_t)t.b * a.H + t.h;
        if (it >= 1) tc::mbar_wait(kv_tmem, (it - 1) & 1);                  // V_{it-1} copied out of sV
        if (it >= 2) tc::mbar_wait(&kst_free[it & 1], ((it >> 1) - 1) & 1);  // item it-2 done with this K buffer
        tc::mbar_arrive_expect_tx(kv_full, 32768);
        tc::tma_load_3d(sKb(it), &tmK, kv_full, t.h * HD, t.kt * BT, t.b);
        tc::tma_load_3d(sV, &tmV, kv_full, t.h * HD, t.kt * BT, t.b);
        for (int ii = 0; ii < t.nq; ++ii, ++g) {
          const int i = t.i0 + ii, st = g % B_QD_STAGES;
          if (g >= B_QD_STAGES) tc::mbar_wait(&qd_empty[st], ((g / B_QD_STAGES) - 1) & 1);
          tc::mbar_arrive_expect_tx(&qd_full[st], 32768 + kExtTile);
          tc::tma_load_3d(sQD + st * 32768, &tmQ, &qd_full[st], t.h * HD, i * BT, t.b);
          tc::tma_load_3d(sQD + st * 32768 + 16384, &tmdO, &qd_full[st], t.h * HD, i * BT, t.b);
          const uint8_t* ge = a.ext + (bh * (a.Npad / BT) + i) * (int64_t)kExtTile;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(sEXT + st * kExtTile)),
                       "l"(ge), "n"(kExtTile), "r"(smem_u32(&qd_full[st]))
                       : "memory");
        }
      }
    }
  } else if (warp == kMMA) {
    {   // all 32 lanes run the issue loop (warp-uniform values); one elected lane issues
      constexpr uint32_t idSS = tc::idesc_bf16_f32(128, 128, 0, 0);  // S^T, dP^T
      constexpr uint32_t idG = tc::idesc_bf16_f32(128, 64, 0, 1);    // dV (A = P^T in TMEM), dK: B (dO / Q) MN-major
      constexpr uint32_t idQ = tc::idesc_bf16_f32(128, 64, 1, 1);    // dQ: A = dS (MN-major view), B = K MN-major
      const uint64_t dOneS = tc::sdesc_noswz(smem_u32(smem + B_SONE) + 128, 128, 384);   // columns 0-1 = 1
      const uint64_t dOneD = tc::sdesc_noswz(smem_u32(smem + B_SONE), 128, 384);         // columns 8-9 = 1
      auto issue_s = [&](int gg) {      // S'_gg^T = K Q_gg^T - lse/scale, K (A) from TMEM
        const int st = gg % B_QD_STAGES;
        tc::mbar_wait(&qd_full[st], (gg / B_QD_STAGES) & 1);
        tc::tc_fence_after();
        const uint32_t aQ = smem_u32(sQD + st * 32768);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc::umma_f16_ts_w(tST, tK + 8 * kk, tc::sdesc_sw128(aQ + kk * 32, 16, 1024), idSS, kk > 0);
        tc::umma_f16_ss_w(tST, dOneS, tc::sdesc_noswz(smem_u32(sEXT + st * kExtTile), 128, 256), idSS, 1u);
        tc::umma_commit_w(s_full);
      };
      auto issue_dp = [&](int gg) {     // dP'_gg^T = V dO_gg^T - delta, V (A) from TMEM (qd_full(gg) already observed)
        const int st = gg % B_QD_STAGES;
        const uint32_t aDO = smem_u32(sQD + st * 32768) + 16384;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc::umma_f16_ts_w(tDPT, tV + 8 * kk, tc::sdesc_sw128(aDO + kk * 32, 16, 1024), idSS, kk > 0);
        tc::umma_f16_ss_w(tDPT, dOneD, tc::sdesc_noswz(smem_u32(sEXT + st * kExtTile), 128, 256), idSS, 1u);
        tc::umma_commit_w(dp_full);
      };
      int g = 0, it = 0;
      for (int w = blockIdx.x; w < a.items; w += stride, ++it) {
        const BwdItem t = bwd_item(a, w);
        const bool has_next = w + stride < a.items;
        const uint32_t aK = smem_u32(sKb(it));
        if (it == 0) {
          tc::mbar_wait(kv_tmem, 0);      // K, V of the first item in TMEM (compute warps copied them)
          tc::tc_fence_after();
          issue_s(0);
          issue_dp(0);
        }
        for (int ii = 0; ii < t.nq; ++ii, ++g) {
          const int st = g % B_QD_STAGES, pb = g & 1;
          const uint32_t aQ = smem_u32(sQD + st * 32768), aDO = aQ + 16384;
          const uint32_t aDS = smem_u32(sDS + pb * 32768);
          const uint32_t acc = (ii > 0) ? 1u : 0u;
          const bool last = ii + 1 == t.nq, nxt = !last || has_next;
          // P_g^T lives over S_g^T and dS_g^T over dP_g^T (packed bf16, TMEM): dV_g / dK_g read them
          // before S_{g+1} / dP_{g+1} overwrite those columns (tcgen05.mma executes in issue order)
          BWD_TRACE(8, g);
          tc::mbar_wait(p_ready, g & 1);
          if (ii == 0 && it > 0) tc::mbar_wait(acc_free, (it - 1) & 1);   // previous item's dK / dV read out
          tc::tc_fence_after();
          BWD_TRACE(0, g);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)     // dV += P^T dO: K step kk = queries [16kk, 16kk+16) = chunk kk/2
            tc::umma_f16_ts_w(tDV, tST + 32 * (kk >> 1) + 8 * (kk & 1), tc::sdesc_sw128(aDO + kk * 2048, 8192, 1024),
                            idG, (acc | kk) ? 1u : 0u);
          BWD_TRACE(9, g);
          // S_{g+1} overwrites P_g^T: dV(g) read it (issue order); the compute warps keep their own
          // copy of P_g in registers for dS, so nothing else reads those columns
          if (last && has_next) tc::mbar_wait(kv_tmem, (it + 1) & 1);   // next item's K / V in TMEM
          tc::tc_fence_after();
          BWD_TRACE(10, g);
          if (nxt) issue_s(g + 1);
          BWD_TRACE(11, g);
          tc::mbar_wait(ds_ready, g & 1);
          tc::tc_fence_after();
          BWD_TRACE(1, g);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)     // dK += dS^T Q (A = dS^T from TMEM)
            tc::umma_f16_ts_w(tDK, tDPT + 32 * (kk >> 1) + 8 * (kk & 1), tc::sdesc_sw128(aQ + kk * 2048, 8192, 1024),
                            idG, (acc | kk) ? 1u : 0u);
          if (nxt) issue_dp(g + 1);
          if (g >= 1) tc::mbar_wait(dq_free, (g - 1) & 1);   // dQ_{g-1} read out of TMEM
          tc::tc_fence_after();
          BWD_TRACE(2, g);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            // A = dS [q][kv]: the dS^T tile (rows kv, 128B-swizzled q chunks) seen MN-major:
            // q chunks 16 KB apart (LBO), 8-row kv groups 1 KB apart (SBO), K step = 16 kv rows
            const uint64_t dA = tc::sdesc_sw128(aDS + kk * 2048, 16384, 1024);
            tc::umma_f16_ss_w(tDQ, dA, tc::sdesc_sw128(aK + kk * 2048, 8192, 1024), idQ, kk > 0);
          }
          BWD_TRACE(12, g);
          tc::umma_commit_w(mma_done);
          tc::umma_commit_w(&qd_empty[st]);
        }
      }
    }
  } else if (warp >= kDrain0) {
    // ------------------------------------------------------------ drain warps (one per TMEM lane quadrant)
    const int quad = warp & 3;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    int g = 0, it = 0;
    for (int w = blockIdx.x; w < a.items; w += stride, ++it) {
      const BwdItem t = bwd_item(a, w);
      for (int ii = 0; ii < t.nq; ++ii, ++g) {
        const int pb = g & 1;
        tc::mbar_wait(mma_done, g & 1);   // dK_g / dQ_g complete: dQ_g final, dS^T_g buffer free
        tc::tc_fence_after();
        if (ii + 1 == t.nq) {
          // the item's dK / dV are final and its K buffer is free (last dQ MMA done): bf16 tiles
          // staged there (this warp's 32 rows = 4 KB, 128B-swizzled) and written by TMA stores,
          // so no warp waits on scattered global stores.  dK (softmax scale folded in: dS was
          // stored without it) is held as bf16 pairs while dV's staging is read out.
          uint8_t* stg = sKb(it) + quad * 4096;
          uint32_t kb[32];
#pragma unroll
          for (int hh = 0; hh < 4; ++hh) {   // dV cols [0,32) [32,64), then dK
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32((hh < 2 ? tDV : tDK) + lane_off + (hh & 1) * 32, r);
            tc::tmem_ld_wait();
            const float osc = hh < 2 ? 1.f : a.scale;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const uint32_t p = pack_bf16x2(__uint_as_float(r[2 * e]) * osc, __uint_as_float(r[2 * e + 1]) * osc);
              if (hh < 2) r[e] = p; else kb[(hh & 1) * 16 + e] = p;
            }
            if (hh < 2) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                *reinterpret_cast<uint4*>(stg + lane * 128 + ((((hh & 1) * 4 + u) ^ (lane & 7)) << 4)) =
                    make_uint4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]);
            }
          }
          tc::tc_fence_before();
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tc::mbar_arrive(acc_free);   // the next item's first dV / dK MMA may overwrite them
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                             reinterpret_cast<uint64_t>(&tmDV)),
                         "r"(smem_u32(stg)), "r"(t.h * HD), "r"(t.kt * BT + quad * 32), "r"(t.b)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<uint4*>(stg + lane * 128 + ((u ^ (lane & 7)) << 4)) =
                make_uint4(kb[4 * u], kb[4 * u + 1], kb[4 * u + 2], kb[4 * u + 3]);
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                             reinterpret_cast<uint64_t>(&tmDK)),
                         "r"(smem_u32(stg)), "r"(t.h * HD), "r"(t.kt * BT + quad * 32), "r"(t.b)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            tc::mbar_arrive(&kst_free[it & 1]);   // the TMA may load K of item it+2 here
          }
          __syncwarp();
          if (warp == kDrain0) BWD_TRACE(23, g);
        }
#ifdef AVB_ATTN_TRACE_HOOKS
        if (a.dbg & 1) {
          __syncwarp();
          if (lane == 0) {
            tc::mbar_arrive(dq_free);
            tc::mbar_arrive(&stage_free[pb]);
          }
          continue;
        }
#endif
        if (a.dq_bf16) {
          // dQ_g (softmax scale folded in: dS carries none) as bf16 pairs in one 4 KB SW128 box per warp
          // (32 query rows x 64), reduce-added by TMA straight into the bf16 dq rows
          uint8_t* stage = sDS + pb * 32768 + quad * 4096;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32(tDQ + lane_off + hh * 32, r);
            tc::tmem_ld_wait();
            if (hh == 1) {
              tc::tc_fence_before();
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(dq_free);
            }
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              pk[e] = pack_bf16x2(__uint_as_float(r[2 * e]) * a.scale, __uint_as_float(r[2 * e + 1]) * a.scale);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              *reinterpret_cast<uint4*>(stage + lane * 128 + ((((hh * 4) + u) ^ (lane & 7)) << 4)) =
                  make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          }
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            const int q0 = (t.i0 + ii) * BT + quad * 32;
            asm volatile(
                "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmDQ)),
                "r"(smem_u32(stage)), "r"(t.h * HD), "r"(q0), "r"(t.b)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            tc::mbar_arrive(&stage_free[pb]);   // the buffer may take dS^T_{g+2}
          }
          __syncwarp();
          continue;
        }
        uint8_t* stage = sDS + pb * 32768 + quad * 8192;   // 32 query rows x 64 fp32, two 4 KB SW128 boxes
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t r[32];
          tc::tmem_ld_32x32b_x32(tDQ + lane_off + hh * 32, r);
          tc::tmem_ld_wait();
          if (hh == 1) {
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(dq_free);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<uint4*>(stage + hh * 4096 + lane * 128 + ((u ^ (lane & 7)) << 4)) =
                make_uint4(r[u * 4], r[u * 4 + 1], r[u * 4 + 2], r[u * 4 + 3]);
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          const int q0 = (t.i0 + ii) * BT + quad * 32;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            if (a.dq_det)   // slice kt of the per-key-tile partials (z = kt * B + b)
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                               reinterpret_cast<uint64_t>(&tmDQ)),
                           "r"(smem_u32(stage + hh * 4096)), "r"(t.h * HD + hh * 32), "r"(q0), "r"(t.kt * a.B + t.b)
                           : "memory");
            else
              asm volatile(
                  "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                      reinterpret_cast<uint64_t>(&tmDQ)),
                  "r"(smem_u32(stage + hh * 4096)), "r"(t.h * HD + hh * 32), "r"(q0), "r"(t.b)
                  : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          tc::mbar_arrive(&stage_free[pb]);   // the buffer may take dS^T_{g+2}
        }
        __syncwarp();
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  } else {
    // ------------------------------------------------------------ compute warps
    // warp w owns TMEM lane quadrant (w & 3) -> key rows, and query chunk c = w >> 2 (32 queries).
    // Per step it forms P^T = exp2(S^T*scale*log2e - lse*log2e) for its chunk, stores it (bf16) over
    // the consumed S^T chunk (dV's A operand) and, keeping P in registers, forms
    // dS^T = P^T (dP^T - delta) once dP^T has landed -> bf16 over the consumed dP^T chunk (dK's A
    // operand) and into the smem tile (dQ's A operand).  All 16 warps take part in both phases, so
    // the exp phase -- on the critical chain exp(g) -> dV(g) -> S(g+1) -> exp(g+1) -- is spread over
    // four warps per SMSP, and dS(g) runs while dV(g) / S(g+1) execute.
    const int quad = warp & 3, c = warp >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float2 sl2 = make_float2(a.scale_log2, a.scale_log2);
    int g = 0, it = 0;
    for (int w = blockIdx.x; w < a.items; w += stride, ++it) {
      const BwdItem t = bwd_item(a, w);
      const int kv0 = t.kt * BT, kvi = kv0 + row;
      if (c < 2) {
        // this item's K (chunk-0 warps) / V (chunk-1 warps) rows -> TMEM (bf16 pairs, 32 columns): the
        // A operands of S^T = K Q^T and dP^T = V dO^T.  The previous item's last S^T / dP^T MMAs are
        // done reading them: this warp's dS of that step waited for its dP^T (issued after S^T).
        tc::mbar_wait(kv_full, it & 1);
        tc::tc_fence_after();
        const uint8_t* src = (c ? sV : sKb(it)) + row * 128;
        uint32_t r[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 q = *reinterpret_cast<const uint4*>(src + ((u ^ (row & 7)) << 4));
          r[4 * u] = q.x; r[4 * u + 1] = q.y; r[4 * u + 2] = q.z; r[4 * u + 3] = q.w;
        }
        tc::tmem_st_32x32b_x32((c ? tV : tK) + lane_off, r);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(kv_tmem);
        if (warp == 0) BWD_TRACE(16, g);
      }
      for (int ii = 0; ii < t.nq; ++ii, ++g) {
        const int i = t.i0 + ii, st = g % B_QD_STAGES;
        const int q0 = i * BT;
        if (warp == 0) {
          BWD_TRACE(4, g);
          BWD_TRACE_NS(15, g);
        }
        // ---- P^T for this chunk
        tc::mbar_wait(s_full, g & 1);   // (the statistics arrive inside S'^T / dP'^T: no smem reads here)
        tc::tc_fence_after();
        if (warp == 0) BWD_TRACE(5, g);
        const bool edge = (q0 + c * 32 + 32 > a.N) || (kv0 + quad * 32 + 32 > a.N) ||
                          (a.causal && q0 + c * 32 < kv0 + quad * 32 + 32);
        uint32_t pk[16];
        {
          uint32_t rs[32];
          if (BWD_DBG(8)) {
#pragma unroll
            for (int e = 0; e < 32; ++e) rs[e] = __float_as_uint(-(float)(lane + e));
          } else {
            tc::tmem_ld_32x32b_x32(tST + lane_off + c * 32, rs);
            tc::tmem_ld_wait();
          }
          if (warp == 0) BWD_TRACE(3, g);
          auto pbody = [&](auto edge_tag) {
            constexpr bool EDGE = decltype(edge_tag)::value;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 sv = make_float2(__uint_as_float(rs[u * 8 + 2 * e]), __uint_as_float(rs[u * 8 + 2 * e + 1]));
                const float2 arg = f2mul(sv, sl2);       // (S - lse/scale)*scale*log2e
                float2 p = BWD_DBG(16) ? arg : (((u * 4 + e) & 7) >= kBwdPoly8From) ? exp2_poly2(arg) : make_float2(ex2(arg.x), ex2(arg.y));
                if (EDGE) {
                  const int qi = q0 + c * 32 + u * 8 + 2 * e;
                  const bool ok0 = (qi < a.N) && (kvi < a.N) && (!a.causal || qi >= kvi);
                  const bool ok1 = (qi + 1 < a.N) && (kvi < a.N) && (!a.causal || qi + 1 >= kvi);
                  p.x = ok0 ? p.x : 0.f;
                  p.y = ok1 ? p.y : 0.f;
                }
                pk[u * 4 + e] = pack_bf16x2(p.x, p.y);
              }
            }
          };
          if (edge) pbody(std::true_type{}); else pbody(std::false_type{});
        }
        if (warp == 0) BWD_TRACE(17, g);
        if (!BWD_DBG(8)) tc::tmem_st_32x32b_x16(tST + lane_off + c * 32, pk);   // P^T over the consumed S^T chunk
        tc::tmem_st_wait();
        if (warp == 0) BWD_TRACE(22, g);
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_ready);
        if (warp == 0) BWD_TRACE(18, g);
        if (warp == 15) BWD_TRACE(21, g);
        // ---- dS^T for this chunk (P from registers)
        tc::mbar_wait(dp_full, g & 1);
        tc::tc_fence_after();
        if (warp == 0) BWD_TRACE(6, g);
        if (g >= 2) tc::mbar_wait(&stage_free[g & 1], ((g - 2) >> 1) & 1);  // dQ_{g-2} staging read out
        uint8_t* ds_t = sDS + (g & 1) * 32768;
        {
          uint32_t rp[32], dsk[16];
          if (BWD_DBG(4)) {
#pragma unroll
            for (int e = 0; e < 32; ++e) rp[e] = __float_as_uint((float)(lane - e));
          } else {
            tc::tmem_ld_32x32b_x32(tDPT + lane_off + c * 32, rp);
            tc::tmem_ld_wait();
          }
          if (warp == 0) BWD_TRACE(19, g);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 wv;
            uint32_t* wp = &wv.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 dp = make_float2(__uint_as_float(rp[u * 8 + 2 * e]), __uint_as_float(rp[u * 8 + 2 * e + 1]));
#if AVB_BWD_DS_BF16X2
              // P (dP - delta) as one bf16x2 multiply of the packed P and the packed dP' (delta folded
              // into the MMA): 2 instructions per pair instead of unpack x2 + FMUL2 + pack
              uint32_t dsp;
              asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(dsp) : "r"(pk[u * 4 + e]), "r"(pack_bf16x2(dp.x, dp.y)));
              wp[e] = dsp;
#else
              const float2 ds = f2mul(unpack_bf16x2(pk[u * 4 + e]), dp);  // P (dP - delta): delta folded into the MMA
              wp[e] = pack_bf16x2(ds.x, ds.y);
#endif
              dsk[u * 4 + e] = wp[e];
            }
            if (!BWD_DBG(2)) st_sw128(ds_t, row, c * 4 + u, wv);   // dQ's A operand (read MN-major from smem)
          }
          if (warp == 0) BWD_TRACE(20, g);
          if (!BWD_DBG(4)) tc::tmem_st_32x32b_x16(tDPT + lane_off + c * 32, dsk);   // dK's A operand, over the consumed dP^T chunk
        }
        tc::tmem_st_wait();
        tc::fence_proxy_async();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(ds_ready);
        if (warp == 0) BWD_TRACE(7, g);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kTMA) BWD_TRACE(14, 0);
  if (warp == kMMA) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// Extension tiles (see kExtTile): row n of (b, h) gets bf16 hi/lo of -lse/scale in columns 0-1 and of
// -rowsum(dO*O) in columns 8-9, zeros elsewhere (padded rows [N, Npad): all zero, so masked elements
// stay finite); also zeroes the dQ accumulator rows.
__device__ __forceinline__ void ext_row(uint8_t* ext, int64_t bh, int Npad, int n, float x, float y) {
  uint8_t* t = ext + (bh * (Npad / BT) + n / BT) * (int64_t)kExtTile;
  const int q = n % BT;
  uint8_t* r = t + (q >> 3) * 256 + (q & 7) * 16;
  const __nv_bfloat16 xh = __float2bfloat16_rn(x), yh = __float2bfloat16_rn(y);
  const __nv_bfloat16 xl = __float2bfloat16_rn(x - __bfloat162float(xh)), yl = __float2bfloat16_rn(y - __bfloat162float(yh));
  const uint32_t px = (uint32_t)__bfloat16_as_ushort(xh) | ((uint32_t)__bfloat16_as_ushort(xl) << 16);
  const uint32_t py = (uint32_t)__bfloat16_as_ushort(yh) | ((uint32_t)__bfloat16_as_ushort(yl) << 16);
  *reinterpret_cast<uint4*>(r) = make_uint4(px, 0u, 0u, 0u);         // k 0..7
  *reinterpret_cast<uint4*>(r + 128) = make_uint4(py, 0u, 0u, 0u);   // k 8..15
}

__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ o, int64_t ld_o, int64_t sb_o,
                                    const __nv_bfloat16* __restrict__ dout, int64_t ld_do, int64_t sb_do,
                                    const float* __restrict__ lse, uint8_t* __restrict__ ext, float inv_scale,
                                    float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dq, int64_t ld_g,
                                    int64_t sb_g, int B, int H, int N, int Npad) {
  // 8 threads per (b, n, h) row of 64 elements
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t item = gid >> 3;
  const int sub = gid & 7;
  const int64_t total = (int64_t)B * N * H;
  if (item >= total) {
    const int64_t pi = gid - total * 8;
    const int npad = Npad - N;
    if (pi < (int64_t)B * H * npad) {
      const int64_t bh = pi / npad;
      ext_row(ext, bh, Npad, N + (int)(pi - bh * npad), 0.f, 0.f);
    }
    return;
  }
  const int h = item % H;
  const int64_t bn = item / H;
  const int n = bn % N;
  const int b = bn / N;
  const uint4 ov = *reinterpret_cast<const uint4*>(o + b * sb_o + (int64_t)n * ld_o + h * HD + sub * 8);
  const uint4 dv = *reinterpret_cast<const uint4*>(dout + b * sb_do + (int64_t)n * ld_do + h * HD + sub * 8);
  const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
  const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 a = __bfloat1622float2(o2[e]), c = __bfloat1622float2(d2[e]);
    s = fmaf(a.x, c.x, fmaf(a.y, c.y, s));
  }
  s += __shfl_xor_sync(0xffffffff, s, 1);
  s += __shfl_xor_sync(0xffffffff, s, 2);
  s += __shfl_xor_sync(0xffffffff, s, 4);
  if (sub == 0) {
    const int64_t bh = (int64_t)b * H + h;
    const float l = lse[bh * Npad + n];
    ext_row(ext, bh, Npad, n, isfinite(l) ? -l * inv_scale : 0.f, -s);
  }
  if (dq_acc) {
    float4* z = reinterpret_cast<float4*>(dq_acc + item * HD + sub * 8);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  } else if (dq) {   // the bf16 dQ rows are the reduce-add target themselves
    *reinterpret_cast<uint4*>(dq + b * sb_g + (int64_t)n * ld_g + h * HD + sub * 8) = make_uint4(0, 0, 0, 0);
  }
}

__global__ void attn_dq_convert_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dq, int64_t ld,
                                       int64_t sb, int B, int H, int N, float scale, int nslices, int causal) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one thread per 8 elements
  const int64_t total = (int64_t)B * N * H * 8;
  if (gid >= total) return;
  const int sub = gid & 7;
  const int64_t item = gid >> 3;
  const int h = item % H;
  const int64_t bn = item / H;
  const int n = bn % N;
  const int b = bn / N;
  // slices summed in key-tile order (deterministic mode; nslices = 1 otherwise); a causal query row n
  // only has contributions from key tiles kt <= n / 128 (the others were never written)
  const int64_t slice = (int64_t)B * N * H * HD;
  const int ns = causal ? min(nslices, n / BT + 1) : nslices;
  float4 x = make_float4(0.f, 0.f, 0.f, 0.f), y = x;
  for (int k = 0; k < ns; ++k) {
    const float4* s = reinterpret_cast<const float4*>(dq_acc + k * slice + item * HD + sub * 8);
    const float4 a0 = s[0], a1 = s[1];
    x = make_float4(x.x + a0.x, x.y + a0.y, x.z + a0.z, x.w + a0.w);
    y = make_float4(y.x + a1.x, y.y + a1.y, y.z + a1.z, y.w + a1.w);
  }
  uint4 v;
  v.x = pack_bf16x2(x.x * scale, x.y * scale);
  v.y = pack_bf16x2(x.z * scale, x.w * scale);
  v.z = pack_bf16x2(y.x * scale, y.y * scale);
  v.w = pack_bf16x2(y.z * scale, y.w * scale);
  *reinterpret_cast<uint4*>(dq + b * sb + (int64_t)n * ld + h * HD + sub * 8) = v;
}

int make_maps(CUtensorMap* m, const void* p, int B, int H, int N, int64_t ld, int64_t sb, uint32_t rows = 128) {
  return avb::make_tmap_3d_bf16(m, p, (uint64_t)H * HD, (uint64_t)N, (uint64_t)B, (uint64_t)ld, (uint64_t)sb, 64, rows,
                                1);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" int avb_attn_fwd(const void* q, const void* k, const void* v, int64_t ld, int64_t sb, void* o, int64_t ld_o,
                            int64_t sb_o, float* lse, int B, int H, int N, int head_dim, float softmax_scale,
                            int causal, void* stream) {
  AVB_CHECK_ARG(head_dim == HD, "head_dim must be 64 (got %d)", head_dim);
  AVB_CHECK_ARG(B >= 0 && H >= 1 && N >= 0, "bad attention dims");
  if (B == 0 || N == 0) return AVB_OK;
  AVB_CHECK_ARG(q && k && v && o && lse, "null pointer");
  AVB_CHECK_ARG(aligned16(q) && aligned16(k) && aligned16(v) && aligned16(o), "q/k/v/o must be 16-byte aligned");
  AVB_CHECK_ARG(ld % 8 == 0 && sb % 8 == 0 && ld_o % 8 == 0, "strides must be multiples of 8 elements");
  AVB_CHECK_ARG(ld >= (int64_t)H * HD && ld_o >= (int64_t)H * HD, "row stride smaller than H*64");
  AVB_CHECK_ARG(B <= 65535 && H <= 65535, "B/H too large");
  CUtensorMap mq, mk, mv;
  int s;
  if ((s = make_maps(&mq, q, B, H, N, ld, sb))) return s;
  if ((s = make_maps(&mk, k, B, H, N, ld, sb, FKB))) return s;
  if ((s = make_maps(&mv, v, B, H, N, ld, sb, FKB))) return s;
  FwdArgs a;
  a.B = B;
  a.H = H;
  a.N = N;
  a.Npad = (N + BT - 1) / BT * BT;
  a.scale_log2 = softmax_scale * kLog2e;
  a.o = reinterpret_cast<__nv_bfloat16*>(o);
  a.ld_o = ld_o;
  a.sb_o = sb_o;
  a.lse = lse;
  a.causal = causal;
  a.trace = nullptr;
#ifdef AVB_ATTN_TRACE_HOOKS   // trace build only: a device buffer address handed over by scripts/trace_attn_fwd.py
  if (const char* tr = getenv("AVB_ATTN_FTRACE")) a.trace = reinterpret_cast<long long*>(strtoull(tr, nullptr, 0));
#endif
  if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(attn_fwd_kernel), F_SMEM, "attn_fwd smem attr"))
    return e;
  dim3 grid((N + 2 * BT - 1) / (2 * BT), H, B);
  attn_fwd_kernel<<<grid, 320, F_SMEM, avb::as_stream(stream)>>>(mq, mk, mv, a);
  return avb::launch_status("avb_attn_fwd");
}

static int attn_bwd_impl(const void* q, const void* k, const void* v, int64_t ld, int64_t sb, const void* o,
                         const void* dout, int64_t ld_o, int64_t sb_o, const float* lse, float* delta, float* dq_acc,
                         void* dq, void* dk, void* dv, int64_t ld_g, int64_t sb_g, int B, int H, int N, int head_dim,
                         float softmax_scale, int causal, int det, void* stream) {
  AVB_CHECK_ARG(head_dim == HD, "head_dim must be 64 (got %d)", head_dim);
  AVB_CHECK_ARG(B >= 0 && H >= 1 && N >= 0, "bad attention dims");
  if (B == 0 || N == 0) return AVB_OK;
  AVB_CHECK_ARG(q && k && v && o && dout && lse && delta && dq && dk && dv, "null pointer");
  AVB_CHECK_ARG(aligned16(q) && aligned16(k) && aligned16(v) && aligned16(o) && aligned16(dout) && aligned16(dq) &&
                    aligned16(dk) && aligned16(dv) && aligned16(lse) && aligned16(delta) &&
                    (!dq_acc || aligned16(dq_acc)),
                "pointers must be 16-byte aligned");
  AVB_CHECK_ARG(ld % 8 == 0 && sb % 8 == 0 && ld_o % 8 == 0 && sb_o % 8 == 0 && ld_g % 8 == 0 && sb_g % 8 == 0,
                "strides must be multiples of 8 elements");
  cudaStream_t st = avb::as_stream(stream);
  const int Npad = (N + BT - 1) / BT * BT;
  {
    const int64_t threads = (int64_t)B * N * H * 8 + (int64_t)B * H * (Npad - N);
    attn_bwd_pre_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(o), ld_o, sb_o, reinterpret_cast<const __nv_bfloat16*>(dout), ld_o,
        sb_o, lse, reinterpret_cast<uint8_t*>(delta), 1.f / softmax_scale, dq_acc, reinterpret_cast<__nv_bfloat16*>(dq),
        ld_g, sb_g, B, H, N, Npad);
    int s = avb::launch_status("attn_bwd_pre");
    if (s) return s;
  }
  CUtensorMap mq, mk, mv, mdo;
  int s;
  if ((s = make_maps(&mq, q, B, H, N, ld, sb))) return s;
  if ((s = make_maps(&mk, k, B, H, N, ld, sb))) return s;
  if ((s = make_maps(&mv, v, B, H, N, ld, sb))) return s;
  if ((s = make_maps(&mdo, dout, B, H, N, ld_o, sb_o))) return s;
  CUtensorMap mdq, mdk, mdv;
  if ((s = make_maps(&mdk, dk, B, H, N, ld_g, sb_g, 32))) return s;   // dK / dV TMA stores: 32-row boxes
  if ((s = make_maps(&mdv, dv, B, H, N, ld_g, sb_g, 32))) return s;
  const int nkt = (N + BT - 1) / BT;
  if (dq_acc) {   // deterministic mode: nkt slices of [B, N, H, 64] (z = kt * B + b)
    if ((s = avb::make_tmap_3d_f32(&mdq, dq_acc, (uint64_t)H * HD, (uint64_t)N, (uint64_t)B * (det ? nkt : 1),
                                   (uint64_t)H * HD, (uint64_t)N * H * HD, 32, 32, 1, 128)))
      return s;
  } else if ((s = make_maps(&mdq, dq, B, H, N, ld_g, sb_g, 32))) {   // bf16 dq rows, 32-row boxes
    return s;
  }
  BwdArgs a;
  a.B = B;
  a.H = H;
  a.N = N;
  a.Npad = Npad;
  a.scale = softmax_scale;
  a.scale_log2 = softmax_scale * kLog2e;
  a.ext = reinterpret_cast<const uint8_t*>(delta);
  a.dk = reinterpret_cast<__nv_bfloat16*>(dk);
  a.dv = reinterpret_cast<__nv_bfloat16*>(dv);
  a.ld_g = ld_g;
  a.sb_g = sb_g;
  a.causal = causal;
  a.nkt = (N + BT - 1) / BT;
  a.items = B * H * a.nkt;
  a.dq_bf16 = dq_acc ? 0 : 1;
  a.dq_det = det;
  a.trace = nullptr;
  a.dbg = 0;
#ifdef AVB_ATTN_TRACE_HOOKS   // trace build only (scripts/trace_attn_bwd.py)
  if (const char* tr = getenv("AVB_ATTN_TRACE")) a.trace = reinterpret_cast<long long*>(strtoull(tr, nullptr, 0));
  a.dbg = getenv("AVB_ATTN_DBG") ? atoi(getenv("AVB_ATTN_DBG")) : 0;
#endif
  // persistent: one CTA per SM walks work items blockIdx.x, +gridDim.x, ... (1 CTA/SM: TMEM 512 cols)
  int grid = std::min(a.items, avb::sm_count());
#ifdef AVB_DEBUG_KNOBS
  if (const char* gs = getenv("AVB_ATTN_BWD_GRID")) grid = std::min(grid, atoi(gs));
#endif
  if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(attn_bwd_kernel), B_SMEM, "attn_bwd smem attr"))
    return e;
  attn_bwd_kernel<<<grid, 32 * kBwdWarps, B_SMEM, st>>>(mq, mk, mv, mdo, mdq, mdk, mdv, a);
  if ((s = avb::launch_status("avb_attn_bwd"))) return s;
  if (!dq_acc) return AVB_OK;   // dQ was reduce-added in bf16 directly
  const int64_t threads = (int64_t)B * N * H * 8;
  attn_dq_convert_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      dq_acc, reinterpret_cast<__nv_bfloat16*>(dq), ld_g, sb_g, B, H, N, softmax_scale, det ? nkt : 1, causal);
  return avb::launch_status("attn_dq_convert");
}

extern "C" int avb_attn_bwd(const void* q, const void* k, const void* v, int64_t ld, int64_t sb, const void* o,
                            const void* dout, int64_t ld_o, int64_t sb_o, const float* lse, float* delta,
                            float* dq_acc, void* dq, void* dk, void* dv, int64_t ld_g, int64_t sb_g, int B, int H,
                            int N, int head_dim, float softmax_scale, int causal, void* stream) {
  return attn_bwd_impl(q, k, v, ld, sb, o, dout, ld_o, sb_o, lse, delta, dq_acc, dq, dk, dv, ld_g, sb_g, B, H, N,
                       head_dim, softmax_scale, causal, 0, stream);
}

extern "C" int avb_attn_bwd_deterministic(const void* q, const void* k, const void* v, int64_t ld, int64_t sb,
                                          const void* o, const void* dout, int64_t ld_o, int64_t sb_o, const float* lse,
                                          float* delta, float* dq_part, void* dq, void* dk, void* dv, int64_t ld_g,
                                          int64_t sb_g, int B, int H, int N, int head_dim, float softmax_scale,
                                          int causal, void* stream) {
  AVB_CHECK_ARG(dq_part, "deterministic attention backward needs the fp32 per-key-tile dQ workspace");
  return attn_bwd_impl(q, k, v, ld, sb, o, dout, ld_o, sb_o, lse, delta, dq_part, dq, dk, dv, ld_g, sb_g, B, H, N,
                       head_dim, softmax_scale, causal, 1, stream);
}
