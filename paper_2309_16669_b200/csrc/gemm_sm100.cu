// K2/K3: persistent warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
//   C[M,N] = epilogue( sum_k A[m,k] * B[n,k] )
//
// Operands are bf16, fed by TMA (128B swizzle) through an mbarrier ring into UMMA
// (tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16), accumulating in TMEM
// (two BN-column accumulators so the epilogue of tile i overlaps the MMAs of tile i+1).
// Each operand may be K-major (A:[M,K], B:[N,K]) or MN-major (A:[K,M], B:[K,N]) so
// forward (X W^T), dgrad (dY W) and wgrad (dY^T X) all run without transposes.
//
// Warp roles (384 threads, 1 CTA/SM; the scheduler prefers the highest warp ids, so the producer
// and MMA issuer sit above the epilogue):
//   warps 0-7  epilogue: TMEM lane quadrant (w & 3) x column half (w >> 2); tcgen05.ld 32 lanes x 32
//              columns -> bias / QuickGELU / residual / dGELU / fp32 split-K reduction -> bf16 tiles
//              staged in 64B-swizzled smem and written by TMA stores (aux tiles TMA-prefetched)
//   warp 8     TMA producer (one elected lane)
//   warp 9     MMA issuer (all lanes run the loop, elect.sync issues)
//   warp 10    TMEM allocator
// CTA-pair mode (cluster of 2, tcgen05 cta_group::2, M = 256) for the large BN = 256 shapes: each
// CTA loads its own 128 A rows and half the B rows; the leader's MMA thread commits to both CTAs.
//
// No reference code exists for this (absent in the reference,
// restated from PAPER.md:258-260,727).
#include "tc_common.cuh"

#include <algorithm>
#include <atomic>

#include <stdlib.h>
#include <string.h>

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 384;   // warps 0-7 epilogue, 8 TMA producer, 9 MMA issuer, 10 TMEM alloc, 11 spare
// (the scheduler prefers the highest warp id: producer and MMA issuer outrank the epilogue)
constexpr int kWProd = 8, kWMma = 9, kWAlloc = 10;
constexpr int kEpiWarps = 8;

struct GemmArgs {
  void* C;
  int64_t ldc;
  int M, N, K;
  int epi;
  const float* bias;     // [N] fp32 or null
  const void* aux;       // bf16 [M, ldaux]: residual (EPI_BF16) or GELU pre-activation (EPI_DGELU)
  int64_t ldaux;
  void* aux_out;         // bf16 [M, ldaux]: pre-activation out (EPI_BIAS_GELU)
  int num_m, num_n, splits, kb_per_split, num_kb;
  int vec_ok;            // 16B-aligned rows for vector epilogue stores
  int tma_out;           // bf16 C (and aux_out) written by TMA stores from swizzled smem
  int tma_aux;           // aux (residual / pre-activation) tiles TMA-prefetched into a smem ring
  float alpha;
  float* rowsum;         // fp32 [M] or null: rowsum[m] += sum_k A[m,k] (the bias gradient of a wgrad)
};

// PAIR: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes a 256 x BN tile; each CTA loads its
// own 128 A rows and half of the BN B rows, so a stage is half as large and the ring twice as deep.
template <int BN, bool A_MN, bool B_MN, int EK, bool PAIR = false>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;               // 16 KB
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;   // 32 KB (BN=256), 16 KB per CTA of a pair
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
// pair-mode plain-epilogue pipeline depth / store slots (compile-time tuning hooks; same-box sweep
// after the issue fix: 6/2 = 5/4 within noise on the step's shapes, 4/4 2-6 % slower)
#ifndef AVB_GEMM_PAIR_STAGES0
#define AVB_GEMM_PAIR_STAGES0 5
#endif
#ifndef AVB_GEMM_PAIR_SSLOTS0
#define AVB_GEMM_PAIR_SSLOTS0 4
#endif
// heavy-epilogue pair rings (stages / store slots / aux slots; same-box sweep with the pair-aux
// change: EK1 4/2/3 + EK2 5/4 (default) vs EK1 5/2/2 + EK2 4/6 vs EK1 4/3/3: defaults best or within noise)
#ifndef AVB_GEMM_PAIR_STAGES1
#define AVB_GEMM_PAIR_STAGES1 4
#endif
#ifndef AVB_GEMM_SSLOTS1
#define AVB_GEMM_SSLOTS1 2
#endif
#ifndef AVB_GEMM_XSLOTS1
#define AVB_GEMM_XSLOTS1 3
#endif
#ifndef AVB_GEMM_PAIR_STAGES2
#define AVB_GEMM_PAIR_STAGES2 5
#endif
#ifndef AVB_GEMM_SSLOTS2
#define AVB_GEMM_SSLOTS2 4
#endif
  static constexpr int STAGES =
      PAIR ? (EK == 0 ? AVB_GEMM_PAIR_STAGES0 : (EK == 1 ? AVB_GEMM_PAIR_STAGES1 : AVB_GEMM_PAIR_STAGES2))
           : ((BN == 256) ? (EK ? 3 : 4) : 6);
  // EK 0: plain; 1: bf16 aux read (residual / GELU pre-activation); 2: second bf16 output (BIAS_GELU)
  static constexpr int SSLOTS =   // TMA-store staging slots per epilogue warp
      EK == 0 ? (PAIR ? AVB_GEMM_PAIR_SSLOTS0 : 2)
              : (EK == 1 ? (PAIR ? AVB_GEMM_SSLOTS1 : 2) : (PAIR ? AVB_GEMM_SSLOTS2 : 4));
  static constexpr int XSLOTS = EK == 1 ? (PAIR ? AVB_GEMM_XSLOTS1 : 3) : 1;   // TMA-load aux ring slots per epilogue warp
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr int EPI_BYTES = (SSLOTS + (EK == 1 ? XSLOTS : 0)) * kEpiWarps * 2048;  // 2 KB slots per epilogue warp
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
  static_assert(SMEM <= 232448, "gemm smem");
  static constexpr uint32_t IDESC = tc::idesc_bf16_f32(PAIR ? 2 * BM : BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
  static constexpr uint32_t IDESC_RS = tc::idesc_bf16_f32(PAIR ? 2 * BM : BM, 16, A_MN ? 1 : 0, 0);   // A x ones[16,K]
};

__device__ __forceinline__ void store_row_chunk(const GemmArgs& a, int row, int col, float (&v)[32]) {
  // v: 32 consecutive columns [col, col+32) of `row`, epilogue already applied
  if (row >= a.M) return;
  const bool full = (col + 32 <= a.N) && a.vec_ok;
  if (a.epi == AVB_EPI_F32_ACCUM) {
    float* c = reinterpret_cast<float*>(a.C) + (int64_t)row * a.ldc + col;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(c + j), "f"(v[j]), "f"(v[j + 1]),
                     "f"(v[j + 2]), "f"(v[j + 3])
                     : "memory");
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < a.N) atomicAdd(c + j, v[j]);
    }
    return;
  }
  if (a.epi == AVB_EPI_F32) {
    float* c = reinterpret_cast<float*>(a.C) + (int64_t)row * a.ldc + col;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < a.N) c[j] = v[j];
    }
    return;
  }
  __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(a.C) + (int64_t)row * a.ldc + col;
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 q;
      q.x = pack_bf16x2(v[j], v[j + 1]);
      q.y = pack_bf16x2(v[j + 2], v[j + 3]);
      q.z = pack_bf16x2(v[j + 4], v[j + 5]);
      q.w = pack_bf16x2(v[j + 6], v[j + 7]);
      *reinterpret_cast<uint4*>(c + j) = q;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col + j < a.N) c[j] = __float2bfloat16_rn(v[j]);
  }
}

__device__ __forceinline__ void load_aux_chunk(const GemmArgs& a, const void* base, int row, int col, float (&o)[32]) {
  const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(base) + (int64_t)row * a.ldaux + col;
  if (row < a.M && col + 32 <= a.N && a.vec_ok) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 q = *reinterpret_cast<const uint4*>(p + j);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(h[e]);
        o[j + 2 * e] = f.x;
        o[j + 2 * e + 1] = f.y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = (row < a.M && col + j < a.N) ? __bfloat162float(p[j]) : 0.f;
  }
}

__device__ __forceinline__ void store_aux_chunk(const GemmArgs& a, int row, int col, const float (&v)[32]) {
  if (row >= a.M) return;
  __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(a.aux_out) + (int64_t)row * a.ldaux + col;
  if (col + 32 <= a.N && a.vec_ok) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 q;
      q.x = pack_bf16x2(v[j], v[j + 1]);
      q.y = pack_bf16x2(v[j + 2], v[j + 3]);
      q.z = pack_bf16x2(v[j + 4], v[j + 5]);
      q.w = pack_bf16x2(v[j + 6], v[j + 7]);
      *reinterpret_cast<uint4*>(c + j) = q;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col + j < a.N) c[j] = __float2bfloat16_rn(v[j]);
  }
}

// ---- CTA-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a local smem object) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// The epilogue's "accumulator drained" arrival on the pair leader's barrier.  Relaxed: what it
// publishes is only that this warp's tcgen05.ld of the accumulator completed (tcgen05.wait::ld +
// tcgen05.fence::before_thread_sync precede it); a .release.cluster arrive would also drain every
// outstanding generic memory operation (MEMBAR.ALL.CTA + MEMBAR.ALL.GPU + ERRBAR in SASS), which
// ncu showed as the epilogue warps' top stall (11 % of samples) in the heavy-epilogue GEMMs.
#ifndef AVB_GEMM_RELAXED_TEMPTY
#define AVB_GEMM_RELAXED_TEMPTY 1
#endif
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
#if AVB_GEMM_RELAXED_TEMPTY
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
// TMA 2D load into this CTA's smem, completion (tx bytes) signalled on an mbarrier of the pair leader
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
// warp-collective forms (all lanes call with uniform operands; one elected lane issues)
__device__ __forceinline__ void umma_f16_ss_cg2_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

// Stage 32 rows x 32 bf16 (thread = row) into a 64B-swizzled 2 KB block and TMA-store it.
template <int PENDING>
__device__ __forceinline__ void tma_store_chunk(uint8_t* stg, const CUtensorMap* map, int lane, const float (&v)[32],
                                                int col, int row0) {
  // the slot we overwrite was used PENDING+1 stores ago: allow PENDING groups in flight
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(PENDING) : "memory");
  __syncwarp();
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint4 q;
    q.x = pack_bf16x2(v[u * 8 + 0], v[u * 8 + 1]);
    q.y = pack_bf16x2(v[u * 8 + 2], v[u * 8 + 3]);
    q.z = pack_bf16x2(v[u * 8 + 4], v[u * 8 + 5]);
    q.w = pack_bf16x2(v[u * 8 + 6], v[u * 8 + 7]);
    st_shared_v4(smem_u32(stg) + lane * 64 + ((u ^ sw) << 4), q);
  }
  tc::fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(stg)), "r"(col), "r"(row0)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

// Both outputs of a BIAS_GELU chunk (pre-activation and activation) staged together: one
// proxy fence and one bulk-group for the two TMA stores.
template <int PENDING>
__device__ __forceinline__ void tma_store_chunk2(uint8_t* stg0, const CUtensorMap* map0, const float (&v0)[32],
                                                 uint8_t* stg1, const CUtensorMap* map1, const float (&v1)[32],
                                                 int lane, int col, int row0) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(PENDING) : "memory");
  __syncwarp();
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint4 q0, q1;
    q0.x = pack_bf16x2(v0[u * 8 + 0], v0[u * 8 + 1]);
    q0.y = pack_bf16x2(v0[u * 8 + 2], v0[u * 8 + 3]);
    q0.z = pack_bf16x2(v0[u * 8 + 4], v0[u * 8 + 5]);
    q0.w = pack_bf16x2(v0[u * 8 + 6], v0[u * 8 + 7]);
    q1.x = pack_bf16x2(v1[u * 8 + 0], v1[u * 8 + 1]);
    q1.y = pack_bf16x2(v1[u * 8 + 2], v1[u * 8 + 3]);
    q1.z = pack_bf16x2(v1[u * 8 + 4], v1[u * 8 + 5]);
    q1.w = pack_bf16x2(v1[u * 8 + 6], v1[u * 8 + 7]);
    st_shared_v4(smem_u32(stg0) + lane * 64 + ((u ^ sw) << 4), q0);
    st_shared_v4(smem_u32(stg1) + lane * 64 + ((u ^ sw) << 4), q1);
  }
  tc::fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map0)),
                 "r"(smem_u32(stg0)), "r"(col), "r"(row0)
                 : "memory");
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map1)),
                 "r"(smem_u32(stg1)), "r"(col), "r"(row0)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

template <int BN, bool A_MN, bool B_MN, int EK, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX, const GemmArgs a) {
  using C = Cfg<BN, A_MN, B_MN, EK, PAIR>;
  static_assert(!PAIR || BN == 256, "pair mode: BN 256");
  // pair mode: tiles are 256 rows (num_m counts 256-row blocks), CTA `rank` owns rows 128*rank..
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int ctas = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;   // tile workers (pairs or CTAs)
  const int cta_id = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  constexpr int TM = PAIR ? 2 * BM : BM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_epi = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* aux_bar = tempty + 2;  // [kEpiWarps][XSLOTS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + kEpiWarps * C::XSLOTS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.num_m * a.num_n * a.splits;
  // Row sums of A ride along as a second accumulator: per K=16 step one extra M=128,N=16 MMA
  // against a constant all-ones B tile (placed in the epilogue staging area, unused by fp32
  // epilogues).  The accumulator sits at TMEM column BN, so the tile accumulator is
  // single-buffered in this mode (wgrad launches own <= 1 tile per CTA anyway).
  const bool rs_mode = a.rowsum != nullptr;
  if (rs_mode) {
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem_epi);
    for (int i = threadIdx.x; i < 512; i += kThreads) ones[i] = 0x3F803F80u;  // bf16 1.0 pairs, 16x64
    tc::fence_proxy_async();
  }

  if (warp == kWProd && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    if (a.tma_out) tc::tma_prefetch(&tmC);
    if (a.tma_out || a.tma_aux) tc::tma_prefetch(&tmX);
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], PAIR ? 2 * kEpiWarps : kEpiWarps);   // pair: both CTAs' epilogues drain
    }
    for (int s = 0; s < kEpiWarps * C::XSLOTS; ++s) tc::mbar_init(&aux_bar[s], 1);
    tc::fence_barrier_init();
  }
  if (warp == kWAlloc) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
    }
  }
  tc::tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWProd) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cta_id; t < total; t += ctas) {
        const int mn = t % (a.num_m * a.num_n);
        const int split = t / (a.num_m * a.num_n);
        const int m0 = (mn / a.num_n) * TM + (int)rank * BM, n0 = (mn % a.num_n) * BN;
        const int kb0 = split * a.kb_per_split;
        const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          const int k0 = kb * BK;
          if constexpr (PAIR) {
            // both CTAs' bytes complete on the leader's full barrier; the leader arms it for both
            const uint32_t fb = map_rank(&full[stage], 0);
            if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            if (A_MN) {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_2d_cg2(sa + j * 8192, &tmA, fb, m0 + 64 * j, k0);
            } else {
              tma_load_2d_cg2(sa, &tmA, fb, k0, m0);
            }
            const int nb = n0 + (int)rank * (BN / 2);
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 128; ++j) tma_load_2d_cg2(sb + j * 8192, &tmB, fb, nb + 64 * j, k0);
            } else {
              tma_load_2d_cg2(sb, &tmB, fb, k0, nb);
            }
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          tc::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tc::tma_load_2d(sa + j * 8192, &tmA, &full[stage], m0 + 64 * j, k0);
          } else {
            tc::tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tc::tma_load_2d(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0);
          } else {
            tc::tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == kWMma) {
    if (leader) {
      // ------------------------------------------------ MMA issuer (pair mode: the leader CTA only);
      // the whole warp runs the loop with uniform values, one elected lane issues each tcgen05 op
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint32_t s0 = smem_u32(smem);
      const uint64_t da0 = A_MN ? tc::sdesc_sw128(s0, 8192, 1024) : tc::sdesc_sw128(s0, 16, 1024);
      const uint64_t db0 = B_MN ? tc::sdesc_sw128(s0 + C::A_BYTES, 8192, 1024) : tc::sdesc_sw128(s0 + C::A_BYTES, 16, 1024);
      for (int t = cta_id; t < total; t += ctas, ++it) {
        const int split = t / (a.num_m * a.num_n);
        const int kb0 = split * a.kb_per_split;
        const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        const int acc = rs_mode ? 0 : (it & 1);
        const uint32_t acc_phase = rs_mode ? (it & 1) : ((it >> 1) & 1);
        // row sums: with split-K, n-tile r of a row block sums the r-th of num_n contiguous parts of the
        // unit's K blocks (the launch waits for its slowest tile; n-tile 0 alone took +12-19 %) and adds
        // its partial sums atomically.  Without split-K (deterministic mode) n-tile 0 sums them all.
        const int rs_n = t % a.num_n, rs_len = kb1 - kb0;
        const int rs_lo = a.splits > 1 ? kb0 + (int)((int64_t)rs_len * rs_n / a.num_n) : (rs_n == 0 ? kb0 : kb1);
        const int rs_hi = a.splits > 1 ? kb0 + (int)((int64_t)rs_len * (rs_n + 1) / a.num_n) : kb1;
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        const uint32_t ones_u32 = smem_u32(smem_epi);
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          // descriptors differ only in the start-address field (bits 0-13, 16-byte units)
          const uint64_t soff = (uint64_t)((stage * C::STAGE_BYTES) >> 4);
#pragma unroll
          const bool do_rs = rs_mode && kb >= rs_lo && kb < rs_hi;
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = da0 + soff + (uint64_t)((A_MN ? k * 2048 : k * 32) >> 4);
            const uint64_t db = db0 + soff + (uint64_t)((B_MN ? k * 2048 : k * 32) >> 4);
            if constexpr (PAIR) {
              umma_f16_ss_cg2_w(d_tmem, da, db, C::IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
              if (do_rs)   // ones tile: each CTA supplies 8 of the 16 B rows (all ones)
                umma_f16_ss_cg2_w(tmem + BN, da, tc::sdesc_sw128(ones_u32 + k * 32, 16, 1024), C::IDESC_RS,
                                (kb > rs_lo || k > 0) ? 1u : 0u);
              continue;
            }
            tc::umma_f16_ss_w(d_tmem, da, db, C::IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
            if (do_rs)
              tc::umma_f16_ss_w(tmem + BN, da, tc::sdesc_sw128(ones_u32 + k * 32, 16, 1024), C::IDESC_RS,
                              (kb > rs_lo || k > 0) ? 1u : 0u);
          }
          if (PAIR) umma_commit_pair_w(&empty[stage]); else tc::umma_commit_w(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (PAIR) umma_commit_pair_w(&tfull[acc]); else tc::umma_commit_w(&tfull[acc]);
      }
    }
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------ epilogue
    // warp w: TMEM lane quadrant (w & 3) = rows 32q..32q+31, column half (w-4)/4 of the tile
    const int ew = warp & 3, eh = warp >> 2, ei = warp;
    constexpr int SS = C::SSLOTS, XS = C::XSLOTS;
    constexpr int NCH = BN / 64;                       // 32-column chunks per warp
    uint8_t* stg = smem_epi + ei * SS * 2048;                            // TMA-store staging slots
    uint8_t* axs = smem_epi + kEpiWarps * SS * 2048 + ei * XS * 2048;    // TMA-loaded aux ring
    uint64_t* axb = aux_bar + ei * XS;
    int sbuf = 0;
    uint32_t auxc = 0;                                 // aux chunks consumed (ring position)
    const bool tma_aux = (EK == 1) && a.tma_aux != 0;
    const uint32_t tlane = (uint32_t)(ew * 32) << 16;
    int it = 0;
    const uint32_t tempty_leader0 = PAIR ? map_rank(&tempty[0], 0) : 0u;
    for (int t = cta_id; t < total; t += ctas, ++it) {
      const int mn = t % (a.num_m * a.num_n);
      const int m0 = (mn / a.num_n) * TM + (int)rank * BM, n0 = (mn % a.num_n) * BN + eh * (BN / 2);
      const int acc = rs_mode ? 0 : (it & 1);
      const uint32_t acc_phase = rs_mode ? (it & 1) : ((it >> 1) & 1);
      const int row0 = m0 + ew * 32;
      if (tma_aux && lane == 0) {
        // prefetch this tile's first XS aux chunks (the ring slots were freed by the last tile)
#pragma unroll
        for (int c = 0; c < XS && c < NCH; ++c) {
          const int slot = (auxc + c) % XS;
          tc::mbar_arrive_expect_tx(&axb[slot], 2048);
          tc::tma_load_2d(axs + slot * 2048, &tmX, &axb[slot], n0 + c * 32, row0);
        }
      }
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      const int row = row0 + lane;
      const uint32_t tbase = tmem + acc * BN + tlane + eh * (BN / 2);
      bool has_rs = false;
      if (rs_mode && eh == 0) {   // the MMA warp's rs_lo < rs_hi for this tile
        const int split = t / (a.num_m * a.num_n);
        const int kb0 = split * a.kb_per_split, kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        const int rn = mn % a.num_n, len = kb1 - kb0;
        has_rs = a.splits > 1 ? ((int64_t)len * (rn + 1) / a.num_n > (int64_t)len * rn / a.num_n) : rn == 0;
      }
      if (has_rs) {
        uint32_t rs;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(rs) : "r"(tmem + BN + tlane));
        tc::tmem_ld_wait();
        if (row < a.M) atomicAdd(a.rowsum + row, __uint_as_float(rs));
      }
      uint32_t rbuf[2][32];
      tc::tmem_ld_32x32b_x32(tbase, rbuf[0]);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = n0 + c * 32;
        uint32_t (&r)[32] = rbuf[c & 1];
        tc::tmem_ld_wait();
        if (c + 1 < NCH) tc::tmem_ld_32x32b_x32(tbase + (c + 1) * 32, rbuf[(c + 1) & 1]);  // overlap next load
        float xa[32];
        if (tma_aux) {
          const int slot = auxc % XS;
          tc::mbar_wait(&axb[slot], (auxc / XS) & 1);
          const uint8_t* src = axs + slot * 2048 + lane * 64;
          const int sw = (lane >> 1) & 3;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 q = ld_shared_v4(smem_u32(src) + ((u ^ sw) << 4));
            const __nv_bfloat162* hq = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(hq[e]);
              xa[u * 8 + 2 * e] = f.x;
              xa[u * 8 + 2 * e + 1] = f.y;
            }
          }
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0 && c + XS < NCH) {
            tc::mbar_arrive_expect_tx(&axb[slot], 2048);
            tc::tma_load_2d(axs + slot * 2048, &tmX, &axb[slot], col + XS * 32, row0);
          }
          ++auxc;
        }
        if (col >= a.N) continue;
        float v[32];
        // the element-wise epilogue math runs on f32x2 pairs (FFMA2 / FMUL2 / FADD2)
        auto pr = [](float (&w)[32], int j) -> float2 { return make_float2(w[j], w[j + 1]); };
        auto pw = [](float (&w)[32], int j, float2 p) { w[j] = p.x; w[j + 1] = p.y; };
        const float2 alpha2 = make_float2(a.alpha, a.alpha);
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          pw(v, j, tc::f2mul(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), alpha2));
        if (a.bias) {
          if (col + 32 <= a.N && a.vec_ok) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 bb = __ldg(reinterpret_cast<const float4*>(a.bias + col + j));
              pw(v, j, tc::f2add(pr(v, j), make_float2(bb.x, bb.y)));
              pw(v, j + 2, tc::f2add(pr(v, j + 2), make_float2(bb.z, bb.w)));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += (col + j < a.N) ? __ldg(a.bias + col + j) : 0.f;
          }
        }
        if (a.epi == AVB_EPI_BF16) {
          if (a.aux) {
            if (!tma_aux) load_aux_chunk(a, a.aux, row, col, xa);
#pragma unroll
            for (int j = 0; j < 32; j += 2) pw(v, j, tc::f2add(pr(v, j), pr(xa, j)));
          }
        } else if (a.epi == AVB_EPI_BIAS_GELU) {
          if (EK == 2 && SS % 2 == 0 && a.tma_out) {   // both outputs in one staged group
#pragma unroll
            for (int j = 0; j < 32; j += 2) pw(xa, j, tc::quick_gelu2(pr(v, j)));
            tma_store_chunk2<SS / 2 - 1>(stg + sbuf * 2048, &tmX, v, stg + ((sbuf + 1) % SS) * 2048, &tmC, xa, lane,
                                         col, row0);
            sbuf = (sbuf + 2) % SS;
            continue;
          }
          if (a.tma_out) {
            tma_store_chunk<SS - 1>(stg + sbuf * 2048, &tmX, lane, v, col, row0);
            sbuf = (sbuf + 1) % SS;
          } else {
            store_aux_chunk(a, row, col, v);
          }
#pragma unroll
          for (int j = 0; j < 32; j += 2) pw(v, j, tc::quick_gelu2(pr(v, j)));
        } else if (a.epi == AVB_EPI_DGELU) {
          if (!tma_aux) load_aux_chunk(a, a.aux, row, col, xa);
#pragma unroll
          for (int j = 0; j < 32; j += 2) pw(v, j, tc::f2mul(pr(v, j), tc::quick_gelu_grad2(pr(xa, j))));
        }
        if (a.tma_out) {
          tma_store_chunk<SS - 1>(stg + sbuf * 2048, &tmC, lane, v, col, row0);
          sbuf = (sbuf + 1) % SS;
        } else {
          store_row_chunk(a, row, col, v);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_cluster(tempty_leader0 + acc * 8u); else tc::mbar_arrive(&tempty[acc]);
      }
    }
  }

  if (warp < kEpiWarps && a.tma_out && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
  tc::tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == kWAlloc) {
    tc::tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
    else
      tc::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// A/B experiment switches (same-box comparisons of the pair / TMA-store / heavy-epilogue paths):
// read from the environment only in a -DAVB_DEBUG_KNOBS build; the product build has none.
inline bool knob(const char* name) {
#ifdef AVB_DEBUG_KNOBS
  return getenv(name) != nullptr;
#else
  (void)name;
  return false;
#endif
}

template <int BN, bool A_MN, bool B_MN, int EK, bool PAIR = false>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tcm, const CUtensorMap& tx,
           const GemmArgs& a, cudaStream_t st) {
  using C = Cfg<BN, A_MN, B_MN, EK, PAIR>;
  auto kern = gemm_kernel<BN, A_MN, B_MN, EK, PAIR>;
  if (int e = avb::ensure_kernel_attrs(reinterpret_cast<const void*>(kern), C::SMEM, "gemm: set smem attribute"))
    return e;
  const int total = a.num_m * a.num_n * a.splits;
  if (!PAIR) {
    const int grid = total < avb::sm_count() ? total : avb::sm_count();
    kern<<<grid, kThreads, C::SMEM, st>>>(ta, tb, tcm, tx, a);
    return avb::launch_status("avb_gemm");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr2[1];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = 2;
  attr2[0].val.clusterDim.y = 1;
  attr2[0].val.clusterDim.z = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = 1;
  // persistent pairs: as many as can be co-resident (a TPC with a harvested SM hosts no pair)
  // (per device and kernel instantiation; a benign race between threads computes the same value)
  static std::atomic<int> max_pairs_dev[64];
  int dev = 0;
  (void)cudaGetDevice(&dev);
  std::atomic<int>& max_pairs = max_pairs_dev[dev & 63];
  if (max_pairs.load(std::memory_order_relaxed) == 0) {
    cfg.gridDim = dim3(avb::sm_count(), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
      (void)cudaGetLastError();
      n = avb::sm_count() / 2;
    }
    max_pairs.store(n, std::memory_order_relaxed);
  }
  const int pairs = std::min(total, max_pairs.load(std::memory_order_relaxed));
  cfg.gridDim = dim3(2 * pairs, 1, 1);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, tx, a);
  if (e != cudaSuccess) return avb::cuda_status(e, "avb_gemm (pair launch)");
  return avb::launch_status("avb_gemm");
}

}  // namespace

// ------------------------------------------------------------------ tensor maps
namespace avb {
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encode() {
  if (g_encode) return AVB_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return AVB_E_CUDA;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return AVB_OK;
}

int make_tmap_2d_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                      uint32_t box_inner, uint32_t box_outer) {
  int s = get_encode();
  if (s) return s;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%llu box=%u,%u", (int)r,
              (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld_elems, box_inner, box_outer);
    return AVB_E_ARG;
  }
  return AVB_OK;
}

int make_tmap_3d_bf16(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_elems,
                      uint64_t s2_elems, uint32_t b0, uint32_t b1, uint32_t b2) {
  int s = get_encode();
  if (s) return s;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_elems * 2, s2_elems * 2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(3d) failed (%d)", (int)r);
    return AVB_E_ARG;
  }
  return AVB_OK;
}
int make_tmap_2d_bf16_sw(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                         uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  int s = get_encode();
  if (s) return s;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(2d bf16 sw%d) failed (%d)", swizzle_bytes, (int)r);
    return AVB_E_ARG;
  }
  return AVB_OK;
}

int make_tmap_3d_f32(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_elems,
                     uint64_t s2_elems, uint32_t b0, uint32_t b1, uint32_t b2, int swizzle_bytes) {
  int s = get_encode();
  if (s) return s;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_elems * 4, s2_elems * 4};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, (swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(3d f32) failed (%d)", (int)r);
    return AVB_E_ARG;
  }
  return AVB_OK;
}
}  // namespace avb

extern "C" int avb_gemm(const void* A, int64_t lda, int a_major, const void* B, int64_t ldb, int b_major, void* C,
                        int64_t ldc, int M, int N, int K, int epilogue, const float* bias, const void* aux,
                        int64_t ldaux, void* aux_out, float alpha, int split_k, float* a_rowsum, void* stream) {
  AVB_CHECK_ARG(M >= 0 && N >= 0 && K >= 0, "negative GEMM dims");
  if (M == 0 || N == 0) return AVB_OK;
  AVB_CHECK_ARG(K >= 1, "K must be >= 1");
  AVB_CHECK_ARG(A && B && C, "null operand");
  AVB_CHECK_ARG(a_major == 0 || a_major == 1, "a_major must be 0 (K-major) or 1 (MN-major)");
  AVB_CHECK_ARG(b_major == 0 || b_major == 1, "b_major must be 0 (K-major) or 1 (MN-major)");
  AVB_CHECK_ARG(epilogue >= AVB_EPI_BF16 && epilogue <= AVB_EPI_F32_ACCUM, "bad epilogue %d", epilogue);
  AVB_CHECK_ARG((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
                "A/B must be 16-byte aligned");
  AVB_CHECK_ARG((lda * 2) % 16 == 0 && (ldb * 2) % 16 == 0, "lda/ldb must be multiples of 8 elements");
  AVB_CHECK_ARG(lda >= (a_major ? M : K) && ldb >= (b_major ? N : K), "leading dimension too small");
  AVB_CHECK_ARG(ldc >= N, "ldc < N");
  AVB_CHECK_ARG(epilogue != AVB_EPI_BIAS_GELU || aux_out, "BIAS_GELU needs aux_out");
  AVB_CHECK_ARG(epilogue != AVB_EPI_DGELU || aux, "DGELU needs aux (pre-activation)");
  AVB_CHECK_ARG(split_k >= 1, "split_k must be >= 1");
  AVB_CHECK_ARG(split_k == 1 || epilogue == AVB_EPI_F32_ACCUM, "split_k > 1 needs EPI_F32_ACCUM");
  AVB_CHECK_ARG(!a_rowsum || epilogue == AVB_EPI_F32 || epilogue == AVB_EPI_F32_ACCUM,
                "a_rowsum needs an fp32 epilogue (EPI_F32 / EPI_F32_ACCUM)");
  AVB_CHECK_ARG(!a_rowsum || (reinterpret_cast<uintptr_t>(a_rowsum) & 3) == 0, "a_rowsum must be 4-byte aligned");

  const int BN = (N <= 128) ? 128 : 256;
  // CTA pairs (cta_group::2, 256 x 256 tiles) for the large-M forward / dgrad shapes
  const bool pair = BN == 256 && M > 128 && !knob("AVB_GEMM_NO_PAIR");
  CUtensorMap ta, tb;
  int s;
  if (a_major == 0)
    s = avb::make_tmap_2d_bf16(&ta, A, K, M, lda, 64, 128);
  else
    s = avb::make_tmap_2d_bf16(&ta, A, M, K, lda, 64, 64);
  if (s) return s;
  if (b_major == 0)
    s = avb::make_tmap_2d_bf16(&tb, B, K, N, ldb, 64, pair ? BN / 2 : BN);
  else
    s = avb::make_tmap_2d_bf16(&tb, B, N, K, ldb, 64, 64);
  if (s) return s;

  GemmArgs g;
  g.C = C;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.epi = epilogue;
  g.bias = bias;
  g.aux = aux;
  g.ldaux = ldaux;
  g.aux_out = aux_out;
  g.alpha = alpha;
  g.rowsum = a_rowsum;
  g.num_m = (M + BM - 1) / BM;   // pair mode re-derives it below
  g.num_n = (N + BN - 1) / BN;
  g.num_kb = (K + BK - 1) / BK;
  int splits = split_k;
  if (splits > g.num_kb) splits = g.num_kb;
  g.kb_per_split = (g.num_kb + splits - 1) / splits;
  g.splits = (g.num_kb + g.kb_per_split - 1) / g.kb_per_split;
  const int esz = (epilogue == AVB_EPI_F32 || epilogue == AVB_EPI_F32_ACCUM) ? 4 : 2;
  g.vec_ok = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((ldc * esz) % 16 == 0) &&
             (!aux || (((reinterpret_cast<uintptr_t>(aux) & 15) == 0) && (ldaux * 2) % 16 == 0)) &&
             (!aux_out || (((reinterpret_cast<uintptr_t>(aux_out) & 15) == 0) && (ldaux * 2) % 16 == 0));
  // bf16 outputs go out through TMA stores (64B-swizzled 32x32 boxes; TMA clips M/N tails)
  CUtensorMap tcm, tx;
  memset(&tcm, 0, sizeof(tcm));
  memset(&tx, 0, sizeof(tx));
  g.tma_out = 0;
  if (g.vec_ok && (epilogue == AVB_EPI_BF16 || epilogue == AVB_EPI_BIAS_GELU || epilogue == AVB_EPI_DGELU) &&
      !knob("AVB_GEMM_NO_TMA_STORE")) {
    int s1 = avb::make_tmap_2d_bf16_sw(&tcm, C, N, M, ldc, 32, 32, 64);
    int s2 = (epilogue == AVB_EPI_BIAS_GELU) ? avb::make_tmap_2d_bf16_sw(&tx, aux_out, N, M, ldaux, 32, 32, 64) : 0;
    if (s1 == AVB_OK && s2 == AVB_OK) g.tma_out = 1;
  }
  g.tma_aux = 0;
  if (g.vec_ok && aux && (epilogue == AVB_EPI_BF16 || epilogue == AVB_EPI_DGELU) && a_major == 0 && N > 128 &&
      !knob("AVB_GEMM_NO_TMA_AUX")) {
    if (avb::make_tmap_2d_bf16_sw(&tx, aux, N, M, ldaux, 32, 32, 64) == AVB_OK) g.tma_aux = 1;
  }
  cudaStream_t st = avb::as_stream(stream);
  const int key = (BN == 256 ? 4 : 0) | (a_major << 1) | b_major;
  // heavy epilogues (bf16 aux read or a second bf16 output) get 3 mainloop stages and 6-deep
  // aux / store rings so TMA latency is covered while the epilogue streams 32-column chunks
  const bool heavy = BN == 256 && a_major == 0 && (g.tma_aux || (g.tma_out && epilogue == AVB_EPI_BIAS_GELU)) &&
                     !knob("AVB_GEMM_NO_HEAVY");
  // aux-reading epilogues run as CTA pairs too: with the staging on st.shared and the relaxed
  // accumulator-empty arrival, the K = 768 shapes gained (same box: fc2 dgrad + dGELU 961 -> 996,
  // proj fwd + residual 962 -> 1031 TFLOP/s; round 1, before those fixes, they were 2-4 % slower)
  if (pair && !knob("AVB_GEMM_NO_PAIR_AUX")) {
    g.num_m = (M + 2 * BM - 1) / (2 * BM);
    if (heavy && g.tma_aux) {
      if (b_major == 0) return launch<256, false, false, 1, true>(ta, tb, tcm, tx, g, st);
      return launch<256, false, true, 1, true>(ta, tb, tcm, tx, g, st);
    }
    if (heavy) {
      if (b_major == 0) return launch<256, false, false, 2, true>(ta, tb, tcm, tx, g, st);
      return launch<256, false, true, 2, true>(ta, tb, tcm, tx, g, st);
    }
    switch ((a_major << 1) | b_major) {
      case 0: return launch<256, false, false, 0, true>(ta, tb, tcm, tx, g, st);
      case 1: return launch<256, false, true, 0, true>(ta, tb, tcm, tx, g, st);
      case 2: return launch<256, true, false, 0, true>(ta, tb, tcm, tx, g, st);
      default: return launch<256, true, true, 0, true>(ta, tb, tcm, tx, g, st);
    }
  }
  if (pair && b_major == 0) {   // single-CTA fallback of a pair-eligible launch: full-height B boxes
    if ((s = avb::make_tmap_2d_bf16(&tb, B, K, N, ldb, 64, BN))) return s;
  }
  if (heavy) {
    if (g.tma_aux) {
      if (b_major == 0) return launch<256, false, false, 1>(ta, tb, tcm, tx, g, st);
      return launch<256, false, true, 1>(ta, tb, tcm, tx, g, st);
    }
    if (b_major == 0) return launch<256, false, false, 2>(ta, tb, tcm, tx, g, st);
    return launch<256, false, true, 2>(ta, tb, tcm, tx, g, st);
  }
  switch (key) {
    case 0: return launch<128, false, false, 0>(ta, tb, tcm, tx, g, st);
    case 1: return launch<128, false, true, 0>(ta, tb, tcm, tx, g, st);
    case 2: return launch<128, true, false, 0>(ta, tb, tcm, tx, g, st);
    case 3: return launch<128, true, true, 0>(ta, tb, tcm, tx, g, st);
    case 4: return launch<256, false, false, 0>(ta, tb, tcm, tx, g, st);
    case 5: return launch<256, false, true, 0>(ta, tb, tcm, tx, g, st);
    case 6: return launch<256, true, false, 0>(ta, tb, tcm, tx, g, st);
    default: return launch<256, true, true, 0>(ta, tb, tcm, tx, g, st);
  }
}
