/*
 * avion_b200.h -- C ABI of the B200-native AVION training hot path.
 *
 * One shared library, paper_2309_16669_b200/libavion_b200.so, built for
 * sm_100a only.  Every entry point:
 *   - takes plain device pointers + sizes/strides (no torch types),
 *   - launches asynchronously on the caller's CUDA stream (`stream` is a
 *     cudaStream_t passed as void*; NULL = legacy default stream),
 *   - never synchronises and never allocates device memory the caller
 *     did not pass in, except the per-process cached TMA descriptors,
 *   - returns AVB_OK (0) or an AVB_E_* code; avb_last_error() gives text.
 * The host-side argument checks run before any launch, so a bad call leaves
 * the output untouched (the reference raises InputError "before any decode",
 * pkg/src/vidpipe/decoder.py:116-119).
 *
 * Reference interfaces replaced (file:line under /root/reference):
 *   avb_rrc_normalize  <- _codec.yuv_to_rgb(y,u,v,hflip,tw,th)
 *                           pkg/src/vidpipe/_codec/codec.cpp:250-275 (binding :806-807)
 *                         VideoReader.current_rgb(x,y,w,h,hflip,tw,th)
 *                           codec.cpp:452-467 (binding :823-825)
 *                         and the Python step that calls them per frame,
 *                           decoder.py:257-271 (crop_planes :282-292),
 *                         extended with the GPU normalize + cast the reference
 *                         defers.
 *   avb_rrc_taps       <- (test hook) the tap table the scaler derives from
 *                         (crop, target); codec.cpp:233-241.
 *   everything else    <- no reference code: the encoder / attention / loss
 *                         the reference only names (README.md:159-161,
 *                         models.py:34-74,127-145).
 */
#ifndef AVION_B200_H
#define AVION_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define AVB_OK             0
#define AVB_E_ARG          1  /* bad dims / strides / dtype / null pointer   */
#define AVB_E_BOX          2  /* crop box not contained in the frame         */
#define AVB_E_UNSUPPORTED  3  /* valid but outside the kernel's envelope     */
#define AVB_E_CUDA         4  /* CUDA runtime / launch error                 */

/* ---- enums ---- */
#define AVB_DTYPE_BF16     0
#define AVB_DTYPE_F32      1

#define AVB_LAYOUT_CTHW    0  /* dst [B,3,T,Ht,Wt]  (encoder input)            */
#define AVB_LAYOUT_TCHW    1  /* dst [B,T,3,Ht,Wt]  (reference Batch.frames)   */
#define AVB_LAYOUT_TUBELET 2  /* dst [B*Np, 3*tt*ph*pw] patch-embed GEMM rows     */

/* GEMM epilogues (avb_gemm) */
#define AVB_EPI_BF16       0  /* C bf16 = alpha*acc (+bias) (+aux residual)                 */
#define AVB_EPI_BIAS_GELU  1  /* aux_out bf16 = alpha*acc+bias; C bf16 = QuickGELU(aux_out)   */
#define AVB_EPI_DGELU      2  /* C bf16 = alpha*acc * QuickGELU'(aux)                       */
#define AVB_EPI_F32        3  /* C fp32 = alpha*acc (+bias)                                 */
#define AVB_EPI_F32_ACCUM  4  /* C fp32 += alpha*acc (red.add; allows split_k > 1)          */

const char* avb_last_error(void);
int avb_version(void);
int avb_device_sm_count(void);

/*
 * K1: fused crop -> hflip -> antialiased bilinear -> normalize -> cast.
 *   src        uint8 frames, element (b,t,y,x,c) at
 *              src[b*s_clip + t*s_t + y*s_h + x*s_w + c*s_c]   (byte strides)
 *              Fast path: s_c == 1 && s_w == 3 (interleaved RGB, THWC).
 *              Any other strides (e.g. the reference's [B,T,3,H,W]) take the
 *              generic path.
 *   boxes_dev  int32 [B,4] device, CropRect order (x, y, crop_w, crop_h)
 *   hflip_dev  uint8 [B] device (nullable = no flip)
 *   boxes_host optional host copy of boxes; when given, every box is checked
 *              against (W,H) and AVB_E_BOX returned before launch.  The kernel
 *              re-checks on device and leaves invalid clips untouched.
 *   mean3, inv_std3  host float[3]; y = (v/255 - mean[c]) * inv_std[c]
 *   dst        device, layout per out_layout, dtype per out_dtype
 */
int avb_rrc_normalize(const uint8_t* src, int64_t B, int T, int H, int W,
                      int64_t s_clip, int64_t s_t, int64_t s_h, int64_t s_w, int64_t s_c,
                      const int32_t* boxes_dev, const uint8_t* hflip_dev,
                      const int32_t* boxes_host, int Ht, int Wt,
                      const float* mean3, const float* inv_std3,
                      int out_dtype, int out_layout, void* dst, void* stream);

/* K1 writing straight into the tubelet patch-embed operand: row n' = ((t/tt)*(Ht/ph) + y/ph)*(Wt/pw)
 * + x/pw of clip b, feature ((c*tt + t%tt)*ph + y%ph)*pw + x%pw (Conv3d weight flattening), so the
 * K2 GEMM reads it with no im2col pass.  tub_w must be even. */
int avb_rrc_normalize_tubelet(const uint8_t* src, int64_t B, int T, int H, int W,
                              int64_t s_clip, int64_t s_t, int64_t s_h, int64_t s_w, int64_t s_c,
                              const int32_t* boxes_dev, const uint8_t* hflip_dev,
                              const int32_t* boxes_host, int Ht, int Wt,
                              const float* mean3, const float* inv_std3, int out_dtype,
                              int tub_t, int tub_h, int tub_w, void* dst, void* stream);

/* Test hook: pin K1's kernel choice for the calling process (path comparisons in the parity tests).
 * AVB_K1_PATH_AUTO (default) picks identity / streaming / strip / generic by shape; GENERIC forces the
 * any-stride kernel, STRIP the strip/band kernel.  Returns the previous setting. */
#define AVB_K1_PATH_AUTO    0
#define AVB_K1_PATH_GENERIC 1
#define AVB_K1_PATH_STRIP   2
int avb_k1_force_path(int path);

/* Test hook: the device-computed tap table for one (crop, target) pair:
 * lo[tgt], hi[tgt] int32 device, weights[tgt*max_taps] float device. */
int avb_rrc_taps(int crop, int tgt, int32_t* lo_dev, int32_t* hi_dev, float* w_dev,
                 int max_taps, void* stream);

/*
 * K2/K3: C[M,N] = epilogue(alpha * sum_k A[m,k] B[n,k]) on tcgen05 (TMEM accumulators, TMA
 * 128B-swizzled operands, persistent warp-specialised, 1 CTA per SM).
 *   A: a_major 0 -> row-major [M,K] (lda >= K);  1 -> row-major [K,M] (lda >= M)
 *   B: b_major 0 -> row-major [N,K] (ldb >= K);  1 -> row-major [K,N] (ldb >= N)
 *   bf16 operands, 16-byte aligned, leading dims multiples of 8 elements.
 *   bias: fp32 [N] or NULL.  aux/aux_out: bf16 [M, ldaux] (see AVB_EPI_*).
 * Used for patch-embed (K2), QKV / out-proj / fc1 / fc2 forward, dgrad (A K-major, B MN-major)
 * and wgrad (both MN-major, EPI_F32_ACCUM, split_k over the token dimension).
 *   a_rowsum: fp32 [M] or NULL (fp32 epilogues only): a_rowsum[m] += sum_k A[m,k], unscaled --
 *   for a wgrad (A = dY^T) that is the bias gradient, computed on the tensor cores from the
 *   A tiles already in shared memory instead of a second pass over dY.  With split_k > 1 the
 *   n-tiles of a row block each sum a contiguous part of the K range and add atomically (order
 *   not fixed); with split_k == 1 one tile adds each row once (bit-reproducible).
 */
int avb_gemm(const void* A, int64_t lda, int a_major, const void* B, int64_t ldb, int b_major,
             void* C, int64_t ldc, int M, int N, int K, int epilogue, const float* bias,
             const void* aux, int64_t ldaux, void* aux_out, float alpha, int split_k,
             float* a_rowsum, void* stream);

/*
 * K4: blockwise attention forward, head_dim 64, fp32 online softmax, O(N) memory.
 *   q,k,v: bf16 [B, N, H, 64] views: element (b,n,h,d) at p[b*sb + n*ld + h*64 + d]
 *          (the packed QKV GEMM output works directly: q=qkv, k=qkv+H*64, v=qkv+2*H*64)
 *   o:     bf16, same form with (ld_o, sb_o)
 *   lse:   fp32 [B*H, Npad] natural-log row log-sum-exp, Npad = roundup(N,128)
 */
int avb_attn_fwd(const void* q, const void* k, const void* v, int64_t ld, int64_t sb,
                 void* o, int64_t ld_o, int64_t sb_o, float* lse, int B, int H, int N,
                 int head_dim, float softmax_scale, int causal, void* stream);

/*
 * K5: blockwise attention backward (recomputes P from lse; no N x N storage).
 *   o, dout share (ld_o, sb_o); dq, dk, dv share (ld_g, sb_g).
 *   delta:  scratch of B*H*Npad*32 bytes, 16-byte aligned (per query row: bf16 hi/lo of -lse/scale and
 *           of -rowsum(dO*O), laid out as the extension tiles of K5's S^T / dP^T MMAs).
 *   dq_acc: NULL (default) -- each key tile's dQ contribution is reduce-added (TMA, bf16 add) straight
 *           into the zeroed bf16 dq rows; or fp32 scratch [B, N, H, 64] -- contributions accumulate in
 *           fp32 and one convert kernel writes dq (one bf16 rounding instead of one per key tile).
 */
int avb_attn_bwd(const void* q, const void* k, const void* v, int64_t ld, int64_t sb,
                 const void* o, const void* dout, int64_t ld_o, int64_t sb_o, const float* lse,
                 float* delta, float* dq_acc, void* dq, void* dk, void* dv, int64_t ld_g, int64_t sb_g,
                 int B, int H, int N, int head_dim, float softmax_scale, int causal, void* stream);

/*
 * K5, bit-reproducible: identical to avb_attn_bwd except that every 128-key tile stores its dQ
 * contribution into its own fp32 slice of dq_part [ceil(N/128), B, N, H, 64] (16-byte aligned) and
 * one pass sums the slices in key-tile order, so dq (like dk, dv) is the same bit pattern run to run.
 * Costs ceil(N/128) x B*N*H*256 bytes of workspace and the extra traffic; meant for debugging.
 */
int avb_attn_bwd_deterministic(const void* q, const void* k, const void* v, int64_t ld, int64_t sb,
                               const void* o, const void* dout, int64_t ld_o, int64_t sb_o, const float* lse,
                               float* delta, float* dq_part, void* dq, void* dk, void* dv, int64_t ld_g,
                               int64_t sb_g, int B, int H, int N, int head_dim, float softmax_scale, int causal,
                               void* stream);

/* K6: LayerNorm over rows of D (<= 1024, multiple of 8) bf16 elements, fp32 gamma/beta/stats. */
int avb_layernorm_fwd(const void* x, int64_t ldx, const float* gamma, const float* beta, void* y,
                      int64_t ldy, float* mean, float* rstd, int M, int D, float eps, void* stream);
/* dx (=|+=) LN'(dy); dgamma/dbeta (nullable) += column reductions; dx_colsum (nullable) += column
 * sums of the resulting dx (the bias gradient of the linear layer whose output is this residual).
 * work: fp32 scratch of avb_layernorm_bwd_workspace(D) floats (per-block partials); every reduction
 * runs in a fixed order, so the result is bit-reproducible. */
int avb_layernorm_bwd(const void* dy, int64_t lddy, const void* x, int64_t ldx, const float* gamma,
                      const float* mean, const float* rstd, void* dx, int64_t lddx, float* dgamma,
                      float* dbeta, float* dx_colsum, float* work, int M, int D, int accumulate, void* stream);
int avb_layernorm_bwd_workspace(int D);

/* out[n] += sum_m X[m,n] (bias gradients); X bf16 [M, ldx]. */
int avb_colsum_accum(const void* X, int64_t ldx, int M, int N, float* out, void* stream);

/* Token assembly with the separable space-time position embedding of PAPER.md:727-729
 * (PE[i] = PE_t[i] + PE_s):  patch n = t*S + s (t < Np/S temporal index, s < S spatial index),
 *   x[b,0]   = cls + pos_s[0]
 *   x[b,1+n] = pe[b*Np+n] + pos_s[1+s] + pos_t[t]
 * pos_s fp32 [1+S, D] (CLIP's spatial table incl. the cls slot), pos_t fp32 [Np/S, D]; bf16 x. */
int avb_tokens_fwd(const void* pe, const float* cls, const float* pos_s, const float* pos_t, void* x, int B,
                   int Np, int S, int D, void* stream);
/* dpe = dx[:,1:] (nullable); dcls += sum_b dx[:,0]; dpos_s[0] += sum_b dx[:,0];
 * dpos_s[1+s] += sum_{b,t} dx[b,1+t*S+s]; dpos_t[t] += sum_{b,s} dx[b,1+t*S+s]  (each nullable).
 * work: fp32 scratch [Np+1, D]; all sums run in a fixed order (no atomics), so the result is
 * bit-reproducible.  dcls / dpos_s / dpos_t / work 16-byte aligned. */
int avb_tokens_bwd(const void* dx, void* dpe, float* dcls, float* dpos_s, float* dpos_t, float* work, int B, int Np,
                   int S, int D, void* stream);

/* Tubelet patchify of normalised clips (the nn.Module path that takes [B,3,T,H,W] input; the training
 * step gets the same rows straight from K1's tubelet layout): x bf16 contiguous [B,3,T,H,W] ->
 * dst [B*Np, 3*tt*th*tw], Conv3d-weight feature order; tw even. */
int avb_patchify(const void* x, int B, int T, int H, int W, int tt, int th, int tw, void* dst, void* stream);

/* softmax cross-entropy: loss += scale*sum_i (lse_i - z_i[y_i]); dlogits bf16 = scale*(softmax - onehot).
 * labels int32; a row whose label is outside [0, C) is ignored (no loss term, zero gradient row). */
int avb_xent(const float* logits, int64_t ld, const int32_t* labels, int B, int C, float scale, float* loss,
             void* dlogits, int64_t ldd, void* stream);

/* K8: AdamW with decoupled weight decay over a flat fp32 buffer; optional bf16 shadow copy;
 * decay_mask (nullable, uint8 per element) selects which elements get weight decay. */
int avb_adamw(float* p, const float* g, float* m, float* v, void* p_bf16, const uint8_t* decay_mask, int64_t n, float lr,
              float beta1, float beta2, float eps, float weight_decay, int step, float grad_scale,
              void* stream);
/* The same update with the step count kept on the device: *step_dev += 1 (a one-thread kernel on the
 * stream), then the bias corrections are computed from *step_dev -- a step captured in a CUDA graph
 * replays with the right step. */
int avb_adamw_dev(float* p, const float* g, float* m, float* v, void* p_bf16, const uint8_t* decay_mask, int64_t n,
                  float lr, float beta1, float beta2, float eps, float weight_decay, int* step_dev, float grad_scale,
                  void* stream);
int avb_cast_bf16(const float* src, void* dst, int64_t n, void* stream);

/*
 * K7: CLIP InfoNCE over a global batch. v, t: fp32 [Bg, E] raw (un-normalised)
 * embeddings; S = s * v^ t^T with s = exp(min(*log_scale, ln 100)) read on the device (no host sync).
 * fwd: norms [Bg], row/col LSE [Bg]; loss += L; dlog_scale (nullable) += dL/dlog_scale.
 * bwd: dv, dt [n, E] (=) grad_scale * dL/d(raw) for global rows / columns [r0, r0+n).
 */
int avb_infonce_fwd(const float* v, const float* t, int Bg, int E, const float* log_scale, float* norms_v,
                    float* norms_t, float* lse_r, float* lse_c, float* loss, float* dlog_scale, void* stream);
int avb_infonce_bwd(const float* v, const float* t, int Bg, int E, const float* log_scale,
                    const float* norms_v, const float* norms_t, const float* lse_r, const float* lse_c,
                    int r0, int n, float grad_scale, float* dv, float* dt, void* stream);

/* text-side token embedding: x[b*L+l] = table[tok] + pos[l] (bf16 out); bwd: dtable[tok] += dx (atomic),
 * dpos[l] += sum_b dx.  Out-of-range ids are clamped to [0, V). */
int avb_embed_fwd(const int32_t* tokens, const float* table, const float* pos, void* x, int B, int L, int D,
                  int V, void* stream);
int avb_embed_bwd(const int32_t* tokens, const void* dx, float* dtable, float* dpos, int B, int L, int D,
                  int V, void* stream);
/* bf16 row gather/scatter: dst[dst_idx ? dst_idx[i] : i] = src[src_idx ? src_idx[i] : i], i < n */
int avb_rows_copy(const void* src, int64_t lds, const int32_t* src_idx, void* dst, int64_t ldd,
                  const int32_t* dst_idx, int n, int D, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AVION_B200_H */
