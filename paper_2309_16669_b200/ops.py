"""Thin torch-facing wrappers over the C ABI (pointers + sizes + current stream).

Every function here validates dtypes/shapes/devices on the host and then calls
one `avb_*` entry point; none of them computes anything in PyTorch.  The
torch.autograd.Function / nn.Module layer on top of these lives in `nn.py`.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import InputError

EPI_BF16, EPI_BIAS_GELU, EPI_DGELU, EPI_F32, EPI_F32_ACCUM = 0, 1, 2, 3, 4


def _ptr(t):
    return None if t is None else t.data_ptr()


def _index(t: torch.Tensor, name: str, n: int | None = None) -> torch.Tensor:
    """Index tensors (labels, token ids, row indices) are read as int32 by the kernels."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InputError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.int32:
        raise InputError(f"{name} must be int32 (got {t.dtype}); the kernels read 32-bit indices")
    if not t.is_contiguous():
        raise InputError(f"{name} must be contiguous")
    if n is not None and t.numel() != n:
        raise InputError(f"{name} must have {n} elements, got {t.numel()}")
    return t


def _rowmajor(t: torch.Tensor, name: str) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise InputError(f"{name} must be a 2-D row-major view, got shape {tuple(t.shape)} strides {t.stride()}")
    return t.stride(0)


def gemm(a: torch.Tensor, b: torch.Tensor, *, a_mn: bool = False, b_mn: bool = False, out: torch.Tensor | None = None,
         epilogue: int = EPI_BF16, bias: torch.Tensor | None = None, aux: torch.Tensor | None = None,
         aux_out: torch.Tensor | None = None, alpha: float = 1.0, split_k: int = 1,
         a_rowsum: torch.Tensor | None = None) -> torch.Tensor:
    """C = epi(alpha * A @ B^T) on the tcgen05 GEMM.

    a: [M,K] (a_mn=False) or [K,M] (a_mn=True); b: [N,K] (b_mn=False) or [K,N] (b_mn=True).
    a_rowsum: fp32 [M], accumulated with sum_k A[m,k] (bias gradient of a wgrad; fp32 epilogues).
    """
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise InputError("gemm operands must be bf16")
    if not (a.is_cuda and b.is_cuda):
        raise InputError("gemm operands must be CUDA tensors")
    lda, ldb = _rowmajor(a, "a"), _rowmajor(b, "b")
    M, K = (a.shape[1], a.shape[0]) if a_mn else (a.shape[0], a.shape[1])
    N, Kb = (b.shape[1], b.shape[0]) if b_mn else (b.shape[0], b.shape[1])
    if K != Kb:
        raise InputError(f"gemm K mismatch {K} vs {Kb}")
    odt = torch.float32 if epilogue in (EPI_F32, EPI_F32_ACCUM) else torch.bfloat16
    if out is None:
        if epilogue == EPI_F32_ACCUM:
            out = torch.zeros((M, N), dtype=odt, device=a.device)
        else:
            out = torch.empty((M, N), dtype=odt, device=a.device)
    if out.dtype != odt or tuple(out.shape) != (M, N):
        raise InputError(f"out must be {odt} [{M},{N}], got {out.dtype} {tuple(out.shape)}")
    ldc = _rowmajor(out, "out")
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != N or not bias.is_contiguous()):
        raise InputError("bias must be contiguous fp32 [N]")
    ldaux = 0
    for t, nm in ((aux, "aux"), (aux_out, "aux_out")):
        if t is not None:
            if t.dtype != torch.bfloat16 or tuple(t.shape) != (M, N):
                raise InputError(f"{nm} must be bf16 [{M},{N}]")
            ldaux = _rowmajor(t, nm)
    if a_rowsum is not None and (a_rowsum.dtype != torch.float32 or a_rowsum.numel() != M
                                 or not a_rowsum.is_contiguous()):
        raise InputError(f"a_rowsum must be contiguous fp32 [{M}]")
    if aux is not None and aux_out is not None and aux.stride(0) != aux_out.stride(0):
        raise InputError("aux and aux_out must share a leading dimension")
    lib = _lib.load()
    st = lib.avb_gemm(a.data_ptr(), lda, int(a_mn), b.data_ptr(), ldb, int(b_mn), out.data_ptr(), ldc, M, N, K,
                      epilogue, _ptr(bias), _ptr(aux), ldaux, _ptr(aux_out), float(alpha), int(split_k),
                      _ptr(a_rowsum), _lib.stream_ptr())
    _lib.check(st, "gemm")
    return out


# ----------------------------------------------------------------------------- attention
def _bnhd(t: torch.Tensor, name: str, H: int):
    """Validate a [B, N, H*64] (or [B, N, H, 64]) bf16 view; return (B, N, ld, sb)."""
    if t.dtype != torch.bfloat16 or not t.is_cuda:
        raise InputError(f"{name} must be a bf16 CUDA tensor")
    if t.dim() == 4:
        if t.shape[2] != H or t.shape[3] != 64 or t.stride(3) != 1 or t.stride(2) != 64:
            raise InputError(f"{name} must be [B,N,H,64] with contiguous heads")
        return t.shape[0], t.shape[1], t.stride(1), t.stride(0)
    if t.dim() != 3 or t.shape[2] != H * 64 or t.stride(2) != 1:
        raise InputError(f"{name} must be [B,N,H*64] with unit last stride")
    return t.shape[0], t.shape[1], t.stride(1), t.stride(0)


def npad(N: int) -> int:
    return (N + 127) // 128 * 128


def attn_fwd(q, k, v, H: int, *, scale: float | None = None, causal: bool = False, out=None, lse=None):
    """O, LSE = blockwise attention over [B,N,H,64] views (q/k/v may be slices of packed QKV)."""
    B, N, ld, sb = _bnhd(q, "q", H)
    for t, nm in ((k, "k"), (v, "v")):
        if _bnhd(t, nm, H) != (B, N, ld, sb):
            raise InputError("q, k, v must share shape and strides")
    if out is None:
        out = torch.empty((B, N, H * 64), dtype=torch.bfloat16, device=q.device)
    _, _, ld_o, sb_o = _bnhd(out, "out", H)
    if lse is None:
        lse = torch.empty((B * H, npad(N)), dtype=torch.float32, device=q.device)
    elif (lse.dtype != torch.float32 or tuple(lse.shape) != (B * H, npad(N)) or not lse.is_contiguous()
          or not lse.is_cuda):
        raise InputError(f"lse must be a contiguous fp32 CUDA tensor [B*H, roundup(N,128)] = [{B * H}, {npad(N)}]")
    if tuple(out.shape[:2]) != (B, N):
        raise InputError("out must match q's [B, N]")
    scale = 64 ** -0.5 if scale is None else float(scale)
    st = _lib.load().avb_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), ld, sb, out.data_ptr(), ld_o, sb_o,
                                  lse.data_ptr(), B, H, N, 64, scale, int(causal), _lib.stream_ptr())
    _lib.check(st, "attn_fwd")
    return out, lse


_DETERMINISTIC = False


def use_deterministic_algorithms(mode: bool = True) -> None:
    """Bit-reproducible training gradients (for debugging), like torch.use_deterministic_algorithms:
    the attention backward stores each key tile's dQ into its own fp32 slice and sums the slices in order,
    and the wgrad GEMMs run without split-K (one fp32 add per gradient element).  LayerNorm's column
    reductions and the token-table gradients are fixed-order in every mode."""
    global _DETERMINISTIC
    _DETERMINISTIC = bool(mode)


def are_deterministic_algorithms_enabled() -> bool:
    return _DETERMINISTIC


def attn_bwd(q, k, v, o, dout, lse, H: int, *, scale: float | None = None, causal: bool = False,
             dq=None, dk=None, dv=None, fp32_dq: bool = False, deterministic: bool | None = None):
    """dQ, dK, dV of blockwise attention (dq/dk/dv may be slices of one packed [B,N,3*H*64] buffer).

    fp32_dq=False (default): every 128-key tile's dQ contribution is reduce-added in bf16 straight into
    dq (no fp32 accumulator, no convert pass); True: fp32 accumulation + one convert kernel.
    deterministic=True: every key tile stores its dQ contribution into its own fp32 slice and one pass
    sums them in key-tile order (bit-reproducible; ceil(N/128) x the fp32 dQ size of workspace)."""
    B, N, ld, sb = _bnhd(q, "q", H)
    for t, nm in ((k, "k"), (v, "v")):
        if _bnhd(t, nm, H) != (B, N, ld, sb):
            raise InputError("q, k, v must share shape and strides (the kernel reads k and v with q's strides)")
    Bo, No, ld_o, sb_o = _bnhd(o, "o", H)
    if (Bo, No) != (B, N) or _bnhd(dout, "dout", H) != (B, N, ld_o, sb_o):
        raise InputError("o and dout must be [B, N, H*64] views sharing strides")
    if (lse.dtype != torch.float32 or tuple(lse.shape) != (B * H, npad(N)) or not lse.is_contiguous()
            or not lse.is_cuda):
        raise InputError(f"lse must be the forward's contiguous fp32 [{B * H}, {npad(N)}] tensor")
    given = [t is not None for t in (dq, dk, dv)]
    if any(given) and not all(given):
        raise InputError("dq, dk, dv must be given together (or all omitted)")
    if dq is None:
        g = torch.empty((B, N, 3, H * 64), dtype=torch.bfloat16, device=q.device)
        dq, dk, dv = g[:, :, 0], g[:, :, 1], g[:, :, 2]
    gq = _bnhd(dq, "dq", H)
    for t, nm in ((dk, "dk"), (dv, "dv")):
        if _bnhd(t, nm, H) != gq:
            raise InputError("dq, dk, dv must share shape and strides (the kernel writes dk and dv with dq's strides)")
    if gq[:2] != (B, N):
        raise InputError("dq/dk/dv must match q's [B, N]")
    _, _, ld_g, sb_g = gq
    delta = torch.empty((B * H * npad(N), 8), dtype=torch.float32, device=q.device)   # 32 B per query row
    if deterministic is None:
        deterministic = _DETERMINISTIC
    if deterministic:
        dq_acc = torch.empty((npad(N) // 128, B, N, H, 64), dtype=torch.float32, device=q.device)
    else:
        dq_acc = torch.empty((B, N, H, 64), dtype=torch.float32, device=q.device) if fp32_dq else None
    scale = 64 ** -0.5 if scale is None else float(scale)
    fn = _lib.load().avb_attn_bwd_deterministic if deterministic else _lib.load().avb_attn_bwd
    st = fn(q.data_ptr(), k.data_ptr(), v.data_ptr(), ld, sb, o.data_ptr(), dout.data_ptr(), ld_o, sb_o,
            lse.data_ptr(), delta.data_ptr(), _ptr(dq_acc), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ld_g, sb_g,
            B, H, N, 64, scale, int(causal), _lib.stream_ptr())
    _lib.check(st, "attn_bwd")
    return dq, dk, dv


# ----------------------------------------------------------------------------- LayerNorm / misc
def layernorm_fwd(x, gamma, beta, eps=1e-5, out=None, mean=None, rstd=None):
    M, D = x.shape
    out = torch.empty_like(x) if out is None else out
    mean = torch.empty(M, dtype=torch.float32, device=x.device) if mean is None else mean
    rstd = torch.empty(M, dtype=torch.float32, device=x.device) if rstd is None else rstd
    st = _lib.load().avb_layernorm_fwd(x.data_ptr(), _rowmajor(x, "x"), gamma.data_ptr(), beta.data_ptr(),
                                       out.data_ptr(), _rowmajor(out, "out"), mean.data_ptr(), rstd.data_ptr(), M, D,
                                       float(eps), _lib.stream_ptr())
    _lib.check(st, "layernorm_fwd")
    return out, mean, rstd


def layernorm_bwd(dy, x, gamma, mean, rstd, dx, dgamma=None, dbeta=None, accumulate=False, dx_colsum=None):
    """dx (=|+=) LN'(dy); dgamma/dbeta/dx_colsum += fixed-order column reductions (bit-reproducible)."""
    M, D = x.shape
    lib = _lib.load()
    work = torch.empty(lib.avb_layernorm_bwd_workspace(D), dtype=torch.float32, device=x.device)
    st = lib.avb_layernorm_bwd(dy.data_ptr(), _rowmajor(dy, "dy"), x.data_ptr(), _rowmajor(x, "x"),
                               gamma.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dx.data_ptr(),
                               _rowmajor(dx, "dx"), _ptr(dgamma), _ptr(dbeta), _ptr(dx_colsum), work.data_ptr(), M, D,
                               int(accumulate), _lib.stream_ptr())
    _lib.check(st, "layernorm_bwd")
    return dx


def colsum_accum(x, out):
    M, N = x.shape
    _lib.check(_lib.load().avb_colsum_accum(x.data_ptr(), _rowmajor(x, "x"), M, N, out.data_ptr(), _lib.stream_ptr()),
               "colsum_accum")
    return out


def tokens_fwd(pe, cls, pos_s, pos_t, B, Np, out):
    """x = [cls | pe] + PE (PE[t*S+s] = pos_t[t] + pos_s[1+s]; cls + pos_s[0])."""
    D = pe.shape[-1]
    S = pos_s.shape[0] - 1
    if pos_t.shape[0] * S != Np or pos_s.shape[1] != D or pos_t.shape[1] != D:
        raise InputError(f"pos_s [1+S, D] and pos_t [T', D] must tile Np={Np} patches (S={S}, T'={pos_t.shape[0]})")
    _lib.check(_lib.load().avb_tokens_fwd(pe.data_ptr(), cls.data_ptr(), pos_s.data_ptr(), pos_t.data_ptr(),
                                          out.data_ptr(), B, Np, S, D, _lib.stream_ptr()), "tokens_fwd")
    return out


def tokens_bwd(dx, dpe, dcls, dpos_s, dpos_t, B, Np, S):
    """Token-embedding backward; fixed-order sums (bit-reproducible), fp32 [Np+1, D] scratch."""
    D = dx.shape[-1]
    work = torch.empty((Np + 1, D), dtype=torch.float32, device=dx.device)
    _lib.check(_lib.load().avb_tokens_bwd(dx.data_ptr(), _ptr(dpe), _ptr(dcls), _ptr(dpos_s), _ptr(dpos_t),
                                          work.data_ptr(), B, Np, S, D, _lib.stream_ptr()), "tokens_bwd")


def patchify(x, tubelet, out=None):
    """bf16 [B,3,T,H,W] clips -> tubelet patch rows [B*Np, 3*t*h*w] (Conv3d feature order)."""
    if x.dtype != torch.bfloat16 or not x.is_cuda or x.dim() != 5 or x.shape[1] != 3 or not x.is_contiguous():
        raise InputError("patchify input must be a contiguous bf16 CUDA tensor [B,3,T,H,W]")
    B, _, T, H, W = x.shape
    tt, th, tw = tubelet
    rows = B * (T // tt) * (H // th) * (W // tw)
    if out is None:
        out = torch.empty((rows, 3 * tt * th * tw), dtype=torch.bfloat16, device=x.device)
    _lib.check(_lib.load().avb_patchify(x.data_ptr(), B, T, H, W, tt, th, tw, out.data_ptr(), _lib.stream_ptr()),
               "patchify")
    return out


def xent(logits, labels, scale, loss, dlogits=None):
    """Softmax CE; labels int32 [B] (a label outside [0, C) ignores its row, see avion_b200.h)."""
    B, C = logits.shape
    _index(labels, "labels", B)
    ldd = dlogits.stride(0) if dlogits is not None else 0
    _lib.check(_lib.load().avb_xent(logits.data_ptr(), logits.stride(0), labels.data_ptr(), B, C, float(scale),
                                    loss.data_ptr(), _ptr(dlogits), ldd, _lib.stream_ptr()), "xent")


def adamw(p, g, m, v, p_bf16, lr, beta1, beta2, eps, wd, step, grad_scale=1.0, decay_mask=None):
    _lib.check(_lib.load().avb_adamw(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), _ptr(p_bf16),
                                     _ptr(decay_mask), p.numel(),
                                     float(lr), float(beta1), float(beta2), float(eps), float(wd), int(step),
                                     float(grad_scale), _lib.stream_ptr()), "adamw")


def adamw_dev(p, g, m, v, p_bf16, lr, beta1, beta2, eps, wd, step_dev, grad_scale=1.0, decay_mask=None):
    """AdamW with the step counter in device memory (int32 [1], incremented by the call): graph-capturable."""
    if step_dev.dtype != torch.int32 or step_dev.numel() != 1 or not step_dev.is_cuda:
        raise InputError("step_dev must be a 1-element int32 CUDA tensor")
    _lib.check(_lib.load().avb_adamw_dev(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), _ptr(p_bf16),
                                         _ptr(decay_mask), p.numel(), float(lr), float(beta1), float(beta2),
                                         float(eps), float(wd), step_dev.data_ptr(), float(grad_scale),
                                         _lib.stream_ptr()), "adamw_dev")


def cast_bf16(src, dst):
    _lib.check(_lib.load().avb_cast_bf16(src.data_ptr(), dst.data_ptr(), src.numel(), _lib.stream_ptr()), "cast_bf16")


# ----------------------------------------------------------------------------- InfoNCE / embeddings
def infonce_fwd(v, t, log_scale, loss, dlog_scale=None):
    """Global-batch CLIP loss: loss += L, dlog_scale += dL/dlog_scale; returns the stats for bwd."""
    if v.dtype != torch.float32 or t.dtype != torch.float32 or v.shape != t.shape or not v.is_contiguous() \
            or not t.is_contiguous():
        raise InputError("v, t must be contiguous fp32 [Bg, E] of equal shape")
    Bg, E = v.shape
    dev = v.device
    st = {"nv": torch.empty(Bg, device=dev), "nt": torch.empty(Bg, device=dev),
          "lr": torch.empty(Bg, device=dev), "lc": torch.empty(Bg, device=dev)}
    _lib.check(_lib.load().avb_infonce_fwd(v.data_ptr(), t.data_ptr(), Bg, E, log_scale.data_ptr(),
                                           st["nv"].data_ptr(), st["nt"].data_ptr(), st["lr"].data_ptr(),
                                           st["lc"].data_ptr(), loss.data_ptr(), _ptr(dlog_scale), _lib.stream_ptr()),
               "infonce_fwd")
    return st


def infonce_bwd(v, t, log_scale, stats, r0, n, grad_scale=1.0, dv=None, dt=None):
    Bg, E = v.shape
    dv = torch.empty(n, E, device=v.device) if dv is None else dv
    dt = torch.empty(n, E, device=v.device) if dt is None else dt
    _lib.check(_lib.load().avb_infonce_bwd(v.data_ptr(), t.data_ptr(), Bg, E, log_scale.data_ptr(),
                                           stats["nv"].data_ptr(), stats["nt"].data_ptr(), stats["lr"].data_ptr(),
                                           stats["lc"].data_ptr(), int(r0), int(n), float(grad_scale), dv.data_ptr(),
                                           dt.data_ptr(), _lib.stream_ptr()), "infonce_bwd")
    return dv, dt


def infonce(v: torch.Tensor, t: torch.Tensor, log_scale: torch.Tensor, r0: int = 0, n: int | None = None,
            grad_scale: float = 1.0):
    """(loss [1], dlog_scale [1], dv [n,E], dt [n,E]) for the CLIP loss over the global batch v, t."""
    Bg = v.shape[0]
    n = Bg - r0 if n is None else n
    loss = torch.zeros(1, device=v.device)
    dls = torch.zeros(1, device=v.device)
    st = infonce_fwd(v, t, log_scale, loss, dls)
    dv, dt = infonce_bwd(v, t, log_scale, st, r0, n, grad_scale)
    return loss, dls, dv, dt


def embed_fwd(tokens, table, pos, out):
    B, L = tokens.shape
    V, D = table.shape
    _index(tokens, "tokens")
    if L > pos.shape[0]:
        raise InputError(f"{L} tokens per caption exceed the position table ({pos.shape[0]})")
    _lib.check(_lib.load().avb_embed_fwd(tokens.data_ptr(), table.data_ptr(), pos.data_ptr(), out.data_ptr(), B, L, D,
                                         V, _lib.stream_ptr()), "embed_fwd")
    return out


def embed_bwd(tokens, dx, dtable, dpos):
    B, L = tokens.shape
    V, D = dtable.shape
    _index(tokens, "tokens")
    _lib.check(_lib.load().avb_embed_bwd(tokens.data_ptr(), dx.data_ptr(), dtable.data_ptr(), _ptr(dpos), B, L, D, V,
                                         _lib.stream_ptr()), "embed_bwd")


def rows_copy(src, dst, src_idx=None, dst_idx=None, n=None):
    n = (src_idx.numel() if src_idx is not None else src.shape[0]) if n is None else n
    for t, nm in ((src_idx, "src_idx"), (dst_idx, "dst_idx")):
        if t is not None:
            _index(t, nm)
            if t.numel() < n:
                raise InputError(f"{nm} has {t.numel()} entries for {n} rows")
    D = src.shape[-1]
    _lib.check(_lib.load().avb_rows_copy(src.data_ptr(), _rowmajor(src, "src"), _ptr(src_idx), dst.data_ptr(),
                                         _rowmajor(dst, "dst"), _ptr(dst_idx), int(n), D, _lib.stream_ptr()),
               "rows_copy")
    return dst
