"""Thin torch-facing wrappers over the C ABI (pointers + sizes + current stream).

Every function here validates dtypes/shapes/devices on the host and then calls
one `avb_*` entry point; none of them computes anything in PyTorch.  Autograd
lives in `nn.py`.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import InputError

EPI_BF16, EPI_BIAS_GELU, EPI_DGELU, EPI_F32, EPI_F32_ACCUM = 0, 1, 2, 3, 4


def _ptr(t):
    return None if t is None else t.data_ptr()


def _rowmajor(t: torch.Tensor, name: str) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise InputError(f"{name} must be a 2-D row-major view, got shape {tuple(t.shape)} strides {t.stride()}")
    return t.stride(0)


def gemm(a: torch.Tensor, b: torch.Tensor, *, a_mn: bool = False, b_mn: bool = False, out: torch.Tensor | None = None,
         epilogue: int = EPI_BF16, bias: torch.Tensor | None = None, aux: torch.Tensor | None = None,
         aux_out: torch.Tensor | None = None, alpha: float = 1.0, split_k: int = 1) -> torch.Tensor:
    """C = epi(alpha * A @ B^T) on the tcgen05 GEMM.

    a: [M,K] (a_mn=False) or [K,M] (a_mn=True); b: [N,K] (b_mn=False) or [K,N] (b_mn=True).
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
    if aux is not None and aux_out is not None and aux.stride(0) != aux_out.stride(0):
        raise InputError("aux and aux_out must share a leading dimension")
    lib = _lib.load()
    st = lib.avb_gemm(a.data_ptr(), lda, int(a_mn), b.data_ptr(), ldb, int(b_mn), out.data_ptr(), ldc, M, N, K,
                      epilogue, _ptr(bias), _ptr(aux), ldaux, _ptr(aux_out), float(alpha), int(split_k),
                      _lib.stream_ptr())
    _lib.check(st, "gemm")
    return out
