"""GPU clip transform: the drop-in for the reference's crop -> flip -> scale step.

Reference contract being mirrored (`pkg/src/vidpipe/decoder.py`):
  * `ClipRequest(crop: CropRect, hflip, target_h, target_w)` (:43-56) -- here one
    box + flip per clip, applied to every frame (`loader.py:161-162`);
  * output written into a caller-provided `out` buffer whose shape/dtype is
    validated, else `InputError` (`_new_output`, :127-134);
  * a crop outside the frame raises `InputError` before any work (:116-119).
The pixel arithmetic (`codec.cpp:187-246`) runs in the sm_100a kernel K1
(`csrc/k1_rrc_normalize.cu`) through `avb_rrc_normalize`; normalize + cast,
which the reference defers to the GPU, are fused into it.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import InputError

CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)
CLIP_STD = (0.26862954, 0.26130258, 0.27577711)

_DT = {torch.bfloat16: _lib.AVB_DTYPE_BF16, torch.float32: _lib.AVB_DTYPE_F32}
_LAYOUT = {"cthw": _lib.AVB_LAYOUT_CTHW, "tchw": _lib.AVB_LAYOUT_TCHW, "tubelet": _lib.AVB_LAYOUT_TUBELET}


def _boxes_to_host(crops) -> np.ndarray:
    if isinstance(crops, torch.Tensor):
        return crops.detach().to("cpu", torch.int32).numpy().reshape(-1, 4)
    if len(crops) and all(hasattr(crops[0], f) for f in ("x", "y", "crop_w", "crop_h")):   # CropRect
        return np.asarray([(c.x, c.y, c.crop_w, c.crop_h) for c in crops], dtype=np.int32)
    return np.asarray(crops, dtype=np.int32).reshape(-1, 4)


def output_shape(B: int, T: int, target: tuple[int, int], layout: str, tubelet=(2, 16, 16)) -> tuple[int, ...]:
    Ht, Wt = target
    if layout == "tubelet":
        tt, ph, pw = tubelet
        return (B * (T // tt) * (Ht // ph) * (Wt // pw), 3 * tt * ph * pw)
    return (B, 3, T, Ht, Wt) if layout == "cthw" else (B, T, 3, Ht, Wt)


def transform(frames: torch.Tensor, crops, hflip=None, target: tuple[int, int] = (224, 224),
              mean: Sequence[float] = CLIP_MEAN, std: Sequence[float] = CLIP_STD, *,
              out: torch.Tensor | None = None, out_dtype: torch.dtype = torch.bfloat16,
              layout: str = "cthw", channels_last: bool = True, validate: bool = True,
              tubelet: tuple[int, int, int] = (2, 16, 16), crops_host=None) -> torch.Tensor:
    """Crop -> hflip -> antialiased bilinear -> normalize -> cast, on the GPU.

    frames:  uint8 CUDA tensor, [B,T,H,W,3] (channels_last, decoded RGB24) or
             [B,T,3,H,W] (`channels_last=False`, the reference `Batch.frames`
             layout, loader.py:99-116).  Any strides are accepted.
    crops:   [B,4] (x, y, crop_w, crop_h) as a CUDA/CPU int tensor, numpy array or
             list of `CropRect`.  One crop per clip.
    hflip:   [B] bools (tensor/array/list) or None.
    out:     optional preallocated CUDA tensor of `output_shape(...)` and `out_dtype`.
    validate: check every box on the host first (needs a host copy of the boxes;
             pass False inside CUDA-graph capture with device boxes -- the kernel
             still skips out-of-frame boxes).
    crops_host: optional host copy of CUDA `crops` (the sampler's own boxes): used for
             validation and for the kernel's exact tap envelope without a device->host
             read.  Without any host copy the kernel assumes the worst-case envelope.
    Returns `out` (layout "cthw" = [B,3,T,Ht,Wt]; "tchw" = [B,T,3,Ht,Wt]; "tubelet" = the
    patch-embed GEMM operand [B*Np, 3*tt*ph*pw] for `tubelet=(tt, ph, pw)`).
    """
    if not isinstance(frames, torch.Tensor) or frames.dtype != torch.uint8:
        raise InputError("frames must be a uint8 torch tensor")
    if not frames.is_cuda:
        raise InputError("frames must be on a CUDA device (the transform has no CPU path)")
    if frames.dim() != 5:
        raise InputError(f"frames must be 5-D, got {tuple(frames.shape)}")
    if layout not in _LAYOUT:
        raise InputError(f"layout must be one of {sorted(_LAYOUT)}")
    if out_dtype not in _DT:
        raise InputError("out_dtype must be torch.bfloat16 or torch.float32")
    if channels_last:
        B, T, H, W, Cn = frames.shape
        s_clip, s_t, s_h, s_w, s_c = frames.stride()
    else:
        B, T, Cn, H, W = frames.shape
        s_clip, s_t, s_c, s_h, s_w = frames.stride()
    if Cn != 3:
        raise InputError(f"expected 3 channels, got {Cn}")
    Ht, Wt = int(target[0]), int(target[1])
    if Ht < 1 or Wt < 1:
        raise InputError("target size must be >= 1 pixel")
    dev = frames.device

    boxes_host = None
    if isinstance(crops, torch.Tensor) and crops.is_cuda:
        boxes_dev = crops.to(torch.int32).contiguous().view(-1, 4)
        if crops_host is not None:
            boxes_host = _boxes_to_host(crops_host)
            if boxes_host.shape != tuple(boxes_dev.shape):
                raise InputError(f"crops_host shape {boxes_host.shape} != crops {tuple(boxes_dev.shape)}")
        elif validate:
            boxes_host = _boxes_to_host(crops)
    else:
        boxes_host = _boxes_to_host(crops)
        boxes_dev = torch.from_numpy(boxes_host).to(dev, non_blocking=False)
    if boxes_dev.shape[0] != B:
        raise InputError(f"need one crop per clip: {boxes_dev.shape[0]} crops for {B} clips")
    if boxes_dev.data_ptr() % 16:
        boxes_dev = boxes_dev.clone()
    if hflip is None:
        flips_dev = None
    elif isinstance(hflip, torch.Tensor) and hflip.is_cuda:
        flips_dev = hflip.to(torch.uint8).contiguous()
    else:
        flips_dev = torch.as_tensor(np.asarray(hflip, dtype=np.uint8).reshape(-1)).to(dev)
    if flips_dev is not None and flips_dev.numel() != B:
        raise InputError(f"need one flip per clip: {flips_dev.numel()} for {B} clips")

    shape = output_shape(B, T, (Ht, Wt), layout, tubelet)
    if out is None:
        out = torch.empty(shape, dtype=out_dtype, device=dev)
    elif tuple(out.shape) != shape or out.dtype != out_dtype or not out.is_contiguous() or out.device != dev:
        raise InputError(f"output buffer must be contiguous {out_dtype} {shape} on {dev}, "
                         f"got {out.dtype} {tuple(out.shape)}")

    bh = np.ascontiguousarray(boxes_host, dtype=np.int32) if boxes_host is not None else None
    inv_std = [1.0 / float(s) for s in std]
    lib = _lib.load()
    fl = flips_dev.data_ptr() if flips_dev is not None else None
    bhp = bh.ctypes.data if bh is not None else None
    with torch.cuda.device(dev):
        if layout == "tubelet":
            st = lib.avb_rrc_normalize_tubelet(
                frames.data_ptr(), B, T, H, W, s_clip, s_t, s_h, s_w, s_c, boxes_dev.data_ptr(), fl, bhp, Ht, Wt,
                _lib.f32x3(mean), _lib.f32x3(inv_std), _DT[out_dtype], int(tubelet[0]), int(tubelet[1]),
                int(tubelet[2]), out.data_ptr(), _lib.stream_ptr())
        else:
            st = lib.avb_rrc_normalize(
                frames.data_ptr(), B, T, H, W, s_clip, s_t, s_h, s_w, s_c, boxes_dev.data_ptr(), fl, bhp, Ht, Wt,
                _lib.f32x3(mean), _lib.f32x3(inv_std), _DT[out_dtype], _LAYOUT[layout], out.data_ptr(),
                _lib.stream_ptr())
    _lib.check(st, "transform")
    return out


def device_taps(crop: int, tgt: int, max_taps: int = 24, device="cuda"):
    """Tap table computed by the kernel's own device function (test hook)."""
    lo = torch.empty(tgt, dtype=torch.int32, device=device)
    hi = torch.empty(tgt, dtype=torch.int32, device=device)
    w = torch.empty(tgt, max_taps, dtype=torch.float32, device=device)
    lib = _lib.load()
    _lib.check(lib.avb_rrc_taps(crop, tgt, lo.data_ptr(), hi.data_ptr(), w.data_ptr(), max_taps,
                                _lib.stream_ptr()), "rrc_taps")
    return lo, hi, w


def algorithmic_bytes(boxes: np.ndarray, T: int, target: tuple[int, int] = (224, 224),
                      out_itemsize: int = 2) -> int:
    """Bytes K1 must move: crop region read once + output written once."""
    Ht, Wt = target
    b = np.asarray(boxes, dtype=np.int64).reshape(-1, 4)
    return int(T * (b[:, 2] * b[:, 3]).sum() * 3 + b.shape[0] * T * 3 * Ht * Wt * out_itemsize)
