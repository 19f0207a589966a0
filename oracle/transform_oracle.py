"""K1 oracle: crop -> hflip -> antialiased bilinear scale -> normalize, float64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it restates
----------------
The reference's only pixel arithmetic on this path is `convert_to_rgb`
(`pkg/src/vidpipe/_codec/codec.cpp:226-246`): the crop is taken by pointer
arithmetic on the decoded planes (`codec.cpp:452-467`, `decoder.py:264,
282-292`), the cropped view is column-reversed when `hflip`
(`hflip_planes`, `codec.cpp:201-224`), then libswscale scales it with
`SWS_BILINEAR|SWS_ACCURATE_RND` (`codec.cpp:28-30`) -- i.e. a tent filter
widened by the downscale factor (antialiased bilinear).  Order is
crop -> hflip -> scale (`codec.cpp:188-191`, `SPEC.md:231`), and
normalization is deferred to the GPU (`SPEC.md:232`, `PAPER.md:666-668`).

libswscale is an un-vendored dependency (version unpinned, `pkg/setup.py:12-26`)
whose 14-bit fixed-point arithmetic is not reproducible bit-for-bit, so this
oracle restates the published separable antialiased-bilinear algorithm
(PIL / torch `antialias=True` semantics) in float64, with the tap ranges in
exact integers:

  s = crop/target, centre c_i = s*(i+1/2)
  downscale (s >= 1):  x_min = max(0, floor((crop(2i-1)+tgt) / 2tgt))
                       x_max = min(crop, floor((crop(2i+3)+tgt) / 2tgt))
                       w_j  ~ max(0, 1 - |j + 1/2 - c_i| / s)
  upscale   (s <  1):  x_min = max(0, floor((crop(2i+1)-tgt) / 2tgt))
                       x_max = min(crop, floor((crop(2i+1)+3tgt) / 2tgt))
                       w_j  ~ max(0, 1 - |j + 1/2 - c_i|)
  weights renormalised to sum 1 per output index.

Normalization (absent in the reference; CLIP constants, an assumption):
  y = (v/255 - mean_c) / std_c.
"""

from __future__ import annotations

import numpy as np

CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)
CLIP_STD = (0.26862954, 0.26130258, 0.27577711)


def tap_ranges(crop: int, tgt: int) -> tuple[np.ndarray, np.ndarray]:
    """Exact-integer [x_min, x_max) per output index."""
    i = np.arange(tgt, dtype=np.int64)
    if crop >= tgt:
        lo = (crop * (2 * i - 1) + tgt) // (2 * tgt)
        hi = (crop * (2 * i + 3) + tgt) // (2 * tgt)
    else:
        lo = (crop * (2 * i + 1) - tgt) // (2 * tgt)
        hi = (crop * (2 * i + 1) + 3 * tgt) // (2 * tgt)
    return np.maximum(lo, 0), np.minimum(hi, crop)


def weight_matrix(crop: int, tgt: int) -> np.ndarray:
    """Dense [tgt, crop] float64 resampling matrix, rows summing to 1."""
    s = crop / tgt
    support_scale = s if s >= 1.0 else 1.0
    lo, hi = tap_ranges(crop, tgt)
    m = np.zeros((tgt, crop), dtype=np.float64)
    for i in range(tgt):
        c = s * (i + 0.5)
        j = np.arange(lo[i], hi[i])
        w = np.maximum(0.0, 1.0 - np.abs(j + 0.5 - c) / support_scale)
        tot = w.sum()
        if tot > 0:
            m[i, lo[i]:hi[i]] = w / tot
    return m


def transform_clip(frames: np.ndarray, box, hflip: bool, target_hw=(224, 224),
                   mean=CLIP_MEAN, std=CLIP_STD, normalize: bool = True) -> np.ndarray:
    """One clip. frames uint8 [T,H,W,3] -> float64 [3,T,Ht,Wt]."""
    x, y, cw, ch = (int(v) for v in box)
    T, H, W, C = frames.shape
    assert C == 3
    if not (x >= 0 and y >= 0 and cw >= 1 and ch >= 1 and x + cw <= W and y + ch <= H):
        raise ValueError(f"crop {box} outside frame {W}x{H}")
    Ht, Wt = target_hw
    crop = frames[:, y:y + ch, x:x + cw, :].astype(np.float64)     # crop (codec.cpp:452-458)
    if hflip:
        crop = crop[:, :, ::-1, :]                                  # hflip (codec.cpp:201-224)
    wy = weight_matrix(ch, Ht)
    wx = weight_matrix(cw, Wt)
    out = np.einsum("ih,thwc,jw->ctij", wy, crop, wx, optimize=True)  # separable scale
    if normalize:
        m = np.asarray(mean, dtype=np.float64).reshape(3, 1, 1, 1)
        s = np.asarray(std, dtype=np.float64).reshape(3, 1, 1, 1)
        out = (out / 255.0 - m) / s
    return out


def transform_batch(frames: np.ndarray, boxes: np.ndarray, flips: np.ndarray,
                    target_hw=(224, 224), mean=CLIP_MEAN, std=CLIP_STD,
                    normalize: bool = True) -> np.ndarray:
    """frames uint8 [B,T,H,W,3] -> float64 [B,3,T,Ht,Wt]."""
    return np.stack([transform_clip(frames[b], boxes[b], bool(flips[b]), target_hw, mean, std,
                                    normalize) for b in range(frames.shape[0])])


def algorithmic_bytes(boxes: np.ndarray, T: int, target_hw=(224, 224), out_itemsize: int = 2) -> int:
    """K1 algorithmic bytes: crop region read once + output written once."""
    Ht, Wt = target_hw
    area = (boxes[:, 2].astype(np.int64) * boxes[:, 3].astype(np.int64)).sum()
    return int(T * area * 3 + boxes.shape[0] * T * 3 * Ht * Wt * out_itemsize)
