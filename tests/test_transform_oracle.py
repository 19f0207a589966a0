"""Pin the K1 oracle before trusting it (CPU only).

* index rule: exact-integer tap ranges == torch's float rule on many shapes;
* values: oracle == torch F.interpolate(bilinear, antialias=True) (PIL semantics)
  to 1e-9 on the golden boxes of config 2 and on edge shapes (upscale, identity,
  mixed, tiny);
* relative semantics the reference tests pin (test_decoder.py:107-150):
  full-frame identity when target == source, and hflip == exact column
  reversal of the unflipped output;
* libswscale cross-check (the reference's actual scaler) when a copy loads:
  interior within 1 LSB.
"""

import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import transform_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rrc_golden.json")))


def torch_ranges(crop, tgt):
    # torch's float computation (UpSampleKernel antialias): int64(center -+ support + 0.5)
    s = crop / tgt
    support = s if s >= 1 else 1.0
    lo, hi = [], []
    for i in range(tgt):
        c = s * (i + 0.5)
        a = max(int(c - support + 0.5), 0)
        b = min(int(c + support + 0.5), crop)
        lo.append(a)
        hi.append(b)
    return np.asarray(lo), np.asarray(hi)


@pytest.mark.parametrize("crop,tgt", [(303, 224), (392, 224), (346, 224), (427, 224), (285, 224),
                                      (448, 224), (100, 224), (224, 224), (7, 3), (5, 9), (568, 224),
                                      (1, 224), (223, 224), (225, 224)])
def test_index_rule_matches_float_rule(crop, tgt):
    lo, hi = O.tap_ranges(crop, tgt)
    tlo, thi = torch_ranges(crop, tgt)
    m = O.weight_matrix(crop, tgt)
    # any tap gained or lost vs the float rule carries exactly zero weight
    for i in range(tgt):
        a, b = set(range(lo[i], hi[i])), set(range(tlo[i], thi[i]))
        for j in a ^ b:
            s = crop / tgt
            w = max(0.0, 1 - abs(j + 0.5 - s * (i + 0.5)) / max(s, 1.0))
            assert w == 0.0
    assert np.allclose(m.sum(1), 1.0)


def _torch_ref(frames, box, flip, target):
    x, y, w, h = box
    t = torch.from_numpy(frames[:, y:y + h, x:x + w, :]).permute(0, 3, 1, 2).double()
    if flip:
        t = t.flip(-1)
    r = F.interpolate(t, size=target, mode="bilinear", align_corners=False, antialias=True)
    return r.permute(1, 0, 2, 3).numpy()


def test_oracle_vs_torch_on_golden_boxes():
    rng = np.random.default_rng(0)
    frames = rng.integers(0, 256, (2, 320, 568, 3), dtype=np.uint8)
    for x, y, w, h, f in GOLD["config2_568x320"][:12]:
        o = O.transform_clip(frames, (x, y, w, h), bool(f), (224, 224), normalize=False)
        r = _torch_ref(frames, (x, y, w, h), bool(f), (224, 224))
        assert np.abs(o - r).max() < 1e-9


@pytest.mark.parametrize("shape", [(100, 150, 224, 224), (224, 224, 224, 224), (336, 224, 224, 224),
                                   (5, 7, 9, 3), (1, 1, 4, 4), (320, 568, 224, 224)])
def test_oracle_vs_torch_edge_shapes(shape):
    h, w, th, tw = shape
    rng = np.random.default_rng(1)
    frames = rng.integers(0, 256, (1, h, w, 3), dtype=np.uint8)
    o = O.transform_clip(frames, (0, 0, w, h), False, (th, tw), normalize=False)
    r = _torch_ref(frames, (0, 0, w, h), False, (th, tw))
    assert np.abs(o - r).max() < 1e-9


def test_identity_and_flip_semantics():
    rng = np.random.default_rng(2)
    frames = rng.integers(0, 256, (3, 256, 320, 3), dtype=np.uint8)
    o = O.transform_clip(frames, (0, 0, 320, 256), False, (256, 320), normalize=False)
    assert np.array_equal(o, frames.transpose(3, 0, 1, 2).astype(np.float64))
    a = O.transform_clip(frames, (40, 32, 128, 16), False, (16, 128), normalize=False)
    b = O.transform_clip(frames, (40, 32, 128, 16), True, (16, 128), normalize=False)
    assert np.array_equal(b, a[..., ::-1])
    # flip commutes with a downscale up to float rounding (symmetric tent)
    a = O.transform_clip(frames, (3, 5, 301, 233), False, (224, 224), normalize=False)
    b = O.transform_clip(frames, (3, 5, 301, 233), True, (224, 224), normalize=False)
    assert np.abs(b - a[..., ::-1]).max() < 1e-9


def test_normalize_constants():
    frames = np.full((1, 4, 4, 3), 255, dtype=np.uint8)
    o = O.transform_clip(frames, (0, 0, 4, 4), False, (2, 2))
    for c in range(3):
        assert np.allclose(o[c], (1.0 - O.CLIP_MEAN[c]) / O.CLIP_STD[c])


def test_bad_box_rejected():
    frames = np.zeros((1, 10, 10, 3), dtype=np.uint8)
    with pytest.raises(ValueError):
        O.transform_clip(frames, (5, 0, 6, 10), False, (4, 4))


def test_swscale_cross_check_interior():
    """Secondary cross-check against libswscale (the reference's scaler, codec.cpp:28-30,233-241), called
    through oracle/swscale_ref.py exactly as convert_to_rgb does (padded planes)."""
    from oracle import swscale_ref as SW
    sws = SW.load()
    if sws is None:
        pytest.skip("no loadable libswscale copy")
    # smooth image: per-pixel differences stay within the fixed-point rounding
    yy, xx = np.mgrid[0:303, 0:392]
    img = np.stack([(127 + 100 * np.sin(xx / 17.0 + c) * np.cos(yy / 13.0)) for c in range(3)], -1)
    img = np.ascontiguousarray(img.astype(np.uint8))
    w, h, tw, th = 392, 303, 224, 224
    out = SW.scale_clip(sws, img[None], (0, 0, w, h), False, (th, tw))[0]
    o = O.transform_clip(img[None], (0, 0, w, h), False, (th, tw), normalize=False)[:, 0].transpose(1, 2, 0)
    d = np.abs(o - out.astype(np.float64))[2:-2, 2:-2]
    assert d.max() <= 1.0 + 1e-9, d.max()
