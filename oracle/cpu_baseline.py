"""CPU baseline timings for bench.py (TEST/BASELINE INFRASTRUCTURE ONLY).

The reference has no GPU path: its CPU implementation of K1's step is
libswscale inside `convert_to_rgb` (codec.cpp:226-246).  Its own extension
needs FFmpeg headers to build (absent here); the scaler itself
is timed through ctypes in `oracle/swscale_ref.py`.  This module times the
torch fp32 restatement of the same algorithm (crop -> hflip -> antialiased
bilinear -> normalize -> bf16), using every host thread -- the `port` baseline
carried beside every augment line.
"""

from __future__ import annotations

import time

import numpy as np

CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)
CLIP_STD = (0.26862954, 0.26130258, 0.27577711)


def transform_clip_torch(frames_thwc, box, flip: bool, target=(224, 224)):
    """frames uint8 torch [T,H,W,3] -> bf16 [3,T,Ht,Wt] on CPU (fp32 math)."""
    import torch
    import torch.nn.functional as F

    x, y, w, h = (int(v) for v in box)
    t = frames_thwc[:, y:y + h, x:x + w, :].permute(0, 3, 1, 2).float()
    if flip:
        t = t.flip(-1)
    r = F.interpolate(t, size=target, mode="bilinear", align_corners=False, antialias=True)
    m = torch.tensor(CLIP_MEAN).view(1, 3, 1, 1)
    s = torch.tensor(CLIP_STD).view(1, 3, 1, 1)
    r = (r / 255.0 - m) / s
    return r.permute(1, 0, 2, 3).to(torch.bfloat16)


def time_augment(boxes, flips, T: int, hw, budget_s: float, threads: int) -> tuple[float, int]:
    """clips/s of the CPU restatement over as many golden-box clips as fit in ~budget_s."""
    import torch

    torch.set_num_threads(threads)
    H, W = hw
    g = torch.Generator().manual_seed(0)
    frames = torch.randint(0, 256, (2, T, H, W, 3), generator=g, dtype=torch.uint8)
    transform_clip_torch(frames[0], boxes[0], bool(flips[0]))  # warm
    n = 0
    t0 = time.perf_counter()
    while True:
        i = n % len(boxes)
        transform_clip_torch(frames[n % 2], boxes[i], bool(flips[i]))
        n += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return n / (time.perf_counter() - t0), n
