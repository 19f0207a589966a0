"""libswscale -- the reference's own scaler -- via ctypes (TEST / BASELINE INFRASTRUCTURE ONLY).

The reference's CPU implementation of K1's step is `convert_to_rgb` (`pkg/src/vidpipe/_codec/
codec.cpp:226-246`): crop by pointer arithmetic on the decoded planes (`codec.cpp:452-467`),
`hflip_planes` (`:201-224`), then `sws_getCachedContext` + `sws_scale` with the pinned flags
`SWS_BILINEAR | SWS_ACCURATE_RND` (`:28-30`, `:233-241`).  The reference's own extension cannot be
built here (no FFmpeg headers), but the image ships a loadable libswscale
(OpenCV's bundled 9.1.100; the reference leaves the version unpinned, `pkg/setup.py:12-26`).  This
module calls it exactly as `convert_to_rgb` does, on RGB24 input (the reference converts from YUV420P
in the same call; RGB24 -> RGB24 isolates the scaler the GPU kernel replaces), for
  * the secondary parity cross-check (tests/test_transform_oracle.py: <= 1 LSB in the interior), and
  * `bench.py --impl reference --workload augment` (the reference's CPU path timed on the host cores).
"""

from __future__ import annotations

import ctypes
import glob
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SWS_BILINEAR, SWS_ACCURATE_RND = 2, 0x40000        # codec.cpp:28-30
AV_PIX_FMT_RGB24 = 2
_LIBDIR_GLOB = "/opt/prime-rl/.venv/lib/python3.12/site-packages/opencv_python_headless.libs"


def load():
    """The swscale CDLL with typed entry points, or None when no copy is loadable."""
    libs = glob.glob(os.path.join(_LIBDIR_GLOB, "libswscale*.so*"))
    if not libs:
        return None
    d = os.path.dirname(libs[0])
    try:
        for p in ("libdrm", "libcrypto", "libavutil"):
            ctypes.CDLL(glob.glob(os.path.join(d, p + "*.so*"))[0], mode=ctypes.RTLD_GLOBAL)
        sws = ctypes.CDLL(libs[0])
    except (OSError, IndexError):
        return None
    sws.sws_getContext.restype = ctypes.c_void_p
    sws.sws_getContext.argtypes = [ctypes.c_int] * 6 + [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                                        ctypes.c_void_p]
    sws.sws_scale.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p, ctypes.c_void_p]
    sws.sws_freeContext.argtypes = [ctypes.c_void_p]
    return sws


def version_tag() -> str:
    libs = glob.glob(os.path.join(_LIBDIR_GLOB, "libswscale*.so*"))
    return os.path.basename(libs[0]) if libs else "absent"


def scale_clip(sws, frames_thwc: np.ndarray, box, flip: bool, target=(224, 224)) -> np.ndarray:
    """One clip: crop -> hflip -> sws_scale per frame, uint8 [T, Ht, Wt, 3] (codec.cpp:226-246 order)."""
    x, y, w, h = (int(v) for v in box)
    T = frames_thwc.shape[0]
    th, tw = target
    ctx = sws.sws_getContext(w, h, AV_PIX_FMT_RGB24, tw, th, AV_PIX_FMT_RGB24, SWS_BILINEAR | SWS_ACCURATE_RND,
                             None, None, None)
    if not ctx:
        raise RuntimeError("sws_getContext failed")
    # FFmpeg's SIMD scalers may read / write up to AV_INPUT_BUFFER_PADDING_SIZE (64) bytes past a plane:
    # both planes live in padded buffers (an unpadded crop copy ending at a page boundary segfaults)
    pad = 64
    src_buf = np.empty(h * w * 3 + pad, dtype=np.uint8)
    dst_buf = np.empty(th * tw * 3 + pad, dtype=np.uint8)
    src = src_buf[:h * w * 3].reshape(h, w, 3)
    dst = dst_buf[:th * tw * 3].reshape(th, tw, 3)
    out = np.empty((T, th, tw, 3), dtype=np.uint8)
    sp = (ctypes.c_void_p * 4)(src_buf.ctypes.data, None, None, None)
    ss = (ctypes.c_int * 4)(w * 3, 0, 0, 0)
    dp = (ctypes.c_void_p * 4)(dst_buf.ctypes.data, None, None, None)
    ds = (ctypes.c_int * 4)(tw * 3, 0, 0, 0)
    try:
        for t in range(T):
            crop = frames_thwc[t, y:y + h, x:x + w]
            # hflip_planes is a reversed copy (codec.cpp:201-224); the crop itself is pointer arithmetic
            np.copyto(src, crop[:, ::-1] if flip else crop)
            sws.sws_scale(ctx, sp, ss, 0, h, dp, ds)   # ctypes releases the GIL around the call
            out[t] = dst
    finally:
        sws.sws_freeContext(ctx)
    return out


def time_augment(boxes, flips, T: int, hw, budget_s: float, threads: int) -> tuple[float, int]:
    """clips/s of crop -> hflip -> sws_scale over golden-box clips, `threads` clips in flight."""
    sws = load()
    if sws is None:
        raise RuntimeError("no loadable libswscale")
    H, W = hw
    rng = np.random.default_rng(0)
    frames = [rng.integers(0, 256, (T, H, W, 3), dtype=np.uint8) for _ in range(2)]
    scale_clip(sws, frames[0], boxes[0], bool(flips[0]))       # warm
    n = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        while time.perf_counter() - t0 < budget_s:
            idx = [(n + k) % len(boxes) for k in range(threads)]
            list(ex.map(lambda i: scale_clip(sws, frames[i % 2], boxes[i], bool(flips[i])), idx))
            n += threads
    return n / (time.perf_counter() - t0), n
