"""Loader -> device hand-off: reference `Batch` objects into K1 on the GPU.

The reference loader yields `Batch.frames`, a host uint8 `[B, T, 3, H, W]` view into a reused ring
buffer that is "valid until the next batch is requested" (`pkg/src/vidpipe/loader.py:99-116`,
`pkg/README.md:159-165`).  `DeviceFeeder` is the component a training loop puts behind
`run_loader`:

  1. `submit(batch)` copies `batch.frames` into the next slot of a pinned host ring *synchronously*
     (so the loader may rewrite its ring as soon as `submit` returns -- the reference's validity
     contract) and enqueues the H2D copy on a dedicated copy stream;
  2. `next()` (or iterating `feed(loader)`) makes the compute stream wait for that copy and launches
     K1 on the device copy: the identity kernel when the frames are already at the target size and
     no crop is given (the fused-decode hand-off, `decoder.py:137-211`: flip +
     normalise + cast + re-layout only), else the crop/flip/antialiased-resize kernel with the
     supplied boxes (`[B, T, 3, H, W]` strides are read directly);
  3. the pinned slot is reused only after its H2D copy has completed (a CUDA event per slot), and a
     device slot only after the K1 launch that read it has run (an event on the compute stream).

With `depth >= 2` the copy of batch i+1 overlaps the compute of batch i.  Output: the normalised
clip tensor in the requested layout (`cthw`, `tchw` or the patch-embed `tubelet` rows).
`channels_last=True` takes decoded RGB24 frames `[B, T, H, W, 3]` instead (full frames + crops: K1's
streaming fast path); a batch that is already a pinned torch tensor is copied to the device directly
(no staging copy -- the caller keeps it unchanged until the next `submit` of that slot returns).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import InputError
from .transform import CLIP_MEAN, CLIP_STD, output_shape, transform


@dataclass
class _Slot:
    host: torch.Tensor          # pinned uint8 [Bmax, T, 3, H, W] (or [Bmax, T, H, W, 3])
    dev: torch.Tensor           # device uint8 [Bmax, T, 3, H, W]
    h2d_done: torch.cuda.Event  # the H2D copy out of `host` finished (host slot reusable)
    consumed: torch.cuda.Event  # K1 read `dev` (device slot reusable)
    boxes_h: torch.Tensor       # pinned int32 [Bmax, 4] / uint8 [Bmax] and their device copies
    flips_h: torch.Tensor
    boxes_d: torch.Tensor
    flips_d: torch.Tensor
    n: int = 0                  # clips in the batch held by this slot
    crops: np.ndarray | None = None
    src: torch.Tensor | None = None   # the pinned tensor of a zero-staging submit (kept alive until reuse)
    busy: bool = False


def _copy_parallel(dst: np.ndarray, src: np.ndarray, threads: int = 8) -> None:
    """Host ring -> pinned slot copy, split by clip over a few threads (numpy releases the GIL)."""
    n = src.shape[0]
    if n < 2 or src.nbytes < (64 << 20):
        np.copyto(dst, src)
        return
    from concurrent.futures import ThreadPoolExecutor

    parts = np.array_split(np.arange(n), min(threads, n))
    with ThreadPoolExecutor(len(parts)) as ex:
        list(ex.map(lambda p: np.copyto(dst[p[0]:p[-1] + 1], src[p[0]:p[-1] + 1]), parts))


class DeviceFeeder:
    """Pinned double-buffered H2D + K1 behind the reference loader's `Batch` stream."""

    def __init__(self, max_batch: int, frames: int, height: int, width: int, target=(224, 224), *,
                 layout: str = "cthw", out_dtype=torch.bfloat16, tubelet=(2, 16, 16), mean=CLIP_MEAN,
                 std=CLIP_STD, depth: int = 2, device=None, channels_last: bool = False):
        if depth < 1:
            raise InputError("depth must be >= 1")
        self.channels_last = bool(channels_last)
        if self.channels_last:
            self.shape = (int(max_batch), int(frames), int(height), int(width), 3)
        else:
            self.shape = (int(max_batch), int(frames), 3, int(height), int(width))
        self.hw = (int(height), int(width))
        self.target = (int(target[0]), int(target[1]))
        self.layout, self.out_dtype, self.tubelet = layout, out_dtype, tuple(tubelet)
        self.mean, self.std = mean, std
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.slots = []
        for _ in range(depth):
            host = torch.empty(self.shape, dtype=torch.uint8, pin_memory=True)
            dev = torch.empty(self.shape, dtype=torch.uint8, device=self.device)
            Bm = self.shape[0]
            s = _Slot(host, dev, torch.cuda.Event(), torch.cuda.Event(),
                      torch.empty((Bm, 4), dtype=torch.int32, pin_memory=True),
                      torch.empty((Bm,), dtype=torch.uint8, pin_memory=True),
                      torch.empty((Bm, 4), dtype=torch.int32, device=self.device),
                      torch.empty((Bm,), dtype=torch.uint8, device=self.device))
            s.h2d_done.record(self.copy_stream)
            s.consumed.record(torch.cuda.current_stream(self.device))
            self.slots.append(s)
        self._put = 0      # next slot submit() fills
        self._get = 0      # next slot next() consumes
        self.h2d_bytes = 0

    # -------------------------------------------------------------- producer side
    def submit(self, batch, crops=None, flips=None) -> None:
        """Stage one reference `Batch` (anything with `.frames`, or the uint8 array itself).

        crops: optional [B, 4] (x, y, crop_w, crop_h) per clip (`CropRect` order) for raw decoded
        frames; None means the frames are already the sampled crop at the target size.
        flips: optional [B] bools (None: no flip, the reference already flipped on the CPU).
        """
        frames = getattr(batch, "frames", batch)
        direct = isinstance(frames, torch.Tensor) and frames.is_pinned() and frames.is_contiguous()
        if isinstance(frames, torch.Tensor) and not direct:
            frames = frames.numpy()
        if frames.dtype not in (np.uint8, torch.uint8) or frames.ndim != 5:
            raise InputError("batch.frames must be a uint8 [B, T, 3, H, W] array")
        B = frames.shape[0]
        if B > self.shape[0] or tuple(frames.shape[1:]) != self.shape[1:]:
            raise InputError(f"batch of shape {frames.shape} does not fit the feeder ring {self.shape}")
        s = self.slots[self._put]
        if s.busy:
            raise InputError("feeder ring full: call next() before submitting more batches than `depth`")
        H, W = self.hw
        if crops is None:
            if (H, W) != self.target:
                raise InputError(f"frames are {H}x{W}, target {self.target}: pass crops= for raw decoded frames")
            box = np.tile(np.asarray([[0, 0, W, H]], dtype=np.int32), (B, 1))     # full frame -> identity K1
        else:
            box = np.ascontiguousarray(np.asarray(crops, dtype=np.int32).reshape(B, 4))
        fl = np.zeros(B, np.uint8) if flips is None else np.asarray(flips, dtype=np.uint8).reshape(B)
        s.h2d_done.synchronize()                          # the previous H2D out of this pinned slot is done
        if direct:
            s.src = frames                                # already pinned: H2D straight from it
        else:
            _copy_parallel(s.host[:B].numpy(), frames)    # the loader may now rewrite its ring buffer
            s.src = s.host[:B]
        np.copyto(s.boxes_h[:B].numpy(), box)
        np.copyto(s.flips_h[:B].numpy(), fl)
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(s.consumed)       # K1 of the slot's previous batch has read `dev`
            s.dev[:B].copy_(s.src, non_blocking=True)
            s.boxes_d[:B].copy_(s.boxes_h[:B], non_blocking=True)
            s.flips_d[:B].copy_(s.flips_h[:B], non_blocking=True)
            s.h2d_done.record(self.copy_stream)
        self.h2d_bytes += frames.nbytes
        s.n = B
        s.crops = box                                     # host copy: validation + K1's exact tap envelope
        s.busy = True
        self._put = (self._put + 1) % len(self.slots)

    # -------------------------------------------------------------- consumer side
    def next(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """K1 on the oldest staged batch, on the current stream; returns the normalised clips."""
        s = self.slots[self._get]
        if not s.busy:
            raise InputError("no staged batch: submit() first")
        stream = torch.cuda.current_stream(self.device)
        stream.wait_event(s.h2d_done)
        B, T = s.n, self.shape[1]
        if out is None:
            out = torch.empty(output_shape(B, T, self.target, self.layout, self.tubelet), dtype=self.out_dtype,
                              device=self.device)
        transform(s.dev[:B], s.boxes_d[:B], s.flips_d[:B], self.target, self.mean, self.std, out=out,
                  out_dtype=self.out_dtype, layout=self.layout, channels_last=self.channels_last,
                  tubelet=self.tubelet, crops_host=s.crops, validate=False)
        s.consumed.record(stream)
        s.busy = False
        self._get = (self._get + 1) % len(self.slots)
        return out

    def feed(self, batches, crops_fn=None):
        """Iterate a reference loader (`run_loader(...)`), one batch of H2D ahead of the compute.

        crops_fn(batch) -> (crops, flips) or None for batches already at the target size.
        """
        it = iter(batches)
        pending = 0
        for b in it:
            cf = crops_fn(b) if crops_fn is not None else None
            self.submit(b, *(cf or (None, None)))
            pending += 1
            if pending == len(self.slots):
                yield self.next()
                pending -= 1
        while pending:
            yield self.next()
            pending -= 1
