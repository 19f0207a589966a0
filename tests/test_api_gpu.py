"""The PyTorch-facing boundary on the GPU.

* `nn.VideoEncoder(cfg)` (nn.Module + autograd) == the explicit forward/backward engine it wraps,
  and both == the fp32 oracle (2e-2); a torch optimizer step refreshes the bf16 weight shadow.
* `nn.attention` (K4/K5 autograd) vs a plain fp32 softmax(QK^T)V reference.
* `nn.clip_loss` (K7 autograd) vs the oracle's CLIP InfoNCE, gradients of v, t and the logit scale.
* `ops.patchify` == the oracle's tubelet patchify (byte-exact permutation).
* `feeder.DeviceFeeder`: reference-style `Batch` objects -> pinned ring -> H2D -> K1, equal to the
  oracle, and the loader's "valid until next iter" contract (the ring may be rewritten after submit).
"""

from dataclasses import dataclass

import numpy as np
import pytest
import torch

from oracle import transform_oracle as TO
from oracle import vit_oracle as VO
from paper_2309_16669_b200 import nn as avnn
from paper_2309_16669_b200 import ops
from paper_2309_16669_b200.feeder import DeviceFeeder
from paper_2309_16669_b200.vit import VitConfig

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


@pytest.fixture(autouse=True)
def _fp32_reference():
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32 = old


CFG = VitConfig(frames=4, height=64, width=96, cube_t=2, cube_h=16, cube_w=16, depth=2, dim=128, heads=2)


def test_patchify_matches_oracle():
    for cfg in (CFG, VitConfig(frames=4, height=56, width=84, cube_t=1, cube_h=14, cube_w=14, depth=1, dim=64,
                               heads=1)):
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.randn(3, 3, cfg.frames, cfg.height, cfg.width, generator=g, device="cuda").to(torch.bfloat16)
        rows = ops.patchify(x, (cfg.cube_t, cfg.cube_h, cfg.cube_w))
        assert torch.equal(rows, VO.patchify(x, cfg))


def test_video_encoder_module_equals_engine_and_oracle():
    torch.manual_seed(0)
    mod = avnn.VideoEncoder(CFG, seed=1)
    with torch.no_grad():
        g = torch.Generator(device="cuda").manual_seed(2)
        mod.flat.add_(torch.randn(mod.flat.numel(), generator=g, device="cuda") * 0.02)   # bumps the version
    B = 3
    clips = torch.randn(B, 3, CFG.frames, CFG.height, CFG.width, generator=g, device="cuda").to(torch.bfloat16)
    R = torch.randn(B, CFG.tokens, CFG.dim, generator=g, device="cuda") / 100.0

    out = mod(clips)                                   # autograd path
    assert out.shape == (B, CFG.tokens, CFG.dim) and out.dtype == torch.bfloat16
    (out.float() * R).sum().backward()
    g_mod = mod.flat.grad.clone()

    rows = ops.patchify(clips, (CFG.cube_t, CFG.cube_h, CFG.cube_w))   # explicit engine path
    mod.store.grad.zero_()
    x, ctx = mod.engine.forward(rows, B)
    assert torch.equal(x.view(B, CFG.tokens, CFG.dim), out)
    mod.engine.backward(R.reshape(-1, CFG.dim).to(torch.bfloat16).contiguous(), ctx)
    assert rel(g_mod, mod.store.grad) < 1e-3          # same kernels; split-K fp32 red.add order only

    P = {n: mod.param(n).detach().clone().requires_grad_(True) for n in mod.names()}
    ref = VO.encoder_forward(P, VO.patchify(clips.float(), CFG), CFG, B).view(B, CFG.tokens, CFG.dim)
    (ref * R).sum().backward()
    assert rel(out, ref) < 2e-2
    for n in mod.names():
        o, shape = mod.store.offsets[n]
        got = g_mod[o:o + P[n].numel()].view(shape)
        assert rel(got, P[n].grad) < 2e-2, n

    # a torch optimizer updates the flat fp32 master; the next forward re-casts the bf16 shadow
    opt = torch.optim.SGD(mod.parameters(), lr=10.0)
    opt.step()
    out2 = mod(clips)
    assert torch.equal(mod.store.shadow, mod.flat.detach().to(torch.bfloat16))
    assert not torch.equal(out2, out)


@pytest.mark.parametrize("N,causal", [(300, False), (1569, False), (77, True)])
def test_attention_autograd(N, causal):
    B, H = 2, 3
    g = torch.Generator(device="cuda").manual_seed(N)
    q, k, v = (torch.randn(B, N, H * 64, generator=g, device="cuda").to(torch.bfloat16).requires_grad_(True)
               for _ in range(3))
    o = avnn.attention(q, k, v, H, causal=causal)
    do = torch.randn(B, N, H * 64, generator=g, device="cuda")
    (o.float() * do).sum().backward()

    qf, kf, vf = (t.detach().float().view(B, N, H, 64).transpose(1, 2).requires_grad_(True) for t in (q, k, v))
    s = qf @ kf.transpose(-1, -2) / 8.0
    if causal:
        s = s.masked_fill(torch.ones(N, N, dtype=torch.bool, device="cuda").triu(1), float("-inf"))
    ref = (torch.softmax(s, -1) @ vf).transpose(1, 2).reshape(B, N, H * 64)
    (ref * do).sum().backward()
    assert rel(o, ref) < 2e-2
    for got, r in ((q.grad, qf.grad), (k.grad, kf.grad), (v.grad, vf.grad)):
        assert rel(got, r.transpose(1, 2).reshape(B, N, H * 64)) < 2e-2


def test_clip_loss_autograd_matches_oracle():
    g = torch.Generator(device="cuda").manual_seed(5)
    v = torch.randn(64, 256, generator=g, device="cuda").requires_grad_(True)
    t = torch.randn(64, 256, generator=g, device="cuda").requires_grad_(True)
    ls = torch.full((1,), float(np.log(1 / 0.07)), device="cuda", requires_grad=True)
    loss = avnn.clip_loss(v, t, ls)
    (2.0 * loss).backward()                                  # a non-unit upstream gradient
    vr, tr = v.detach().clone().requires_grad_(True), t.detach().clone().requires_grad_(True)
    lr_ = ls.detach().clone().requires_grad_(True)
    ref = VO.clip_loss(vr, tr, lr_.exp().squeeze())
    (2.0 * ref).backward()
    assert abs(loss.item() - ref.item()) < 1e-4 * max(1.0, abs(ref.item()))
    assert rel(v.grad, vr.grad) < 1e-4 and rel(t.grad, tr.grad) < 1e-4
    assert abs(ls.grad.item() - lr_.grad.item()) < 1e-4 * max(1.0, abs(lr_.grad.item()))


@dataclass
class Batch:                      # the fields of vidpipe.loader.Batch the hand-off reads (loader.py:99-116)
    frames: np.ndarray
    sample_ids: list
    batch_index: int


def test_feeder_identity_handoff_and_ring_contract():
    rng = np.random.default_rng(0)
    ring = [rng.integers(0, 256, (4, 4, 3, 224, 224), dtype=np.uint8) for _ in range(2)]
    snap = [r.copy() for r in ring]
    fd = DeviceFeeder(4, 4, 224, 224, layout="cthw", depth=2)
    outs = []
    for i in range(5):                                       # more batches than ring slots
        fd.submit(Batch(ring[i % 2], [0, 1, 2, 3], i))
        ring[i % 2][:] = 255 - ring[i % 2]                   # the loader rewrites its ring after submit()
        outs.append((i, fd.next()))
    torch.cuda.synchronize()
    # batch i saw ring[i % 2] as it was at submit time: flipped (255 - x) once per earlier reuse
    for i, out in outs:
        src = snap[i % 2] if (i // 2) % 2 == 0 else 255 - snap[i % 2]
        thwc = src.transpose(0, 1, 3, 4, 2)                   # [B,T,H,W,3] for the oracle
        boxes = np.tile(np.asarray([[0, 0, 224, 224]], np.int32), (4, 1))
        ref = TO.transform_batch(thwc, boxes, np.zeros(4, np.uint8))
        assert np.abs(out.float().cpu().numpy() - ref).max() <= 0.02   # bf16 output


def test_feeder_raw_frames_with_crops_channels_last():
    rng = np.random.default_rng(1)
    frames = rng.integers(0, 256, (3, 4, 320, 568, 3), dtype=np.uint8)
    boxes = np.asarray([[65, 15, 392, 303], [40, 32, 346, 281], [50, 4, 327, 297]], np.int32)
    flips = np.asarray([0, 1, 0], np.uint8)
    fd = DeviceFeeder(3, 4, 320, 568, layout="cthw", out_dtype=torch.float32, channels_last=True)
    fd.submit(frames, boxes, flips)
    out = fd.next()
    ref = TO.transform_batch(frames, boxes, flips)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3
    pinned = torch.from_numpy(frames).pin_memory()           # zero-staging submit of a pinned tensor
    fd.submit(pinned, boxes, flips)
    assert np.abs(fd.next().cpu().numpy() - ref).max() <= 1e-3
