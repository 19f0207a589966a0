"""K1 parity on the GPU: CUDA kernel vs the float64 numpy oracle on identical inputs + boxes.

Tolerances (BASELINE.json north_star / SURVEY.md 8(c)):
  * tap index ranges: bit-exact; gather at identity scale: exact;
  * fp32 output: <= 1e-3 absolute;
  * bf16 output: <= 1 bf16 ulp of the oracle value.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import transform_oracle as O
from paper_2309_16669_b200 import transform as T
from paper_2309_16669_b200.errors import InputError

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rrc_golden.json")))
CFG2 = np.asarray(GOLD["config2_568x320"], dtype=np.int32)


def frames_u8(B, Tn, H, W, seed=0):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (B, Tn, H, W, 3), generator=g, dtype=torch.uint8)


def bf16_ulp(x):
    a = np.abs(x).astype(np.float64)
    e = np.floor(np.log2(np.maximum(a, 1e-30)))
    return np.where(a > 0, 2.0 ** (e - 7), 2.0 ** -133)


@pytest.mark.parametrize("crop,tgt", [(303, 224), (392, 224), (427, 224), (448, 224), (100, 224), (224, 224),
                                      (7, 3), (5, 9), (568, 224), (1, 224)])
def test_device_taps_bit_exact(crop, tgt):
    lo, hi, w = T.device_taps(crop, tgt)
    elo, ehi = O.tap_ranges(crop, tgt)
    assert np.array_equal(lo.cpu().numpy(), elo)
    assert np.array_equal(hi.cpu().numpy(), ehi)
    m = O.weight_matrix(crop, tgt)
    wd = w.cpu().numpy()
    for i in range(tgt):
        n = ehi[i] - elo[i]
        assert np.allclose(wd[i, :n], m[i, elo[i]:ehi[i]], atol=1e-7, rtol=0)


def test_identity_gather_exact():
    fr = frames_u8(2, 3, 64, 80, seed=1)
    boxes = np.asarray([[0, 0, 80, 64], [0, 0, 80, 64]], dtype=np.int32)
    out = T.transform(fr.cuda(), boxes, [0, 1], (64, 80), mean=(0, 0, 0), std=(1, 1, 1), out_dtype=torch.float32)
    ref = fr.numpy().transpose(0, 4, 1, 2, 3).astype(np.float64) / 255.0
    ref[1] = ref[1][..., ::-1]
    assert np.abs(out.cpu().numpy() - ref).max() < 1e-6
    # byte-exact gather: recover the source bytes
    back = np.rint(out.cpu().numpy() * 255.0)
    assert np.array_equal(back[0], fr.numpy()[0].transpose(3, 0, 1, 2))


@pytest.mark.parametrize("layout", ["cthw", "tchw"])
def test_config2_boxes_fp32_and_bf16(layout):
    B, Tn = 6, 4
    fr = frames_u8(B, Tn, 320, 568, seed=2)
    boxes, flips = CFG2[:B, :4], CFG2[:B, 4]
    ref = O.transform_batch(fr.numpy(), boxes, flips)                     # [B,3,T,224,224]
    if layout == "tchw":
        ref = ref.transpose(0, 2, 1, 3, 4)
    d = fr.cuda()
    o32 = T.transform(d, boxes, flips, out_dtype=torch.float32, layout=layout).cpu().numpy()
    assert np.abs(o32 - ref).max() <= 1e-3
    o16 = T.transform(d, boxes, flips, out_dtype=torch.bfloat16, layout=layout).float().cpu().numpy()
    assert np.all(np.abs(o16 - ref) <= bf16_ulp(ref) + 1e-6)


def test_generic_strides_reference_batch_layout():
    """[B,T,3,H,W] planar (reference Batch.frames) takes the generic-stride path."""
    B, Tn = 3, 2
    fr = frames_u8(B, Tn, 120, 200, seed=3)
    planar = fr.permute(0, 1, 4, 2, 3).contiguous().cuda()               # [B,T,3,H,W]
    boxes = np.asarray([[3, 5, 150, 101], [0, 0, 200, 120], [50, 19, 77, 99]], dtype=np.int32)
    flips = np.asarray([1, 0, 1])
    out = T.transform(planar, boxes, flips, (64, 96), channels_last=False, out_dtype=torch.float32)
    ref = O.transform_batch(fr.numpy(), boxes, flips, (64, 96))
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3


@pytest.mark.parametrize("layout", ["cthw", "tubelet"])
def test_planar_v4_config2_boxes(layout):
    """Reference-layout [B,T,3,H,W] clips with host boxes (downscales, 16-byte-aligned planes) stream
    through v4 with one bulk copy per channel plane: same tolerances as the interleaved path, and the
    same values as the forced generic kernel."""
    B, Tn = 4, 4
    fr = frames_u8(B, Tn, 320, 568, seed=21)
    planar = fr.permute(0, 1, 4, 2, 3).contiguous().cuda()                   # [B,T,3,H,W]
    boxes, flips = CFG2[:B, :4], CFG2[:B, 4]
    ref = O.transform_batch(fr.numpy(), boxes, flips)                       # [B,3,T,224,224]
    kw = dict(channels_last=False, crops_host=boxes, layout=layout)
    if layout == "tubelet":   # [B, T/2, 14, 14, 3, 2, 16, 16] -> rows (t', py, px), features (c, dt, y, x)
        kw["tubelet"] = (2, 16, 16)
        ref = ref.reshape(B, 3, Tn // 2, 2, 14, 16, 14, 16).transpose(0, 2, 4, 6, 1, 3, 5, 7).reshape(-1, 1536)
    o32 = T.transform(planar, boxes, flips, out_dtype=torch.float32, **kw).cpu().numpy()
    o16 = T.transform(planar, boxes, flips, **kw).float().cpu().numpy()
    assert np.abs(o32 - ref).max() <= 1e-3
    assert np.all(np.abs(o16 - ref) <= bf16_ulp(ref) + 1e-6)
    from paper_2309_16669_b200 import _lib
    with _Path(_lib.AVB_K1_PATH_GENERIC):
        g32 = T.transform(planar, boxes, flips, out_dtype=torch.float32, **kw).cpu().numpy()
    assert np.abs(o32 - g32).max() <= 2e-5


def test_planar_v4_tensor_end_and_unaligned_planes():
    """Planar clip whose last channel row ends at the tensor end (zero-filled tail copies), and planes
    that are not 16-byte aligned (generic fallback) -- both against the oracle."""
    fr = frames_u8(1, 2, 230, 304, seed=22)                                 # plane 69920 B = 16 * 4370
    b2 = np.asarray([[80, 6, 224, 224]], dtype=np.int32)
    planar = fr.permute(0, 1, 4, 2, 3).contiguous()
    out = T.transform(planar.cuda(), b2, [1], channels_last=False, crops_host=b2, out_dtype=torch.float32)
    ref = O.transform_batch(fr.numpy(), b2, np.asarray([1]))
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3
    fr2 = frames_u8(2, 2, 231, 301, seed=23)                                # plane 69531 B: unaligned
    b3 = np.asarray([[0, 0, 300, 230], [40, 3, 250, 228]], dtype=np.int32)
    pl2 = fr2.permute(0, 1, 4, 2, 3).contiguous()
    out = T.transform(pl2.cuda(), b3, [0, 1], channels_last=False, crops_host=b3, out_dtype=torch.float32)
    ref = O.transform_batch(fr2.numpy(), b3, np.asarray([0, 1]))
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3


@pytest.mark.parametrize("H,W,Ht,Wt,box", [(40, 50, 97, 131, (3, 2, 41, 33)),   # upscale, odd Wt
                                           (33, 47, 33, 47, (0, 0, 47, 33)),    # identity, odd
                                           (9, 9, 1, 1, (0, 0, 9, 9)),          # to 1 pixel
                                           (600, 1000, 224, 224, (10, 20, 980, 570))])  # 4.4x down
def test_edge_shapes(H, W, Ht, Wt, box):
    fr = frames_u8(1, 2, H, W, seed=4)
    out = T.transform(fr.cuda(), np.asarray([box], dtype=np.int32), [1], (Ht, Wt), out_dtype=torch.float32)
    ref = O.transform_batch(fr.numpy(), np.asarray([box]), np.asarray([1]), (Ht, Wt))
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3


def test_out_buffer_and_errors():
    fr = frames_u8(2, 2, 50, 60).cuda()
    boxes = np.asarray([[0, 0, 60, 50], [10, 10, 50, 40]], dtype=np.int32)
    buf = torch.full((2, 3, 2, 32, 32), 7.0, dtype=torch.bfloat16, device="cuda")
    r = T.transform(fr, boxes, None, (32, 32), out=buf)
    assert r.data_ptr() == buf.data_ptr()
    with pytest.raises(InputError):
        T.transform(fr, boxes, None, (32, 31), out=buf)                     # shape mismatch
    bad = np.asarray([[0, 0, 60, 50], [11, 10, 50, 40]], dtype=np.int32)  # x + w = 61 > 60
    before = buf.clone()
    with pytest.raises(InputError):
        T.transform(fr, bad, None, (32, 32), out=buf)
    torch.cuda.synchronize()
    assert torch.equal(before, buf)                                          # untouched on error
    with pytest.raises(InputError):
        T.transform(fr.cpu(), boxes, None, (32, 32))                        # no CPU path


def test_full_config2_size_properties():
    """B=64, T=16, 568x320 -> 224^2 bf16: spot-check clips vs oracle + flip/mirror property."""
    B, Tn = 64, 16
    g = torch.Generator(device="cuda").manual_seed(0)
    fr = torch.randint(0, 256, (B, Tn, 320, 568, 3), generator=g, dtype=torch.uint8, device="cuda")
    boxes, flips = CFG2[:B, :4], CFG2[:B, 4]
    out = T.transform(fr, boxes, flips)
    assert out.shape == (B, 3, Tn, 224, 224) and torch.isfinite(out.float()).all()
    for b in (0, 1, 37, 63):
        ref = O.transform_clip(fr[b, :4].cpu().numpy(), boxes[b], bool(flips[b]))
        o = out[b, :, :4].float().cpu().numpy()
        assert np.all(np.abs(o - ref) <= bf16_ulp(ref) + 1e-6)
    # flipping the flip bit mirrors the output columns (up to bf16 rounding of equal values)
    out2 = T.transform(fr, boxes, 1 - flips)
    assert (out2.float() - out.float().flip(-1)).abs().max().item() <= 0.02


# ---------------------------------------------------------------- v4 (default streaming kernel) coverage
class _Path:
    """Pin K1's kernel choice for the process (avb_k1_force_path test hook), restored on exit."""

    def __init__(self, path):
        self.path = path

    def __enter__(self):
        from paper_2309_16669_b200 import _lib
        self.old = _lib.load().avb_k1_force_path(self.path)

    def __exit__(self, *a):
        from paper_2309_16669_b200 import _lib
        _lib.load().avb_k1_force_path(self.old)


@pytest.mark.parametrize("Tn", [1, 3, 4])
def test_v4_matches_v2_and_oracle(Tn):
    """v4 (default) and v2 (AVB_K1_V2) agree to fp32 rounding; odd T leaves a partial frame group."""
    B = 5
    fr = frames_u8(B, Tn, 320, 568, seed=7)
    boxes, flips = CFG2[8:8 + B, :4], CFG2[8:8 + B, 4]
    ref = O.transform_batch(fr.numpy(), boxes, flips)
    d = fr.cuda()
    o4 = T.transform(d, boxes, flips, out_dtype=torch.float32)
    from paper_2309_16669_b200 import _lib
    with _Path(_lib.AVB_K1_PATH_STRIP):
        o2 = T.transform(d, boxes, flips, out_dtype=torch.float32)
    assert np.abs(o4.cpu().numpy() - ref).max() <= 1e-3
    assert (o4 - o2).abs().max().item() <= 2e-5


def test_v4_tubelet_layout():
    B, Tn = 3, 4
    fr = frames_u8(B, Tn, 320, 568, seed=8)
    boxes, flips = CFG2[20:20 + B, :4], CFG2[20:20 + B, 4]
    ref = O.transform_batch(fr.numpy(), boxes, flips)                      # [B,3,T,224,224]
    tub = T.transform(fr.cuda(), boxes, flips, out_dtype=torch.float32, layout="tubelet", tubelet=(2, 16, 16))
    # [B, T/2, 14, 14, 3, 2, 16, 16] -> rows (t', py, px), features (c, dt, y, x)
    r = ref.reshape(B, 3, Tn // 2, 2, 14, 16, 14, 16).transpose(0, 2, 4, 6, 1, 3, 5, 7).reshape(-1, 1536)
    assert np.abs(tub.cpu().numpy() - r).max() <= 1e-3


@pytest.mark.parametrize("tub", [(1, 16, 16), (2, 14, 14), (2, 16, 16)])
def test_tubelet_layouts_configs_3_4_5(tub):
    """The patch-embed operand for config 3 (1x16x16), config 4 (2x16x16) and config 5 (2x14x14)."""
    from oracle import vit_oracle as VO
    from paper_2309_16669_b200.vit import VitConfig
    tt, ph, pw = tub
    B, Tn = 3, 4
    fr = frames_u8(B, Tn, 320, 568, seed=30 + pw)
    boxes, flips = CFG2[40:40 + B, :4], CFG2[40:40 + B, 4]
    ref = O.transform_batch(fr.numpy(), boxes, flips)                      # [B,3,T,224,224] float64
    cfg = VitConfig(frames=Tn, cube_t=tt, cube_h=ph, cube_w=pw)
    r = VO.patchify(torch.from_numpy(ref), cfg).numpy()
    tubf = T.transform(fr.cuda(), boxes, flips, out_dtype=torch.float32, layout="tubelet", tubelet=tub)
    assert tubf.shape == (B * cfg.patches, cfg.patch_dim)
    assert np.abs(tubf.cpu().numpy() - r).max() <= 1e-3
    tubh = T.transform(fr.cuda(), boxes, flips, layout="tubelet", tubelet=tub).float().cpu().numpy()
    assert np.all(np.abs(tubh - r) <= bf16_ulp(r) + 1e-6)


def test_forced_generic_path_matches_oracle():
    from paper_2309_16669_b200 import _lib
    fr = frames_u8(2, 3, 320, 568, seed=33)
    boxes, flips = CFG2[50:52, :4], CFG2[50:52, 4]
    ref = O.transform_batch(fr.numpy(), boxes, flips)
    with _Path(_lib.AVB_K1_PATH_GENERIC):
        out = T.transform(fr.cuda(), boxes, flips, out_dtype=torch.float32)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3


@pytest.mark.parametrize("H,W,Ht,Wt,box,flip", [
    (120, 200, 57, 81, (3, 5, 150, 101), 1),     # odd target width (last thread has one column)
    (90, 180, 30, 64, (1, 2, 171, 87), 0),       # many frames per CTA, ~2.7x down (NT 6)
    (64, 64, 60, 62, (0, 1, 63, 63), 1),         # barely-downscale
    (50, 70, 50, 70, (0, 0, 70, 50), 1),         # identity scale (crop == target)
    (260, 900, 64, 240, (5, 7, 881, 250), 0),    # 3.7x down horizontally (NT 8)
])
def test_v4_shapes(H, W, Ht, Wt, box, flip):
    Tn = 5
    fr = frames_u8(2, Tn, H, W, seed=9)
    boxes = np.asarray([box, box], dtype=np.int32)
    flips = np.asarray([flip, 1 - flip])
    ref = O.transform_batch(fr.numpy(), boxes, flips, (Ht, Wt))
    out = T.transform(fr.cuda(), boxes, flips, (Ht, Wt), out_dtype=torch.float32)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3
    o16 = T.transform(fr.cuda(), boxes, flips, (Ht, Wt)).float().cpu().numpy()
    assert np.all(np.abs(o16 - ref) <= bf16_ulp(ref) + 1e-6)


def test_v4_strided_view_and_tensor_end():
    """A sliced (non-contiguous-clip) view; the last row of the last frame ends at the tensor end."""
    full = frames_u8(4, 3, 300, 410, seed=10)                              # row pitch 1230 = 14 mod 16
    boxes = np.asarray([[0, 0, 405, 280], [100, 50, 305, 230]], dtype=np.int32)
    flips = np.asarray([0, 1])
    fd = full.cuda()
    for sl in (np.s_[2:4], np.s_[1:3, :, 20:, 5:]):                        # 16B-aligned slice / unaligned view
        view = full[sl]
        ref = O.transform_batch(view.numpy(), boxes, flips)
        out = T.transform(fd[sl], boxes, flips, out_dtype=torch.float32)
        assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3
    tail = frames_u8(1, 2, 230, 300, seed=11)                               # box touches the last byte
    b2 = np.asarray([[76, 6, 224, 224]], dtype=np.int32)
    out = T.transform(tail.cuda(), b2, [1], out_dtype=torch.float32)
    ref = O.transform_batch(tail.numpy(), b2, np.asarray([1]))
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3


def test_v4_device_boxes_mixed_scales():
    """Device-only boxes (validate=False): v4 takes the downscale clips with the worst-case tap
    envelope, a complement v2 launch takes the upscale clip; every clip matches the oracle."""
    fr = frames_u8(3, 3, 320, 568, seed=12)
    boxes = np.asarray([[65, 15, 392, 303], [300, 200, 150, 100], [0, 0, 568, 320]], dtype=np.int32)
    flips = np.asarray([1, 0, 1])
    ref = O.transform_batch(fr.numpy(), boxes, flips)
    bd = torch.from_numpy(boxes).cuda()
    fd = torch.from_numpy(flips.astype(np.uint8)).cuda()
    out = T.transform(fr.cuda(), bd, fd, out_dtype=torch.float32, validate=False)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3


@pytest.mark.parametrize("layout", ["cthw", "tchw", "tubelet"])
def test_identity_planar_fused_decode_handoff(layout):
    """CPU fused decode already cropped/scaled to 224^2 -> [B,T,3,224,224] uint8
    (reference Batch.frames); K1's identity kernel only flips, normalizes, casts and re-lays out."""
    B, Tn = 3, 4
    fr = frames_u8(B, Tn, 224, 224, seed=13)                                 # [B,T,H,W,3]
    planar = fr.permute(0, 1, 4, 2, 3).contiguous()                          # [B,T,3,H,W]
    boxes = np.asarray([[0, 0, 224, 224]] * B, dtype=np.int32)
    flips = np.asarray([0, 1, 1])
    ref = O.transform_batch(fr.numpy(), boxes, flips)                        # [B,3,T,224,224]
    kw = dict(layout=layout, channels_last=False)
    if layout == "tubelet":
        kw["tubelet"] = (2, 16, 16)
        ref = ref.reshape(B, 3, Tn // 2, 2, 14, 16, 14, 16).transpose(0, 2, 4, 6, 1, 3, 5, 7).reshape(-1, 1536)
    elif layout == "tchw":
        ref = ref.transpose(0, 2, 1, 3, 4)
    o32 = T.transform(planar.cuda(), boxes, flips, out_dtype=torch.float32, **kw).cpu().numpy()
    assert np.abs(o32 - ref).max() <= 1e-3
    o16 = T.transform(planar.cuda(), boxes, flips, **kw).float().cpu().numpy()
    assert np.all(np.abs(o16 - ref) <= bf16_ulp(ref) + 1e-6)
    # byte-exact gather through the identity path: recover the source bytes
    back = T.transform(planar.cuda(), boxes, None, mean=(0, 0, 0), std=(1, 1, 1), out_dtype=torch.float32,
                       channels_last=False)
    assert np.array_equal(np.rint(back.cpu().numpy() * 255.0), fr.numpy().transpose(0, 4, 1, 2, 3))
