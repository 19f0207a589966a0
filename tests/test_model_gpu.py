"""Encoder + head + loss + gradients on the GPU kernels vs the fp32 torch oracle (oracle/vit_oracle.py).

Same inputs (patch rows), same fp32 master weights.  Tolerance (north_star): loss,
outputs and every parameter gradient within 2e-2 norm-relative of fp32.
"""

import pytest
import torch

from oracle import vit_oracle as VO
from paper_2309_16669_b200 import ops
from paper_2309_16669_b200.vit import CONFIG1_TINY, FineTuneModel, VitConfig

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float().cpu() - b.float().cpu()).norm() / b.float().cpu().norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("cfg,B,C", [(VitConfig(frames=4, height=64, width=64, cube_t=2, depth=2, dim=128, heads=2), 3, 10),
                                     (CONFIG1_TINY, 4, 400)])
def test_finetune_step_matches_oracle(cfg, B, C):
    torch.manual_seed(0)
    model = FineTuneModel(cfg, num_classes=C, seed=1)
    # make every parameter non-trivial (biases / LN / cls start at constants)
    g = torch.Generator(device="cuda").manual_seed(2)
    model.store.data.add_(torch.randn(model.store.n, generator=g, device="cuda") * 0.02)
    ops.cast_bf16(model.store.data, model.store.shadow)
    patches = torch.randn(B * cfg.patches, cfg.patch_dim, generator=g, device="cuda").to(torch.bfloat16)
    labels = torch.randint(0, C, (B,), generator=g, device="cuda", dtype=torch.int32)
    loss = torch.zeros(1, device="cuda")
    model.zero_grad()
    model.forward_backward(patches, labels, B, loss)
    torch.cuda.synchronize()

    names = [s[0] for s in model.store.specs]
    P = {n: model.store.p(n).detach().cpu().clone().requires_grad_(True) for n in names}
    x = VO.encoder_forward(P, patches.float().cpu(), cfg, B)
    ref_loss, _ = VO.head_loss(P, x, B, cfg.tokens, labels.cpu(), C)
    ref_loss.backward()
    assert abs(loss.item() - ref_loss.item()) / abs(ref_loss.item()) < 2e-2
    bad = []
    for n in names:
        ref = P[n].grad
        if ref is None or ref.norm() < 1e-12:
            continue
        got = model.store.g(n)
        if n == "head.w" or n == "head.b":
            got, ref = got[:C], ref[:C]
        r = rel(got, ref)
        if r > 2e-2:
            bad.append((n, r))
    assert not bad, bad


@pytest.mark.parametrize("n,off", [(10_000, 0), (10_003, 0), (10_003, 1)])
def test_adamw_kernel_matches_torch(n, off):
    # off = 1: every buffer is a view one element in (not 16-byte aligned) -> scalar kernel;
    # n = 10_003: vectorised body + scalar tail
    g0 = torch.Generator(device="cuda").manual_seed(3)
    p = torch.randn(n + off, device="cuda", generator=g0)[off:]
    grads = [torch.randn(n, device="cuda", generator=g0) for _ in range(3)]
    m, v = torch.zeros(n + off, device="cuda")[off:], torch.zeros(n + off, device="cuda")[off:]
    sh = torch.empty(n + off, dtype=torch.bfloat16, device="cuda")[off:]
    mask = (torch.arange(n, device="cuda") % 3 != 0).to(torch.uint8)
    tp_d = p.clone().requires_grad_(True)
    tp_n = p.clone().requires_grad_(True)
    opt = torch.optim.AdamW([{"params": [tp_d], "weight_decay": 0.01}, {"params": [tp_n], "weight_decay": 0.0}],
                            lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    for i, gr in enumerate(grads):
        ops.adamw(p, gr, m, v, sh, 1e-3, 0.9, 0.999, 1e-8, 0.01, i + 1, decay_mask=mask)
        tp_d.grad, tp_n.grad = gr.clone(), gr.clone()
        opt.step()
    ref = torch.where(mask.bool(), tp_d.detach(), tp_n.detach())
    assert (p - ref).abs().max().item() < 1e-6
    assert torch.equal(sh, p.to(torch.bfloat16))


@pytest.mark.parametrize("M,D,acc", [(1000, 768, True), (1, 768, True), (1003, 256, False), (20011, 1024, True),
                                     (4099, 512, False), (3001, 520, True), (777, 200, False), (5000, 1000, True)])
def test_layernorm_and_colsum(M, D, acc):
    # ragged row counts (M % 8 != 0) exercise the partial last row block of the TMA-staged kernels
    g0 = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn(M, D, device="cuda", generator=g0).to(torch.bfloat16)
    gam = torch.randn(D, device="cuda", generator=g0)
    bet = torch.randn(D, device="cuda", generator=g0)
    y, mu, rs = ops.layernorm_fwd(x, gam, bet)
    xf = x.float().requires_grad_(True)
    gf, bf = gam.clone().requires_grad_(True), bet.clone().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xf, (D,), gf, bf, 1e-5)
    assert rel(y, ref) < 1e-2
    dy = torch.randn(M, D, device="cuda", generator=g0).to(torch.bfloat16)
    ref.backward(dy.float())
    dx = torch.randn(M, D, device="cuda", generator=g0).to(torch.bfloat16)
    if not acc:
        dx.zero_()
    dx0 = dx.float().clone()
    dg = torch.zeros(D, device="cuda")
    db = torch.zeros(D, device="cuda")
    csum = torch.zeros(D, device="cuda")
    ops.layernorm_bwd(dy, x, gam, mu, rs, dx, dg, db, accumulate=acc, dx_colsum=csum)
    assert rel(dx.float() - dx0, xf.grad) < 2e-2
    assert rel(csum, dx.float().sum(0)) < 1e-4
    assert rel(dg, gf.grad) < 1e-3 and rel(db, bf.grad) < 1e-3
    cs = torch.zeros(D, device="cuda")
    ops.colsum_accum(dy, cs)
    assert rel(cs, dy.float().sum(0)) < 1e-4


def test_tubelet_layout_matches_patchify():
    import numpy as np
    from oracle import transform_oracle as TO
    from paper_2309_16669_b200 import transform as TR
    cfg = VitConfig(frames=4, height=64, width=96, cube_t=2, cube_h=16, cube_w=16, depth=1, dim=64, heads=1)
    B = 2
    g0 = torch.Generator().manual_seed(5)
    fr = torch.randint(0, 256, (B, 4, 120, 160, 3), generator=g0, dtype=torch.uint8)
    boxes = np.asarray([[3, 4, 150, 101], [10, 0, 140, 120]], dtype=np.int32)
    flips = np.asarray([1, 0], dtype=np.uint8)
    cthw = TR.transform(fr.cuda(), boxes, flips, (64, 96), out_dtype=torch.float32)
    tub = TR.transform(fr.cuda(), boxes, flips, (64, 96), out_dtype=torch.float32, layout="tubelet", tubelet=(2, 16, 16))
    assert torch.equal(tub, VO.patchify(cthw, cfg))


def test_adamw_dev_counter_matches_host_step():
    """avb_adamw_dev (step count on the device, incremented per call) == avb_adamw with host steps."""
    g0 = torch.Generator(device="cuda").manual_seed(8)
    n = 4099
    p1 = torch.randn(n, device="cuda", generator=g0)
    p2 = p1.clone()
    m1, v1, m2, v2 = (torch.zeros(n, device="cuda") for _ in range(4))
    step = torch.zeros(1, dtype=torch.int32, device="cuda")
    for i in range(3):
        gr = torch.randn(n, device="cuda", generator=g0)
        ops.adamw(p1, gr, m1, v1, None, 1e-3, 0.9, 0.999, 1e-8, 0.01, i + 1)
        ops.adamw_dev(p2, gr, m2, v2, None, 1e-3, 0.9, 0.999, 1e-8, 0.01, step)
    assert step.item() == 3
    assert (p1 - p2).abs().max().item() < 1e-7


def test_captured_train_step_matches_eager():
    """FineTuneModel.capture_train_step: 1 warm-up step + 2 graph replays == 3 eager steps."""
    cfg = VitConfig(frames=4, height=64, width=64, cube_t=2, depth=2, dim=128, heads=2)
    B, C = 3, 10
    g = torch.Generator(device="cuda").manual_seed(9)
    patches = torch.randn(B * cfg.patches, cfg.patch_dim, generator=g, device="cuda").to(torch.bfloat16)
    labels = torch.randint(0, C, (B,), generator=g, device="cuda", dtype=torch.int32)
    eager = FineTuneModel(cfg, num_classes=C, seed=1)
    graphed = FineTuneModel(cfg, num_classes=C, seed=1)
    loss_e = torch.zeros(1, device="cuda")
    for _ in range(3):
        eager.zero_grad()
        loss_e.zero_()
        eager.forward_backward(patches, labels, B, loss_e)
        eager.optimizer_step()
    loss_g = torch.zeros(1, device="cuda")
    step = graphed.capture_train_step(patches, labels, B, loss_g, warmup=1)
    step()
    step()
    torch.cuda.synchronize()
    assert graphed.store.step_dev.item() == 3
    d = (graphed.store.data - eager.store.data).abs().max().item()
    assert d < 1e-5, d
    assert abs(loss_g.item() - loss_e.item()) < 1e-4 * abs(loss_e.item())
