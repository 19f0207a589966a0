"""One tiny training step of the whole hot path on cuda:0, checked against the CPU oracle.

Used by `__graft_entry__.smoke()`: uint8 clips -> K1 (crop + flip + antialiased resize + normalize,
written straight into the tubelet patch-embed operand) -> ViT encoder forward (tcgen05 GEMMs,
LayerNorm, blockwise attention) -> classification head + cross-entropy -> full backward ->
AdamW.  The loss and the parameter gradients are compared with the fp32 torch restatement
(oracle/vit_oracle.py) on the same patch rows and weights (tolerance 2e-2, north_star).
The oracle is the checker only; everything measured runs through libavion_b200.so.
"""

from __future__ import annotations

import numpy as np
import torch


def run(tol: float = 2e-2) -> dict:
    from oracle import vit_oracle as VO

    from . import ops
    from .vit import FineTuneModel, VitConfig

    cfg = VitConfig(frames=4, height=64, width=64, cube_t=2, depth=2, dim=128, heads=2)
    B, C = 2, 10
    model = FineTuneModel(cfg, num_classes=C, seed=1)
    g = torch.Generator(device="cuda").manual_seed(2)
    model.store.data.add_(torch.randn(model.store.n, generator=g, device="cuda") * 0.02)
    ops.cast_bf16(model.store.data, model.store.shadow)
    frames = torch.randint(0, 256, (B, cfg.frames, 96, 120, 3), generator=g, device="cuda", dtype=torch.uint8)
    boxes = np.asarray([[5, 3, 100, 80], [0, 0, 120, 96]], dtype=np.int32)
    patches = model.patches_from_clips(frames, torch.from_numpy(boxes).cuda(),
                                       torch.tensor([1, 0], dtype=torch.uint8, device="cuda"), boxes_host=boxes)
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
    loss_rel = abs(loss.item() - ref_loss.item()) / abs(ref_loss.item())
    worst = 0.0
    for n in names:
        ref = P[n].grad
        if ref is None or ref.norm() < 1e-12:
            continue
        got = model.store.g(n).float().cpu()
        if n in ("head.w", "head.b"):
            got, ref = got[:C], ref[:C]
        worst = max(worst, ((got - ref).norm() / ref.norm()).item())
    assert loss_rel < tol and worst < tol, f"model smoke: loss rel {loss_rel:.3e}, worst grad rel {worst:.3e}"
    model.optimizer_step()   # fused AdamW on the flat fp32 master buffer
    torch.cuda.synchronize()
    assert torch.isfinite(model.store.data).all()
    return {"loss": loss.item(), "loss_rel": loss_rel, "worst_grad_rel": worst}
