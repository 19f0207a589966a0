"""K7 fused InfoNCE vs the fp32 torch oracle (oracle/vit_oracle.clip_loss) incl. DP local-row gradients."""

import pytest
import torch

from oracle import vit_oracle as VO
from paper_2309_16669_b200 import ops

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float().cpu() - b.float().cpu()).norm() / b.float().cpu().norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("Bg,E,r0,n", [(4, 256, 0, 4), (1024, 256, 128, 128), (300, 64, 0, 300), (96, 512, 40, 17)])
def test_infonce_matches_oracle(Bg, E, r0, n):
    g = torch.Generator().manual_seed(Bg + E)
    v = torch.randn(Bg, E, generator=g)
    t = torch.randn(Bg, E, generator=g)
    s = 1 / 0.07
    vr, tr = v.clone().requires_grad_(True), t.clone().requires_grad_(True)
    sr = torch.tensor(s, requires_grad=True)
    ref = VO.clip_loss(vr, tr, sr)
    ref.backward()
    import math
    ls = torch.tensor([math.log(s)], device="cuda")
    loss, dls, dv, dt = ops.infonce(v.cuda(), t.cuda(), ls, r0, n, grad_scale=2.0)
    assert abs(loss.item() - ref.item()) / ref.item() < 1e-4
    # d/dlog_scale = s * d/ds
    assert abs(dls.item() - s * sr.grad.item()) < 1e-4 * max(1.0, abs(s * sr.grad.item()))
    assert rel(dv, 2.0 * vr.grad[r0:r0 + n]) < 1e-4
    assert rel(dt, 2.0 * tr.grad[r0:r0 + n]) < 1e-4
