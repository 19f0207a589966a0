"""Race hunt: repeat the small fine-tune step of test_dp_gloo (single process, default mode) and
compare every step's gradient with the first one (the default paths differ only in fp32 summation
order, ~1e-7).  Prints the per-group error of any step that is off by more than 1e-5.

usage: python scripts/stress_step.py [steps] [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16669_b200.vit import FineTuneModel, VitConfig

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = VitConfig(frames=4, height=64, width=64, cube_t=2, depth=2, dim=128, heads=2)
C = 10
g = torch.Generator(device="cuda").manual_seed(7)
patches = torch.randn(B * cfg.patches, cfg.patch_dim, generator=g, device="cuda").to(torch.bfloat16)
labels = torch.randint(0, C, (B,), generator=g, device="cuda", dtype=torch.int32)
model = FineTuneModel(cfg, num_classes=C, seed=1)
st = model.store


def step():
    loss = torch.zeros(1, device="cuda")
    model.zero_grad()
    model.forward_backward(patches, labels, B, loss, loss_scale=1.0 / B)
    torch.cuda.synchronize()
    return st.grad.clone()


ref = step()
bad = 0
for i in range(steps):
    gr = step()
    tot = ((gr - ref).norm() / ref.norm()).item()
    if tot > 1e-5:
        bad += 1
        per = {}
        for name in st.groups:
            a, b = st.group_slice(name)
            per[name] = f"{((gr[a:b] - ref[a:b]).norm() / ref[a:b].norm().clamp_min(1e-30)).item():.1e}"
        print(f"step {i}: rel {tot:.3e} {per}", flush=True)
print(f"{bad} of {steps} steps off by > 1e-5 (B={B})", flush=True)
