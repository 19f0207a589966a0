import sys, os
sys.path.insert(0, os.getcwd())
import torch, math
from oracle import vit_oracle as VO
from paper_2309_16669_b200 import ops
from paper_2309_16669_b200.clip import CLIPModel
from paper_2309_16669_b200.vit import TextConfig, VitConfig
def rel(a, b):
    return ((a.float().cpu() - b.float().cpu()).norm() / b.float().cpu().norm().clamp_min(1e-30)).item()
for seed, ls in [(3, None), (5, None), (3, 0.0)]:
    vcfg = VitConfig(frames=2, height=32, width=48, cube_t=1, depth=2, dim=128, heads=2)
    tcfg = TextConfig(vocab=300, context=13, dim=128, heads=2, depth=2)
    B = 6
    m = CLIPModel(vcfg, tcfg, embed_dim=64, seed=seed)
    g = torch.Generator(device="cuda").manual_seed(4)
    m.store.data.add_(torch.randn(m.store.n, generator=g, device="cuda") * 0.02)
    if ls is not None: m.store.p("clip.logit_scale").fill_(ls)
    ops.cast_bf16(m.store.data, m.store.shadow)
    patches = torch.randn(B * vcfg.patches, vcfg.patch_dim, generator=g, device="cuda").to(torch.bfloat16)
    tokens = torch.randint(0, tcfg.vocab, (B, tcfg.context), generator=g, device="cuda", dtype=torch.int32)
    eot = (torch.arange(B, device="cuda", dtype=torch.int32) * tcfg.context + tokens.argmax(1).to(torch.int32))
    loss = torch.zeros(1, device="cuda")
    m.zero_grad()
    m.forward_backward(patches, tokens, eot, loss)
    torch.cuda.synchronize()
    names = [s[0] for s in m.store.specs]
    P = {n: m.store.p(n).detach().cpu().clone().requires_grad_(True) for n in names}
    ref = VO.clip_forward_loss(P, patches.float().cpu(), tokens.cpu(), eot.cpu(), vcfg, tcfg)
    ref.backward()
    print("seed", seed, "ls", ls, "loss", loss.item(), ref.item())
    errs = [(n, round(rel(m.store.g(n), P[n].grad), 4)) for n in names if P[n].grad is not None and P[n].grad.norm() > 1e-10]
    print(sorted(errs, key=lambda x: -x[1])[:12])
    print("median", sorted(e for _, e in errs)[len(errs)//2])
