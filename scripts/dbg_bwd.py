import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_attn_gpu import packed, ref_attn, rel
from paper_2309_16669_b200 import ops
for (B, N, H) in [(1, 128, 1), (2, 197, 3), (2, 300, 1), (1, 1569, 2), (2, 300, 1), (2, 785, 2)]:
    qkv = packed(B, N, H, seed=7 + N)
    q, k, v = (qkv[:, :, i].contiguous() for i in range(3))
    D = H * 64
    o, lse = ops.attn_fwd(q.view(B, N, D), k.view(B, N, D), v.view(B, N, D), H)
    g = torch.Generator(device="cuda").manual_seed(99)
    do = torch.randn(B, N, D, generator=g, device="cuda").to(torch.bfloat16)
    dq, dk, dv = ops.attn_bwd(q.view(B, N, D), k.view(B, N, D), v.view(B, N, D), o, do, lse, H)
    qf, kf, vf = (t.float().requires_grad_(True) for t in (q, k, v))
    ro, _ = ref_attn(qf, kf, vf, 0.125, False)
    ro.backward(do.float().view(B, N, H, 64))
    res = []
    for name, got, ref in (("dq", dq, qf.grad), ("dk", dk, kf.grad), ("dv", dv, vf.grad)):
        gg = got.reshape(B, N, H, 64).float(); 
        err = (gg - ref).norm(dim=-1) / ref.norm(dim=-1).clamp_min(1e-6)   # per (b, n, h)
        bad = (err > 0.05).nonzero()
        if bad.shape[0]: torch.save({'got': gg.cpu(), 'ref': ref.detach().cpu()}, f'gpurun_out/bad_{name}_{N}.pt')
        res.append(f"{name} rel={rel(gg, ref):.3e} nbad={bad.shape[0]} first={bad[:4].tolist()}")
    print(B, N, H, " | ".join(res))
