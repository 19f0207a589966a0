import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2309_16669_b200 import ops
for (B, N, H) in [(4, 1569, 6), (2, 2049, 4)]:
    D = H * 64
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = (torch.randn(B, N, D, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    o, lse = ops.attn_fwd(q, k, v, H)
    do = torch.randn(B, N, D, generator=g, device="cuda").to(torch.bfloat16)
    dq_bf = ops.attn_bwd(q, k, v, o, do, lse, H)[0].clone()
    dq_32 = ops.attn_bwd(q, k, v, o, do, lse, H, fp32_dq=True)[0].clone()
    qf, kf, vf = (t.float().view(B, N, H, 64).transpose(1, 2).requires_grad_(True) for t in (q, k, v))
    ref = torch.softmax(qf @ kf.transpose(-1, -2) / 8.0, -1) @ vf
    ref.backward(do.float().view(B, N, H, 64).transpose(1, 2))
    r = qf.grad.transpose(1, 2).reshape(B, N, D)
    rel = lambda a: ((a.float() - r).norm() / r.norm()).item()
    print(B, N, H, "dq rel err bf16-direct", rel(dq_bf), "fp32-acc", rel(dq_32))
