"""Tiny K4/K5 run with a parity check (for quick same-box A/B of experimental builds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_16669_b200 import ops
torch.manual_seed(0)
for (B, N, H) in [(2, 300, 2), (4, 1569, 12)]:
    D = H * 64
    qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
    o, lse = ops.attn_fwd(q, k, v, H)
    torch.cuda.synchronize()
    qf, kf, vf = (t.float().view(B, N, H, 64).transpose(1, 2) for t in (q, k, v))
    ref = torch.softmax(qf @ kf.transpose(-1, -2) / 8.0, -1) @ vf
    err = (o.float().view(B, N, H, 64).transpose(1, 2) - ref).abs().max().item()
    print("shape", (B, N, H), "fwd max err", err, flush=True)
