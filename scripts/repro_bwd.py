"""Run one K5 case (B N H causal from argv) and report errors / parity vs the fp32 reference."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16669_b200 import ops

B, N, H, causal = (int(x) for x in sys.argv[1:5])
g = torch.Generator(device="cuda").manual_seed(7)
q, k, v = ((torch.randn(B, N, H * 64, generator=g, device="cuda")).to(torch.bfloat16) for _ in range(3))
o, lse = ops.attn_fwd(q, k, v, H, causal=bool(causal))
do = torch.randn(B, N, H * 64, generator=g, device="cuda").to(torch.bfloat16)
dq, dk, dv = ops.attn_bwd(q, k, v, o, do, lse, H, causal=bool(causal))
torch.cuda.synchronize()
qf, kf, vf = (t.float().view(B, N, H, 64).transpose(1, 2).requires_grad_(True) for t in (q, k, v))
s = qf @ kf.transpose(-1, -2) / 8.0
if causal:
    s = s.masked_fill(torch.ones(N, N, dtype=torch.bool, device="cuda").triu(1), float("-inf"))
ref = torch.softmax(s, -1) @ vf
ref.backward(do.float().view(B, N, H, 64).transpose(1, 2))
for nm, got, r in (("dq", dq, qf.grad), ("dk", dk, kf.grad), ("dv", dv, vf.grad)):
    r = r.transpose(1, 2).reshape(B, N, H * 64)
    print(nm, ((got.float() - r).norm() / r.norm()).item())
