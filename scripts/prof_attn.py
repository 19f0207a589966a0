"""One K4 + K5 launch at the config-4 shape (for `ncu -k regex:attn_` captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16669_b200 import ops

B, N, H = (int(x) for x in os.environ.get("SHAPE", "64,1569,12").split(","))
D = H * 64
qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
o, lse = ops.attn_fwd(q, k, v, H)
do = torch.randn_like(o)
for _ in range(2):
    ops.attn_fwd(q, k, v, H, out=o, lse=lse)
    ops.attn_bwd(q, k, v, o, do, lse, H)
torch.cuda.synchronize()
