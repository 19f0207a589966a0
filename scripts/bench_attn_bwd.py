"""K5 and K4 at the config-4 and config-5 shapes: ms and TFLOP/s (algorithmic)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16669_b200 import ops


def tm(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for (B, N, H) in [(64, 1569, 12), (24, 2049, 16)]:
    D = H * 64
    qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
    o, lse = ops.attn_fwd(q, k, v, H)
    do = torch.randn_like(o)
    g = torch.empty(B, N, 3, D, dtype=torch.bfloat16, device="cuda")
    fl = 4.0 * B * H * N * N * 64
    res = {"shape": [B, N, H], "fwd_ms": tm(lambda: ops.attn_fwd(q, k, v, H, out=o, lse=lse))}
    res["bwd_ms"] = tm(lambda: ops.attn_bwd(q, k, v, o, do, lse, H, dq=g[:, :, 0], dk=g[:, :, 1], dv=g[:, :, 2]))
    res["bwd_tflops"] = 2 * fl / res["bwd_ms"] / 1e9
    res["fwd_tflops"] = fl / res["fwd_ms"] / 1e9
    print(json.dumps(res), flush=True)
