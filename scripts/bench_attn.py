"""Time K4/K5 on the config-4 (N=1569, 12 heads, 64 clips) and config-5 shapes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_16669_b200 import ops

for (B, N, H) in [(64, 1569, 12), (24, 2049, 16), (128, 785, 12)]:
    D = H * 64
    qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
    o, lse = ops.attn_fwd(q, k, v, H)
    do = torch.randn_like(o)
    g = torch.empty(B, N, 3, D, dtype=torch.bfloat16, device="cuda")
    f = lambda: ops.attn_fwd(q, k, v, H, out=o, lse=lse)
    bw = lambda: ops.attn_bwd(q, k, v, o, do, lse, H, dq=g[:, :, 0], dk=g[:, :, 1], dv=g[:, :, 2])
    res = {"B": B, "N": N, "H": H}
    for name, fn, mult in (("fwd", f, 1.0), ("bwd", bw, 2.5)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        fl = 4.0 * B * H * N * N * 64 * mult
        res[name + "_ms"] = ms
        res[name + "_tflops"] = fl / ms / 1e9
    # torch SDPA (cuDNN/flash) for context
    qh, kh, vh = (t.reshape(B, N, H, 64).transpose(1, 2) for t in (q, k, v))
    sd = lambda: torch.nn.functional.scaled_dot_product_attention(qh, kh, vh)
    for _ in range(3): sd()
    e0.record()
    for _ in range(5): sd()
    e1.record(); torch.cuda.synchronize()
    res["sdpa_fwd_tflops"] = 4.0 * B * H * N * N * 64 / (e0.elapsed_time(e1) / 5) / 1e9
    print(json.dumps(res), flush=True)
