"""K4/K5 vs torch SDPA (cuDNN / flash backends) fwd+bwd on the config-4 shape."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_16669_b200 import ops

def tm(fn, n=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

for (B, N, H) in [(64, 1569, 12)]:
    D = H * 64
    qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
    o, lse = ops.attn_fwd(q, k, v, H)
    do = torch.randn_like(o)
    g = torch.empty(B, N, 3, D, dtype=torch.bfloat16, device="cuda")
    fl = 4.0 * B * H * N * N * 64
    res = {"fwd_ms": tm(lambda: ops.attn_fwd(q, k, v, H, out=o, lse=lse)),
           "bwd_ms": tm(lambda: ops.attn_bwd(q, k, v, o, do, lse, H, dq=g[:, :, 0], dk=g[:, :, 1], dv=g[:, :, 2]))}
    qh, kh, vh = (t.reshape(B, N, H, 64).transpose(1, 2).detach().requires_grad_() for t in (q, k, v))
    from torch.nn.attention import sdpa_kernel, SDPBackend
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel(be):
                out = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh)
                dout = torch.randn_like(out)
                f_ms = tm(lambda: torch.nn.functional.scaled_dot_product_attention(qh, kh, vh))
                def fb():
                    out = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh)
                    torch.autograd.grad(out, (qh, kh, vh), dout)
                fb_ms = tm(fb)
            res[str(be).split('.')[-1]] = {"fwd_ms": f_ms, "bwd_ms": fb_ms - f_ms}
        except Exception as e:
            res[str(be).split('.')[-1]] = repr(e)[:120]
    res["fwd_tflops"] = fl / res["fwd_ms"] / 1e9
    res["bwd_tflops_2x"] = 2 * fl / res["bwd_ms"] / 1e9
    print(json.dumps(res), flush=True)
