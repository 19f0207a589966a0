"""LayerNorm fwd/bwd at the config-4 shape (M = 64*1569, D = 768): time and achieved HBM GB/s."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_16669_b200 import ops
M, D = 64 * 1569, 768
x = torch.randn(M, D, device="cuda").to(torch.bfloat16)
dy = torch.randn(M, D, device="cuda").to(torch.bfloat16)
g = torch.randn(D, device="cuda"); b = torch.randn(D, device="cuda")
y = torch.empty_like(x); mu = torch.empty(M, device="cuda"); rs = torch.empty(M, device="cuda")
dx = torch.zeros_like(x); dg = torch.zeros(D, device="cuda"); db = torch.zeros(D, device="cuda")
def tm(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
f_ms = tm(lambda: ops.layernorm_fwd(x, g, b, out=y, mean=mu, rstd=rs) if 'out' in ops.layernorm_fwd.__code__.co_varnames else ops.layernorm_fwd(x, g, b))
b_ms = tm(lambda: ops.layernorm_bwd(dy, x, g, mu, rs, dx, dg, db, accumulate=True))
print(json.dumps({"fwd_ms": f_ms, "fwd_GBs": 2 * M * D * 2 / f_ms / 1e6, "bwd_ms": b_ms, "bwd_GBs": 4 * M * D * 2 / b_ms / 1e6}))
