"""wgrad GEMMs of a config-4 layer with and without the fused bias-gradient row sums (a_rowsum)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16669_b200 import ops
from paper_2309_16669_b200.vit import wgrad_split

M = 64 * 1569


def tm(fn, n=20):
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


for name, mo, no in (("fc2", 768, 3072), ("fc1", 3072, 768), ("qkv", 2304, 768), ("proj", 768, 768)):
    dy = torch.randn(M, mo, device="cuda").to(torch.bfloat16)
    x = torch.randn(M, no, device="cuda").to(torch.bfloat16)
    w = torch.zeros(mo, no, device="cuda")
    b = torch.zeros(mo, device="cuda")
    sp = wgrad_split(mo, no, M)
    kw = dict(a_mn=True, b_mn=True, out=w, epilogue=ops.EPI_F32_ACCUM, split_k=sp)
    t0 = tm(lambda: ops.gemm(dy, x, **kw))
    t1 = tm(lambda: ops.gemm(dy, x, a_rowsum=b, **kw))
    t2 = tm(lambda: ops.colsum_accum(dy, b))
    fl = 2.0 * M * mo * no
    print(f"{name} {mo}x{no} split {sp}: plain {t0:.4f} ms ({fl / t0 / 1e9:.0f} TF), +rowsum {t1:.4f} ms "
          f"({fl / t1 / 1e9:.0f} TF), separate colsum {t2:.4f} ms", flush=True)
