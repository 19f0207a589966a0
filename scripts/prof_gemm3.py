import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_16669_b200 import ops
M, D = 64 * 1569, 768
dy = torch.randn(M, D, device="cuda").to(torch.bfloat16)
w2 = torch.randn(D, 4 * D, device="cuda").to(torch.bfloat16)   # fc2.w [out=D, in=4D]
pre = torch.randn(M, 4 * D, device="cuda").to(torch.bfloat16)
out = torch.empty(M, 4 * D, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    ops.gemm(dy, w2, b_mn=True, out=out, epilogue=ops.EPI_DGELU, aux=pre)
torch.cuda.synchronize()
