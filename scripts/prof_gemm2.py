import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_16669_b200 import ops
M, D = 64 * 1569, 768
x = torch.randn(M, D, device="cuda").to(torch.bfloat16)
wq = torch.randn(3 * D, D, device="cuda").to(torch.bfloat16)
q = torch.empty(M, 3 * D, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    ops.gemm(x, wq, out=q)
torch.cuda.synchronize()
