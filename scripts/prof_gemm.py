"""The three heaviest config-4 GEMM launches of a training step, once each (for ncu captures):
fc1 forward with bias+QuickGELU (two bf16 outputs), fc2 dgrad with dGELU (bf16 aux read), qkv forward."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16669_b200 import ops

M, D = 64 * 1569, 768
x = torch.randn(M, D, device="cuda").to(torch.bfloat16)
w1 = (torch.randn(4 * D, D, device="cuda") * 0.05).to(torch.bfloat16)
wq = (torch.randn(3 * D, D, device="cuda") * 0.05).to(torch.bfloat16)
w2 = (torch.randn(D, 4 * D, device="cuda") * 0.05).to(torch.bfloat16)
b1 = torch.randn(4 * D, device="cuda")
pre = torch.empty(M, 4 * D, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    act = ops.gemm(x, w1, bias=b1, epilogue=ops.EPI_BIAS_GELU, aux_out=pre)
    dpre = ops.gemm(x, w2, b_mn=True, epilogue=ops.EPI_DGELU, aux=pre)
    qkv = ops.gemm(x, wq)
torch.cuda.synchronize()
