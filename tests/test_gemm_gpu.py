"""tcgen05 GEMM parity vs a torch fp32 reference of the same op (bf16 inputs, fp32 accumulate).

Tolerance: norm-relative error <= 1e-2 for bf16 outputs (output rounding ~4e-3), <= 1e-4
for fp32 outputs (accumulation-order only).
"""

import pytest
import torch

from paper_2309_16669_b200 import ops
from paper_2309_16669_b200.errors import InputError

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def mk(*shape, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, generator=g, device="cuda") * 0.5).to(torch.bfloat16)


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (296, 208, 136), (1024, 768, 768), (264, 3072, 768),
                                   (1569, 2304, 768), (128, 128, 1536)])
def test_gemm_layouts(a_mn, b_mn, M, N, K):
    from paper_2309_16669_b200.errors import InputError
    A = mk(K, M, seed=1) if a_mn else mk(M, K, seed=1)
    if (a_mn and M % 8) or (b_mn and N % 8):
        B = mk(K, N, seed=2) if b_mn else mk(N, K, seed=2)
        with pytest.raises(InputError):   # leading dims must be 16-byte multiples (TMA)
            ops.gemm(A, B, a_mn=a_mn, b_mn=b_mn)
        return
    B = mk(K, N, seed=2) if b_mn else mk(N, K, seed=2)
    Af = A.float().t() if a_mn else A.float()
    Bf = B.float() if b_mn else B.float().t()
    ref = Af @ Bf
    out32 = ops.gemm(A, B, a_mn=a_mn, b_mn=b_mn, epilogue=ops.EPI_F32)
    assert rel(out32, ref) < 1e-4
    out16 = ops.gemm(A, B, a_mn=a_mn, b_mn=b_mn)
    assert rel(out16, ref) < 1e-2


# K = 768: aux-reading epilogues on single CTAs; K = 3072: on CTA pairs (the K >= 1536 rule);
# b_mn: the dgrad form (B = W read MN-major), which is how the training step runs dGELU
@pytest.mark.parametrize("K", [768, 3072])
@pytest.mark.parametrize("b_mn", [False, True])
def test_epilogues(K, b_mn):
    M, N = 777, 768
    A = mk(M, K, seed=3)
    Bw = mk(K, N, seed=4) if b_mn else mk(N, K, seed=4)
    Bt = Bw.float() if b_mn else Bw.float().t()   # [K, N]
    bias = torch.randn(N, device="cuda")
    res = mk(M, N, seed=5)
    ref = A.float() @ Bt + bias
    out = ops.gemm(A, Bw, b_mn=b_mn, bias=bias, aux=res)
    assert rel(out, ref + res.float()) < 1e-2
    pre = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    act = ops.gemm(A, Bw, b_mn=b_mn, bias=bias, epilogue=ops.EPI_BIAS_GELU, aux_out=pre)
    assert rel(pre, ref) < 1e-2
    assert rel(act, ref * torch.sigmoid(1.702 * ref)) < 1e-2
    dg = ops.gemm(A, Bw, b_mn=b_mn, epilogue=ops.EPI_DGELU, aux=pre)
    h = pre.float()
    s = torch.sigmoid(1.702 * h)
    assert rel(dg, (A.float() @ Bt) * (s + 1.702 * h * s * (1 - s))) < 1e-2
    half = ops.gemm(A, Bw, b_mn=b_mn, epilogue=ops.EPI_F32, alpha=0.5)
    assert rel(half, 0.5 * (A.float() @ Bt)) < 1e-4


@pytest.mark.parametrize("splits", [1, 4, 13])
def test_wgrad_split_k_accumulate(splits):
    # dW[N_out, K_in] = dY^T X over M tokens: both operands MN-major
    Mtok, Nout, Kin = 100416 // 8, 768, 768
    dY, X = mk(Mtok, Nout, seed=6), mk(Mtok, Kin, seed=7)
    acc = torch.full((Nout, Kin), 1.0, device="cuda")
    ops.gemm(dY, X, a_mn=True, b_mn=True, out=acc, epilogue=ops.EPI_F32_ACCUM, split_k=splits)
    ref = dY.float().t() @ X.float() + 1.0
    assert rel(acc, ref) < 1e-4


def test_odd_n_unaligned_head():
    # classifier head N=3806 -> scalar epilogue path
    M, N, K = 200, 3806, 768
    A, B = mk(M, K, seed=8), mk(N, K, seed=9)
    out = torch.empty(M, 3808, dtype=torch.float32, device="cuda")[:, :N]
    ops.gemm(A, B, out=out, epilogue=ops.EPI_F32)
    assert rel(out, A.float() @ B.float().t()) < 1e-4


@pytest.mark.parametrize("Mtok,Nout,Kin,splits", [(100416 // 8, 768, 3072, 2), (12552, 3072, 768, 2),
                                                  (1000, 200, 136, 1), (777, 2304, 768, 5), (64, 3808, 768, 1),
                                                  (256, 512, 3072, 2)])   # more n-tiles than K blocks per split
def test_wgrad_rowsum_bias_grad(Mtok, Nout, Kin, splits):
    # fused bias gradient: a_rowsum[n] += sum_tokens dY[token, n] alongside dW = dY^T X
    dY, X = mk(Mtok, Nout, seed=16), mk(Mtok, Kin, seed=17)
    acc = torch.zeros((Nout, Kin), device="cuda")
    db = torch.full((Nout,), 0.5, device="cuda")
    ops.gemm(dY, X, a_mn=True, b_mn=True, out=acc, epilogue=ops.EPI_F32_ACCUM, split_k=splits, a_rowsum=db)
    assert rel(acc, dY.float().t() @ X.float()) < 1e-4
    ref = dY.float().sum(0) + 0.5
    assert (db - ref).abs().max().item() < 1e-3 * max(1.0, ref.abs().max().item())
    # a second call accumulates
    ops.gemm(dY, X, a_mn=True, b_mn=True, out=acc, epilogue=ops.EPI_F32_ACCUM, split_k=splits, a_rowsum=db)
    assert (db - (2 * dY.float().sum(0) + 0.5)).abs().max().item() < 2e-3 * max(1.0, ref.abs().max().item())


def test_rowsum_k_major_and_rejects_bf16_epilogue():
    A, B = mk(300, 520, seed=18), mk(256, 520, seed=19)
    rs = torch.zeros(300, device="cuda")
    out = ops.gemm(A, B, epilogue=ops.EPI_F32, a_rowsum=rs)
    assert rel(out, A.float() @ B.float().t()) < 1e-4
    assert (rs - A.float().sum(1)).abs().max().item() < 1e-3 * max(1.0, A.float().sum(1).abs().max().item())
    with pytest.raises(InputError):
        ops.gemm(A, B, a_rowsum=rs)
