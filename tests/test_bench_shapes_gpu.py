"""Parity at the shapes the benchmark runs (VERDICT r1 "what's weak" 1-2).

* Every GEMM epilogue at M = 100,416 (config 4: 64 clips x 1569 tokens), so each persistent CTA
  (pair) walks 16-64 tiles and the accumulator double-buffer / aux-ring / store-ring phases wrap
  many times -- against a torch fp32 matmul of the same bf16 operands on the GPU.
* The config-5 patch-embed GEMM (K = 1176, not a multiple of the 64-wide k-block).
* One full config-4 transformer layer (B = 2, N = 1569, D = 768, 12 heads) and one config-5 layer
  (N = 2049, D = 1024, 16 heads, hidden 4096), forward and backward, against the fp32 oracle
  (oracle/vit_oracle.py) evaluated on the GPU with the same fp32 master weights.
* The config-4 and config-5 encoders end to end at depth 1 (patch-embed, PE_t + PE_s tokens, head).

Tolerances (north_star): bf16 outputs / gradients within 2e-2 norm-relative of fp32; fp32 GEMM
outputs within 1e-4 (accumulation order only).
"""

import pytest
import torch

from oracle import vit_oracle as VO
from paper_2309_16669_b200 import ops
from paper_2309_16669_b200.vit import FineTuneModel, ParamStore, TransformerStack, VitConfig, wgrad_split

pytestmark = pytest.mark.gpu
M4 = 64 * 1569


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def mk(*shape, seed=0, scale=0.5):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, generator=g, device="cuda") * scale).to(torch.bfloat16)


@pytest.fixture(autouse=True)
def _fp32_reference():
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32 = old
    torch.cuda.empty_cache()


# ----------------------------------------------------------------------------- GEMMs at M = 100,416
@pytest.mark.parametrize("N,K", [(2304, 768), (768, 3072)])
def test_fwd_plain_and_residual_at_bench_M(N, K):
    """qkv fwd (bias) / fc2 fwd (bias + residual aux ring), CTA pairs, many tiles per pair."""
    A, W = mk(M4, K, seed=1), mk(N, K, seed=2, scale=0.05)
    bias = torch.randn(N, device="cuda")
    ref = A.float() @ W.float().t() + bias
    out = ops.gemm(A, W, bias=bias)
    assert rel(out, ref) < 1e-2
    if N == 768:
        res = mk(M4, N, seed=3)
        out = ops.gemm(A, W, bias=bias, aux=res)
        assert rel(out, ref + res.float()) < 1e-2


def test_fc1_bias_gelu_at_bench_M():
    A, W = mk(M4, 768, seed=4), mk(3072, 768, seed=5, scale=0.05)
    bias = torch.randn(3072, device="cuda") * 0.1
    pre = torch.empty(M4, 3072, dtype=torch.bfloat16, device="cuda")
    act = ops.gemm(A, W, bias=bias, epilogue=ops.EPI_BIAS_GELU, aux_out=pre)
    ref = A.float() @ W.float().t() + bias
    assert rel(pre, ref) < 1e-2
    assert rel(act, ref * torch.sigmoid(1.702 * ref)) < 1e-2


def test_proj_residual_k768_at_bench_M():
    A, W = mk(M4, 768, seed=6), mk(768, 768, seed=7, scale=0.05)
    bias = torch.randn(768, device="cuda")
    res = mk(M4, 768, seed=8)
    out = ops.gemm(A, W, bias=bias, aux=res)
    assert rel(out, A.float() @ W.float().t() + bias + res.float()) < 1e-2


def test_fc2_dgrad_dgelu_at_bench_M():
    """dpre = (dY W2) * QuickGELU'(pre): A = dY [M,768] K-major, B = W2 [768,3072] read MN-major."""
    dY, W2 = mk(M4, 768, seed=9), mk(768, 3072, seed=10, scale=0.05)
    pre = mk(M4, 3072, seed=11, scale=2.0)
    out = ops.gemm(dY, W2, b_mn=True, epilogue=ops.EPI_DGELU, aux=pre)
    h = pre.float()
    s = torch.sigmoid(1.702 * h)
    ref = (dY.float() @ W2.float()) * (s + 1.702 * h * s * (1 - s))
    assert rel(out, ref) < 1e-2


@pytest.mark.parametrize("Nout,Kin", [(768, 3072), (2304, 768)])
def test_dgrad_plain_at_bench_M(Nout, Kin):
    """fc1 / qkv dgrad: dX = dY W, W read MN-major."""
    dY, W = mk(M4, Nout, seed=12), mk(Nout, Kin, seed=13, scale=0.05)
    out = ops.gemm(dY, W, b_mn=True)
    assert rel(out, dY.float() @ W.float()) < 1e-2


@pytest.mark.parametrize("Nout,Kin", [(3072, 768), (768, 768)])
def test_wgrad_split_bias_grad_at_bench_M(Nout, Kin):
    """fp32 split-K wgrad over 100,416 tokens with the fused bias gradient, the split the step uses."""
    dY, X = mk(M4, Nout, seed=14), mk(M4, Kin, seed=15)
    acc = torch.zeros(Nout, Kin, device="cuda")
    db = torch.zeros(Nout, device="cuda")
    ops.gemm(dY, X, a_mn=True, b_mn=True, out=acc, epilogue=ops.EPI_F32_ACCUM,
             split_k=wgrad_split(Nout, Kin, M4), a_rowsum=db)
    assert rel(acc, dY.float().t() @ X.float()) < 1e-4
    ref = dY.float().sum(0)
    assert (db - ref).abs().max().item() < 1e-3 * max(1.0, ref.abs().max().item())


def test_patch_embed_k1176_config5():
    """ViT-L/14 patch embed: K = 3*2*14*14 = 1176 (18.4 k-blocks: the TMA zero-fills the tail)."""
    M = 24 * 2048
    A, W = mk(M, 1176, seed=16), mk(1024, 1176, seed=17, scale=0.05)
    bias = torch.randn(1024, device="cuda")
    out = ops.gemm(A, W, bias=bias)
    assert rel(out, A.float() @ W.float().t() + bias) < 1e-2
    dY = mk(M, 1024, seed=18)
    acc = torch.zeros(1024, 1176, device="cuda")
    db = torch.zeros(1024, device="cuda")
    ops.gemm(dY, A, a_mn=True, b_mn=True, out=acc, epilogue=ops.EPI_F32_ACCUM, split_k=wgrad_split(1024, 1176, M),
             a_rowsum=db)
    assert rel(acc, dY.float().t() @ A.float()) < 1e-4


# ----------------------------------------------------------------------------- full layers vs the oracle
def _layer_check(D, heads, B, N, seed):
    store = ParamStore(torch.device("cuda"))
    stack = TransformerStack(D, heads, 1, 4 * D, store, "enc")
    store.allocate(seed)
    g = torch.Generator(device="cuda").manual_seed(seed + 1)
    store.data.add_(torch.randn(store.n, generator=g, device="cuda") * 0.02)   # non-trivial LN / biases
    ops.cast_bf16(store.data, store.shadow)
    x = (torch.randn(B * N, D, generator=g, device="cuda")).to(torch.bfloat16)
    R = torch.randn(B * N, D, generator=g, device="cuda") / (B * N * D) ** 0.5   # loss = <out, R>
    out, saved = stack.forward(x, B, N)
    dx = R.to(torch.bfloat16).contiguous()
    store.grad.zero_()
    dx = stack.backward(dx, saved, B, N)
    torch.cuda.synchronize()

    names = [s[0] for s in store.specs]
    P = {n: store.p(n).detach().clone().requires_grad_(True) for n in names}
    xf = x.float().requires_grad_(True)
    ref = VO.blocks(P, xf, B, N, D, heads, 1, "enc")
    (ref * R).sum().backward()
    assert rel(out, ref) < 2e-2
    assert rel(dx, xf.grad) < 2e-2
    bad = [(n, rel(store.g(n), P[n].grad)) for n in names if rel(store.g(n), P[n].grad) > 2e-2]
    assert not bad, bad


def test_config4_layer_fwd_bwd_vs_oracle():
    _layer_check(768, 12, 2, 1569, seed=20)


def test_config5_layer_fwd_bwd_vs_oracle():
    _layer_check(1024, 16, 1, 2049, seed=21)


@pytest.mark.parametrize("cfg,B", [(VitConfig(frames=16, cube_t=2, depth=1), 2),
                                   (VitConfig(frames=16, cube_t=2, cube_h=14, cube_w=14, depth=1, dim=1024,
                                              heads=16), 1)])
def test_encoder_head_step_vs_oracle(cfg, B):
    """Patch-embed (K = 1536 / 1176) + PE_t + PE_s tokens + one block + head CE, loss and every
    parameter gradient, at the config-4 / config-5 token counts."""
    C = 3806
    model = FineTuneModel(cfg, num_classes=C, seed=3)
    g = torch.Generator(device="cuda").manual_seed(4)
    model.store.data.add_(torch.randn(model.store.n, generator=g, device="cuda") * 0.02)
    ops.cast_bf16(model.store.data, model.store.shadow)
    patches = torch.randn(B * cfg.patches, cfg.patch_dim, generator=g, device="cuda").to(torch.bfloat16)
    labels = torch.randint(0, C, (B,), generator=g, device="cuda", dtype=torch.int32)
    loss = torch.zeros(1, device="cuda")
    model.zero_grad()
    model.forward_backward(patches, labels, B, loss)
    torch.cuda.synchronize()
    names = [s[0] for s in model.store.specs]
    P = {n: model.store.p(n).detach().clone().requires_grad_(True) for n in names}
    x = VO.encoder_forward(P, patches.float(), cfg, B)
    ref_loss, _ = VO.head_loss(P, x, B, cfg.tokens, labels, C)
    ref_loss.backward()
    assert abs(loss.item() - ref_loss.item()) / abs(ref_loss.item()) < 2e-2
    bad = []
    for n in names:
        ref = P[n].grad
        if ref is None or ref.norm() < 1e-12:
            continue
        got = model.store.g(n)
        if n in ("head.w", "head.b"):
            got, ref = got[:C], ref[:C]
        if rel(got, ref) > 2e-2:
            bad.append((n, rel(got, ref)))
    assert not bad, bad
