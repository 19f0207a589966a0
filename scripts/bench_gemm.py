"""Time the tcgen05 GEMM on the ViT-B/16 (config 4) shapes vs cuBLAS (torch.matmul) for context."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_16669_b200 import ops

M = 64 * 1569
D = 768
shapes = [  # name, M, N, K, a_mn, b_mn, epi
    ("qkv_fwd", M, 3 * D, D, False, False, ops.EPI_BF16),
    ("proj_fwd", M, D, D, False, False, ops.EPI_BF16),
    ("fc1_fwd", M, 4 * D, D, False, False, ops.EPI_BF16),
    ("fc1_fwd_gelu", M, 4 * D, D, False, False, ops.EPI_BIAS_GELU),
    ("fc2_dgrad_dgelu", M, 4 * D, D, False, True, ops.EPI_DGELU),
    ("fc2_fwd", M, D, 4 * D, False, False, ops.EPI_BF16),
    ("fc2_fwd_res", M, D, 4 * D, False, False, ops.EPI_BF16),
    ("proj_fwd_res", M, D, D, False, False, ops.EPI_BF16),
    ("fc1_dgrad", M, D, 4 * D, False, True, ops.EPI_BF16),
    ("fc2_dgrad", M, 4 * D, D, False, True, ops.EPI_BF16),
    ("fc1_wgrad", 4 * D, D, M, True, True, ops.EPI_F32_ACCUM),
    ("qkv_wgrad", 3 * D, D, M, True, True, ops.EPI_F32_ACCUM),
    ("proj_wgrad", D, D, M, True, True, ops.EPI_F32_ACCUM),
    ("sq8192", 8192, 8192, 8192, False, False, ops.EPI_BF16),
]
res = []
for name, m, n, k, amn, bmn, epi in shapes:
    A = torch.randn((k, m) if amn else (m, k), device="cuda").to(torch.bfloat16)
    B = torch.randn((k, n) if bmn else (n, k), device="cuda").to(torch.bfloat16)
    out = torch.zeros((m, n), device="cuda", dtype=torch.float32 if epi == ops.EPI_F32_ACCUM else torch.bfloat16)
    split = 1
    if epi == ops.EPI_F32_ACCUM:
        from paper_2309_16669_b200.vit import wgrad_split
        split = wgrad_split(m, n, k)
    kw = {}
    if epi == ops.EPI_BIAS_GELU:
        kw = dict(bias=torch.randn(n, device="cuda"), aux_out=torch.empty((m, n), device="cuda", dtype=torch.bfloat16))
    if epi == ops.EPI_DGELU:
        kw = dict(aux=torch.randn((m, n), device="cuda").to(torch.bfloat16))
    if name.endswith("_res"):   # bias + residual add (the training step's proj / fc2 forward)
        kw = dict(bias=torch.randn(n, device="cuda"), aux=torch.randn((m, n), device="cuda").to(torch.bfloat16))
    f = lambda: ops.gemm(A, B, a_mn=amn, b_mn=bmn, out=out, epilogue=epi, split_k=split, **kw)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    Af = A.t() if amn else A
    Bf = B if bmn else B.t()
    g = lambda: torch.matmul(Af, Bf)
    for _ in range(3): g()
    e0.record()
    for _ in range(it): g()
    e1.record(); torch.cuda.synchronize()
    ms_cublas = e0.elapsed_time(e1) / it
    fl = 2.0 * m * n * k
    r = {"name": name, "M": m, "N": n, "K": k, "ms": ms, "tflops": fl / ms / 1e9, "cublas_tflops": fl / ms_cublas / 1e9, "split": split}
    print(json.dumps(r), flush=True)
