"""Space-time ViT video encoder (tubelet patch-embed + pre-LN blocks) on the sm_100a kernels.

Shape contract: `VitConfig` keeps the reference's field names and token rule
(`pkg/src/vidpipe/models.py:34-74`): N = (frames/cube_t)(height/cube_h)(width/cube_w)
+ extra_tokens.  The architecture itself is absent from the reference and is
restated from PAPER.md: non-overlapping t x h x w cubes linearly projected to D
with the separable position embedding PE[i] = PE_t[i] + PE_s (:258-259, :727-729;
PE_s is CLIP's spatial table incl. its cls slot, PE_t one row per temporal token
index, linearly interpolated when T changes -- `interpolate_temporal_pe`), a cls
token (extra_tokens = 1), L pre-LN blocks x += Proj(MHA(LN x)); x += FC2(act(FC1(LN x)))
with CLIP's QuickGELU (:259-260, :727), blockwise attention (:265-272).

Execution model (B200-first):
  * all parameters live in ONE flat fp32 master buffer laid out layer by layer, with a
    flat fp32 gradient buffer, AdamW moments and a bf16 shadow the GEMMs read -- so the
    optimizer is one fused kernel and the DP all-reduce works on contiguous per-layer
    slices that become final as the backward walks down the stack;
  * forward/backward are explicit kernel sequences (no autograd graph in the hot loop);
    weight gradients accumulate straight into the fp32 buffer with split-K tcgen05 wgrad
    GEMMs (red.global.add), bias gradients via column sums;
  * activations saved for backward follow the flash contract of models.py:137-140:
    O + per-row LSE for attention, never an N x N tensor.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from . import ops
from .errors import ConfigurationError


@dataclass(frozen=True)
class VitConfig:
    """Field names/defaults and validation as reference `VitConfig` (models.py:34-74)."""

    frames: int = 4
    height: int = 224
    width: int = 224
    cube_t: int = 1
    cube_h: int = 16
    cube_w: int = 16
    depth: int = 12
    dim: int = 768
    heads: int = 12
    bytes_per_elem: int = 2
    mlp_ratio: float = 4.0
    extra_tokens: int = 1

    def validate(self) -> None:
        for name in ("frames", "height", "width", "cube_t", "cube_h", "cube_w", "depth", "dim", "heads",
                     "bytes_per_elem"):
            if getattr(self, name) < 1:
                raise ConfigurationError(f"{name} must be >= 1")
        if self.frames % self.cube_t or self.height % self.cube_h or self.width % self.cube_w:
            raise ConfigurationError(
                f"input {self.frames}x{self.height}x{self.width} not divisible by cube "
                f"{self.cube_t}x{self.cube_h}x{self.cube_w}")
        if self.mlp_ratio <= 0:
            raise ConfigurationError("mlp_ratio must be > 0")
        if self.extra_tokens < 0:
            raise ConfigurationError("extra_tokens must be >= 0")
        # B200 kernel envelope
        if self.dim != self.heads * 64:
            raise ConfigurationError("head_dim must be 64 (dim == 64 * heads)")
        if self.extra_tokens != 1:
            raise ConfigurationError("the encoder uses exactly one cls token (extra_tokens=1)")
        if self.cube_w % 2:
            raise ConfigurationError("cube_w must be even (tubelet writes bf16 pairs)")

    @property
    def tokens(self) -> int:
        return (self.frames // self.cube_t) * (self.height // self.cube_h) * (self.width // self.cube_w) \
            + self.extra_tokens

    @property
    def patches(self) -> int:
        return self.tokens - self.extra_tokens

    @property
    def spatial_tokens(self) -> int:
        return (self.height // self.cube_h) * (self.width // self.cube_w)

    @property
    def temporal_tokens(self) -> int:
        return self.frames // self.cube_t

    @property
    def patch_dim(self) -> int:
        return 3 * self.cube_t * self.cube_h * self.cube_w

    @property
    def hidden(self) -> int:
        return int(self.dim * self.mlp_ratio)

    def forward_flops_per_clip(self) -> float:
        """GEMM 2MNK + attention 4 N^2 d per head (BASELINE.md 3 conventions)."""
        N, D, L = self.tokens, self.dim, self.depth
        pe = 2.0 * self.patches * self.patch_dim * D
        per_layer = 2.0 * N * D * (3 * D + D + 2 * self.hidden) + 4.0 * N * N * D
        return pe + L * per_layer

    def attention_forward_flops_per_clip(self) -> float:
        return self.depth * 4.0 * self.tokens ** 2 * self.dim


# BASELINE.json configs
CONFIG1_TINY = VitConfig(frames=4, height=112, width=112, depth=4, dim=192, heads=3)
CONFIG3_VIT_B = VitConfig()                                   # 4x224^2, 1x16x16, N=785
CONFIG4_VIT_B_16F = VitConfig(frames=16, cube_t=2)            # 16x224^2, 2x16x16, N=1569
CONFIG5_VIT_L_16F = VitConfig(frames=16, cube_t=2, cube_h=14, cube_w=14, depth=24, dim=1024, heads=16)


# ----------------------------------------------------------------------------- parameters
@dataclass
class ParamStore:
    """One flat fp32 master buffer (+grad, AdamW moments, bf16 shadow, decay mask)."""

    device: torch.device
    specs: list = field(default_factory=list)     # (name, shape, decay, init, group)
    offsets: dict = field(default_factory=dict)
    groups: dict = field(default_factory=dict)    # group -> (start, end)
    n: int = 0

    ALIGN = 64  # elements; keeps every view 128-byte aligned for TMA / vector loads

    def add(self, name, shape, decay: bool, init: str, group: str):
        self.specs.append((name, tuple(shape), decay, init, group))

    def allocate(self, seed: int = 0):
        off = 0
        for name, shape, decay, init, group in self.specs:
            numel = math.prod(shape)
            self.offsets[name] = (off, shape)
            g0, g1 = self.groups.get(group, (off, off))
            self.groups[group] = (min(g0, off), off + numel)
            off += (numel + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        self.n = off
        dev = self.device
        self.data = torch.zeros(off, dtype=torch.float32, device=dev)
        self.grad = torch.zeros(off, dtype=torch.float32, device=dev)
        self.m = torch.zeros(off, dtype=torch.float32, device=dev)
        self.v = torch.zeros(off, dtype=torch.float32, device=dev)
        self.shadow = torch.zeros(off, dtype=torch.bfloat16, device=dev)
        mask = torch.zeros(off, dtype=torch.uint8)
        gen = torch.Generator().manual_seed(seed)
        host = torch.zeros(off, dtype=torch.float32)
        for name, shape, decay, init, group in self.specs:
            o, _ = self.offsets[name]
            numel = math.prod(shape)
            if init == "normal":
                t = torch.empty(numel)
                torch.nn.init.trunc_normal_(t, std=0.02, a=-0.04, b=0.04, generator=gen)
                host[o:o + numel] = t
            elif init == "ones":
                host[o:o + numel] = 1.0
            if decay:
                mask[o:o + numel] = 1
        self.data.copy_(host)
        self.decay_mask = mask.to(dev)
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=dev)   # AdamW step count (device side)
        ops.cast_bf16(self.data, self.shadow)

    def p(self, name):
        o, shape = self.offsets[name]
        return self.data[o:o + math.prod(shape)].view(shape)

    def g(self, name):
        o, shape = self.offsets[name]
        return self.grad[o:o + math.prod(shape)].view(shape)

    def w(self, name):
        o, shape = self.offsets[name]
        return self.shadow[o:o + math.prod(shape)].view(shape)

    def group_slice(self, group):
        a, b = self.groups[group]
        return a, (b + self.ALIGN - 1) // self.ALIGN * self.ALIGN


def wgrad_split(m_out: int, n_out: int, k_tokens: int | None = None, sms: int = 148) -> int:
    """Split-K factor for a wgrad over k_tokens: minimise waves x (k-blocks per item + epilogue).

    The fused bias-gradient mode runs a single-buffered accumulator, so every extra work item
    per CTA pays its fp32 reduce epilogue (~35 k-block equivalents) un-overlapped.
    """
    if ops.are_deterministic_algorithms_enabled():
        return 1   # one fp32 add per gradient element: bit-reproducible
    if n_out > 128 and m_out > 128:   # CTA-pair GEMM: 256 x 256 tiles, one worker per SM pair
        tiles, sms = ((m_out + 255) // 256) * ((n_out + 255) // 256), sms // 2
    else:
        tiles = ((m_out + 127) // 128) * ((n_out + 255) // 256 if n_out > 128 else 1)
    if k_tokens is None:
        return max(1, sms // tiles)
    kb = (k_tokens + 63) // 64
    best, best_cost = 1, None
    for s in range(1, 17):
        if s > kb:
            break
        waves = -(-tiles * s // sms)
        cost = waves * (-(-kb // s) + 35)
        if best_cost is None or cost < best_cost:
            best, best_cost = s, cost
    return best


# ----------------------------------------------------------------------------- blocks
class TransformerStack:
    """L pre-LN blocks over a residual stream [B*N, D] bf16.

    Shared by the video encoder (bidirectional) and the text encoder (causal).
    """

    def __init__(self, dim: int, heads: int, depth: int, hidden: int, store: ParamStore, prefix: str,
                 causal: bool = False):
        if dim != 64 * heads:
            raise ConfigurationError("head_dim must be 64")
        self.D, self.H, self.L, self.Hd = dim, heads, depth, hidden
        self.s, self.pre, self.causal = store, prefix, causal
        D, Hd = dim, hidden
        for l in range(depth):
            g = f"{prefix}.blk{l}"
            store.add(f"{g}.ln1.g", (D,), False, "ones", g)
            store.add(f"{g}.ln1.b", (D,), False, "zeros", g)
            store.add(f"{g}.qkv.w", (3 * D, D), True, "normal", g)
            store.add(f"{g}.qkv.b", (3 * D,), False, "zeros", g)
            store.add(f"{g}.proj.w", (D, D), True, "normal", g)
            store.add(f"{g}.proj.b", (D,), False, "zeros", g)
            store.add(f"{g}.ln2.g", (D,), False, "ones", g)
            store.add(f"{g}.ln2.b", (D,), False, "zeros", g)
            store.add(f"{g}.fc1.w", (Hd, D), True, "normal", g)
            store.add(f"{g}.fc1.b", (Hd,), False, "zeros", g)
            store.add(f"{g}.fc2.w", (D, Hd), True, "normal", g)
            store.add(f"{g}.fc2.b", (D,), False, "zeros", g)

    def forward(self, x: torch.Tensor, B: int, N: int, save: bool = True):
        s, P, D, H = self.s, self.pre, self.D, self.H
        M = B * N
        dev = x.device
        saved = []
        for l in range(self.L):
            g = f"{P}.blk{l}"
            h1, mu1, rs1 = ops.layernorm_fwd(x, s.p(f"{g}.ln1.g"), s.p(f"{g}.ln1.b"))
            qkv = ops.gemm(h1, s.w(f"{g}.qkv.w"), bias=s.p(f"{g}.qkv.b"))
            q3 = qkv.view(B, N, 3 * D)
            o, lse = ops.attn_fwd(q3[:, :, :D], q3[:, :, D:2 * D], q3[:, :, 2 * D:], H, causal=self.causal)
            o2 = o.view(M, D)
            x2 = ops.gemm(o2, s.w(f"{g}.proj.w"), bias=s.p(f"{g}.proj.b"), aux=x)
            h2, mu2, rs2 = ops.layernorm_fwd(x2, s.p(f"{g}.ln2.g"), s.p(f"{g}.ln2.b"))
            pre = torch.empty((M, self.Hd), dtype=torch.bfloat16, device=dev)
            a = ops.gemm(h2, s.w(f"{g}.fc1.w"), bias=s.p(f"{g}.fc1.b"), epilogue=ops.EPI_BIAS_GELU, aux_out=pre)
            x3 = ops.gemm(a, s.w(f"{g}.fc2.w"), bias=s.p(f"{g}.fc2.b"), aux=x2)
            if save:
                saved.append((x, h1, mu1, rs1, qkv, o2, lse, x2, h2, mu2, rs2, pre, a))
            x = x3
        return x, saved

    def backward(self, dx: torch.Tensor, saved: list, B: int, N: int, on_layer_done=None):
        """dx: grad of the stack output [B*N, D] bf16; consumed in place, returns grad of the input."""
        s, P, D, H, Hd = self.s, self.pre, self.D, self.H, self.Hd
        M = B * N
        dev = dx.device
        for l in reversed(range(self.L)):
            g = f"{P}.blk{l}"
            x, h1, mu1, rs1, qkv, o2, lse, x2, h2, mu2, rs2, pre, a = saved[l]
            # fc2: x3 = x2 + a W2^T + b2.  Bias gradients that are column sums of the residual-stream
            # gradient dx come out of the LayerNorm backward that produced dx (fixed-order, nearly free
            # there; as an extra N=16 MMA per K step they cost the wgrad GEMM 12-16 %): fc2.b of block l
            # from block l+1's ln1 backward, proj.b from this block's ln2 backward.  Only the top
            # block's fc2.b (dx from the caller) uses the GEMM row sums.
            ops.gemm(dx, a, a_mn=True, b_mn=True, out=s.g(f"{g}.fc2.w"), epilogue=ops.EPI_F32_ACCUM,
                     split_k=wgrad_split(D, Hd, M), a_rowsum=s.g(f"{g}.fc2.b") if l == self.L - 1 else None)
            dpre = ops.gemm(dx, s.w(f"{g}.fc2.w"), b_mn=True, epilogue=ops.EPI_DGELU, aux=pre)
            # fc1: pre = h2 W1^T + b1
            ops.gemm(dpre, h2, a_mn=True, b_mn=True, out=s.g(f"{g}.fc1.w"), epilogue=ops.EPI_F32_ACCUM,
                     split_k=wgrad_split(Hd, D, M), a_rowsum=s.g(f"{g}.fc1.b"))
            dh2 = ops.gemm(dpre, s.w(f"{g}.fc1.w"), b_mn=True)
            del dpre
            ops.layernorm_bwd(dh2, x2, s.p(f"{g}.ln2.g"), mu2, rs2, dx, s.g(f"{g}.ln2.g"), s.g(f"{g}.ln2.b"),
                              accumulate=True, dx_colsum=s.g(f"{g}.proj.b"))
            del dh2
            # proj: x2 = x + o Wo^T + bo (bias gradient: the column sums above)
            ops.gemm(dx, o2, a_mn=True, b_mn=True, out=s.g(f"{g}.proj.w"), epilogue=ops.EPI_F32_ACCUM,
                     split_k=wgrad_split(D, D, M))
            do = ops.gemm(dx, s.w(f"{g}.proj.w"), b_mn=True)
            q3 = qkv.view(B, N, 3 * D)
            dqkv = torch.empty((M, 3 * D), dtype=torch.bfloat16, device=dev)
            d3 = dqkv.view(B, N, 3 * D)
            ops.attn_bwd(q3[:, :, :D], q3[:, :, D:2 * D], q3[:, :, 2 * D:], o2.view(B, N, D), do.view(B, N, D), lse,
                         H, causal=self.causal, dq=d3[:, :, :D], dk=d3[:, :, D:2 * D], dv=d3[:, :, 2 * D:])
            del do
            ops.gemm(dqkv, h1, a_mn=True, b_mn=True, out=s.g(f"{g}.qkv.w"), epilogue=ops.EPI_F32_ACCUM,
                     split_k=wgrad_split(3 * D, D, M), a_rowsum=s.g(f"{g}.qkv.b"))
            dh1 = ops.gemm(dqkv, s.w(f"{g}.qkv.w"), b_mn=True)
            del dqkv
            ops.layernorm_bwd(dh1, x, s.p(f"{g}.ln1.g"), mu1, rs1, dx, s.g(f"{g}.ln1.g"), s.g(f"{g}.ln1.b"),
                              accumulate=True, dx_colsum=s.g(f"{P}.blk{l - 1}.fc2.b") if l > 0 else None)
            del dh1
            saved[l] = None
            if on_layer_done is not None:
                on_layer_done(g)
        return dx


# ----------------------------------------------------------------------------- encoders
class VideoEncoder:
    """ViT video encoder over tubelet-patch rows (the K1 "tubelet" layout).

    forward(patches [B*Np, 3*t*h*w] bf16) -> final residual stream [B*N, D] bf16
    backward(dx) accumulates every parameter gradient into `store.grad`.
    """

    def __init__(self, cfg: VitConfig, store: ParamStore, prefix: str = "enc"):
        cfg.validate()
        self.cfg = cfg
        self.s = store
        self.pre = prefix
        D, F = cfg.dim, cfg.patch_dim
        s, P = store, prefix
        s.add(f"{P}.pe.w", (D, F), True, "normal", f"{P}.embed")
        s.add(f"{P}.pe.b", (D,), False, "zeros", f"{P}.embed")
        s.add(f"{P}.cls", (D,), False, "normal", f"{P}.embed")
        s.add(f"{P}.pos_s", (1 + cfg.spatial_tokens, D), False, "normal", f"{P}.embed")   # PE_s (+ cls slot)
        s.add(f"{P}.pos_t", (cfg.temporal_tokens, D), False, "normal", f"{P}.embed")      # PE_t
        self.stack = TransformerStack(D, cfg.heads, cfg.depth, cfg.hidden, store, P)

    def forward(self, patches: torch.Tensor, B: int, save: bool = True):
        cfg, s, P = self.cfg, self.s, self.pre
        N, Np, D = cfg.tokens, cfg.patches, cfg.dim
        pe = ops.gemm(patches, s.w(f"{P}.pe.w"), bias=s.p(f"{P}.pe.b"))
        x = torch.empty((B * N, D), dtype=torch.bfloat16, device=patches.device)
        ops.tokens_fwd(pe, s.p(f"{P}.cls"), s.p(f"{P}.pos_s"), s.p(f"{P}.pos_t"), B, Np, x)
        del pe
        x, saved = self.stack.forward(x, B, N, save)
        return x, {"patches": patches, "B": B, "saved": saved}

    def backward(self, dx: torch.Tensor, ctx: dict, on_layer_done=None):
        """dx: grad of the final residual stream [B*N, D] bf16 (consumed in place)."""
        cfg, s, P = self.cfg, self.s, self.pre
        B = ctx["B"]
        N, Np, D = cfg.tokens, cfg.patches, cfg.dim
        dx = self.stack.backward(dx, ctx["saved"], B, N, on_layer_done)
        dpe = torch.empty((B * Np, D), dtype=torch.bfloat16, device=dx.device)
        ops.tokens_bwd(dx, dpe, s.g(f"{P}.cls"), s.g(f"{P}.pos_s"), s.g(f"{P}.pos_t"), B, Np, cfg.spatial_tokens)
        ops.gemm(dpe, ctx["patches"], a_mn=True, b_mn=True, out=s.g(f"{P}.pe.w"), epilogue=ops.EPI_F32_ACCUM,
                 split_k=wgrad_split(D, cfg.patch_dim, B * Np), a_rowsum=s.g(f"{P}.pe.b"))
        if on_layer_done is not None:
            on_layer_done(f"{P}.embed")


def interpolate_temporal_pe(pe_t, new_t: int):
    """PE_t [T0, D] -> [new_t, D] by linear interpolation along time (T grows from 4 to 16
    when fine-tuning).  Half-pixel-centre sampling (align_corners=False), i.e. the source coordinate of
    row i is (i + 0.5) * T0 / new_t - 0.5, clamped to [0, T0 - 1].  A load-time parameter transform on
    the host (numpy float64), not a training-step op."""
    import numpy as np

    src = np.asarray(pe_t.detach().cpu() if isinstance(pe_t, torch.Tensor) else pe_t, dtype=np.float64)
    T0 = src.shape[0]
    x = np.clip((np.arange(new_t) + 0.5) * T0 / new_t - 0.5, 0.0, T0 - 1)
    i0 = np.floor(x).astype(np.int64)
    i1 = np.minimum(i0 + 1, T0 - 1)
    w = (x - i0)[:, None]
    out = src[i0] * (1.0 - w) + src[i1] * w
    return torch.from_numpy(out.astype(np.float32))


@dataclass(frozen=True)
class TextConfig:
    """CLIP text tower (12-layer GPT-like, <= 77 BPE tokens; width 512 assumed)."""

    vocab: int = 49408
    context: int = 77
    dim: int = 512
    heads: int = 8
    depth: int = 12
    mlp_ratio: float = 4.0

    @property
    def hidden(self) -> int:
        return int(self.dim * self.mlp_ratio)


class TextEncoder:
    """Token embedding + causal transformer stack; pooled at the EOT position per caption."""

    def __init__(self, cfg: TextConfig, store: ParamStore, prefix: str = "txt"):
        self.cfg, self.s, self.pre = cfg, store, prefix
        store.add(f"{prefix}.tok", (cfg.vocab, cfg.dim), False, "normal", f"{prefix}.embed")
        store.add(f"{prefix}.pos", (cfg.context, cfg.dim), False, "normal", f"{prefix}.embed")
        self.stack = TransformerStack(cfg.dim, cfg.heads, cfg.depth, cfg.hidden, store, prefix, causal=True)

    def forward(self, tokens: torch.Tensor, save: bool = True):
        B, L = tokens.shape
        s, P = self.s, self.pre
        x = torch.empty((B * L, self.cfg.dim), dtype=torch.bfloat16, device=tokens.device)
        ops.embed_fwd(tokens, s.p(f"{P}.tok"), s.p(f"{P}.pos"), x)
        x, saved = self.stack.forward(x, B, L, save)
        return x, {"tokens": tokens, "B": B, "saved": saved}

    def backward(self, dx: torch.Tensor, ctx: dict, on_layer_done=None):
        s, P = self.s, self.pre
        B, L = ctx["tokens"].shape
        dx = self.stack.backward(dx, ctx["saved"], B, L, on_layer_done)
        ops.embed_bwd(ctx["tokens"], dx, s.g(f"{P}.tok"), s.g(f"{P}.pos"))
        if on_layer_done is not None:
            on_layer_done(f"{P}.embed")


class ClassifierHead:
    """Fine-tune head (config 4): LayerNorm on the cls token -> Linear(D, C) -> softmax CE."""

    def __init__(self, dim: int, num_classes: int, store: ParamStore, prefix: str = "head"):
        self.D, self.C = dim, num_classes
        self.Cp = (num_classes + 7) // 8 * 8  # 16-byte aligned rows
        self.s, self.pre = store, prefix
        store.add(f"{prefix}.ln.g", (dim,), False, "ones", prefix)
        store.add(f"{prefix}.ln.b", (dim,), False, "zeros", prefix)
        store.add(f"{prefix}.w", (self.Cp, dim), True, "normal", prefix)
        store.add(f"{prefix}.b", (self.Cp,), False, "zeros", prefix)

    def forward_backward(self, x: torch.Tensor, B: int, N: int, labels: torch.Tensor, loss: torch.Tensor,
                         loss_scale: float):
        """x: final residual [B*N, D]; returns dx (zeros except cls rows); loss += mean CE."""
        s, P, D = self.s, self.pre, self.D
        dev = x.device
        cls = x.view(B, N, D)[:, 0]                       # strided [B, D] view (ld = N*D)
        z, mu, rs = ops.layernorm_fwd(cls, s.p(f"{P}.ln.g"), s.p(f"{P}.ln.b"),
                                      out=torch.empty((B, D), dtype=torch.bfloat16, device=dev))
        logits = ops.gemm(z, s.w(f"{P}.w"), epilogue=ops.EPI_F32, bias=s.p(f"{P}.b"))
        dlogits = torch.zeros((B, self.Cp), dtype=torch.bfloat16, device=dev)
        ops.xent(logits[:, :self.C], labels, loss_scale, loss, dlogits)
        ops.gemm(dlogits, z, a_mn=True, b_mn=True, out=s.g(f"{P}.w"), epilogue=ops.EPI_F32_ACCUM,
                 a_rowsum=s.g(f"{P}.b"))
        dz = ops.gemm(dlogits, s.w(f"{P}.w"), b_mn=True)
        dx = torch.zeros((B * N, D), dtype=torch.bfloat16, device=dev)
        ops.layernorm_bwd(dz, cls, s.p(f"{P}.ln.g"), mu, rs, dx.view(B, N, D)[:, 0], s.g(f"{P}.ln.g"),
                          s.g(f"{P}.ln.b"), accumulate=False)
        return dx, logits


@dataclass
class AdamWConfig:
    """beta (0.9, 0.999), weight decay 0.01, lr 3e-5."""

    lr: float = 3e-5
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01


class FineTuneModel:
    """Config-4 training step: K1 -> encoder -> cls head CE -> (DP all-reduce) -> AdamW."""

    def __init__(self, cfg: VitConfig, num_classes: int = 3806, device="cuda", seed: int = 0,
                 opt: AdamWConfig | None = None):
        self.cfg = cfg
        self.device = torch.device(device)
        self.store = ParamStore(self.device)
        self.encoder = VideoEncoder(cfg, self.store)
        self.head = ClassifierHead(cfg.dim, num_classes, self.store)
        self.store.allocate(seed)
        self.opt = opt or AdamWConfig()
        self.step_num = 0

    def patches_from_clips(self, frames, boxes, flips, out=None, boxes_host=None):
        from . import transform as TR

        cfg = self.cfg
        return TR.transform(frames, boxes, flips, (cfg.height, cfg.width), out=out, layout="tubelet",
                            tubelet=(cfg.cube_t, cfg.cube_h, cfg.cube_w), validate=False, crops_host=boxes_host)

    def forward_backward(self, patches: torch.Tensor, labels: torch.Tensor, B: int, loss: torch.Tensor,
                         loss_scale: float | None = None, on_layer_done=None):
        cfg = self.cfg
        x, ctx = self.encoder.forward(patches, B)
        dx, _ = self.head.forward_backward(x, B, cfg.tokens, labels, loss, loss_scale or 1.0 / B)
        if on_layer_done is not None:
            on_layer_done("head")
        del x
        self.encoder.backward(dx, ctx, on_layer_done)

    def optimizer_step(self, grad_scale: float = 1.0):
        """Fused AdamW (K8); the step count lives on the device (graph-capturable), `step_num` mirrors it."""
        self.step_num += 1
        s, o = self.store, self.opt
        ops.adamw_dev(s.data, s.grad, s.m, s.v, s.shadow, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay, s.step_dev,
                      grad_scale, s.decay_mask)

    def zero_grad(self):
        self.store.grad.zero_()

    def capture_train_step(self, patches: torch.Tensor, labels: torch.Tensor, B: int, loss: torch.Tensor,
                           grad_scale: float = 1.0, warmup: int = 3):
        """The whole model step -- zero grads, forward, head + CE, backward, fused AdamW -- captured into one
        CUDA graph over the static buffers `patches` / `labels` / `loss` (K1 writes the next clips into
        `patches` in place).  Replaying it launches the same ~250 kernels with no host work per launch.
        `warmup` eager steps run first (on a side stream, as graph capture requires) and do train.
        Single-process only: the DP gradient all-reduce is not captured."""
        def body():
            self.zero_grad()
            loss.zero_()
            self.forward_backward(patches, labels, B, loss)
            self.optimizer_step(grad_scale)
        return CapturedStep(body, warmup)


class CapturedStep:
    """A training-step callable captured into one CUDA graph and replayed on the current stream."""

    def __init__(self, fn, warmup: int = 3):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()

    def __call__(self):
        self.graph.replay()
