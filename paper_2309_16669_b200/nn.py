"""PyTorch-facing boundary: autograd Functions and nn.Modules over the sm_100a kernels.

The reference's training call site is `train_step(batch.frames)` (`pkg/README.md:159-161`) with the
shape contract of `VitConfig` (`pkg/src/vidpipe/models.py:34-74`); the paper's loss is the CLIP
InfoNCE (`PAPER.md:291`, `:1196`).  This module gives a PyTorch training loop the three calls it needs:

  * `VideoEncoder(cfg)` -- an `nn.Module` that owns its flat fp32 `ParamStore` (one `nn.Parameter`
    aliasing the master buffer) and whose `forward(x)` accepts normalised clips `[B,3,T,H,W]` or K1's
    tubelet patch rows; its backward is the explicit kernel sequence of `vit.VideoEncoder.backward`
    (tcgen05 dgrad/wgrad GEMMs, K5 attention backward, LayerNorm backward), wrapped in one
    `torch.autograd.Function`, so it composes with any loss and optimizer;
  * `attention(q, k, v, heads, causal=False)` -- K4/K5 as an autograd Function;
  * `clip_loss(v, t, logit_scale)` -- the fused InfoNCE kernel (K7) as an autograd Function, with the
    data-parallel form (embedding all_gather, local-row gradients) when a process group is active;
  * `transform(...)` -- re-exported K1 (uint8 input: no gradient flows into decoded pixels).

Nothing here computes in PyTorch except gradient plumbing (zero-initialised buffers, the upstream
scalar applied to the InfoNCE gradients); every op is a libavion_b200 kernel.
"""

from __future__ import annotations

import torch

from . import dp, ops
from .errors import InputError
from .transform import transform  # noqa: F401  (re-export: the K1 drop-in)
from .vit import AdamWConfig, ParamStore, VitConfig
from .vit import VideoEncoder as _Engine


# ----------------------------------------------------------------------------- attention
class _AttentionFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, heads: int, causal: bool, scale):
        o, lse = ops.attn_fwd(q, k, v, heads, causal=causal, scale=scale)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.heads, ctx.causal, ctx.scale = heads, causal, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        do = do.to(torch.bfloat16)
        if do.stride() != o.stride():
            do = do.contiguous() if o.is_contiguous() else do.clone(memory_format=torch.contiguous_format)
        if do.stride() != o.stride():
            raise InputError("attention backward: upstream gradient layout differs from the output's")
        dq, dk, dv = ops.attn_bwd(q, k, v, o, do, lse, ctx.heads, causal=ctx.causal, scale=ctx.scale)
        return dq, dk, dv, None, None, None


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, heads: int, causal: bool = False,
              scale: float | None = None) -> torch.Tensor:
    """softmax(q k^T * scale) v over [B, N, heads*64] bf16 views (blockwise, O(N) memory).

    q, k, v must share shape and strides (e.g. slices of one packed QKV tensor or three contiguous
    tensors); the gradients come back as views of one packed [B, N, 3, heads*64] buffer.
    """
    return _AttentionFn.apply(q, k, v, int(heads), bool(causal), scale)


# ----------------------------------------------------------------------------- CLIP loss
class _ClipLossFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, v, t, logit_scale, group):
        if v.dtype != torch.float32 or t.dtype != torch.float32:
            raise InputError("clip_loss embeddings must be fp32 [B, E]")
        if logit_scale.dtype != torch.float32 or logit_scale.numel() != 1 or not logit_scale.is_cuda:
            raise InputError("logit_scale must be a 1-element fp32 CUDA tensor (log-domain, CLIP's parameter)")
        v, t = v.contiguous(), t.contiguous()
        B = v.shape[0]
        v_all, t_all = dp.gather_embeddings(v, t, group=group)       # [W*B, E] global contrastive batch
        loss = torch.zeros(1, dtype=torch.float32, device=v.device)
        dls = torch.zeros(1, dtype=torch.float32, device=v.device)
        ls = logit_scale.reshape(1).contiguous()
        stats = ops.infonce_fwd(v_all, t_all, ls, loss, dls)
        ctx.save_for_backward(v_all, t_all, ls, dls, *stats.values())
        ctx.keys = list(stats.keys())
        ctx.B = B
        ctx.shape_ls = logit_scale.shape
        return loss.reshape(())

    @staticmethod
    def backward(ctx, gl):
        v_all, t_all, ls, dls, *st = ctx.saved_tensors
        stats = dict(zip(ctx.keys, st))
        r0, n = dp.local_rows(ctx.B)
        # every rank evaluates the full global loss but differentiates only its own rows: encoder
        # gradients must be SUMMED over ranks, so with a mean all-reduce they are scaled by world
        # here; the replicated logit-scale gradient is left as is (dp.py)
        dv, dt = ops.infonce_bwd(v_all, t_all, ls, stats, r0, n, grad_scale=dp.local_grad_scale())
        dv.mul_(gl)
        dt.mul_(gl)
        return dv, dt, (dls * gl).reshape(ctx.shape_ls), None


def clip_loss(v: torch.Tensor, t: torch.Tensor, logit_scale: torch.Tensor, group=None) -> torch.Tensor:
    """L = 1/2 [CE_rows(s v^ t^T) + CE_cols(s v^ t^T)], v^/t^ L2-normalised, s = exp(min(logit_scale, ln 100)).

    v, t: fp32 [B, E] raw embeddings of this rank's pairs; `logit_scale` is CLIP's learnable
    log-temperature parameter (initialised to ln(1/0.07)).  With an initialised process group the
    embeddings are all-gathered into the global batch (one fused [B, 2E] all_gather) and gradients
    flow into the local rows only (see `_ClipLossFn.backward`).
    """
    return _ClipLossFn.apply(v, t, logit_scale, group)


# ----------------------------------------------------------------------------- encoder module
class _EncoderFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, patches, flat, mod: "VideoEncoder"):
        mod._sync_shadow()
        B = patches.shape[0] // mod.cfg.patches
        x, saved = mod.engine.forward(patches, B, save=True)
        ctx.mod, ctx.saved = mod, saved
        return x.view(B, mod.cfg.tokens, mod.cfg.dim)

    @staticmethod
    def backward(ctx, gx):
        mod = ctx.mod
        store = mod.store
        cfg = mod.cfg
        dx = gx.reshape(-1, cfg.dim).to(torch.bfloat16).contiguous().clone()   # consumed in place by the engine
        gflat = torch.zeros_like(store.data)
        keep = store.grad
        store.grad = gflat          # the engine's wgrad GEMMs accumulate (fp32 red.add) into store.grad
        try:
            mod.engine.backward(dx, ctx.saved)
        finally:
            store.grad = keep
        ctx.saved = None
        return None, gflat, None


class VideoEncoder(torch.nn.Module):
    """Space-time ViT video encoder as an nn.Module (`VitConfig` field names, models.py:34-74).

    forward(x): x is either normalised clips bf16 [B, 3, T, H, W] (patchified on the GPU) or K1's
    tubelet rows bf16 [B*Np, 3*t*h*w]; returns the final residual stream bf16 [B, N, D] (token 0 is
    cls).  `flat` is the single fp32 master parameter (views by name via `param(name)`); any torch
    optimizer may update it -- the bf16 shadow the GEMMs read is refreshed automatically when
    `flat` changed -- or `fused_adamw_step()` runs the fused K8 kernel.
    """

    def __init__(self, cfg: VitConfig, device="cuda", seed: int = 0):
        super().__init__()
        cfg.validate()
        self.cfg = cfg
        self.store = ParamStore(torch.device(device))
        self.engine = _Engine(cfg, self.store)
        self.store.allocate(seed)
        self.flat = torch.nn.Parameter(self.store.data, requires_grad=True)
        self.store.data = self.flat        # one tensor: optimizer updates bump the version the shadow sync reads
        self._shadow_version = self.flat._version
        self._adamw_step = 0

    def param(self, name: str) -> torch.Tensor:
        """fp32 view of one named parameter, e.g. 'enc.blk0.qkv.w' (see `names()`)."""
        return self.store.p(name)

    def names(self) -> list[str]:
        return [s[0] for s in self.store.specs]

    def _sync_shadow(self):
        if self.flat._version != self._shadow_version:
            ops.cast_bf16(self.store.data, self.store.shadow)
            self._shadow_version = self.flat._version

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        cfg = self.cfg
        if x.dim() == 5:
            if tuple(x.shape[1:]) != (3, cfg.frames, cfg.height, cfg.width):
                raise InputError(f"clips must be [B, 3, {cfg.frames}, {cfg.height}, {cfg.width}], got {tuple(x.shape)}")
            x = ops.patchify(x.to(torch.bfloat16).contiguous(), (cfg.cube_t, cfg.cube_h, cfg.cube_w))
        if x.dim() != 2 or x.shape[1] != cfg.patch_dim or x.shape[0] % cfg.patches or x.dtype != torch.bfloat16:
            raise InputError(f"patch rows must be bf16 [B*{cfg.patches}, {cfg.patch_dim}]")
        return _EncoderFn.apply(x.contiguous(), self.flat, self)

    @torch.no_grad()
    def fused_adamw_step(self, opt: AdamWConfig | None = None, grad_scale: float = 1.0):
        """AdamW (K8) on the flat buffer with `flat.grad`, refreshing the bf16 shadow in the same pass."""
        o = opt or AdamWConfig()
        if self.flat.grad is None:
            return
        self._adamw_step += 1
        s = self.store
        ops.adamw_dev(s.data, self.flat.grad, s.m, s.v, s.shadow, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay,
                      s.step_dev, grad_scale, s.decay_mask)
        self._shadow_version = self.flat._version
