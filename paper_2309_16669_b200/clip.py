"""CLIP-style dual encoder (config 3): video ViT + causal text transformer + InfoNCE over the global batch.

PAPER.md:726-732 (ViT-B/16 video encoder from CLIP, 12-layer GPT-like text encoder, <=77 tokens),
:1196 (projection to 256-d), :291/:857 (contrastive loss), :1198-1199 (large global batch over
8 GPUs).  Per rank: K1 -> video encoder on its clips, text encoder on its captions, pooled
(cls / EOT) -> LayerNorm -> projection -> one fused all_gather of [B, 2E] embeddings -> fused
InfoNCE kernel on the full global batch -> gradients for the local rows only (scaled by world
so the mean all-reduce yields the exact sum, dp.py) -> backward through both towers.
"""

from __future__ import annotations

import math

import torch

from . import dp, ops
from .vit import (CONFIG3_VIT_B, AdamWConfig, ParamStore, TextConfig, TextEncoder, VideoEncoder, VitConfig)


class CLIPModel:
    def __init__(self, vcfg: VitConfig = CONFIG3_VIT_B, tcfg: TextConfig = TextConfig(), embed_dim: int = 256,
                 device="cuda", seed: int = 0, opt: AdamWConfig | None = None):
        self.vcfg, self.tcfg, self.E = vcfg, tcfg, embed_dim
        self.device = torch.device(device)
        s = self.store = ParamStore(self.device)
        self.video = VideoEncoder(vcfg, s, "enc")
        self.text = TextEncoder(tcfg, s, "txt")
        s.add("clip.vln.g", (vcfg.dim,), False, "ones", "clip")
        s.add("clip.vln.b", (vcfg.dim,), False, "zeros", "clip")
        s.add("clip.vproj", (embed_dim, vcfg.dim), True, "normal", "clip")
        s.add("clip.tln.g", (tcfg.dim,), False, "ones", "clip")
        s.add("clip.tln.b", (tcfg.dim,), False, "zeros", "clip")
        s.add("clip.tproj", (embed_dim, tcfg.dim), True, "normal", "clip")
        s.add("clip.logit_scale", (1,), False, "zeros", "clip")
        s.allocate(seed)
        s.p("clip.logit_scale").fill_(math.log(1 / 0.07))   # CLIP init (an assumption; not in the paper)
        self.opt = opt or AdamWConfig()
        self.step_num = 0

    def patches_from_clips(self, frames, boxes, flips, out=None, boxes_host=None):
        from . import transform as TR

        c = self.vcfg
        return TR.transform(frames, boxes, flips, (c.height, c.width), out=out, layout="tubelet",
                            tubelet=(c.cube_t, c.cube_h, c.cube_w), validate=False, crops_host=boxes_host)

    def _head_fwd(self, rows, ln_g, ln_b, proj):
        s = self.store
        z, mu, rs = ops.layernorm_fwd(rows, s.p(ln_g), s.p(ln_b),
                                      out=torch.empty(rows.shape, dtype=torch.bfloat16, device=rows.device))
        e = ops.gemm(z, s.w(proj), epilogue=ops.EPI_F32)
        return z, mu, rs, e

    def _head_bwd(self, de, rows, z, mu, rs, ln_g, ln_b, proj, drows):
        s = self.store
        de16 = torch.empty(de.shape, dtype=torch.bfloat16, device=de.device)
        ops.cast_bf16(de, de16)
        ops.gemm(de16, z, a_mn=True, b_mn=True, out=s.g(proj), epilogue=ops.EPI_F32_ACCUM)
        dz = ops.gemm(de16, s.w(proj), b_mn=True)
        ops.layernorm_bwd(dz, rows, s.p(ln_g), mu, rs, drows, s.g(ln_g), s.g(ln_b), accumulate=False)

    def forward_backward(self, patches: torch.Tensor, tokens: torch.Tensor, eot: torch.Tensor, loss: torch.Tensor,
                         on_layer_done=None):
        """patches: K1 tubelet rows of the local clips; tokens int32 [B, L]; eot int32 [B] = b*L + EOT position."""
        vc, tc_ = self.vcfg, self.tcfg
        B, L = tokens.shape
        s = self.store
        dev = patches.device
        xv, cv = self.video.forward(patches, B)
        vrows = xv.view(B, vc.tokens, vc.dim)[:, 0]                       # cls rows (strided view)
        zv, muv, rsv, ev = self._head_fwd(vrows, "clip.vln.g", "clip.vln.b", "clip.vproj")
        xt, ct = self.text.forward(tokens)
        trows = ops.rows_copy(xt, torch.empty((B, tc_.dim), dtype=torch.bfloat16, device=dev), src_idx=eot)
        zt, mut, rst, et = self._head_fwd(trows, "clip.tln.g", "clip.tln.b", "clip.tproj")
        v_all, t_all = dp.gather_embeddings(ev, et)
        ls = s.p("clip.logit_scale")
        stats = ops.infonce_fwd(v_all, t_all, ls, loss, s.g("clip.logit_scale"))
        r0, n = dp.local_rows(B)
        dv, dt = ops.infonce_bwd(v_all, t_all, ls, stats, r0, n, grad_scale=dp.local_grad_scale())
        dxv = torch.zeros_like(xv)
        self._head_bwd(dv, vrows, zv, muv, rsv, "clip.vln.g", "clip.vln.b", "clip.vproj",
                       dxv.view(B, vc.tokens, vc.dim)[:, 0])
        dtrows = torch.empty((B, tc_.dim), dtype=torch.bfloat16, device=dev)
        self._head_bwd(dt, trows, zt, mut, rst, "clip.tln.g", "clip.tln.b", "clip.tproj", dtrows)
        dxt = torch.zeros_like(xt)
        ops.rows_copy(dtrows, dxt, dst_idx=eot)
        if on_layer_done is not None:
            on_layer_done("clip")
        del xv, xt
        self.text.backward(dxt, ct, on_layer_done)
        self.video.backward(dxv, cv, on_layer_done)

    def optimizer_step(self, grad_scale: float = 1.0):
        self.step_num += 1
        s, o = self.store, self.opt
        ops.adamw_dev(s.data, s.grad, s.m, s.v, s.shadow, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay, s.step_dev,
                      grad_scale, s.decay_mask)

    def zero_grad(self):
        self.store.grad.zero_()
