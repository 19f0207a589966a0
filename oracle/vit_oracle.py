"""Encoder / attention / loss oracle: plain torch fp32 (TEST INFRASTRUCTURE ONLY).

The reference package has no encoder, attention or loss code and no tests for them
(SURVEY.md 0.3, 8(c)), so there is no reference output to pin against; this restates
PAPER.md directly, and tests/test_vit_oracle_pins.py checks it against independent public
formulations (F.scaled_dot_product_attention, nn.Conv3d tubelet embedding,
nn.TransformerEncoderLayer(norm_first=True), open_clip's ClipLoss formula):
  * tubelet patch-embed: non-overlapping t x h x w cubes -> Linear(3*t*h*w, D), plus the
    separable position embedding PE[t*S + s] = PE_t[t] + PE_s[1 + s] (cls: PE_s[0]) and a cls
    token;
  * pre-LN ViT block: x += Proj(MHA(LN x)); x += FC2(QuickGELU(FC1(LN x)))
    (QuickGELU = CLIP's activation, an assumption);
  * attention softmax(QK^T/sqrt(d)) V computed densely here (the kernels are blockwise;
    the math is the same);
  * fine-tune head: LN(cls) -> Linear(D, C) -> cross-entropy;
  * CLIP InfoNCE: L = 1/2 [CE_rows(s v t^T) + CE_cols(s v t^T)] on L2-normalised
    embeddings.
Token count follows the reference's VitConfig.tokens (models.py:71-74).
"""

from __future__ import annotations

import math
import os
import time

import torch
import torch.nn.functional as F


def quick_gelu(x):
    return x * torch.sigmoid(1.702 * x)


def patchify(clips, cfg):
    """clips [B,3,T,H,W] -> [B*Np, 3*t*h*w] rows in Conv3d-weight feature order."""
    B, C, T, H, W = clips.shape
    t, h, w = cfg.cube_t, cfg.cube_h, cfg.cube_w
    x = clips.reshape(B, C, T // t, t, H // h, h, W // w, w)
    x = x.permute(0, 2, 4, 6, 1, 3, 5, 7)  # B, T', H', W', C, t, h, w
    return x.reshape(B * (T // t) * (H // h) * (W // w), C * t * h * w)


def attention(qkv, B, N, H, causal=False):
    D = H * 64
    q, k, v = qkv.view(B, N, 3, H, 64).permute(2, 0, 3, 1, 4)
    s = q @ k.transpose(-1, -2) / math.sqrt(64)
    if causal:
        s = s.masked_fill(torch.ones(N, N, dtype=torch.bool).triu(1), float("-inf"))
    o = torch.softmax(s, -1) @ v
    return o.permute(0, 2, 1, 3).reshape(B * N, D)


def blocks(P: dict, x, B, N, D, heads, depth, prefix, causal=False):
    for l in range(depth):
        g = f"{prefix}.blk{l}"
        h = F.layer_norm(x, (D,), P[f"{g}.ln1.g"], P[f"{g}.ln1.b"], 1e-5)
        qkv = h @ P[f"{g}.qkv.w"].t() + P[f"{g}.qkv.b"]
        x = x + attention(qkv, B, N, heads, causal) @ P[f"{g}.proj.w"].t() + P[f"{g}.proj.b"]
        h = F.layer_norm(x, (D,), P[f"{g}.ln2.g"], P[f"{g}.ln2.b"], 1e-5)
        a = quick_gelu(h @ P[f"{g}.fc1.w"].t() + P[f"{g}.fc1.b"])
        x = x + a @ P[f"{g}.fc2.w"].t() + P[f"{g}.fc2.b"]
    return x


def encoder_forward(P: dict, patches, cfg, B, prefix="enc"):
    N, D = cfg.tokens, cfg.dim
    pe = patches @ P[f"{prefix}.pe.w"].t() + P[f"{prefix}.pe.b"]
    pe = pe.view(B, N - 1, D)
    cls = P[f"{prefix}.cls"].view(1, 1, D).expand(B, 1, D)
    ps, pt = P[f"{prefix}.pos_s"], P[f"{prefix}.pos_t"]                       # [1+S, D], [T', D]
    S = ps.shape[0] - 1
    pos = torch.cat([ps[:1], (pt.view(-1, 1, D) + ps[1:].view(1, S, D)).reshape(-1, D)], 0)
    x = (torch.cat([cls, pe], 1) + pos.view(1, N, D)).reshape(B * N, D)
    return blocks(P, x, B, N, D, cfg.heads, cfg.depth, prefix)


def text_forward(P: dict, tokens, tcfg, prefix="txt"):
    """Causal GPT-like text tower: token + position embedding -> blocks."""
    B, L = tokens.shape
    x = (P[f"{prefix}.tok"][tokens.long()] + P[f"{prefix}.pos"][:L]).reshape(B * L, tcfg.dim)
    return blocks(P, x, B, L, tcfg.dim, tcfg.heads, tcfg.depth, prefix, causal=True)


def clip_forward_loss(P: dict, patches, tokens, eot, vcfg, tcfg):
    """Dual-encoder CLIP loss: cls / EOT pooling -> LN -> projection -> InfoNCE (logit scale = exp(param))."""
    B, L = tokens.shape
    xv = encoder_forward(P, patches, vcfg, B)
    v = F.layer_norm(xv.view(B, vcfg.tokens, vcfg.dim)[:, 0], (vcfg.dim,), P["clip.vln.g"], P["clip.vln.b"], 1e-5)
    v = v @ P["clip.vproj"].t()
    xt = text_forward(P, tokens, tcfg)
    t = F.layer_norm(xt[eot.long()], (tcfg.dim,), P["clip.tln.g"], P["clip.tln.b"], 1e-5)
    t = t @ P["clip.tproj"].t()
    return clip_loss(v, t, P["clip.logit_scale"].exp().squeeze())


def head_loss(P: dict, x, B, N, labels, num_classes, prefix="head"):
    D = x.shape[-1]
    cls = x.view(B, N, D)[:, 0]
    z = F.layer_norm(cls, (D,), P[f"{prefix}.ln.g"], P[f"{prefix}.ln.b"], 1e-5)
    logits = z @ P[f"{prefix}.w"][:num_classes].t() + P[f"{prefix}.b"][:num_classes]
    return F.cross_entropy(logits, labels.long()), logits


def clip_loss(v, t, logit_scale):
    """CLIP InfoNCE over a (global) batch: v, t [Bg, E] raw embeddings."""
    v = F.normalize(v, dim=-1)
    t = F.normalize(t, dim=-1)
    s = logit_scale * v @ t.t()
    y = torch.arange(v.shape[0], device=v.device)
    return 0.5 * (F.cross_entropy(s, y) + F.cross_entropy(s.t(), y))


# ----------------------------------------------------------------------------- CPU baseline
def _encoder_param_shapes(cfg, prefix="enc"):
    D, Fd, Hd = cfg.dim, cfg.patch_dim, cfg.hidden
    P = {f"{prefix}.pe.w": (D, Fd), f"{prefix}.pe.b": (D,), f"{prefix}.cls": (D,),
         f"{prefix}.pos_s": (1 + cfg.spatial_tokens, D), f"{prefix}.pos_t": (cfg.temporal_tokens, D)}
    P.update(_block_param_shapes(D, Hd, cfg.depth, prefix))
    return P


def _block_param_shapes(D, Hd, depth, prefix):
    P = {}
    for l in range(depth):
        g = f"{prefix}.blk{l}"
        P.update({f"{g}.ln1.g": (D,), f"{g}.ln1.b": (D,), f"{g}.qkv.w": (3 * D, D), f"{g}.qkv.b": (3 * D,),
                  f"{g}.proj.w": (D, D), f"{g}.proj.b": (D,), f"{g}.ln2.g": (D,), f"{g}.ln2.b": (D,),
                  f"{g}.fc1.w": (Hd, D), f"{g}.fc1.b": (Hd,), f"{g}.fc2.w": (D, Hd), f"{g}.fc2.b": (D,)})
    return P


class CpuTrainStep:
    """One fp32 training step (fwd + bwd + AdamW) of the restatement on the host cores.

    kind "finetune": config-4/5 encoder + cls head CE over `num_classes`;
    kind "clip":     config-3 video + text towers + InfoNCE.
    Built once (weights, optimizer, synthetic inputs); `step()` runs exactly one step.
    """

    def __init__(self, cfg, clips: int, threads: int, kind: str = "finetune", num_classes: int = 3806,
                 tcfg=None, embed_dim: int = 256):
        torch.set_num_threads(threads)
        gen = torch.Generator().manual_seed(0)
        self.cfg, self.clips, self.kind, self.C = cfg, clips, kind, num_classes
        D = cfg.dim
        P = _encoder_param_shapes(cfg)
        if kind == "finetune":
            P.update({"head.ln.g": (D,), "head.ln.b": (D,), "head.w": (num_classes, D), "head.b": (num_classes,)})
        else:
            self.tcfg = tcfg
            P.update({"txt.tok": (tcfg.vocab, tcfg.dim), "txt.pos": (tcfg.context, tcfg.dim)})
            P.update(_block_param_shapes(tcfg.dim, tcfg.hidden, tcfg.depth, "txt"))
            P.update({"clip.vln.g": (D,), "clip.vln.b": (D,), "clip.vproj": (embed_dim, D),
                      "clip.tln.g": (tcfg.dim,), "clip.tln.b": (tcfg.dim,), "clip.tproj": (embed_dim, tcfg.dim),
                      "clip.logit_scale": (1,)})
        self.params = {k: (torch.randn(*s, generator=gen) * 0.02).requires_grad_(True) for k, s in P.items()}
        self.opt = torch.optim.AdamW(self.params.values(), lr=3e-5, weight_decay=0.01)
        self.clips_t = torch.randn(clips, 3, cfg.frames, cfg.height, cfg.width, generator=gen)
        self.labels = torch.randint(0, num_classes, (clips,), generator=gen)
        if kind == "clip":
            self.tokens = torch.randint(0, tcfg.vocab, (clips, tcfg.context), generator=gen)
            self.eot = torch.arange(clips) * tcfg.context + tcfg.context - 1

    def step(self) -> float:
        P, cfg = self.params, self.cfg
        if self.kind == "finetune":
            x = encoder_forward(P, patchify(self.clips_t, cfg), cfg, self.clips)
            loss, _ = head_loss(P, x, self.clips, cfg.tokens, self.labels, self.C)
        else:
            loss = clip_forward_loss(P, patchify(self.clips_t, cfg), self.tokens, self.eot, cfg, self.tcfg)
        self.opt.zero_grad()
        loss.backward()
        self.opt.step()
        return float(loss.detach())


def cpu_train_step_time(cfg, num_classes: int, clips: int, threads: int, steps: int = 1):
    """Seconds per fp32 fine-tune step (min over `steps` after one untimed step)."""
    st = CpuTrainStep(cfg, clips, threads, "finetune", num_classes)
    st.step()
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        st.step()
        times.append(time.perf_counter() - t0)
    return min(times)
