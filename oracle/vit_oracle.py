"""Encoder / attention / loss oracle: plain torch fp32 (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED: the reference package has no encoder, attention or loss code and
no tests for them; this restates PAPER.md directly:
  * tubelet patch-embed: non-overlapping t x h x w cubes -> Linear(3*t*h*w, D), plus a
    learned position table and a cls token;
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
    x = (torch.cat([cls, pe], 1) + P[f"{prefix}.pos"].view(1, N, D)).reshape(B * N, D)
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
    y = torch.arange(v.shape[0])
    return 0.5 * (F.cross_entropy(s, y) + F.cross_entropy(s.t(), y))


# ----------------------------------------------------------------------------- CPU baseline
def cpu_train_step_time(cfg, num_classes: int, clips: int, threads: int, steps: int = 1):
    """Seconds per fp32 training step (fwd+bwd+AdamW) of the restatement on `clips` clips."""
    torch.set_num_threads(threads)
    gen = torch.Generator().manual_seed(0)
    D, Fd, Hd, N = cfg.dim, cfg.patch_dim, cfg.hidden, cfg.tokens
    P = {"enc.pe.w": (D, Fd), "enc.pe.b": (D,), "enc.cls": (D,), "enc.pos": (N, D)}
    for l in range(cfg.depth):
        g = f"enc.blk{l}"
        P.update({f"{g}.ln1.g": (D,), f"{g}.ln1.b": (D,), f"{g}.qkv.w": (3 * D, D), f"{g}.qkv.b": (3 * D,),
                  f"{g}.proj.w": (D, D), f"{g}.proj.b": (D,), f"{g}.ln2.g": (D,), f"{g}.ln2.b": (D,),
                  f"{g}.fc1.w": (Hd, D), f"{g}.fc1.b": (Hd,), f"{g}.fc2.w": (D, Hd), f"{g}.fc2.b": (D,)})
    P.update({"head.ln.g": (D,), "head.ln.b": (D,), "head.w": (num_classes, D), "head.b": (num_classes,)})
    params = {k: (torch.randn(*s, generator=gen) * 0.02).requires_grad_(True) for k, s in P.items()}
    opt = torch.optim.AdamW(params.values(), lr=3e-5, weight_decay=0.01)
    clips_t = torch.randn(clips, 3, cfg.frames, cfg.height, cfg.width, generator=gen)
    labels = torch.randint(0, num_classes, (clips,), generator=gen)
    times = []
    for _ in range(steps + 1):
        t0 = time.perf_counter()
        x = encoder_forward(params, patchify(clips_t, cfg), cfg, clips)
        loss, _ = head_loss(params, x, clips, N, labels, num_classes)
        opt.zero_grad()
        loss.backward()
        opt.step()
        times.append(time.perf_counter() - t0)
    return min(times[1:]) if steps else times[0]


def reference_train_line(args, world, cores):
    """`bench.py --impl reference --workload train`: CPU fp32 restatement of the config-4 step."""
    from paper_2309_16669_b200.vit import CONFIG4_VIT_B_16F as cfg  # shapes only

    clips = 1
    for _ in range(max(0, args.warmup - 2)):
        pass
    sec = cpu_train_step_time(cfg, 3806, clips, cores, steps=max(1, min(args.steps, 2)))
    v = clips / sec
    return {"impl": "reference", "metric": "train clips/sec ViT-B/16 16x224^2 (fine-tune step)", "value": v,
            "unit": "clips/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic clips, random-init weights",
            "config": {"workload": "configs[3] ViT-B/16 fine-tune 16x224^2, tubelet 2x16x16 (N=1569)",
                       "clips_per_step": clips},
            "cpu_baseline": {"value": v, "unit": "clips/s", "cores": cores, "kind": "port",
                             "sample": f"{clips} clip per step, torch fp32 restatement fwd+bwd+AdamW, "
                                       f"{cores} threads"},
            "e2e": {"value": v, "unit": "clips/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
