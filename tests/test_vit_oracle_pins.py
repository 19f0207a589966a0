"""Pin the encoder/attention/loss oracle (oracle/vit_oracle.py) against independent formulations.

The reference has no encoder code (parity unpinned), so the restatement is checked
against public semantics it must agree with:
  * attention  == torch.nn.functional.scaled_dot_product_attention (math backend), causal and not;
  * patchify + Linear == nn.Conv3d(kernel = stride = tubelet) with the same weights (the ViT
    tubelet embedding);
  * the separable position embedding == an explicit per-token loop of PE_t[t] + PE_s[1+s] (cls: PE_s[0]);
  * clip_loss == open_clip's ClipLoss formula (scaled normalised logits, symmetric CE, mean);
  * one pre-LN block == torch.nn.TransformerEncoderLayer(norm_first=True) with QuickGELU;
  * a 2-layer stack == transformers' CLIPEncoder (the CLIP ViT block AVION starts from).
CPU only, fp64 where the comparison is exact.
"""

import math

import torch
import torch.nn.functional as F

from oracle import vit_oracle as VO
from paper_2309_16669_b200.vit import VitConfig


def test_attention_matches_sdpa():
    torch.manual_seed(0)
    B, N, H = 2, 37, 3
    qkv = torch.randn(B, N, 3 * H * 64, dtype=torch.float64)
    for causal in (False, True):
        got = VO.attention(qkv, B, N, H, causal=causal).view(B, N, H, 64)
        q, k, v = qkv.view(B, N, 3, H, 64).permute(2, 0, 3, 1, 4)
        ref = F.scaled_dot_product_attention(q, k, v, is_causal=causal).permute(0, 2, 1, 3)
        assert (got - ref).abs().max().item() < 1e-12


def test_patchify_linear_is_conv3d():
    torch.manual_seed(1)
    cfg = VitConfig(frames=4, height=32, width=48, cube_t=2, cube_h=16, cube_w=16, depth=1, dim=64, heads=1)
    x = torch.randn(2, 3, cfg.frames, cfg.height, cfg.width, dtype=torch.float64)
    conv = torch.nn.Conv3d(3, cfg.dim, (cfg.cube_t, cfg.cube_h, cfg.cube_w), stride=(cfg.cube_t, cfg.cube_h, cfg.cube_w),
                           dtype=torch.float64)
    ref = conv(x).flatten(2).transpose(1, 2).reshape(-1, cfg.dim)          # [B*Np, D], tokens (t, y, x)
    got = VO.patchify(x, cfg) @ conv.weight.reshape(cfg.dim, -1).t() + conv.bias
    assert (got - ref).abs().max().item() < 1e-10


def test_separable_position_embedding():
    torch.manual_seed(2)
    cfg = VitConfig(frames=4, height=32, width=48, cube_t=2, cube_h=16, cube_w=16, depth=0, dim=8, heads=1)
    D, S, Tp, B = cfg.dim, cfg.spatial_tokens, cfg.temporal_tokens, 2
    P = {"enc.pe.w": torch.zeros(D, cfg.patch_dim, dtype=torch.float64), "enc.pe.b": torch.zeros(D, dtype=torch.float64),
         "enc.cls": torch.randn(D, dtype=torch.float64), "enc.pos_s": torch.randn(1 + S, D, dtype=torch.float64),
         "enc.pos_t": torch.randn(Tp, D, dtype=torch.float64)}
    x = VO.encoder_forward(P, torch.zeros(B * cfg.patches, cfg.patch_dim, dtype=torch.float64), cfg, B).view(B, -1, D)
    assert torch.allclose(x[:, 0], P["enc.cls"] + P["enc.pos_s"][0])
    for t in range(Tp):
        for s in range(S):
            assert torch.allclose(x[:, 1 + t * S + s], P["enc.pos_t"][t] + P["enc.pos_s"][1 + s])


def test_clip_loss_matches_open_clip_formula():
    torch.manual_seed(3)
    img, txt = torch.randn(16, 32, dtype=torch.float64), torch.randn(16, 32, dtype=torch.float64)
    scale = torch.tensor(1 / 0.07, dtype=torch.float64)
    i_n, t_n = img / img.norm(dim=-1, keepdim=True), txt / txt.norm(dim=-1, keepdim=True)
    logits_per_image = scale * i_n @ t_n.t()
    logits_per_text = scale * t_n @ i_n.t()
    labels = torch.arange(16)
    ref = (F.cross_entropy(logits_per_image, labels) + F.cross_entropy(logits_per_text, labels)) / 2
    assert abs(VO.clip_loss(img, txt, scale).item() - ref.item()) < 1e-12


def test_block_matches_torch_encoder_layer():
    torch.manual_seed(4)
    D, H, B, N = 128, 2, 2, 11
    layer = torch.nn.TransformerEncoderLayer(D, H, 4 * D, dropout=0.0, activation=VO.quick_gelu, batch_first=True,
                                             norm_first=True, dtype=torch.float64)
    layer.eval()
    g = "enc.blk0"
    P = {f"{g}.ln1.g": layer.norm1.weight, f"{g}.ln1.b": layer.norm1.bias,
         f"{g}.qkv.w": layer.self_attn.in_proj_weight, f"{g}.qkv.b": layer.self_attn.in_proj_bias,
         f"{g}.proj.w": layer.self_attn.out_proj.weight, f"{g}.proj.b": layer.self_attn.out_proj.bias,
         f"{g}.ln2.g": layer.norm2.weight, f"{g}.ln2.b": layer.norm2.bias,
         f"{g}.fc1.w": layer.linear1.weight, f"{g}.fc1.b": layer.linear1.bias,
         f"{g}.fc2.w": layer.linear2.weight, f"{g}.fc2.b": layer.linear2.bias}
    x = torch.randn(B, N, D, dtype=torch.float64)
    with torch.no_grad():
        ref = layer(x)
        got = VO.blocks(P, x.reshape(B * N, D), B, N, D, H, 1, "enc").view(B, N, D)
    assert (got - ref).abs().max().item() < 1e-10
    assert math.isfinite(got.sum().item())


def test_blocks_match_transformers_clip_encoder():
    """A 2-layer stack == transformers' CLIPEncoder (pre-LN, QuickGELU): the CLIP ViT-B/16 block that
    AVION initialises its video encoder from, an independent public implementation."""
    from transformers.models.clip.configuration_clip import CLIPVisionConfig
    from transformers.models.clip.modeling_clip import CLIPEncoder

    torch.manual_seed(5)
    D, H, L, B, N = 128, 2, 2, 2, 13   # head_dim 64 (the kernels' and the oracle's)
    cfg = CLIPVisionConfig(hidden_size=D, num_attention_heads=H, intermediate_size=4 * D, num_hidden_layers=L,
                           hidden_act="quick_gelu", attention_dropout=0.0)
    cfg._attn_implementation = "eager"
    enc = CLIPEncoder(cfg).to(torch.float64).eval()
    P = {}
    for l, layer in enumerate(enc.layers):
        g = f"enc.blk{l}"
        a = layer.self_attn
        for t in (layer.layer_norm1, layer.layer_norm2, a.q_proj, a.k_proj, a.v_proj, a.out_proj, layer.mlp.fc1,
                  layer.mlp.fc2):
            torch.nn.init.normal_(t.weight, std=0.2 if isinstance(t, torch.nn.LayerNorm) else 0.05)
            torch.nn.init.normal_(t.bias, std=0.05)
            if isinstance(t, torch.nn.LayerNorm):
                t.weight.data += 1.0
        P.update({f"{g}.ln1.g": layer.layer_norm1.weight, f"{g}.ln1.b": layer.layer_norm1.bias,
                  f"{g}.qkv.w": torch.cat([a.q_proj.weight, a.k_proj.weight, a.v_proj.weight]),
                  f"{g}.qkv.b": torch.cat([a.q_proj.bias, a.k_proj.bias, a.v_proj.bias]),
                  f"{g}.proj.w": a.out_proj.weight, f"{g}.proj.b": a.out_proj.bias,
                  f"{g}.ln2.g": layer.layer_norm2.weight, f"{g}.ln2.b": layer.layer_norm2.bias,
                  f"{g}.fc1.w": layer.mlp.fc1.weight, f"{g}.fc1.b": layer.mlp.fc1.bias,
                  f"{g}.fc2.w": layer.mlp.fc2.weight, f"{g}.fc2.b": layer.mlp.fc2.bias})
    x = torch.randn(B, N, D, dtype=torch.float64)
    with torch.no_grad():
        out = enc(inputs_embeds=x)
        ref = out.last_hidden_state if hasattr(out, "last_hidden_state") else out[0]
        got = VO.blocks(P, x.reshape(B * N, D), B, N, D, H, L, "enc").view(B, N, D)
    # transformers' eager attention takes the softmax in fp32 even in an fp64 model: ~1e-8 differences
    assert (got - ref).abs().max().item() < 1e-6
