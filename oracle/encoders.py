"""fp32 PyTorch CPU encoders -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates the public definitions the north star names (the reference has no
encoder: SPEC.md:8, :106 -- parity unpinned by the reference):

* MiniCPM-V 2.6 vision path: SigLIP ViT (Conv2d patch embed + learned position
  embedding; pre-LN blocks with q/k/v/o projections and GELU-tanh MLP;
  post-LayerNorm) and the perceiver resampler (kv_proj, ln_kv, ln_q(query),
  nn.MultiheadAttention with key = x + 2-D sincos position, value = x, ln_post,
  ``x @ proj``).
* InternVL2 vision path: InternViT (CLS token + position embedding; pre-LN blocks
  with fused qkv, layer scale ls1/ls2, GELU MLP; last hidden state), CLS drop,
  ``pixel_shuffle(x, 0.5)`` (ps_version v2) and mlp1 (LayerNorm, Linear, GELU,
  Linear).

Inputs: uint8 tiles [n, S, S, C]; weights: the canonical dict produced by
paper_2501_05460_b200.weights.init_weights (same names and shapes).
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def _attn(q, k, v, heads):
    """q [n, Tq, E], k/v [n, Tk, E] -> [n, Tq, E] softmax(q k^T / sqrt(d)) v."""
    n, tq, e = q.shape
    tk = k.shape[1]
    d = e // heads
    q = q.view(n, tq, heads, d).transpose(1, 2)
    k = k.view(n, tk, heads, d).transpose(1, 2)
    v = v.view(n, tk, heads, d).transpose(1, 2)
    p = torch.softmax((q @ k.transpose(-1, -2)) / math.sqrt(d), dim=-1)
    return (p @ v).transpose(1, 2).reshape(n, tq, e)


def _embed(cfg, w, tiles):
    x = tiles.float() / 255.0
    x = (x - torch.tensor(cfg.mean[: cfg.channels])) / torch.tensor(cfg.std[: cfg.channels])
    x = x.permute(0, 3, 1, 2)
    x = F.conv2d(x, w["patch_embed.weight"], w["patch_embed.bias"], stride=cfg.patch_size)
    return x.flatten(2).transpose(1, 2)  # [n, grid*grid, D]


def siglip_resampler(cfg, w, tiles: torch.Tensor) -> torch.Tensor:
    D, eps = cfg.hidden, cfg.ln_eps
    x = _embed(cfg, w, tiles) + w["pos_embed"]
    for l in range(cfg.layers):
        p = f"layers.{l}."
        h = F.layer_norm(x, (D,), w[p + "ln1.weight"], w[p + "ln1.bias"], eps)
        q = F.linear(h, w[p + "attn.q.weight"], w[p + "attn.q.bias"])
        k = F.linear(h, w[p + "attn.k.weight"], w[p + "attn.k.bias"])
        v = F.linear(h, w[p + "attn.v.weight"], w[p + "attn.v.bias"])
        x = x + F.linear(_attn(q, k, v, cfg.heads), w[p + "attn.o.weight"], w[p + "attn.o.bias"])
        h = F.layer_norm(x, (D,), w[p + "ln2.weight"], w[p + "ln2.bias"], eps)
        h = F.gelu(F.linear(h, w[p + "mlp.fc1.weight"], w[p + "mlp.fc1.bias"]), approximate="tanh")
        x = x + F.linear(h, w[p + "mlp.fc2.weight"], w[p + "mlp.fc2.bias"])
    x = F.layer_norm(x, (D,), w["post_ln.weight"], w["post_ln.bias"], eps)
    # resampler (MiniCPM-V 2.6): LayerNorms use eps 1e-6
    E = cfg.out_dim
    kv = F.linear(x, w["rs.kv_proj.weight"])
    kv = F.layer_norm(kv, (E,), w["rs.ln_kv.weight"], w["rs.ln_kv.bias"], 1e-6)
    q = F.layer_norm(w["rs.query"], (E,), w["rs.ln_q.weight"], w["rs.ln_q.bias"], 1e-6)
    n = tiles.shape[0]
    q = F.linear(q, w["rs.attn.q.weight"], w["rs.attn.q.bias"]).unsqueeze(0).expand(n, -1, -1)
    k = F.linear(kv + w["rs.pos_embed"], w["rs.attn.k.weight"], w["rs.attn.k.bias"])
    v = F.linear(kv, w["rs.attn.v.weight"], w["rs.attn.v.bias"])
    o = F.linear(_attn(q, k, v, cfg.out_heads), w["rs.attn.o.weight"], w["rs.attn.o.bias"])
    o = F.layer_norm(o, (E,), w["rs.ln_post.weight"], w["rs.ln_post.bias"], 1e-6)
    return o @ w["rs.proj"]


def pixel_shuffle(x: torch.Tensor, scale_factor: float = 0.5) -> torch.Tensor:
    """InternVL pixel_shuffle, ps_version 'v2' (view/permute sequence of the public code)."""
    n, wd, h, c = x.size()
    x = x.view(n, wd, int(h * scale_factor), int(c / scale_factor))
    x = x.permute(0, 2, 1, 3).contiguous()
    x = x.view(n, int(h * scale_factor), int(wd * scale_factor), int(c / (scale_factor * scale_factor)))
    x = x.permute(0, 2, 1, 3).contiguous()
    return x


def internvit_mlp(cfg, w, tiles: torch.Tensor) -> torch.Tensor:
    D, eps = cfg.hidden, cfg.ln_eps
    x = _embed(cfg, w, tiles)
    n = x.shape[0]
    cls = w["cls_token"].view(1, 1, D).expand(n, 1, D)
    x = torch.cat([cls, x], dim=1) + w["pos_embed"]
    for l in range(cfg.layers):
        p = f"layers.{l}."
        h = F.layer_norm(x, (D,), w[p + "ln1.weight"], w[p + "ln1.bias"], eps)
        qkv = F.linear(h, w[p + "attn.qkv.weight"], w[p + "attn.qkv.bias"])
        q, k, v = qkv.split(D, dim=-1)
        a = F.linear(_attn(q, k, v, cfg.heads), w[p + "attn.o.weight"], w[p + "attn.o.bias"])
        x = x + w[p + "ls1"] * a
        h = F.layer_norm(x, (D,), w[p + "ln2.weight"], w[p + "ln2.bias"], eps)
        h = F.gelu(F.linear(h, w[p + "mlp.fc1.weight"], w[p + "mlp.fc1.bias"]))
        x = x + w[p + "ls2"] * F.linear(h, w[p + "mlp.fc2.weight"], w[p + "mlp.fc2.bias"])
    x = x[:, 1:, :]
    g = int(round(math.sqrt(x.shape[1])))
    x = pixel_shuffle(x.reshape(n, g, g, D), 0.5).reshape(n, -1, 4 * D)
    x = F.layer_norm(x, (4 * D,), w["mlp1.ln.weight"], w["mlp1.ln.bias"], 1e-5)
    x = F.gelu(F.linear(x, w["mlp1.fc1.weight"], w["mlp1.fc1.bias"]))
    return F.linear(x, w["mlp1.fc2.weight"], w["mlp1.fc2.bias"])


def encode(cfg, weights: dict, tiles: torch.Tensor) -> torch.Tensor:
    """fp32 MM tokens [n, out_tokens, out_dim] for uint8 tiles [n, S, S, C] (CPU)."""
    from paper_2501_05460_b200._lib import FAMILY_INTERNVIT_MLP, FAMILY_SIGLIP_RESAMPLER
    tiles = tiles.cpu()
    with torch.no_grad():
        if cfg.family == FAMILY_SIGLIP_RESAMPLER:
            return siglip_resampler(cfg, weights, tiles)
        if cfg.family == FAMILY_INTERNVIT_MLP:
            return internvit_mlp(cfg, weights, tiles)
    raise ValueError("unknown encoder family")


def bf16_weights(weights: dict) -> dict:
    """The canonical weights rounded to the bf16 values the GPU path stores (kept in fp32)."""
    return {k: v.to(torch.bfloat16).float() for k, v in weights.items()}


def relerr(y: torch.Tensor, ref: torch.Tensor) -> float:
    """North-star metric: max|y - ref| / max|ref| over the whole tensor."""
    y = y.float().cpu()
    ref = ref.float().cpu()
    return float((y - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
