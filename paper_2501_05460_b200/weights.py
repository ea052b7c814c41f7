"""Deterministic random-init weights in the canonical (framework) layout.

The schema (names, shapes, order) is owned by the C library
(``epd_encoder_weight_info``); this module fills it from a seeded CPU
generator so the GPU path and the fp32 CPU oracle consume identical tensors
(N(0, 0.02) weights; LayerNorm gamma near 1 and beta near 0;
layer scale near 0.1; the resampler key positions are the fixed 2-D sincos
table of MiniCPM-V's resampler).
"""
from __future__ import annotations

import numpy as np
import torch


def sincos_2d(embed_dim: int, grid_h: int, grid_w: int) -> np.ndarray:
    """MiniCPM-V resampler position table for a (grid_h x grid_w) patch grid.

    Restates the public get_2d_sincos_pos_embed (meshgrid with w first; half of the
    channels encode the w coordinate, half the h coordinate; sin then cos), flattened
    row-major to [grid_h * grid_w, embed_dim].
    """
    def one_d(dim: int, pos: np.ndarray) -> np.ndarray:
        omega = np.arange(dim // 2, dtype=np.float32)
        omega /= dim / 2.0
        omega = 1.0 / 10000 ** omega
        out = np.einsum("hw,d->hwd", pos, omega)
        return np.concatenate([np.sin(out), np.cos(out)], axis=-1)

    gh = np.arange(grid_h, dtype=np.float32)
    gw = np.arange(grid_w, dtype=np.float32)
    grid = np.stack(np.meshgrid(gw, gh), axis=0)  # [2, H, W]; grid[0] = w coordinate
    emb = np.concatenate([one_d(embed_dim // 2, grid[0]), one_d(embed_dim // 2, grid[1])], axis=-1)
    return emb.reshape(grid_h * grid_w, embed_dim).astype(np.float32)


def _is_ln(name: str) -> bool:
    parts = name.split(".")
    return len(parts) >= 2 and (parts[-2].startswith("ln") or parts[-2] == "post_ln")


def weight_schema(cfg) -> list[tuple[str, tuple[int, ...]]]:
    """The canonical weight list (names, shapes, order) in pure Python.

    Mirrors ``Encoder::validate_and_build_schema`` (csrc/encoder.cu) so host-only
    callers -- the CPU reference arm of bench.py, fixture scripts -- never open
    libepd.so; ``tests/test_abi_cpu.py`` checks the two agree for every config.
    """
    from ._lib import FAMILY_INTERNVIT_MLP, FAMILY_SIGLIP_RESAMPLER
    D, F, E, P, Ch = cfg.hidden, cfg.mlp, cfg.out_dim, cfg.patch_size, cfg.channels
    grid = cfg.image_size // cfg.patch_size
    siglip = cfg.family == FAMILY_SIGLIP_RESAMPLER
    if not siglip and cfg.family != FAMILY_INTERNVIT_MLP:
        raise ValueError("unknown encoder family")
    T = grid * grid + (0 if siglip else 1)
    s: list[tuple[str, tuple[int, ...]]] = [("patch_embed.weight", (D, Ch, P, P)), ("patch_embed.bias", (D,))]
    if not siglip:
        s.append(("cls_token", (D,)))
    s.append(("pos_embed", (T, D)))
    for l in range(cfg.layers):
        p = f"layers.{l}."
        s += [(p + "ln1.weight", (D,)), (p + "ln1.bias", (D,))]
        if siglip:
            for m in "qkv":
                s += [(p + f"attn.{m}.weight", (D, D)), (p + f"attn.{m}.bias", (D,))]
        else:
            s += [(p + "attn.qkv.weight", (3 * D, D)), (p + "attn.qkv.bias", (3 * D,))]
        s += [(p + "attn.o.weight", (D, D)), (p + "attn.o.bias", (D,))]
        if not siglip:
            s.append((p + "ls1", (D,)))
        s += [(p + "ln2.weight", (D,)), (p + "ln2.bias", (D,)),
              (p + "mlp.fc1.weight", (F, D)), (p + "mlp.fc1.bias", (F,)),
              (p + "mlp.fc2.weight", (D, F)), (p + "mlp.fc2.bias", (D,))]
        if not siglip:
            s.append((p + "ls2", (D,)))
    if siglip:
        Q = cfg.out_tokens
        s += [("post_ln.weight", (D,)), ("post_ln.bias", (D,)), ("rs.query", (Q, E)),
              ("rs.kv_proj.weight", (E, D)), ("rs.ln_q.weight", (E,)), ("rs.ln_q.bias", (E,)),
              ("rs.ln_kv.weight", (E,)), ("rs.ln_kv.bias", (E,))]
        for m in "qkvo":
            s += [(f"rs.attn.{m}.weight", (E, E)), (f"rs.attn.{m}.bias", (E,))]
        s += [("rs.ln_post.weight", (E,)), ("rs.ln_post.bias", (E,)), ("rs.proj", (E, E)),
              ("rs.pos_embed", (T, E))]
    else:
        C4 = 4 * D
        s += [("mlp1.ln.weight", (C4,)), ("mlp1.ln.bias", (C4,)), ("mlp1.fc1.weight", (E, C4)),
              ("mlp1.fc1.bias", (E,)), ("mlp1.fc2.weight", (E, E)), ("mlp1.fc2.bias", (E,))]
    return s


def canonical_weights(cfg, seed: int) -> dict[str, torch.Tensor]:
    """The fp32 canonical weights of ``cfg`` without loading the C library."""
    return init_weights(weight_schema(cfg), cfg, seed)


def init_weights(schema: list[tuple[str, tuple[int, ...]]], cfg, seed: int) -> dict[str, torch.Tensor]:
    """Canonical fp32 CPU tensors for every schema entry, drawn in schema order."""
    g = torch.Generator().manual_seed(seed)
    out: dict[str, torch.Tensor] = {}
    for name, shape in schema:
        if name == "rs.pos_embed":
            grid = cfg.image_size // cfg.patch_size
            t = torch.from_numpy(sincos_2d(shape[1], grid, grid))
        elif _is_ln(name) and name.endswith(".weight"):
            t = 1.0 + 0.02 * torch.randn(shape, generator=g)
        elif name.split(".")[-1] in ("ls1", "ls2"):
            t = 0.1 + 0.01 * torch.randn(shape, generator=g)
        else:
            t = 0.02 * torch.randn(shape, generator=g)
        out[name] = t.float().contiguous()
    return out
