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
