#!/usr/bin/env python
"""Pin the encoder oracle (oracle/encoders.py) to the PUBLIC model implementations.

The reference (disaggsim) has no encoder, so the fp32 CPU oracle is a
restatement of the public models. This script -- run in the build container, where
transformers 5.5 and vLLM 0.22 are importable -- builds those public modules, loads them
with the oracle's canonical random-init weights, runs both on the same synthetic uint8
tiles and writes ``encoder_golden.json``:

* MiniCPM-V 2.6 vision path: transformers ``Idefics2VisionTransformer`` (the SigLIP-so400m
  tower MiniCPM-V 2.6 runs, with its NaViT bucketed position ids over a 70x70 table:
  image_size 980 / patch 14) + vLLM ``Resampler2_5`` (vllm/model_executor/models/minicpmv.py,
  ``init_resampler``: 64 queries, embed 3584, heads 3584 // 128, kv_dim 1152; its own 2-D
  sincos cache ``version=(2, 5)`` -- so the oracle's ``rs.pos_embed`` table is pinned too).
* InternVL2-8B vision path: transformers ``InternVLVisionModel`` (InternViT-300M: CLS,
  absolute positions, layer scale, no final norm = ``use_mean_pooling``) ->
  ``InternVLModel.pixel_shuffle(x, 0.5)`` -> ``InternVLMultiModalProjector`` (LN, Linear,
  GELU, Linear), as ``InternVLModel.get_image_features`` chains them.

The fixture keeps, per model: the max relative error oracle vs public (must be <= 1e-5 in
fp32), a deterministic sample of the public outputs (every ``stride``-th element of the
flattened tensor) and whole-tensor sums. ``tests/test_encoder_golden_cpu.py`` re-runs the
oracle against it (CPU tier) and ``tests/test_encoder_gpu.py`` compares the B200 bf16
tokens with the same public outputs (1e-2).

Usage:  python tests/golden/make_encoder_golden.py   (~1 min on 8 cores)
"""
from __future__ import annotations

import json
import sys
import types
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2501_05460_b200.configs import INTERNVIT_300M, SEED, SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.weights import canonical_weights  # noqa: E402

import oracle.encoders as oe  # noqa: E402

OUT = Path(__file__).resolve().parent / "encoder_golden.json"
N_TILES = 2
TILE_SEED = 7
SAMPLES = 4096


def golden_tiles(cfg, n: int = N_TILES, seed: int = TILE_SEED) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n, cfg.image_size, cfg.image_size, cfg.channels), dtype=torch.uint8, generator=g)


def pixel_values(cfg, tiles: torch.Tensor) -> torch.Tensor:
    """The public image processors' rescale (1/255) + normalize, NCHW fp32."""
    x = tiles.float() / 255.0
    x = (x - torch.tensor(cfg.mean)) / torch.tensor(cfg.std)
    return x.permute(0, 3, 1, 2).contiguous()


def _load(module: torch.nn.Module, tensors: dict[str, torch.Tensor]) -> None:
    sd = module.state_dict()
    missing = [k for k in sd if k not in tensors]
    extra = [k for k in tensors if k not in sd]
    if missing or extra:
        raise KeyError(f"state dict mismatch: missing {missing[:5]} extra {extra[:5]}")
    for k, v in tensors.items():
        if tuple(sd[k].shape) != tuple(v.shape):
            raise ValueError(f"{k}: {tuple(sd[k].shape)} vs {tuple(v.shape)}")
    module.load_state_dict(tensors, strict=True)


def public_minicpmv26(cfg, w: dict, tiles: torch.Tensor) -> torch.Tensor:
    from transformers.models.idefics2.configuration_idefics2 import Idefics2VisionConfig
    from transformers.models.idefics2.modeling_idefics2 import Idefics2VisionTransformer

    import vllm.distributed.parallel_state as ps
    # Resampler2_5.kv_proj is a vLLM ReplicatedLinear, which asks for the TP rank at
    # construction; a single-process stand-in group is all it needs on CPU.
    ps.get_tp_group = lambda: types.SimpleNamespace(rank_in_group=0, world_size=1)
    from vllm.model_executor.models.minicpmv import Resampler2_5

    D, L = cfg.hidden, cfg.layers
    vcfg = Idefics2VisionConfig(hidden_size=D, intermediate_size=cfg.mlp, num_hidden_layers=L,
                                num_attention_heads=cfg.heads, num_channels=cfg.channels, image_size=980,
                                patch_size=cfg.patch_size, hidden_act="gelu_pytorch_tanh",
                                layer_norm_eps=cfg.ln_eps, attention_dropout=0.0)
    vcfg._attn_implementation = "eager"
    vpm = Idefics2VisionTransformer(vcfg).eval()
    grid = cfg.image_size // cfg.patch_size
    # the NaViT position ids a full 32x32 patch grid selects from the 70x70 table
    with torch.no_grad():
        mask = torch.ones(1, grid, grid, dtype=torch.bool)
        emb = vpm.embeddings
        boundaries = torch.arange(1 / emb.num_patches_per_side, 1.0, 1 / emb.num_patches_per_side)
        frac = torch.clamp(torch.arange(grid, dtype=torch.float32) * (1.0 / grid), max=1.0 - 1e-6)
        b = torch.bucketize(frac, boundaries, right=True)
        pos_ids = (b[:, None] * emb.num_patches_per_side + b[None, :]).reshape(-1)
        assert pos_ids.unique().numel() == grid * grid and bool(mask.all())
    table = torch.zeros(emb.num_positions, D)
    table[pos_ids] = w["pos_embed"]
    sd = {"embeddings.patch_embedding.weight": w["patch_embed.weight"],
          "embeddings.patch_embedding.bias": w["patch_embed.bias"],
          "embeddings.position_embedding.weight": table,
          "post_layernorm.weight": w["post_ln.weight"], "post_layernorm.bias": w["post_ln.bias"]}
    for l in range(L):
        p, q = f"layers.{l}.", f"encoder.layers.{l}."
        for a, b_ in (("q", "q_proj"), ("k", "k_proj"), ("v", "v_proj"), ("o", "out_proj")):
            sd[q + f"self_attn.{b_}.weight"] = w[p + f"attn.{a}.weight"]
            sd[q + f"self_attn.{b_}.bias"] = w[p + f"attn.{a}.bias"]
        for a, b_ in (("ln1", "layer_norm1"), ("ln2", "layer_norm2")):
            sd[q + f"{b_}.weight"] = w[p + f"{a}.weight"]
            sd[q + f"{b_}.bias"] = w[p + f"{a}.bias"]
        for f in ("fc1", "fc2"):
            sd[q + f"mlp.{f}.weight"] = w[p + f"mlp.{f}.weight"]
            sd[q + f"mlp.{f}.bias"] = w[p + f"mlp.{f}.bias"]
    _load(vpm, sd)

    E = cfg.out_dim
    rs = Resampler2_5(num_queries=cfg.out_tokens, embed_dim=E, num_heads=E // 128, kv_dim=D).float().eval()
    assert E // 128 == cfg.out_heads
    rsd = {"query": w["rs.query"], "proj": w["rs.proj"], "kv_proj.weight": w["rs.kv_proj.weight"],
           "attn.in_proj_weight": torch.cat([w[f"rs.attn.{m}.weight"] for m in "qkv"]),
           "attn.in_proj_bias": torch.cat([w[f"rs.attn.{m}.bias"] for m in "qkv"]),
           "attn.out_proj.weight": w["rs.attn.o.weight"], "attn.out_proj.bias": w["rs.attn.o.bias"]}
    for ln in ("ln_q", "ln_kv", "ln_post"):
        rsd[f"{ln}.weight"] = w[f"rs.{ln}.weight"]
        rsd[f"{ln}.bias"] = w[f"rs.{ln}.bias"]
    _load(rs, rsd)
    with torch.no_grad():
        x = vpm(pixel_values=pixel_values(cfg, tiles)).last_hidden_state
        n = tiles.shape[0]
        # the resampler's own sincos cache must equal the oracle's rs.pos_embed
        own = rs.pos_embed[:grid, :grid, :].reshape(grid * grid, -1).float()
        pos_err = float((own - w["rs.pos_embed"]).abs().max())
        return rs(x, torch.tensor([[grid, grid]] * n)), pos_err


def public_internvl2(cfg, w: dict, tiles: torch.Tensor) -> torch.Tensor:
    from transformers.models.internvl.configuration_internvl import InternVLConfig, InternVLVisionConfig
    from transformers.models.internvl.modeling_internvl import (InternVLModel, InternVLMultiModalProjector,
                                                                InternVLVisionModel)

    D, L = cfg.hidden, cfg.layers
    vcfg = InternVLVisionConfig(hidden_size=D, intermediate_size=cfg.mlp, num_hidden_layers=L,
                                num_attention_heads=cfg.heads, num_channels=cfg.channels,
                                image_size=[cfg.image_size, cfg.image_size], patch_size=[cfg.patch_size] * 2,
                                attention_bias=True, use_qk_norm=False, norm_type="layer_norm",
                                layer_norm_eps=cfg.ln_eps, hidden_act="gelu", use_mean_pooling=True,
                                layer_scale_init_value=0.1, use_absolute_position_embeddings=True,
                                attention_dropout=0.0, projection_dropout=0.0, hidden_dropout_prob=0.0)
    vcfg._attn_implementation = "eager"
    vit = InternVLVisionModel(vcfg).eval()
    sd = {"embeddings.cls_token": w["cls_token"].view(1, 1, D),
          "embeddings.position_embeddings": w["pos_embed"].unsqueeze(0),
          "embeddings.patch_embeddings.projection.weight": w["patch_embed.weight"],
          "embeddings.patch_embeddings.projection.bias": w["patch_embed.bias"]}
    for l in range(L):
        p, q = f"layers.{l}.", f"encoder.layer.{l}."
        qw, kw, vw = w[p + "attn.qkv.weight"].split(D)
        qb, kb, vb = w[p + "attn.qkv.bias"].split(D)
        sd.update({q + "attention.q_proj.weight": qw, q + "attention.q_proj.bias": qb,
                   q + "attention.k_proj.weight": kw, q + "attention.k_proj.bias": kb,
                   q + "attention.v_proj.weight": vw, q + "attention.v_proj.bias": vb,
                   q + "attention.projection_layer.weight": w[p + "attn.o.weight"],
                   q + "attention.projection_layer.bias": w[p + "attn.o.bias"],
                   q + "layernorm_before.weight": w[p + "ln1.weight"], q + "layernorm_before.bias": w[p + "ln1.bias"],
                   q + "layernorm_after.weight": w[p + "ln2.weight"], q + "layernorm_after.bias": w[p + "ln2.bias"],
                   q + "lambda_1": w[p + "ls1"], q + "lambda_2": w[p + "ls2"],
                   q + "mlp.fc1.weight": w[p + "mlp.fc1.weight"], q + "mlp.fc1.bias": w[p + "mlp.fc1.bias"],
                   q + "mlp.fc2.weight": w[p + "mlp.fc2.weight"], q + "mlp.fc2.bias": w[p + "mlp.fc2.bias"]})
    _load(vit, sd)
    full = InternVLConfig(vision_config=vcfg.to_dict(),
                          text_config={"model_type": "qwen2", "hidden_size": cfg.out_dim},
                          downsample_ratio=0.5, projector_hidden_act="gelu")
    proj = InternVLMultiModalProjector(full).eval()
    _load(proj, {"layer_norm.weight": w["mlp1.ln.weight"], "layer_norm.bias": w["mlp1.ln.bias"],
                 "linear_1.weight": w["mlp1.fc1.weight"], "linear_1.bias": w["mlp1.fc1.bias"],
                 "linear_2.weight": w["mlp1.fc2.weight"], "linear_2.bias": w["mlp1.fc2.bias"]})
    with torch.no_grad():
        # InternVLModel.get_image_features with vision_feature_layer -1, strategy "default"
        x = vit(pixel_values=pixel_values(cfg, tiles)).last_hidden_state[:, 1:, :]
        n, t, c = x.shape
        g = int(t ** 0.5)
        x = InternVLModel.pixel_shuffle(None, x.reshape(n, g, g, c), scale_factor=0.5)
        return proj(x.reshape(n, -1, x.shape[-1])), 0.0


def sample_positions(numel: int, k: int = SAMPLES) -> torch.Tensor:
    """Deterministic, well-spread flat indices: a fixed odd stride through the tensor."""
    stride = max(1, numel // k) | 1
    return torch.arange(0, numel, stride)[:k]


def record(name: str, cfg, fn) -> dict:
    torch.manual_seed(0)
    w = canonical_weights(cfg, SEED)
    tiles = golden_tiles(cfg)
    pub, pos_err = fn(cfg, w, tiles)
    ora = oe.encode(cfg, w, tiles)
    assert pub.shape == ora.shape, (pub.shape, ora.shape)
    err = oe.relerr(ora, pub)
    flat = pub.reshape(-1).double()
    idx = sample_positions(flat.numel())
    print(f"{name}: layers {cfg.layers}, {tuple(pub.shape)}, oracle vs public relerr {err:.3e}, "
          f"pos table err {pos_err:.1e}")
    return {"config": cfg.name, "layers": cfg.layers, "weight_seed": SEED, "tile_seed": TILE_SEED,
            "n_tiles": N_TILES, "shape": list(pub.shape), "oracle_relerr": err, "pos_table_maxabs": pos_err,
            "max_abs": float(flat.abs().max()), "sum": float(flat.sum()), "abs_sum": float(flat.abs().sum()),
            "sample_stride": int(idx[1] - idx[0]), "samples": [float(v) for v in flat[idx].float()]}


def main() -> None:
    torch.set_num_threads(max(1, torch.get_num_threads()))
    import transformers
    import vllm
    out = {"generator": "tests/golden/make_encoder_golden.py",
           "public_impls": {"transformers": transformers.__version__, "vllm": vllm.__version__,
                            "minicpm-v-2.6": "transformers Idefics2VisionTransformer + vllm minicpmv.Resampler2_5",
                            "internvl2-8b": "transformers InternVLVisionModel + InternVLModel.pixel_shuffle + "
                                            "InternVLMultiModalProjector"},
           "models": {}}
    out["models"]["siglip"] = record("minicpm-v-2.6", SIGLIP_MINICPM, public_minicpmv26)
    out["models"]["internvit"] = record("internvl2-8b", INTERNVIT_300M, public_internvl2)
    for m in out["models"].values():
        assert m["oracle_relerr"] <= 1e-5, m["oracle_relerr"]
        assert m["pos_table_maxabs"] <= 1e-6
    OUT.write_text(json.dumps(out, indent=0) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
