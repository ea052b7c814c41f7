"""Model geometry for the encode path.

Two kinds of numbers live here:

* the reference's own catalog values (``disaggsim/data/models.cfg:6-40``) that the
  path must agree with bit-exactly: tiles per image resolution (``patch_table``),
  tokens per tile (``tokens_per_patch``), MM-token width (``hidden_dim``) and the
  KV geometry (``num_layers``, ``kv_heads``, ``head_dim``) used for byte counts;
* the encoder shapes (ViT width/depth/heads, MLP width, resampler/projector),
  which the reference does not carry (it has only ``encoder_params``); they follow
  the public model cards of SigLIP-so400m (MiniCPM-V 2.6) and InternViT-300M
  (InternVL2-8B), cf. SURVEY.md section 2b.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from ._lib import FAMILY_INTERNVIT_MLP, FAMILY_SIGLIP_RESAMPLER

SEED = 20260808  # reference preset seed (presets.py:149)


@dataclass(frozen=True)
class ModelGeometry:
    """Reference catalog entry (models.cfg) fields the encode path depends on."""

    name: str
    num_layers: int
    kv_heads: int
    head_dim: int
    hidden_dim: int
    tokens_per_patch: int
    max_context_tokens: int
    patch_table: dict = field(default_factory=dict)
    bytes_per_param: int = 2

    def kv_bytes_per_token(self) -> int:  # models.py:128-130
        return 2 * self.num_layers * self.kv_heads * self.head_dim * self.bytes_per_param

    def mm_bytes_per_token(self) -> int:  # models.py:133-135
        return self.hidden_dim * self.bytes_per_param

    def tiles_for_image(self, resolution) -> int:  # models.py:138-143
        try:
            return self.patch_table[tuple(resolution)]
        except KeyError:
            raise UnknownResolution(f"{self.name}: no patch count for resolution {tuple(resolution)}") from None

    def tokens_for_request(self, images, prompt_tokens: int) -> tuple[int, int]:  # models.py:146-155
        mm = sum(self.tiles_for_image(r) * self.tokens_per_patch for r in images)
        return mm, mm + prompt_tokens


class UnknownResolution(KeyError):
    """Mirror of disaggsim.models.UnknownResolution (models.py:53-54)."""


MINICPM_V26 = ModelGeometry(
    name="minicpm-v-2.6", num_layers=28, kv_heads=4, head_dim=128, hidden_dim=3584,
    tokens_per_patch=64, max_context_tokens=32768,
    patch_table={(313, 234): 1, (787, 444): 3, (4032, 3024): 10})
INTERNVL2_8B = ModelGeometry(
    name="internvl2-8b", num_layers=32, kv_heads=8, head_dim=128, hidden_dim=4096,
    tokens_per_patch=256, max_context_tokens=65536,
    patch_table={(313, 234): 13, (787, 444): 3, (4032, 3024): 13})
# PR1 oracle geometry: the reference test fixture toy_model (tests/conftest.py:7-22) with a
# 64x64 image mapped to 4 tiles.
TOY = ModelGeometry(
    name="toy", num_layers=2, kv_heads=2, head_dim=4, hidden_dim=8, tokens_per_patch=4,
    max_context_tokens=10_000, patch_table={(64, 64): 4, (100, 100): 6, (200, 200): 12})


@dataclass(frozen=True)
class EncoderConfig:
    """Vision-encoder shape, passed to the C ABI as epd_encoder_desc_t."""

    name: str
    family: int
    image_size: int
    patch_size: int
    hidden: int
    layers: int
    heads: int
    mlp: int
    out_tokens: int
    out_dim: int
    out_heads: int
    ln_eps: float
    mean: tuple
    std: tuple
    channels: int = 3
    geometry: ModelGeometry = MINICPM_V26

    @property
    def tile_bytes(self) -> int:
        return self.image_size * self.image_size * self.channels

    @property
    def out_bytes_per_tile(self) -> int:
        return self.out_tokens * self.out_dim * 2

    def with_layers(self, layers: int) -> "EncoderConfig":
        from dataclasses import replace
        return replace(self, layers=layers, name=f"{self.name}-L{layers}")


# MiniCPM-V 2.6 vision tower: SigLIP-so400m-patch14 (27 layers, 1152 wide, 16 heads x 72,
# MLP 4304, GELU-tanh, LN eps 1e-6) on 448x448 slices + perceiver resampler (64 queries,
# 3584 wide, 28 heads x 128). Image normalisation mean = std = 0.5.
SIGLIP_MINICPM = EncoderConfig(
    name="siglip400m-minicpmv26", family=FAMILY_SIGLIP_RESAMPLER, image_size=448, patch_size=14,
    hidden=1152, layers=27, heads=16, mlp=4304, out_tokens=64, out_dim=3584, out_heads=28,
    ln_eps=1e-6, mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5), geometry=MINICPM_V26)

# InternVL2-8B vision tower: InternViT-300M-448px (24 layers, 1024 wide, 16 heads x 64,
# MLP 4096, GELU, LN eps 1e-6, layer scale, CLS) + pixel shuffle 0.5 + mlp1 -> 256 x 4096.
INTERNVIT_300M = EncoderConfig(
    name="internvit300m-internvl2-8b", family=FAMILY_INTERNVIT_MLP, image_size=448, patch_size=14,
    hidden=1024, layers=24, heads=16, mlp=4096, out_tokens=256, out_dim=4096, out_heads=0,
    ln_eps=1e-6, mean=(0.485, 0.456, 0.406), std=(0.229, 0.224, 0.225), geometry=INTERNVL2_8B)

# PR1 tiny ViT (BASELINE config 1): 56x56 tiles (4x4 patches), 2 layers, emits the toy
# model's 4 tokens x 8 dims per tile.
TINY_VIT = EncoderConfig(
    name="tiny-vit", family=FAMILY_SIGLIP_RESAMPLER, image_size=56, patch_size=14, hidden=64,
    layers=2, heads=1, mlp=128, out_tokens=4, out_dim=8, out_heads=1, ln_eps=1e-6,
    mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5), geometry=TOY)

CONFIGS = {c.name: c for c in (SIGLIP_MINICPM, INTERNVIT_300M, TINY_VIT)}
