"""CPU tier: the fp32 encoder oracle is pinned to the public model implementations.

``tests/golden/encoder_golden.json`` was produced by ``tests/golden/make_encoder_golden.py``
from transformers' Idefics2VisionTransformer + vLLM's MiniCPM-V ``Resampler2_5`` and
transformers' InternVLVisionModel + pixel_shuffle + InternVLMultiModalProjector, loaded with
the canonical random-init weights. Here the oracle re-runs at full depth on the same tiles
and must agree with the recorded public outputs within 1e-5 (fp32)."""
import json
from pathlib import Path

import pytest
import torch

from paper_2501_05460_b200.configs import CONFIGS, SEED
from paper_2501_05460_b200.weights import canonical_weights

GOLDEN = Path(__file__).resolve().parent / "golden" / "encoder_golden.json"


def golden():
    return json.loads(GOLDEN.read_text())


def golden_tiles(cfg, g):
    gen = torch.Generator().manual_seed(g["tile_seed"])
    return torch.randint(0, 256, (g["n_tiles"], cfg.image_size, cfg.image_size, cfg.channels), dtype=torch.uint8,
                         generator=gen)


def sampled(y: torch.Tensor, g) -> torch.Tensor:
    flat = y.reshape(-1).float()
    idx = torch.arange(0, flat.numel(), g["sample_stride"])[:len(g["samples"])]
    return flat[idx]


def test_fixture_records_pinned_oracle():
    d = golden()
    assert set(d["models"]) == {"siglip", "internvit"}
    for m in d["models"].values():
        assert m["oracle_relerr"] <= 1e-5
        assert m["weight_seed"] == SEED
        assert len(m["samples"]) >= 2048


@pytest.mark.parametrize("key", ["siglip", "internvit"])
def test_oracle_matches_public_implementation(key):
    import oracle.encoders as oe
    g = golden()["models"][key]
    cfg = CONFIGS[g["config"]]
    assert cfg.layers == g["layers"]
    torch.set_num_threads(max(1, torch.get_num_threads()))
    w = canonical_weights(cfg, SEED)
    y = oe.encode(cfg, w, golden_tiles(cfg, g))
    assert list(y.shape) == g["shape"]
    ref = torch.tensor(g["samples"])
    err = float((sampled(y, g) - ref).abs().max()) / g["max_abs"]
    assert err <= 1e-5, f"oracle drifted from the public {key} implementation: {err:.3e}"
    assert float(y.double().sum()) == pytest.approx(g["sum"], rel=1e-4, abs=1e-3 * g["max_abs"])
