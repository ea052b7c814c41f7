"""End-to-end encoder parity on the B200: the sm_100a encode path (through the
C ABI) against the fp32 CPU oracle on identical random-init weights and
synthetic uint8 tiles.

Tolerance (BASELINE.json north_star): max|y - y_ref| / max|y_ref| <= 1e-2 (bf16 compute).
"""
import pytest
import torch

from paper_2501_05460_b200.configs import INTERNVIT_300M, SEED, SIGLIP_MINICPM, TINY_VIT

pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2

_cache = {}


def _setup(cfg, cuda, max_tiles=4):
    key = (cfg.name, max_tiles)
    if key not in _cache:
        from paper_2501_05460_b200.encoder import VisionEncoder, canonical_weights
        w = canonical_weights(cfg, SEED)
        enc = VisionEncoder(cfg, cuda, max_tiles=max_tiles, weights=w)
        _cache[key] = (w, enc)
    return _cache[key]


def _tiles(cfg, n, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n, cfg.image_size, cfg.image_size, cfg.channels), dtype=torch.uint8,
                         generator=g)


@pytest.mark.parametrize("cfg,n", [
    (TINY_VIT, 4),                         # PR1 config: 1 request x 4 tiles
    (SIGLIP_MINICPM.with_layers(2), 2),
    (INTERNVIT_300M.with_layers(2), 2),
    (SIGLIP_MINICPM, 1),                   # full 27-layer SigLIP + resampler
    (INTERNVIT_300M, 1),                   # full 24-layer InternViT + mlp1
])
def test_encoder_matches_oracle(cuda, cfg, n):
    import oracle.encoders as oe
    w, enc = _setup(cfg, cuda)
    tiles = _tiles(cfg, n, seed=SEED + n)
    y = enc.encode(tiles.to(cuda))
    torch.cuda.synchronize()
    # The deployed weights are bf16: the oracle computes the same (bf16-valued) weights in fp32.
    ref = oe.encode(cfg, oe.bf16_weights(w), tiles)
    assert y.shape == (n, cfg.out_tokens, cfg.out_dim)
    err = oe.relerr(y, ref)
    err32 = oe.relerr(y, oe.encode(cfg, w, tiles))
    print(f"{cfg.name}: n={n} relerr={err:.3e} (vs fp32-valued weights {err32:.3e})")
    assert err <= TOL_BF16


def test_encoder_chunking_and_tile_independence(cuda):
    """Tiles are independent sequences: encoding [a, b, c] in one call (split across
    max_tiles chunks) equals encoding each alone, bit for bit."""
    cfg = SIGLIP_MINICPM.with_layers(2)
    w, enc = _setup(cfg, cuda, max_tiles=2)
    tiles = _tiles(cfg, 3, seed=7).to(cuda)
    together = enc.encode(tiles)
    alone = torch.cat([enc.encode(tiles[i:i + 1].contiguous()) for i in range(3)])
    torch.cuda.synchronize()
    assert torch.equal(together, alone)


def test_graph_replay_equals_direct_launches(cuda):
    """The CUDA-graph replay path (default) is bit-identical to direct launches."""
    from paper_2501_05460_b200 import _lib
    cfg = SIGLIP_MINICPM.with_layers(2)
    w, enc = _setup(cfg, cuda, max_tiles=2)
    tiles = _tiles(cfg, 3, seed=9).to(cuda)
    g1 = enc.encode(tiles)
    g2 = enc.encode(tiles)
    _lib.call("epd_encoder_set_graphs", enc._h, 0)
    d = enc.encode(tiles)
    _lib.call("epd_encoder_set_graphs", enc._h, 1)
    torch.cuda.synchronize()
    assert torch.equal(g1, d) and torch.equal(g2, d)


def test_encoder_rejects_bad_input(cuda):
    cfg = TINY_VIT
    _, enc = _setup(cfg, cuda)
    with pytest.raises(ValueError):
        enc.encode(torch.zeros(1, 8, 8, 3, dtype=torch.uint8, device=cuda))
    with pytest.raises(ValueError):
        enc.encode_latency(None, -1)
    assert enc.encode_latency(None, 0) == 0.0


# ---- fp32 check mode (north star: <= 1e-4 for an fp32 check mode) -----------------
TOL_FP32 = 1e-4


@pytest.mark.parametrize("cfg,n", [
    (TINY_VIT, 4),
    (SIGLIP_MINICPM.with_layers(2), 2),
    (INTERNVIT_300M.with_layers(2), 2),
    (SIGLIP_MINICPM, 1),
    (INTERNVIT_300M, 1),
])
def test_fp32_check_mode_matches_oracle(cuda, cfg, n):
    """The fp32 check path runs the deployed layouts and fusions (head padding, fused
    QKV, folded key positions / CLS row, pixel-shuffle gather) without rounding; it
    must match the fp32 oracle on the fp32 weights to 1e-4."""
    import oracle.encoders as oe
    from paper_2501_05460_b200.encoder import VisionEncoder, canonical_weights
    w = canonical_weights(cfg, SEED)
    enc = VisionEncoder(cfg, cuda, max_tiles=4, weights=w, check_fp32=True)
    tiles = _tiles(cfg, n, seed=SEED + 100 + n)
    y = enc.encode_f32(tiles.to(cuda))
    yb = enc.encode(tiles.to(cuda))
    torch.cuda.synchronize()
    ref = oe.encode(cfg, w, tiles)
    err = oe.relerr(y, ref)
    errb = oe.relerr(yb, oe.encode(cfg, oe.bf16_weights(w), tiles))
    print(f"{cfg.name}: fp32 check relerr={err:.3e}, bf16 path relerr={errb:.3e}")
    assert y.dtype == torch.float32 and y.shape == (n, cfg.out_tokens, cfg.out_dim)
    assert err <= TOL_FP32
    assert errb <= TOL_BF16
    enc.close()


def test_fp32_check_mode_requires_opt_in(cuda):
    _, enc = _setup(TINY_VIT, cuda)
    with pytest.raises(RuntimeError):
        enc.encode_f32(torch.zeros(1, TINY_VIT.image_size, TINY_VIT.image_size, 3, dtype=torch.uint8, device=cuda))


# ---- parity at the benched request sizes (C2 = 10 SigLIP tiles, C5 = 13 InternViT tiles)
@pytest.mark.parametrize("cfg,n", [(SIGLIP_MINICPM, 10), (INTERNVIT_300M, 13)])
def test_encoder_matches_oracle_at_bench_size(cuda, cfg, n):
    """The whole benched request in one encoder call (max_tiles = n, the bench's GEMM tile
    schedules and attention item mix) against the fp32 oracle on the bf16-valued weights."""
    import oracle.encoders as oe
    from paper_2501_05460_b200.stage import tiles_for_request
    w, enc = _setup(cfg, cuda, max_tiles=n)
    tiles = tiles_for_request(n, cfg, seed=SEED)
    y = enc.encode(tiles.to(cuda))
    torch.cuda.synchronize()
    torch.set_num_threads(max(1, torch.get_num_threads()))
    err = oe.relerr(y, oe.encode(cfg, oe.bf16_weights(w), tiles))
    print(f"{cfg.name}: n={n} relerr={err:.3e}")
    assert err <= TOL_BF16


@pytest.mark.parametrize("cfg,n", [(SIGLIP_MINICPM, 10), (INTERNVIT_300M, 13)])
def test_irp_shards_equal_slices_of_the_whole_request(cuda, cfg, n):
    """IRP at any width returns the single-GPU tokens bit for bit: every shard encode of
    irp_shard(n, w), w = 2/4/8, equals its slice of the n-tile encode (batch invariance
    across the 1/2/3/5/7-tile GEMM and attention schedules)."""
    from paper_2501_05460_b200.routing import shard_ranges
    from paper_2501_05460_b200.stage import tiles_for_request
    _, enc = _setup(cfg, cuda, max_tiles=n)
    tiles = tiles_for_request(n, cfg, seed=SEED + 1).to(cuda)
    whole = enc.encode(tiles)
    for w_ in (2, 4, 8):
        for first, count in shard_ranges(n, w_):
            if count:
                part = enc.encode(tiles[first:first + count].contiguous())
                assert torch.equal(part, whole[first:first + count]), (w_, first, count)
    torch.cuda.synchronize()


@pytest.mark.parametrize("key", ["siglip", "internvit"])
def test_encoder_matches_public_implementation(cuda, key):
    """Direct pin against the public model code: the B200 tokens vs the outputs of
    transformers' Idefics2VisionTransformer + vLLM Resampler2_5 / transformers' InternVL
    vision tower + projector recorded in tests/golden/encoder_golden.json (fp32-valued
    weights; bf16 compute budget 1e-2)."""
    import json
    from pathlib import Path

    from paper_2501_05460_b200.configs import CONFIGS
    g = json.loads((Path(__file__).resolve().parent / "golden" / "encoder_golden.json").read_text())["models"][key]
    cfg = CONFIGS[g["config"]]
    _, enc = _setup(cfg, cuda, max_tiles=4)
    gen = torch.Generator().manual_seed(g["tile_seed"])
    tiles = torch.randint(0, 256, (g["n_tiles"], cfg.image_size, cfg.image_size, cfg.channels), dtype=torch.uint8,
                          generator=gen)
    y = enc.encode(tiles.to(cuda)).float().cpu().reshape(-1)
    idx = torch.arange(0, y.numel(), g["sample_stride"])[:len(g["samples"])]
    err = float((y[idx] - torch.tensor(g["samples"])).abs().max()) / g["max_abs"]
    print(f"{key}: B200 vs public implementation (sampled) relerr {err:.3e}")
    assert err <= TOL_BF16
