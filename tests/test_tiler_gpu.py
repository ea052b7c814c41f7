"""On-device tiler vs the reference tile counts and a torch fp32 antialiased-bilinear
reference (interpolate(..., antialias=True) on the same image), within 1 LSB."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref_tiles(img, model, S=448):
    from paper_2501_05460_b200.tiler import plan
    H, W, _ = img.shape
    cols, rows, thumb, thumb_first = plan(model, W, H)
    x = img.permute(2, 0, 1)[None].float()

    def rs(h, w):
        return torch.nn.functional.interpolate(x, size=(h, w), mode="bilinear", align_corners=False,
                                               antialias=True)[0].permute(1, 2, 0)
    grid = []
    if cols * rows:
        big = rs(rows * S, cols * S)
        grid = [big[j * S:(j + 1) * S, i * S:(i + 1) * S] for j in range(rows) for i in range(cols)]
    th = [rs(S, S)] if thumb else []
    tiles = th + grid if thumb_first else grid + th
    return torch.stack(tiles).round().clamp(0, 255)


@pytest.mark.parametrize("model,w,h", [("minicpm-v-2.6", 4032, 3024), ("minicpm-v-2.6", 787, 444),
                                       ("minicpm-v-2.6", 313, 234), ("internvl2-8b", 4032, 3024),
                                       ("internvl2-8b", 787, 444), ("internvl2-8b", 313, 234)])
def test_tile_image_matches_reference(cuda, model, w, h):
    from paper_2501_05460_b200.configs import INTERNVL2_8B, MINICPM_V26
    from paper_2501_05460_b200.tiler import tile_image
    g = torch.Generator().manual_seed(w + h)
    # smooth-ish synthetic photo: low-frequency pattern + noise (exercises every filter tap)
    yy, xx = torch.meshgrid(torch.arange(h, dtype=torch.float32), torch.arange(w, dtype=torch.float32), indexing="ij")
    base = 127 + 60 * torch.sin(xx / 37.0)[..., None] * torch.cos(yy / 23.0)[..., None] * torch.tensor([1.0, 0.7, -0.5])
    img = (base + torch.randn(h, w, 3, generator=g) * 25).round().clamp(0, 255).to(torch.uint8)
    tiles = tile_image(img.to(cuda), model)
    torch.cuda.synchronize()
    geom = MINICPM_V26 if model.startswith("minicpm") else INTERNVL2_8B
    assert tiles.shape == (geom.patch_table[(w, h)], 448, 448, 3)
    ref = _ref_tiles(img.to(cuda), model)
    diff = (tiles.float() - ref).abs()
    assert float(diff.max()) <= 1.0
    assert float((diff > 0).float().mean()) < 1e-3  # only rounding ties may differ


def test_stage_process_image_equals_tiles_path(cuda):
    """process_image (upload photo -> GPU tiles -> encode) packs exactly the tokens that
    encoding the same GPU-cut tiles directly gives."""
    from paper_2501_05460_b200.configs import TINY_VIT
    from paper_2501_05460_b200.encoder import VisionEncoder
    from paper_2501_05460_b200.stage import EncodeStage
    from paper_2501_05460_b200.tiler import tile_image
    enc = VisionEncoder(TINY_VIT, cuda, max_tiles=16)
    stage = EncodeStage(enc, cuda)
    g = torch.Generator().manual_seed(3)
    img = torch.randint(0, 256, (1100, 1500, 3), dtype=torch.uint8, generator=g).pin_memory()
    res = stage.process_image(img, "minicpm-v-2.6")
    tiles = tile_image(img.to(cuda), "minicpm-v-2.6", tile=TINY_VIT.image_size)
    ref = enc.encode(tiles)
    torch.cuda.synchronize()
    assert res.tokens.shape[0] == tiles.shape[0] and torch.equal(res.tokens, ref)
