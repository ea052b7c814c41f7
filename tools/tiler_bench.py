"""Tiler timing: one 4032x3024 photo -> the model's tiles on the GPU."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.tiler import tile_image  # noqa: E402

img = torch.randint(0, 256, (3024, 4032, 3), dtype=torch.uint8, device="cuda")
for model in ("minicpm-v-2.6", "internvl2-8b"):
    for _ in range(3):
        t = tile_image(img, model)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        tile_image(img, model, out=t)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"{model}: {t.shape[0]} tiles in {ms * 1e3:.1f} us ({img.numel() / ms / 1e6:.0f} GB/s of source image)")
