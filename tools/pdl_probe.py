"""Encode time per request, graphs on/off, for PDL A/B (EPD_PDL env)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import _lib  # noqa: E402
from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402

for cfg, n in [(INTERNVIT_300M, 12), (SIGLIP_MINICPM, 10)]:
    enc = VisionEncoder(cfg, 0, max_tiles=n)
    tiles = torch.randint(0, 256, (n, cfg.image_size, cfg.image_size, 3), dtype=torch.uint8, device="cuda")
    res = []
    for graphs in (1, 0):
        _lib.call("epd_encoder_set_graphs", enc._h, graphs)
        for _ in range(3):
            enc.encode(tiles)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            enc.encode(tiles)
        e.record()
        torch.cuda.synchronize()
        res.append(f"graphs={graphs}: {s.elapsed_time(e) / 10:.2f} ms")
    print(f"PDL={os.environ.get('EPD_PDL', '1')} {cfg.name}: " + " | ".join(res))
    enc.close()
