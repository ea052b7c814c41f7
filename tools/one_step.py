"""One encoder request inside a cudaProfilerStart/Stop range, after warm-up: the ncu target
(`ncu --profile-from-start off ...`). usage: python tools/one_step.py [siglip|internvit] [tiles]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "siglip"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = SIGLIP_MINICPM if fam == "siglip" else INTERNVIT_300M
enc = VisionEncoder(cfg, 0, max_tiles=n)
tiles = torch.randint(0, 256, (n, cfg.image_size, cfg.image_size, 3), dtype=torch.uint8, device="cuda")
for _ in range(3):
    enc.encode(tiles)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
enc.encode(tiles)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
