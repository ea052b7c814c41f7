"""Pipelined e2e loop of C2 from a 4032x3024 photo (c2i): device tiles/s and host time per call, against the tile-upload loop and the raw H2D rate."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.configs import SIGLIP_MINICPM
from paper_2501_05460_b200.encoder import VisionEncoder
from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request
cfg, n = SIGLIP_MINICPM, 10
dev = torch.device("cuda", 0)
enc = VisionEncoder(cfg, dev, max_tiles=n)
stage = EncodeStage(enc, dev)
g = torch.Generator().manual_seed(1)
img = torch.randint(0, 256, (3024, 4032, 3), dtype=torch.uint8, generator=g).pin_memory()
print("pinned", img.is_pinned())
oh = torch.empty(n, cfg.out_tokens, cfg.out_dim, dtype=torch.bfloat16).pin_memory()
th = tiles_for_request(n, cfg, seed=1).pin_memory()
for _ in range(5):
    stage.process_image(img, cfg.geometry.name, out_host=oh)
torch.cuda.synchronize()
for rep in range(3):
    for mode in ("image", "tiles", "image_noout"):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hts = []
        a.record()
        for _ in range(20):
            t0 = time.perf_counter()
            if mode == "image": stage.process_image(img, cfg.geometry.name, out_host=oh)
            elif mode == "tiles": stage.process(th, out_host=oh)
            else: stage.process_image(img, cfg.geometry.name)
            hts.append((time.perf_counter() - t0) * 1e3)
        stage.join()
        b.record()
        torch.cuda.synchronize()
        print(f"rep {rep} {mode:12s}: {20 * n / (a.elapsed_time(b) / 1e3):7.1f} tiles/s  host ms/call median {sorted(hts)[10]:.2f} max {max(hts):.2f}")
# raw copy bandwidth
buf = torch.empty_like(img, device=dev)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): buf.copy_(img, non_blocking=True)
b.record(); torch.cuda.synchronize()
print("H2D GB/s", 10 * img.numel() / (a.elapsed_time(b) / 1e3) / 1e9)
