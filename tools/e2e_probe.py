"""Repeated pipelined e2e loops (C2) to characterise run-to-run variance and attribute the
e2e cost (h2d: uploads only, d2h: readbacks only)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.configs import SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402
from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request  # noqa: E402

cfg, n = SIGLIP_MINICPM, 10
dev = torch.device("cuda", 0)
enc = VisionEncoder(cfg, dev, max_tiles=n)
stage = EncodeStage(enc, dev)
th = tiles_for_request(n, cfg, seed=1).pin_memory()
td = th.to(dev)
oh = torch.empty(n, cfg.out_tokens, cfg.out_dim, dtype=torch.bfloat16).pin_memory()
for _ in range(5):
    stage.process(th, out_host=oh)
    stage.process(None, tiles_dev=td)
torch.cuda.synchronize()
for rep in range(6):
    for mode in ("resident", "e2e", "h2d", "d2h"):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            if mode == "e2e":
                stage.process(th, out_host=oh)
            elif mode == "h2d":
                stage.process(th)
            elif mode == "d2h":
                stage.process(None, tiles_dev=td, out_host=oh)
            else:
                stage.process(None, tiles_dev=td)
        stage.join()
        b.record()
        torch.cuda.synchronize()
        print(f"rep {rep} {mode:8s}: {20 * n / (a.elapsed_time(b) / 1e3):7.1f} tiles/s")
