"""Device time of one encoder call for small IRP shards (p tiles resident, CUDA-graph
path), median of 20 calls after warm-up. These are the per-rank encode times that set
TTFT at IRP widths 4 and 8 (a 10-tile request leaves 1-3 tiles per rank).

usage: python tools/small_shard.py [siglip|internvit] p1,p2,...
"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402


def main():
    fam = sys.argv[1] if len(sys.argv) > 1 else "siglip"
    ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,5,10").split(",")]
    cfg = SIGLIP_MINICPM if fam == "siglip" else INTERNVIT_300M
    enc = VisionEncoder(cfg, 0, max_tiles=max(ps))
    res = []
    for p in ps:
        tiles = torch.randint(0, 256, (p, cfg.image_size, cfg.image_size, 3), dtype=torch.uint8, device="cuda")
        out = torch.empty(p, cfg.out_tokens, cfg.out_dim, dtype=torch.bfloat16, device="cuda")
        for _ in range(5):
            enc.encode(tiles, out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            enc.encode(tiles, out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        med = statistics.median(ts)
        res.append((p, med))
        print(f"{cfg.name} p={p:3d}: {med:.3f} ms  ({med / p:.3f} ms/tile, {p / med * 1e3:.0f} tiles/s)", flush=True)
    return res


if __name__ == "__main__":
    main()
