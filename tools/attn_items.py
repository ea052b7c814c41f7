"""Attention kernel time vs image count and item schedule (EPD_ATTN_SPLIT=auto/0/1 runs
set by the caller). Launches are queued behind a device sleep so the events time the
kernels back to back, not the Python launch path.

usage: EPD_ATTN_SPLIT=<mode> python tools/attn_items.py [siglip|internvit]"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402


def main():
    fam = sys.argv[1] if len(sys.argv) > 1 else "siglip"
    H, T, Dv = (16, 1024, 72) if fam == "siglip" else (16, 1025, 64)
    dev = torch.device("cuda")
    res = []
    for B in (1, 2, 3, 5, 10):
        qkv = torch.randn(B * T, 3 * H * Dv, device=dev).to(torch.bfloat16)
        q, k, v = qkv[:, :H * Dv], qkv[:, H * Dv:2 * H * Dv], qkv[:, 2 * H * Dv:]
        out = torch.empty(B * T, H * Dv, device=dev, dtype=torch.bfloat16)
        f = lambda: kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5, out=out)  # noqa: E731
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        n = 40
        torch.cuda._sleep(100_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            f()
        e.record()
        torch.cuda.synchronize()
        res.append(f"B={B} {s.elapsed_time(e) / n * 1e3:6.1f}us")
    print(f"{fam} split={os.environ.get('EPD_ATTN_SPLIT', 'auto')}: " + " | ".join(res))


if __name__ == "__main__":
    main()
