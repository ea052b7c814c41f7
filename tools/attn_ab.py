"""Attention timing for A/B runs: python tools/attn_ab.py [ones]  (library from EPD_LIB_PATH)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402


def timeit(fn, iters=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


tag = Path(os.environ.get("EPD_LIB_PATH", "libepd.so")).stem
dev = torch.device("cuda")
for (B, H, T, Dv) in [(10, 16, 1024, 72), (12, 16, 1025, 64)]:
    qkv = torch.randn(B * T, 3 * H * Dv, device=dev).to(torch.bfloat16)
    q, k, v = qkv[:, :H * Dv], qkv[:, H * Dv:2 * H * Dv], qkv[:, 2 * H * Dv:]
    out = torch.empty(B * T, H * Dv, device=dev, dtype=torch.bfloat16)
    ms = timeit(lambda: kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5, out=out))
    fl = 4 * B * H * T * T * Dv
    print(f"{tag:6s} B={B} T={T} Dv={Dv}: {ms * 1e3:7.1f} us {fl / ms / 1e9:6.1f} TF/s")
