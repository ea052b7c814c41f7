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


ones = len(sys.argv) > 1 and sys.argv[1] == "ones"
tag = Path(os.environ.get("EPD_LIB_PATH", "libepd.so")).stem
dev = torch.device("cuda")
for (B, H, T, Dv, Dp) in [(10, 16, 1024, 72, 80), (12, 16, 1025, 64, 64)]:
    q = torch.randn(B * H, T, Dp, device=dev).to(torch.bfloat16)
    k = torch.randn(B * H, T, Dp, device=dev).to(torch.bfloat16)
    v = torch.randn(B * H, T, Dp, device=dev).to(torch.bfloat16)
    if Dp > Dv:
        q[..., Dv:] = 0
        k[..., Dv:] = 0
        v[..., Dv:] = 0
    use_ones = ones and Dv < Dp
    if use_ones:
        v[..., Dv] = 1.0
    out = torch.empty(B * T, H * Dv, device=dev, dtype=torch.bfloat16)
    ms = timeit(lambda: kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5, out=out, v_ones_col=use_ones))
    fl = 4 * B * H * T * T * Dv
    print(f"{tag:6s} ones={int(use_ones)} B={B} T={T} Dv={Dv}: {ms * 1e3:7.1f} us {fl / ms / 1e9:6.1f} TF/s")
