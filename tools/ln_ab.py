"""Residual-stream LayerNorm timing (fp32 in, bf16 out) for A/B runs (library from EPD_LIB_PATH)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402

tag = Path(os.environ.get("EPD_LIB_PATH", "libepd.so")).stem
dev = torch.device("cuda")
res = []
for rows, D in [(10240, 1152), (12300, 1024)]:
    xs = [torch.randn(rows, D, device=dev) for _ in range(4)]  # 4 x 47 MB rotate through the 126 MB L2
    g = torch.ones(D, device=dev, dtype=torch.bfloat16)
    y = torch.empty(rows, D, device=dev, dtype=torch.bfloat16)
    for i in range(5):
        kernels.layernorm_f32(xs[i % 4], g, g, 1e-6, out=y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(100_000_000)  # launches queue behind it: events time kernels, not the host
    s.record()
    for i in range(48):
        kernels.layernorm_f32(xs[i % 4], g, g, 1e-6, out=y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 48
    res.append(f"{rows}x{D}: {ms * 1e3:6.1f} us {rows * D * 6 / ms / 1e6:6.0f} GB/s")
print(f"{tag:6s} " + " | ".join(res))
