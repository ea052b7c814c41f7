"""Split-K reduce-add GEMM timing at the LLM prefill shapes (EPD_GEMM_SPLIT forces the count)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402

dev = torch.device("cuda")
line = []
for (M, N, K) in [(662, 3584, 18944), (662, 3584, 3584), (3350, 4096, 14336)]:
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev) * K ** -0.5).to(torch.bfloat16)
    h = torch.zeros(M, N, device=dev)
    for _ in range(5):
        kernels.linear_acc(a, w, h, max_split=16)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(30):
        kernels.linear_acc(a, w, h, max_split=16)
    e.record()
    torch.cuda.synchronize()
    line.append(f"{M}x{N}x{K} {s.elapsed_time(e) / 30 * 1e3:6.1f}us")
print(f"split={os.environ.get('EPD_GEMM_SPLIT', 'auto')}: " + " | ".join(line), flush=True)
