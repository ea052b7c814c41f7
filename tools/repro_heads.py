"""Minimal repro of a heads-mode projection (debug helper)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402

M, T, H, Dp, S = [int(x) for x in sys.argv[1:6]]
trans = tuple(s == 2 for s in range(S))
a = torch.randn(M, 256, device="cuda").to(torch.bfloat16)
w = torch.randn(S * H * Dp, 256, device="cuda").to(torch.bfloat16)
outs = kernels.linear_heads(a, w, H, Dp, T, S, trans=trans)
torch.cuda.synchronize()
print("ok")
