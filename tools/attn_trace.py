"""Print the per-event timeline of one attention CTA (needs a TRACE-instrumented build)."""
import ctypes as C
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import _lib, kernels  # noqa: E402

dev = torch.device("cuda")
B, H, T, Dv, Dp = 10, 16, 1024, 72, 80
q = torch.randn(B * H, T, Dp, device=dev).to(torch.bfloat16)
k = torch.randn(B * H, T, Dp, device=dev).to(torch.bfloat16)
v = torch.randn(B * H, T, Dp, device=dev).to(torch.bfloat16)
out = torch.empty(B * T, H * Dv, device=dev, dtype=torch.bfloat16)
L = _lib.lib()
L.epd_debug_trace.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 8192)()
for it in range(3):
    kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5, out=out)
    torch.cuda.synchronize()
n = L.epd_debug_trace(buf, 8192)
ev = sorted(((b >> 16), (b >> 8) & 0xff, (b >> 2) & 63, b & 3) for b in buf[:n])
t0 = ev[0][0]
names = {3: "S: issue", 4: "S: issued", 5: "PV: wait p_ready", 6: "PV: wait v_full", 7: "PV: issue",
         8: "PV: issued"}
for t, c, j, g in ev:
    print(f"{t - t0:8d}  {names[c]:14s} j={j} g={g}")
