"""Timeline of one attention CTA (experiment build with -DEPD_ATTN_TRACE=1):
python tools/attn_trace.py   (EPD_LIB_PATH=ab/trace.so)

Prints, per key block of CTA 0's first items, when each softmax warp saw S (s_full), when it
handed P over (p_ready), and when the MMA warp saw p_ready and finished issuing PV + S(j+2),
in SM cycles relative to the first event."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import _lib, kernels  # noqa: E402

dev = torch.device("cuda")
B, H, T, Dv = 10, 16, 1024, 72
qkv = torch.randn(B * T, 3 * H * Dv, device=dev).to(torch.bfloat16)
q, k, v = qkv[:, :H * Dv], qkv[:, H * Dv:2 * H * Dv], qkv[:, 2 * H * Dv:]
out = torch.empty(B * T, H * Dv, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5, out=out)
torch.cuda.synchronize()
buf = np.zeros((8, 8, 48), dtype=np.uint32)
lib = _lib.lib()
lib.epd_debug_attn_trace.argtypes = [C.c_void_p]
assert lib.epd_debug_attn_trace(buf.ctypes.data) == 0
t = buf.astype(np.int64)
t0 = t[0, :, 0].min()
t = (t - t0) & 0xFFFFFFFF
sf, pr, mw, mi = t[0], t[1], t[2, :2], t[3, :2]
print("blk | tile0: sfull(min..max) softmax(max) | tile1: sfull softmax | mma: seen0 issued0 seen1 issued1")
for b in range(48):
    s0, s1 = sf[0:4, b], sf[4:8, b]
    p0, p1 = pr[0:4, b], pr[4:8, b]
    print(f"{b:3d} | {s0.min():7d}..{s0.max():7d} {int((p0 - s0).max()):5d} | {s1.min():7d}..{s1.max():7d} "
          f"{int((p1 - s1).max()):5d} | {mw[0, b]:7d} {mi[0, b]:7d} {mw[1, b]:7d} {mi[1, b]:7d}")
print("\nper softmax warp (warp id = 2 + index; SMSP = warp % 4): s_full seen / p_ready arrive")
for b in range(18, 24):
    print(f"blk {b}: " + "  ".join(f"w{2 + i}:{sf[i, b]}/{pr[i, b]}" for i in range(8)))
print("\nMMA warp: p_ready(b) seen / S(b+2) issued, tile 0 and 1")
for b in range(18, 24):
    print(f"blk {b}: t0 {mw[0, b]}/{mi[0, b]}  t1 {mw[1, b]}/{mi[1, b]}   last arrive t0 {pr[0:4, b].max()} t1 {pr[4:8, b].max()}")

print("\nsoftmax phases per warp (cycles): ld-wait | max+vote | exp loop | st+wait | fence+arrive ; blocks 18-23")
for b in range(18, 24):
    row = []
    for i in range(8):
        s0, ld, mx, ex, st, arr = t[0, i, b], t[4, i, b], t[5, i, b], t[6, i, b], t[7, i, b], t[1, i, b]
        row.append(f"w{2 + i}:{ld - s0}|{mx - ld}|{ex - mx}|{st - ex}|{arr - st}")
    print(f"blk {b}: " + "  ".join(row))
