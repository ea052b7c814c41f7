"""Per-event timeline of one attention CTA. Needs a trace build:
   tools/build_variant.sh libT -DEPD_ATTN_TRACE && EPD_LIB_PATH=ab/libT.so python tools/attn_trace.py"""
import ctypes as C
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import _lib, kernels  # noqa: E402

dev = torch.device("cuda")
B, H, T, Dv, Dp = 10, 16, 1024, 72, 80
qkv = torch.randn(B * T, 3 * H * Dv, device=dev).to(torch.bfloat16)
q, k, v = qkv[:, :H * Dv], qkv[:, H * Dv:2 * H * Dv], qkv[:, 2 * H * Dv:]
out = torch.empty(B * T, H * Dv, device=dev, dtype=torch.bfloat16)
L = _lib.lib()
L.epd_debug_trace.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_uint * 1024)()
for it in range(3):
    kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5, out=out)
    torch.cuda.synchronize()
L.epd_debug_trace(buf, 1024)
ev = []
for code in range(32):
    for j in range(16):
        for g in range(2):
            x = buf[(code * 16 + j) * 2 + g]
            if x:
                ev.append((x, code, j, g))
ev.sort()
t0 = ev[0][0]
names = {3: "MMA S issue", 4: "MMA S issued", 5: "MMA wait p_ready", 6: "MMA p_ready ok", 7: "MMA PV issue",
         8: "MMA PV issued", 9: "SM wait s_full", 10: "SM s_full ok", 11: "SM S loaded", 12: "SM max done",
         13: "SM bar done", 14: "SM exps done", 15: "SM p_ready (w0)", 16: "SM p_ready (w7)"}
for t, c, j, g in ev:
    print(f"{t - t0:8d}  {names.get(c, c):18s} j={j} g={g}")
at = defaultdict(dict)
for t, c, j, g in ev:
    at[(g, j)][c] = t
ph = defaultdict(list)
for (g, j), d in at.items():
    for a, b2, name in [(10, 11, "tmem ld S"), (11, 12, "max"), (12, 13, "bar"), (13, 14, "rescale+exps"),
                        (14, 15, "st P + arrive"), (10, 15, "softmax total"), (15, 6, "p_ready->MMA sees"),
                        (7, 8, "PV+S issue"), (4, 10, "S commit->SM sees")]:
        if a in d and b2 in d:
            ph[name].append(d[b2] - d[a])
for name, xs in ph.items():
    print(f"{name:20s} mean {sum(xs) / len(xs):8.1f} cycles  (n={len(xs)})")
