"""Per-launch breakdown of one encoder forward (CUDA events around every launch).

usage: python tools/enc_breakdown.py [siglip|internvit] [tiles] [cta_policy]
Prints per-kernel-role totals (summed over layers) with achieved TFLOP/s.
"""
import ctypes as C
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import _lib  # noqa: E402
from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402

ROLES_LAYER = ["ln1", "qkv", "attn", "o_proj", "ln2", "fc1", "fc2"]
ROLES_SIGLIP_TAIL = ["post_ln", "kv_proj", "ln_kv", "kv_in", "rs_attn", "rs_o", "ln_post", "proj"]
ROLES_INTERN_TAIL = ["shuffle_ln", "mlp_fc1", "mlp_fc2"]


def main():
    fam = sys.argv[1] if len(sys.argv) > 1 else "siglip"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    if len(sys.argv) > 3:
        _lib.call("epd_set_gemm_cta_group", int(sys.argv[3]))
    cfg = SIGLIP_MINICPM if fam == "siglip" else INTERNVIT_300M
    enc = VisionEncoder(cfg, 0, max_tiles=n)
    tiles = torch.randint(0, 256, (n, cfg.image_size, cfg.image_size, 3), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        enc.encode(tiles)
    torch.cuda.synchronize()
    _lib.call("epd_encoder_profile", enc._h, 1)
    reps = 3
    agg = defaultdict(lambda: [0.0, 0.0, 0])
    for _ in range(reps):
        torch.cuda._sleep(60_000_000)  # launches queue behind it: events time kernels, not host gaps
        enc.encode(tiles)
        nc = 5
        ms = (C.c_double * nc)(); fl = (C.c_double * nc)(); by = (C.c_double * nc)(); cnt = (C.c_int64 * nc)()
        _lib.call("epd_encoder_profile_read", enc._h, ms, fl, by, cnt, nc)
        cap = 4096
        cls = (C.c_int32 * cap)(); lms = (C.c_float * cap)(); lfl = (C.c_double * cap)()
        k = _lib.lib().epd_encoder_profile_launches(enc._h, cls, lms, lfl, cap)
        head = 3 if cfg.family == 2 else 2  # (memset,) patchify, patch GEMM
        names = (["memset"] if cfg.family == 2 else []) + ["patchify", "patch_embed"]
        names += ROLES_LAYER * cfg.layers
        names += ROLES_SIGLIP_TAIL if cfg.family == 1 else ROLES_INTERN_TAIL
        assert len(names) == k, (len(names), k, head)
        for i in range(k):
            a = agg[names[i]]
            a[0] += lms[i] / reps
            a[1] += lfl[i] / reps
            a[2] += 1
    total = sum(v[0] for v in agg.values())
    print(f"{cfg.name} n={n}: total {total:.3f} ms (profiled, serialised)")
    for name, (t, f, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        tf = f / t / 1e9 if t and f else 0.0
        print(f"  {name:12s} {t:8.3f} ms {100 * t / total:5.1f}%  x{c // reps:3d}  {tf:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
