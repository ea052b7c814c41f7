"""GEMM timing for A/B runs over the encoder's shapes (library from EPD_LIB_PATH)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402


def timeit(fn, iters=30, warm=5):
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
BN = int(os.environ.get("BN", "0"))
CL = int(os.environ.get("CL", "0"))
if CL:
    from paper_2501_05460_b200._lib import call as _call
    _call("epd_set_gemm_cta_group", CL)
tag += f"/bn{BN}/cl{CL}/M{os.environ.get('M', '10240')}"
dev = torch.device("cuda")
M = int(os.environ.get("M", "10240"))
line = []
for (N, K, act, name, acc) in [(3840, 1152, "none", "qkv", False), (1152, 1152, "none", "o+acc", True),
                               (4304, 1152, "gelu_tanh", "fc1", False), (4304, 1152, "none", "fc1-none", False), (1152, 4304, "none", "fc2+acc", True),
                               (4096, 1024, "gelu_erf", "ivit_fc1", False)]:
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev) * K ** -0.5).to(torch.bfloat16)
    b = torch.randn(N, device=dev).to(torch.bfloat16)
    if acc:
        h = torch.zeros(M, N, device=dev)
        ms = timeit(lambda: kernels.linear_acc(a, w, h, bias=b, bn=BN))
    else:
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        ms = timeit(lambda: kernels.linear(a, w, bias=b, act=act, out=out, bn=BN))
    line.append(f"{name} {ms * 1e3:6.1f}us {2 * M * N * K / ms / 1e9:6.0f}TF")
# QKV in heads mode (SigLIP: H=16, Dp=80, T=1024), natural layouts for all sections
from paper_2501_05460_b200._lib import call  # noqa: E402
H, Dp, T, K = 16, 80, 1024, 1152
N = 3 * H * Dp
a = torch.randn(M, K, device=dev).to(torch.bfloat16)
w = (torch.randn(N, K, device=dev) * K ** -0.5).to(torch.bfloat16)
b = torch.randn(N, device=dev).to(torch.bfloat16)
outs = [torch.empty(M // T * H, T, Dp, device=dev, dtype=torch.bfloat16) for _ in range(3)]
ms = timeit(lambda: call("epd_linear_heads_bf16", a.data_ptr(), K, w.data_ptr(), K, M, N, K, b.data_ptr(), None, 0,
                         0, H, Dp, T, T, H * Dp, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), 0,
                         torch.cuda.current_stream().cuda_stream))
line.append(f"qkv_heads {ms * 1e3:6.1f}us {2 * M * N * K / ms / 1e9:6.0f}TF")
print(f"{tag:6s} " + " | ".join(line))
