"""Our tcgen05 GEMM against cuBLAS (torch.matmul, bf16) on the encoder and prefill shapes:
python tools/gemm_vs_cublas.py. Plain GEMM (no bias / activation) on both sides, L2 flushed
between timed calls, so the comparison is kernel against kernel."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402

dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / iters


shapes = [("siglip qkv", 10240, 3456, 1152), ("siglip attn-out", 10240, 1152, 1152), ("siglip fc1", 10240, 4304, 1152),
          ("siglip fc2", 10240, 1152, 4304), ("resampler kv", 10240, 3584, 3584), ("ivit fc1", 12300, 4096, 1024),
          ("qwen2 qkv", 662, 4608, 3584), ("qwen2 gate/up", 662, 37888, 3584), ("qwen2 down", 662, 3584, 18944),
          ("square 8192", 8192, 8192, 8192)]
for name, M, N, K in shapes:
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev) * K ** -0.5).to(torch.bfloat16)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    if name.endswith("+acc"):  # fp32 residual accumulate
        h = torch.zeros(M, N, device=dev)
        ours = timeit(lambda: kernels.linear_acc(a, w, h))
    else:
        ours = timeit(lambda: kernels.linear(a, w, out=out))
    lib = timeit(lambda: torch.matmul(a, w.t(), out=out))
    fl = 2 * M * N * K
    print(f"{name:16s} {M:6d}x{N:6d}x{K:6d}: ours {ours * 1e3:8.1f} us {fl / ours / 1e9:6.0f} TF | "
          f"cuBLAS {lib * 1e3:8.1f} us {fl / lib / 1e9:6.0f} TF | ratio {lib / ours:5.2f}")
