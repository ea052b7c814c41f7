"""Kernel micro-benchmarks (CUDA events, warm L2 unless noted) for the encoder's hot kernels."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402


def timeit(fn, iters=20, warm=3):
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


def main():
    from paper_2501_05460_b200._lib import call
    dev = torch.device("cuda")
    cg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    call("epd_set_gemm_cta_group", cg)
    print(f"gemm cta-group policy {cg}")
    M = 10240
    for (N, K, act, name) in [(3840, 1152, "none", "qkv"), (1152, 1152, "none", "o"),
                              (4304, 1152, "gelu_tanh", "fc1"), (1152, 4304, "none", "fc2"),
                              (3584, 1152, "none", "kv_proj"), (7168, 3584, "none", "kv_in")]:
        a = torch.randn(M, K, device=dev).to(torch.bfloat16)
        w = (torch.randn(N, K, device=dev) * K ** -0.5).to(torch.bfloat16)
        b = torch.randn(N, device=dev).to(torch.bfloat16)
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        for bn in (0, 128, 192, 256):
            ms = timeit(lambda: kernels.linear(a, w, bias=b, act=act, out=out, bn=bn))
            tf = 2 * M * N * K / ms / 1e9
            print(f"gemm {name:8s} M={M} N={N} K={K} bn={bn:3d}: {ms*1e3:8.1f} us  {tf:7.1f} TFLOP/s")
        ms = timeit(lambda: torch.matmul(a, w.t(), out=out))
        print(f"  torch/cuBLAS {name}: {ms*1e3:8.1f} us  {2*M*N*K/ms/1e9:7.1f} TFLOP/s")
        if name in ("o", "fc2"):
            h = torch.zeros(M, N, device=dev)
            for bn in (0, 128, 192, 256):
                ms = timeit(lambda: kernels.linear_acc(a, w, h, bias=b, bn=bn))
                print(f"gemm {name}+acc_f32 bn={bn:3d}: {ms*1e3:8.1f} us  {2*M*N*K/ms/1e9:7.1f} TFLOP/s")
    for (B, H, T, Dv, Tq, qs) in [(10, 16, 1024, 72, 1024, False), (10, 28, 1024, 128, 64, True)]:
        kv = torch.randn(B * T, 2 * H * Dv, device=dev).to(torch.bfloat16)
        k, v = kv[:, :H * Dv], kv[:, H * Dv:]
        q = torch.randn(Tq if qs else B * Tq, H * Dv, device=dev).to(torch.bfloat16)
        out = torch.empty(B * Tq, H * Dv, device=dev, dtype=torch.bfloat16)
        ms = timeit(lambda: kernels.attention(q, k, v, B, H, Tq, T, Dv, Dv ** -0.5, q_shared=qs, out=out))
        fl = 4 * B * H * Tq * T * Dv
        print(f"attn B={B} H={H} Tq={Tq} Tk={T} Dv={Dv}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOP/s (algorithmic)")
    x = torch.randn(M, 1152, device=dev).to(torch.bfloat16)
    g = torch.ones(1152, device=dev, dtype=torch.bfloat16)
    y = torch.empty_like(x)
    ms = timeit(lambda: kernels.layernorm(x, g, g, 1e-6, out=y))
    print(f"layernorm {M}x1152: {ms*1e3:.1f} us  {2*x.numel()*2/ms/1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
