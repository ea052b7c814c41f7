"""Attention-only micro-benchmark (long runs, clocks reported) for A/B experiments."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402


def main():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    dev = torch.device("cuda")
    for (B, H, T, Dv, Tq, qs) in [(10, 16, 1024, 72, 1024, False), (10, 16, 1025, 64, 1025, False),
                                  (10, 28, 1024, 128, 64, True)]:
        kv = torch.randn(B * T, 2 * H * Dv, device=dev).to(torch.bfloat16)
        k, v = kv[:, :H * Dv], kv[:, H * Dv:]
        q = torch.randn(Tq if qs else B * Tq, H * Dv, device=dev).to(torch.bfloat16)
        out = torch.empty(B * Tq, H * Dv, device=dev, dtype=torch.bfloat16)
        f = lambda: kernels.attention(q, k, v, B, H, Tq, T, Dv, Dv ** -0.5, q_shared=qs, out=out)  # noqa: E731
        for _ in range(50):
            f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(200):
            f()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 200
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        fl = 4 * B * H * Tq * T * Dv
        print(f"attn B={B} H={H} T={Tq}x{T} Dv={Dv}: {ms*1e3:7.1f} us {fl/ms/1e9:6.1f} TF/s  sm={clk} MHz")


if __name__ == "__main__":
    main()
