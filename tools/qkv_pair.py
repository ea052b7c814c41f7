"""One rows-mode and one heads-mode QKV GEMM (SigLIP shape) after warm-up: ncu target."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402
from paper_2501_05460_b200._lib import call  # noqa: E402

dev = torch.device("cuda")
M, H, Dp, T, K = 10240, 16, 80, 1024, 1152
N = 3 * H * Dp
a = torch.randn(M, K, device=dev).to(torch.bfloat16)
w = (torch.randn(N, K, device=dev) * K ** -0.5).to(torch.bfloat16)
b = torch.randn(N, device=dev).to(torch.bfloat16)
out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
outs = [torch.empty(M // T * H, T, Dp, device=dev, dtype=torch.bfloat16) for _ in range(3)]


def heads():
    call("epd_linear_heads_bf16", a.data_ptr(), K, w.data_ptr(), K, M, N, K, b.data_ptr(), None, 0, 0, H, Dp, T, T,
         H * Dp, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), 0, torch.cuda.current_stream().cuda_stream)


for _ in range(3):
    kernels.linear(a, w, bias=b, out=out)
    heads()
torch.cuda.synchronize()
kernels.linear(a, w, bias=b, out=out)
heads()
torch.cuda.synchronize()
