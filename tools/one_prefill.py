"""One Qwen2-7B prefill (662 tokens) inside a cudaProfilerStart/Stop range: ncu target."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.prefill import QWEN2_7B, Prefiller  # noqa: E402

pf = Prefiller(QWEN2_7B, 0, max_tokens=662, use_graphs=False)
mm = (torch.randn(640, QWEN2_7B.hidden, device="cuda") * 0.5).to(torch.bfloat16)
ids = torch.randint(0, QWEN2_7B.vocab, (22,), dtype=torch.int32, device="cuda")
for _ in range(2):
    pf.prefill(mm, ids)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
pf.prefill(mm, ids)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
