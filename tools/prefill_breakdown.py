"""Per-op device time of one prefill (direct launches, CUDA events around each op)."""
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200 import kernels  # noqa: E402
from paper_2501_05460_b200.prefill import INTERNLM25_7B, QWEN2_7B, Prefiller  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "qwen"
if len(sys.argv) > 2:
    from paper_2501_05460_b200._lib import call
    call("epd_set_gemm_cta_group", int(sys.argv[2]))
cfg = QWEN2_7B if which == "qwen" else INTERNLM25_7B
T_mm = 640 if which == "qwen" else 3072
pf = Prefiller(cfg, 0, max_tokens=T_mm + 22, use_graphs=False)
mm = (torch.randn(T_mm, cfg.hidden, device="cuda") * 0.5).to(torch.bfloat16)
ids = torch.randint(0, cfg.vocab, (22,), dtype=torch.int32, device="cuda")
for _ in range(2):
    pf.prefill(mm, ids)
torch.cuda.synchronize()
times = defaultdict(float)
orig = {}
for name in ("rmsnorm_f32", "linear", "rope_", "attention", "linear_acc", "silu_mul", "gather_rows_f32", "argmax"):
    fn = getattr(kernels, name)
    orig[name] = fn

    def wrap(*a, _fn=fn, _name=name, **k):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)  # the op's launch queues behind it: the events time the GPU only
        s.record()
        r = _fn(*a, **k)
        e.record()
        e.synchronize()
        key = _name
        if _name in ("linear", "linear_acc"):
            key = f"{_name} N={a[1].shape[0]} K={a[1].shape[1]}"
        times[key] += s.elapsed_time(e)
        return r
    setattr(kernels, name, wrap)
pf.prefill(mm, ids)
tot = sum(times.values())
print(f"{cfg.name} T={T_mm + 22}: {tot:.2f} ms (serialised)")
for k, v in sorted(times.items(), key=lambda kv: -kv[1]):
    print(f"  {k:40s} {v:7.3f} ms {100 * v / tot:5.1f}%")
