"""Measured B200 prefill latency (seconds for T tokens, one GPU) of the two LLMs the encode
path feeds -- Qwen2-7B (MiniCPM-V 2.6) and InternLM2.5-7B (InternVL2-8B) -- through
prefill.Prefiller (CUDA graph per shape, random-init weights of the public geometry). The
reference charges prefill with costs.prefill_latency (costs.py:93-99); tools/calibrate_reference.py
fits its polynomial from these samples.
Writes argv[1] (default profiles/r02/prefill_latency_b200.json)."""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2501_05460_b200.prefill import INTERNLM25_7B, QWEN2_7B, Prefiller  # noqa: E402

TOKENS = [128, 256, 662, 1024, 2048, 3350, 4096, 6144, 8192]
PROMPT = 22

out = {"device": torch.cuda.get_device_name(0),
       "note": "seconds per prefill of T tokens ([T - 22 MM tokens | 22 prompt tokens]) to the first token, "
               "one GPU, CUDA graph, median of 5 after a warm-up", "models": {}}
dev = torch.device("cuda", 0)
for ref_name, cfg in [("minicpm-v-2.6", QWEN2_7B), ("internvl2-8b", INTERNLM25_7B)]:
    pf = Prefiller(cfg, dev, max_tokens=max(TOKENS))
    g = torch.Generator(device=dev).manual_seed(1)
    samples = []
    for T in TOKENS:
        mm = (torch.randn(T - PROMPT, cfg.hidden, generator=g, device=dev) * 0.5).to(torch.bfloat16)
        ids = torch.randint(0, cfg.vocab, (PROMPT,), generator=g, device=dev, dtype=torch.int32)
        pf.prefill(mm, ids)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            pf.prefill(mm, ids)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        samples.append([T, statistics.median(ts)])
        print(ref_name, T, round(samples[-1][1] * 1e3, 3), "ms", flush=True)
    out["models"][ref_name] = {"llm": cfg.name, "samples": samples}
    del pf
    torch.cuda.empty_cache()
path = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r02" / "prefill_latency_b200.json"
path.write_text(json.dumps(out, indent=1))
print(path)
