"""CPU tier: the LLM-prefill oracle (oracle/llm.py) against transformers' Qwen2ForCausalLM
outputs recorded in tests/golden/llm_golden.json (tests/golden/make_llm_golden.py) for the
product's canonical weights of a 2-layer reduced-width Qwen2-shaped LLM with [MM rows | prompt]
input. This pins the prefill consumer's reference semantics (RMSNorm gains, QKV bias, GQA,
rotate-half RoPE, SwiGLU, final norm, LM head) to a public implementation; the GPU tier
(tests/test_prefill_gpu.py) holds the B200 prefill to this oracle."""
import importlib.util
import json
from pathlib import Path

import torch

GOLDEN = Path(__file__).parent / "golden"


def _inputs():
    spec = importlib.util.spec_from_file_location("make_llm_golden", GOLDEN / "make_llm_golden.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.golden_inputs()


def test_llm_oracle_matches_transformers_qwen2():
    import oracle.llm as ol
    fx = json.loads((GOLDEN / "llm_golden.json").read_text())
    cfg, w, mm, ids = _inputs()
    assert fx["T_mm"] == mm.shape[0] and fx["prompt"] == ids.tolist()
    o = ol.prefill(cfg, w, mm, ids)
    lg = o["logits"]
    ref = torch.tensor(fx["logits"])
    assert (lg[torch.tensor(fx["logits_idx"])] - ref).abs().max() <= 1e-5 * fx["logits_absmax"]
    assert abs(float(lg.sum()) - fx["logits_sum"]) <= 1e-4 * fx["logits_absmax"] * cfg.vocab ** 0.5
    assert o["token"] == fx["token"]
    normed = ol.rms(o["hidden"], w["final_norm"].float(), cfg.rms_eps)
    got = normed[fx["hidden_rows"], :16]
    want = torch.tensor(fx["hidden"])
    assert (got - want).abs().max() <= 1e-5 * max(1.0, want.abs().max().item())
