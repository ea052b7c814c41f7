"""Pin the LLM-prefill oracle (oracle/llm.py) to the public Qwen2 implementation.

Builds transformers' Qwen2ForCausalLM (transformers 5.5, fp32, eager attention) with the
product's canonical random weights for a 2-layer, reduced-width Qwen2-shaped LLM (prefill.TINY_LLM
geometry: GQA 4 / 2 heads of 64, SwiGLU 512, QKV bias, rotate-half RoPE) -- norm gains
randomised so they are pinned too -- runs [MM rows | prompt] through it as inputs_embeds and
records the final hidden state and last-position logits. tests/test_llm_golden_cpu.py
recomputes oracle/llm.py on the same weights and inputs against this fixture.

usage: python tests/golden/make_llm_golden.py   (writes tests/golden/llm_golden.json)
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def golden_inputs():
    """Weights (oracle layout) and inputs shared by this script and the CPU test."""
    from paper_2501_05460_b200.prefill import TINY_LLM, llm_weights
    cfg = TINY_LLM
    w = llm_weights(cfg, "cpu", seed=20260808)
    g = torch.Generator().manual_seed(7)
    for k in list(w):
        if k.endswith("norm"):  # pin the gains as well: 1 + 0.1 N(0, 1)
            w[k] = (1 + 0.1 * torch.randn(w[k].shape, generator=g)).to(torch.bfloat16)
    mm = (torch.randn(24, cfg.hidden, generator=g) * 0.5).to(torch.bfloat16)  # 24 MM rows
    ids = torch.randint(0, cfg.vocab, (9,), generator=g, dtype=torch.int64)  # 9 prompt tokens
    return cfg, w, mm, ids


def hf_forward(cfg, w, mm, ids):
    from transformers import Qwen2Config, Qwen2ForCausalLM
    hc = Qwen2Config(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
                     num_hidden_layers=cfg.layers, num_attention_heads=cfg.q_heads,
                     num_key_value_heads=cfg.kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.rms_eps,
                     rope_theta=cfg.rope_theta, tie_word_embeddings=False, attn_implementation="eager",
                     max_position_embeddings=4096, use_sliding_window=False)
    m = Qwen2ForCausalLM(hc).float().eval()
    f = {k: v.float() for k, v in w.items()}
    Hq, Hk, hd, F = cfg.q_heads, cfg.kv_heads, cfg.head_dim, cfg.ffn
    sd = {"model.embed_tokens.weight": f["embed"], "model.norm.weight": f["final_norm"],
          "lm_head.weight": f["lm_head"][:cfg.vocab]}
    for i in range(cfg.layers):
        p, q = f"layers.{i}.", f"model.layers.{i}."
        wq, wk, wv = f[p + "wqkv"].split([Hq * hd, Hk * hd, Hk * hd], 0)
        bq, bk, bv = f[p + "bqkv"].split([Hq * hd, Hk * hd, Hk * hd], 0)
        wg = f[p + "wgu"].view(F // 32, 2, 32, -1)
        sd.update({q + "input_layernorm.weight": f[p + "attn_norm"],
                   q + "post_attention_layernorm.weight": f[p + "mlp_norm"],
                   q + "self_attn.q_proj.weight": wq, q + "self_attn.q_proj.bias": bq,
                   q + "self_attn.k_proj.weight": wk, q + "self_attn.k_proj.bias": bk,
                   q + "self_attn.v_proj.weight": wv, q + "self_attn.v_proj.bias": bv,
                   q + "self_attn.o_proj.weight": f[p + "wo"],
                   q + "mlp.gate_proj.weight": wg[:, 0].reshape(F, -1),
                   q + "mlp.up_proj.weight": wg[:, 1].reshape(F, -1),
                   q + "mlp.down_proj.weight": f[p + "wd"]})
    missing, unexpected = m.load_state_dict(sd, strict=False)
    missing = [k for k in missing if "rotary" not in k]
    if missing or unexpected:
        raise RuntimeError(f"state dict mismatch: missing {missing}, unexpected {unexpected}")
    x = torch.cat([mm.float(), f["embed"][ids]], 0)[None]
    with torch.no_grad():
        out = m(inputs_embeds=x, output_hidden_states=True)
    # transformers' last hidden state is taken after the final RMSNorm; the oracle returns the
    # residual before it, so the comparison normalises the oracle's
    return {"logits": out.logits[0, -1], "final_normed_hidden": out.hidden_states[-1][0]}


def main():
    cfg, w, mm, ids = golden_inputs()
    hf = hf_forward(cfg, w, mm, ids)
    import oracle.llm as ol
    o = ol.prefill(cfg, w, mm, ids)
    normed = ol.rms(o["hidden"], w["final_norm"].float(), cfg.rms_eps)
    rel_l = float((o["logits"] - hf["logits"]).abs().max() / hf["logits"].abs().max())
    rel_h = float((normed - hf["final_normed_hidden"]).abs().max() / hf["final_normed_hidden"].abs().max())
    print(f"oracle vs transformers Qwen2: logits {rel_l:.2e}, final-normed hidden {rel_h:.2e}")
    idx = torch.linspace(0, cfg.vocab - 1, 64).long()
    fx = {"source": "transformers " + __import__("transformers").__version__ + " Qwen2ForCausalLM (fp32, eager)",
          "config": cfg.name, "T_mm": int(mm.shape[0]), "prompt": ids.tolist(),
          "logits_idx": idx.tolist(), "logits": hf["logits"][idx].tolist(),
          "logits_sum": float(hf["logits"].sum()), "logits_absmax": float(hf["logits"].abs().max()),
          "token": int(hf["logits"].argmax()),
          "hidden_rows": [0, 23, 24, 32], "hidden": hf["final_normed_hidden"][[0, 23, 24, 32], :16].tolist(),
          "hidden_sum": float(hf["final_normed_hidden"].sum()),
          "oracle_rel_err": {"logits": rel_l, "final_normed_hidden": rel_h}}
    path = Path(__file__).with_name("llm_golden.json")
    path.write_text(json.dumps(fx, indent=1))
    print(path)


if __name__ == "__main__":
    main()
