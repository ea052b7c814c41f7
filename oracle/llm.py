"""TEST INFRASTRUCTURE ONLY -- fp32 CPU oracle of the prefill consumer
(paper_2501_05460_b200/prefill.py). Not on any product path.

A plain restatement of a Qwen2 / InternLM2-style decoder prefill (public model
definitions; the reference models prefill only as costs.prefill_latency,
costs.py:93-99): RMSNorm, fused QKV (+bias), rotate-half RoPE with base theta,
causal grouped-KV attention, SwiGLU MLP, final RMSNorm, LM head. Sequence =
[MM tokens | prompt tokens], positions 0..T-1. The reference has no LLM code; this
restatement is pinned to transformers' Qwen2ForCausalLM (tests/golden/make_llm_golden.py ->
llm_golden.json, checked by tests/test_llm_golden_cpu.py: 6.7e-7 max rel err in fp32), and
the B200 prefill is held to it by tests/test_prefill_gpu.py.
"""
from __future__ import annotations

import torch


def rms(x: torch.Tensor, g: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def rope(x: torch.Tensor, theta: float) -> torch.Tensor:
    """x: [T, heads, hd], positions 0..T-1."""
    T, _, hd = x.shape
    pos = torch.arange(T, dtype=torch.float64)[:, None]
    inv = theta ** (-torch.arange(0, hd, 2, dtype=torch.float64) / hd)
    ang = pos * inv[None, :]
    cos, sin = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    a, b = x[..., :hd // 2], x[..., hd // 2:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)


def prefill(cfg, w: dict, mm_tokens: torch.Tensor | None, text_ids: torch.Tensor) -> dict:
    """fp32 forward. Returns {"hidden": final-norm input [T, H], "logits": [vocab],
    "token": int, "k": [layers][T, kv_heads*hd], "v": ...}."""
    f = {k: v.detach().float().cpu() for k, v in w.items()}
    parts = []
    if mm_tokens is not None and mm_tokens.shape[0]:
        parts.append(mm_tokens.detach().float().cpu())
    if text_ids.numel():
        parts.append(f["embed"][text_ids.cpu().long()])
    h = torch.cat(parts, 0)
    T = h.shape[0]
    Hq, Hk, hd = cfg.q_heads, cfg.kv_heads, cfg.head_dim
    ks, vs = [], []
    mask = torch.ones(T, T, dtype=torch.bool).tril()
    for i in range(cfg.layers):
        p = f"layers.{i}."
        x = rms(h, f[p + "attn_norm"], cfg.rms_eps)
        qkv = x @ f[p + "wqkv"].t() + f[p + "bqkv"]
        q = rope(qkv[:, :Hq * hd].reshape(T, Hq, hd), cfg.rope_theta)
        k = rope(qkv[:, Hq * hd:(Hq + Hk) * hd].reshape(T, Hk, hd), cfg.rope_theta)
        v = qkv[:, (Hq + Hk) * hd:].reshape(T, Hk, hd)
        ks.append(k.reshape(T, Hk * hd))
        vs.append(v.reshape(T, Hk * hd))
        kr = k.repeat_interleave(Hq // Hk, dim=1)
        vr = v.repeat_interleave(Hq // Hk, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, kr) * hd ** -0.5
        s = s.masked_fill(~mask, float("-inf"))
        a = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), vr).reshape(T, Hq * hd)
        h = h + a @ f[p + "wo"].t()
        x = rms(h, f[p + "mlp_norm"], cfg.rms_eps)
        # wgu rows alternate 32-row gate / up groups (prefill.py stores them that way)
        wg = f[p + "wgu"].view(cfg.ffn // 32, 2, 32, -1)
        gate, up = x @ wg[:, 0].reshape(cfg.ffn, -1).t(), x @ wg[:, 1].reshape(cfg.ffn, -1).t()
        h = h + (torch.nn.functional.silu(gate) * up) @ f[p + "wd"].t()
    last = rms(h[-1:], f["final_norm"], cfg.rms_eps)
    logits = (last @ f["lm_head"][:cfg.vocab].t())[0]
    return {"hidden": h, "logits": logits, "token": int(logits.argmax()), "k": ks, "v": vs}
