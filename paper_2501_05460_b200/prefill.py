"""Prefill consumer of the packed MM tokens.

The reference models prefill as ``costs.prefill_latency(params, total_tokens)``
(costs.py:93-99) and the first token as the end of that batch (``_on_batch_end``,
engine.py:385-407): TTFT = arrival -> encode -> EP transfer -> prefill end. Here the
prefill GPU runs a real decoder of the model's LLM shape on ``[MM tokens | prompt]``
and produces the first token, so TTFT is measured end to end. Weights are random-init
N(0, 0.02) (norm gains 1) of the public LLM geometry; the reference catalog fixes
layers / KV heads / head dim / hidden (models.cfg), the model cards the rest.

Every op runs on the sm_100a kernels of ``libepd`` (tcgen05 GEMMs with fused bias, SwiGLU
and fp32 residual reduce-add, causal grouped-KV attention, RMSNorm, RoPE, paged KV write,
argmax); PyTorch only owns the buffers and captures the launch sequence in one
CUDA graph per prompt shape. K/V land in the paged pool that the P->D handoff
(handoff.py) moves, so the decode side receives real prefill KV.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from . import kernels
from .configs import INTERNVL2_8B, MINICPM_V26, SEED, ModelGeometry


@dataclass(frozen=True)
class LLMConfig:
    name: str
    layers: int
    hidden: int
    q_heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float
    rms_eps: float
    qkv_bias: bool
    geometry: ModelGeometry | None = None

    @property
    def qkv_dim(self) -> int:
        return (self.q_heads + 2 * self.kv_heads) * self.head_dim

    @property
    def vocab_padded(self) -> int:  # GEMM N granularity; argmax only reads [0, vocab)
        return (self.vocab + 7) // 8 * 8

    def with_layers(self, layers: int) -> "LLMConfig":
        from dataclasses import replace
        return replace(self, layers=layers, name=f"{self.name}-L{layers}")

    def flops(self, T: int) -> float:
        """Algorithmic FLOPs of one prefill of T tokens (causal attention counted at T^2/2)."""
        hd, H = self.head_dim, self.hidden
        per_layer = (2.0 * T * H * self.qkv_dim + 2.0 * T * self.q_heads * hd * H
                     + 2.0 * 2.0 * T * T / 2 * self.q_heads * hd + 2.0 * T * H * 2 * self.ffn + 2.0 * T * self.ffn * H)
        return self.layers * per_layer + 2.0 * H * self.vocab


# MiniCPM-V 2.6's LLM (Qwen2-7B) and InternVL2-8B's (InternLM2.5-7B): catalog geometry
# (models.cfg) + public model cards (q heads, FFN, vocab, RoPE base, norm eps, QKV bias).
QWEN2_7B = LLMConfig("qwen2-7b", 28, 3584, 28, 4, 128, 18944, 152064, 1e6, 1e-6, True, MINICPM_V26)
INTERNLM25_7B = LLMConfig("internlm2.5-7b", 32, 4096, 32, 8, 128, 14336, 92553, 1e6, 1e-5, False, INTERNVL2_8B)
TINY_LLM = LLMConfig("tiny-llm", 2, 256, 4, 2, 64, 512, 1000, 1e4, 1e-6, True)

# The O and down projections run at M = prompt length (662 tokens for C2): their output tiles
# alone leave CTA pairs idle, so they may split K (epd_linear_acc_f32_split; deterministic
# order). The encoder never splits (its results are batch invariant).
PREFILL_MAX_SPLIT = int(os.environ.get("EPD_PREFILL_MAX_SPLIT", "8"))  # A/B: 0 = never split


def llm_weights(cfg: LLMConfig, device, seed: int = SEED) -> dict[str, torch.Tensor]:
    """Random-init bf16 weights on the device: N(0, 0.02), norm gains 1, biases N(0, 0.02)."""
    g = torch.Generator(device=device).manual_seed(seed)

    def rnd(*shape):
        return (torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * 0.02).to(torch.bfloat16)

    H, hd = cfg.hidden, cfg.head_dim
    w = {"embed": rnd(cfg.vocab, H), "final_norm": torch.ones(H, dtype=torch.bfloat16, device=device)}
    lm = torch.zeros(cfg.vocab_padded, H, dtype=torch.bfloat16, device=device)
    lm[:cfg.vocab] = rnd(cfg.vocab, H)
    w["lm_head"] = lm
    for i in range(cfg.layers):
        p = f"layers.{i}."
        w[p + "attn_norm"] = torch.ones(H, dtype=torch.bfloat16, device=device)
        w[p + "wqkv"] = rnd(cfg.qkv_dim, H)
        w[p + "bqkv"] = rnd(cfg.qkv_dim) if cfg.qkv_bias else torch.zeros(cfg.qkv_dim, dtype=torch.bfloat16,
                                                                          device=device)
        w[p + "wo"] = rnd(H, cfg.q_heads * hd)
        w[p + "mlp_norm"] = torch.ones(H, dtype=torch.bfloat16, device=device)
        # gate / up rows interleaved in 32-row groups: the GEMM epilogue applies SwiGLU
        w[p + "wgu"] = kernels.swiglu_interleave(rnd(cfg.ffn, H), rnd(cfg.ffn, H))
        w[p + "wd"] = rnd(H, cfg.ffn)
    return w


class Prefiller:
    """One prefill GPU's LLM: ``prefill(mm_tokens, text_ids)`` -> first token id.

    Sequence = [MM tokens | prompt tokens], positions 0..T-1. With ``kv`` (a
    :class:`~.handoff.PagedKVCache`) and ``block_ids``, every layer's post-RoPE K/V rows
    are written into those blocks (the P->D handoff payload).
    """

    def __init__(self, cfg: LLMConfig, device, max_tokens: int = 1024, weights: dict | None = None,
                 seed: int = SEED, use_graphs: bool = True):
        self.cfg = cfg
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("Prefiller runs on a CUDA device only (no CPU fallback)")
        self.max_tokens = max_tokens
        self.w = weights if weights is not None else llm_weights(cfg, self.device, seed)
        bf, dev, T, H = torch.bfloat16, self.device, max_tokens, cfg.hidden
        self.h = torch.zeros(T, H, dtype=torch.float32, device=dev)
        self.xn = torch.zeros(T, H, dtype=bf, device=dev)
        self.qkv = torch.zeros(T, cfg.qkv_dim, dtype=bf, device=dev)
        self.attn = torch.zeros(T, cfg.q_heads * cfg.head_dim, dtype=bf, device=dev)
        self.act = torch.zeros(T, cfg.ffn, dtype=bf, device=dev)
        self.logits = torch.zeros(1, cfg.vocab_padded, dtype=bf, device=dev)
        self.token = torch.zeros(1, dtype=torch.int32, device=dev)
        self.mm_in = torch.zeros(T, H, dtype=bf, device=dev)
        self.ids_in = torch.zeros(T, dtype=torch.int32, device=dev)
        self.blocks_in = torch.zeros(T, dtype=torch.int32, device=dev)
        self.mm_rows = torch.zeros(T, dtype=torch.int32, device=dev)  # paged MM input: pool row per token
        self.iota = torch.arange(T, dtype=torch.int32, device=dev)
        # RoPE (cos, sin) for positions 0..max_tokens-1, built once
        self.rope_cs = kernels.rope_table(T, cfg.head_dim, cfg.rope_theta, device=dev)
        self.use_graphs = use_graphs
        self._graphs: dict = {}

    # -- one forward over the static buffers -------------------------------------------
    def _forward(self, n_mm: int, n_text: int, kv, mm_pool=None) -> None:
        cfg, w = self.cfg, self.w
        T, hd, Hq, Hk = n_mm + n_text, cfg.head_dim, cfg.q_heads, cfg.kv_heads
        h = self.h[:T]
        if n_mm and mm_pool is not None:
            # MM tokens straight from the prefill instance's paged MM pool (runtime.py)
            kernels.gather_rows_f32(mm_pool, self.mm_rows[:n_mm], self.h[:n_mm])
        elif n_mm:
            kernels.gather_rows_f32(self.mm_in, self.iota[:n_mm], self.h[:n_mm])
        if n_text:
            kernels.gather_rows_f32(w["embed"], self.ids_in[:n_text], self.h[n_mm:T])
        xn, qkv, attn, act = self.xn[:T], self.qkv[:T], self.attn[:T], self.act[:T]
        for i in range(cfg.layers):
            p = f"layers.{i}."
            kernels.rmsnorm_f32(h, w[p + "attn_norm"], cfg.rms_eps, out=xn)
            kernels.linear(xn, w[p + "wqkv"], bias=w[p + "bqkv"], out=qkv)
            kernels.rope_(qkv, 0, Hq + Hk, hd, cfg.rope_theta, table=self.rope_cs)
            if kv is not None:
                kernels.kv_write_paged(qkv[:, Hq * hd:], Hk * hd, Hk * hd, self.blocks_in, kv.block_size, kv.pool, i)
            kernels.attention(qkv[:, :Hq * hd], qkv[:, Hq * hd:(Hq + Hk) * hd], qkv[:, (Hq + Hk) * hd:], 1, Hq, T, T,
                              hd, hd ** -0.5, out=attn, kv_heads=Hk, causal=True)
            kernels.linear_acc(attn, w[p + "wo"], h, max_split=PREFILL_MAX_SPLIT)
            kernels.rmsnorm_f32(h, w[p + "mlp_norm"], cfg.rms_eps, out=xn)
            kernels.linear(xn, w[p + "wgu"], act="swiglu", out=act)  # silu(gate) * up in the epilogue
            kernels.linear_acc(act, w[p + "wd"], h, max_split=PREFILL_MAX_SPLIT)
        kernels.rmsnorm_f32(h[T - 1:T], w["final_norm"], cfg.rms_eps, out=xn[:1])
        kernels.linear(xn[:1], w["lm_head"], out=self.logits)
        kernels.argmax(self.logits[0, :cfg.vocab], out=self.token)

    def prefill(self, mm_tokens: torch.Tensor | None, text_ids: torch.Tensor, kv=None,
                block_ids: list[int] | torch.Tensor | None = None, mm_pool: torch.Tensor | None = None,
                mm_rows: torch.Tensor | None = None) -> torch.Tensor:
        """mm_tokens: bf16 [n_mm, hidden] on the device (the packed encode output, flattened);
        or, paged, ``mm_pool`` (bf16 [rows, hidden]) with ``mm_rows`` (int32, the pool row of
        each MM token, in request order). text_ids: int32 [n_text] on the device. Returns the
        first token id (int32 [1], device)."""
        cfg = self.cfg
        if mm_pool is not None:
            if mm_tokens is not None or mm_rows is None:
                raise ValueError("paged prefill takes mm_pool + mm_rows instead of mm_tokens")
            if mm_pool.dtype != torch.bfloat16 or mm_pool.shape[1] != cfg.hidden:
                raise ValueError(f"the MM pool must be bf16 [rows, {cfg.hidden}]")
        n_mm = mm_rows.numel() if mm_pool is not None else (0 if mm_tokens is None else mm_tokens.shape[0])
        n_text = text_ids.numel()
        T = n_mm + n_text
        if T < 1 or T > self.max_tokens:
            raise ValueError(f"prefill needs 1..{self.max_tokens} tokens, got {T}")
        if mm_tokens is not None and (mm_tokens.shape[1] != cfg.hidden or mm_tokens.dtype != torch.bfloat16):
            raise ValueError(f"MM tokens must be bf16 [n, {cfg.hidden}]")
        if kv is not None:
            nb = -(-T // kv.block_size)
            ids = torch.as_tensor(block_ids, dtype=torch.int32)
            if ids.numel() < nb:
                raise ValueError(f"{T} tokens need {nb} KV blocks, got {ids.numel()}")
            self.blocks_in[:nb].copy_(ids[:nb], non_blocking=True)
        if n_mm and mm_pool is not None:
            self.mm_rows[:n_mm].copy_(mm_rows, non_blocking=True)
        elif n_mm:
            self.mm_in[:n_mm].copy_(mm_tokens)
        if n_text:
            self.ids_in[:n_text].copy_(text_ids.to(torch.int32))
        key = (n_mm, n_text, kv is not None, id(kv) if kv is not None else 0,
               id(mm_pool) if mm_pool is not None else 0)
        if not self.use_graphs:
            self._forward(n_mm, n_text, kv, mm_pool)
            return self.token
        g = self._graphs.get(key)
        if g is None:
            self._forward(n_mm, n_text, kv, mm_pool)  # warm-up (kernel attributes, tensor maps) outside capture
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self._forward(n_mm, n_text, kv, mm_pool)
            torch.cuda.current_stream(self.device).wait_stream(s)
            self._graphs[key] = g
        g.replay()
        return self.token


__all__ = ["LLMConfig", "QWEN2_7B", "INTERNLM25_7B", "TINY_LLM", "llm_weights", "Prefiller"]
