"""Prefill consumer on the B200 against the fp32 CPU oracle
(oracle/llm.py): final hidden state and logits within 1e-2 (bf16 compute, fp32 residual
stream), the paged KV pool holding every layer's post-RoPE K/V, graph replay bit-exact."""
import pytest
import torch

from paper_2501_05460_b200.configs import SEED

pytestmark = pytest.mark.gpu

TOL = 1e-2
# Final hidden state (max-normalised): a CPU emulation of this pipeline's bf16 rounding points
# (xn, qkv, P, attention out, gate/up, SwiGLU out; fp32 residual) scores 1.22e-2 against the
# fp32 oracle at the Qwen2-7B width (2 layers, 662 tokens); the kernels measure 1.11e-2.
TOL_H = 2e-2


def relerr(y, ref):
    y, ref = y.float().cpu(), ref.float().cpu()
    return float((y - ref).abs().max() / ref.abs().max().clamp_min(1e-12))


def _inputs(cfg, n_mm, n_text, dev, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    mm = (torch.randn(n_mm, cfg.hidden, generator=g, device=dev) * 0.5).to(torch.bfloat16) if n_mm else None
    ids = torch.randint(0, cfg.vocab, (n_text,), generator=g, device=dev, dtype=torch.int32)
    return mm, ids


@pytest.mark.parametrize("which,n_mm,n_text", [("tiny", 48, 22), ("tiny", 0, 5), ("qwen2-L2", 640, 22),
                                               ("internlm-L2", 3328, 22)])
def test_prefill_matches_oracle(cuda, which, n_mm, n_text):
    """qwen2-L2: the C2 prefill width (662 tokens); internlm-L2: the C5 one (13 tiles x 256 MM
    tokens + prompt = 3350 tokens, grouped K/V 32 / 8 heads)."""
    import oracle.llm as ol
    from paper_2501_05460_b200.handoff import PagedKVCache
    from paper_2501_05460_b200.prefill import INTERNLM25_7B, QWEN2_7B, TINY_LLM, Prefiller
    cfg = {"tiny": TINY_LLM, "qwen2-L2": QWEN2_7B.with_layers(2), "internlm-L2": INTERNLM25_7B.with_layers(2)}[which]
    pf = Prefiller(cfg, cuda, max_tokens=max(704, n_mm + n_text))
    mm, ids = _inputs(cfg, n_mm, n_text, cuda, SEED + n_mm)
    T = n_mm + n_text
    kv = PagedKVCache(cfg.layers, cfg.kv_heads, cfg.head_dim, 16, max(64, -(-(n_mm + n_text) // 16)), cuda)
    blocks = kv.manager.allocate(1, T)
    tok = int(pf.prefill(mm, ids, kv=kv, block_ids=blocks))
    torch.cuda.synchronize()
    ref = ol.prefill(cfg, pf.w, mm, ids)
    err_h = relerr(pf.h[:T], ref["hidden"])
    err_l = relerr(pf.logits[0, :cfg.vocab], ref["logits"])
    print(f"{cfg.name} T={T}: hidden relerr {err_h:.2e}, logits relerr {err_l:.2e}, token {tok} vs {ref['token']}")
    assert err_h <= TOL_H and err_l <= TOL_H, (err_h, err_l)
    assert tok == int(pf.logits[0, :cfg.vocab].float().argmax())
    top2 = ref["logits"].topk(2).values
    if float(top2[0] - top2[1]) > 2 * TOL_H * float(ref["logits"].abs().max()):
        assert tok == ref["token"]  # the first token, when the oracle's margin exceeds the error bound
    # paged KV: token t of layer l at block blocks[t // 16], slot t % 16
    row = cfg.kv_heads * cfg.head_dim
    for layer in range(cfg.layers):
        got_k = torch.stack([kv.pool[2 * layer, blocks[t // 16], (t % 16) * row:(t % 16 + 1) * row] for t in range(T)])
        got_v = torch.stack([kv.pool[2 * layer + 1, blocks[t // 16], (t % 16) * row:(t % 16 + 1) * row]
                             for t in range(T)])
        # layer 0's K/V carry only their own bf16 rounding; later layers also carry the hidden
        # state's accumulated rounding (bounded like the hidden state)
        tol = TOL if layer == 0 else TOL_H
        assert relerr(got_k, ref["k"][layer]) <= tol and relerr(got_v, ref["v"][layer]) <= tol


def test_prefill_graph_equals_direct_and_rejects_bad_input(cuda):
    from paper_2501_05460_b200.prefill import TINY_LLM, Prefiller
    cfg = TINY_LLM
    w = None
    outs = []
    for graphs in (True, False):
        pf = Prefiller(cfg, cuda, max_tokens=128, weights=w, use_graphs=graphs)
        w = pf.w
        mm, ids = _inputs(cfg, 40, 9, cuda, 3)
        pf.prefill(mm, ids)
        pf.prefill(mm, ids)  # replay
        torch.cuda.synchronize()
        outs.append(pf.h[:49].clone())
    assert torch.equal(outs[0], outs[1])
    with pytest.raises(ValueError):
        pf.prefill(None, torch.zeros(200, dtype=torch.int32, device=cuda))
    with pytest.raises(ValueError):
        pf.prefill(torch.zeros(3, 7, dtype=torch.bfloat16, device=cuda), ids)


def test_paged_mm_input_equals_packed(cuda):
    """The runtime's paged MM input (rows gathered from the prefill instance's MM blocks in
    any block order) gives the same hidden state, bit for bit, as the packed input."""
    from paper_2501_05460_b200.prefill import QWEN2_7B, Prefiller
    cfg = QWEN2_7B.with_layers(2)
    pf = Prefiller(cfg, cuda, max_tokens=704)
    mm, ids = _inputs(cfg, 640, 22, cuda, 5)
    pf.prefill(mm, ids)
    torch.cuda.synchronize()
    packed = pf.h[:662].clone()
    blocks = torch.randperm(100, generator=torch.Generator().manual_seed(1))[:40]  # 40 blocks of 16 tokens
    pool = torch.zeros(100 * 16, cfg.hidden, dtype=torch.bfloat16, device=cuda)
    rows = (blocks.view(-1, 1) * 16 + torch.arange(16)).view(-1)
    pool[rows.to(cuda)] = mm
    pf.prefill(None, ids, mm_pool=pool, mm_rows=rows.to(torch.int32))
    torch.cuda.synchronize()
    assert torch.equal(pf.h[:662], packed)


def test_prefill_matches_transformers_fixture(cuda):
    """The B200 prefill on the golden weights and inputs of tests/golden/llm_golden.json
    (transformers Qwen2ForCausalLM, fp32): last-position logits within the bf16 bound."""
    import importlib.util
    import json
    from pathlib import Path

    from paper_2501_05460_b200.prefill import Prefiller
    golden = Path(__file__).parent / "golden"
    spec = importlib.util.spec_from_file_location("make_llm_golden", golden / "make_llm_golden.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    cfg, w, mm, ids = mod.golden_inputs()
    fx = json.loads((golden / "llm_golden.json").read_text())
    pf = Prefiller(cfg, cuda, max_tokens=64, weights={k: v.to(cuda) for k, v in w.items()})
    tok = int(pf.prefill(mm.to(cuda), ids.to(cuda, torch.int32)))
    torch.cuda.synchronize()
    lg = pf.logits[0, :cfg.vocab].float().cpu()
    err = float((lg[torch.tensor(fx["logits_idx"])] - torch.tensor(fx["logits"])).abs().max()) / fx["logits_absmax"]
    print(f"B200 prefill vs transformers Qwen2: logits {err:.2e}, token {tok} vs {fx['token']}")
    assert err <= TOL_H
