"""CPU tier for the C ABI: libepd.so loads, exports every symbol include/epd.h declares,
host-only entry points work without a GPU, and status codes map onto the reference's
exception classes."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2501_05460_b200 import _lib
from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM, TINY_VIT

HEADER = Path(__file__).resolve().parent.parent / "include" / "epd.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(epd_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported_and_bound():
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), f"libepd.so does not export {s}"
    assert set(syms) == set(_lib.EXPORTED), "ctypes bindings and header disagree"


def test_abi_version():
    assert _lib.lib().epd_abi_version() == 1


def test_status_mapping():
    counts = (C.c_int64 * 1)()
    with pytest.raises(ValueError):
        _lib.call("epd_irp_shard", 10, 0, counts)
    assert "width" in _lib.lib().epd_last_error().decode()
    with pytest.raises(ValueError):
        _lib.call("epd_irp_shard", -1, 2, counts)


@pytest.mark.parametrize("cfg,params,flops", [
    (SIGLIP_MINICPM, 485_616_368, 1040.660299776e9),
    (INTERNVIT_300M, 337_583_104, 740.77290496e9),
    (TINY_VIT, None, None),
])
def test_encoder_schema_host_only(cfg, params, flops):
    from paper_2501_05460_b200.encoder import EncoderSchema
    s = EncoderSchema(cfg)
    sch = s.schema()
    names = [n for n, _ in sch]
    assert len(names) == len(set(names))
    total = sum(int(__import__("math").prod(shape)) for _, shape in sch)
    if params is not None:
        assert total == params
        # SURVEY.md 8(d) algorithmic work per tile
        assert s.flops_per_tile() == pytest.approx(flops, rel=1e-9)
    assert s.launches(10) > 0
    from paper_2501_05460_b200.weights import weight_schema
    assert weight_schema(cfg) == sch  # the pure-Python schema the CPU reference arm uses
    s.close()


def test_encoder_rejects_unsupported_shapes():
    from dataclasses import replace

    from paper_2501_05460_b200.encoder import EncoderSchema
    with pytest.raises(ValueError):
        EncoderSchema(replace(SIGLIP_MINICPM, heads=5))       # 1152 / 5 not integral
    with pytest.raises(ValueError):
        EncoderSchema(replace(SIGLIP_MINICPM, hidden=1152 * 2, heads=8))  # head_dim 288 > 128
    with pytest.raises(ValueError):
        EncoderSchema(replace(INTERNVIT_300M, out_tokens=64))


def test_fp32_check_mode_host_state():
    """Opting into the fp32 check mode is host-only; encoding before finalize fails
    with the reference's RuntimeError mapping, not a crash."""
    import ctypes as C

    from paper_2501_05460_b200.encoder import EncoderSchema
    s = EncoderSchema(TINY_VIT, 1)
    _lib.call("epd_encoder_enable_fp32_check", s._h)
    with pytest.raises(RuntimeError):
        _lib.call("epd_encode_tiles_f32", s._h, C.c_void_p(1), 1, C.c_void_p(1), C.c_void_p(0))
    s.close()


def test_weights_deterministic_and_shaped():
    import torch

    from paper_2501_05460_b200.encoder import canonical_weights
    a = canonical_weights(TINY_VIT, 123)
    b = canonical_weights(TINY_VIT, 123)
    c = canonical_weights(TINY_VIT, 124)
    assert all(torch.equal(a[k], b[k]) for k in a)
    assert any(not torch.equal(a[k], c[k]) for k in a)
    assert torch.allclose(a["layers.0.ln1.weight"].mean(), torch.tensor(1.0), atol=0.05)


def test_sincos_table_matches_public_formula_shape():
    import numpy as np

    from paper_2501_05460_b200.weights import sincos_2d
    t = sincos_2d(3584, 32, 32)
    assert t.shape == (1024, 3584)
    # position (h=0, w=0): sin(0)=0 for the first quarter, cos(0)=1 for the second
    assert np.allclose(t[0, :896], 0) and np.allclose(t[0, 896:1792], 1)
    # the first half encodes the w coordinate: row 1 is (h=0, w=1)
    assert np.isclose(t[1, 0], np.sin(1.0))
    assert np.isclose(t[32, 1792], np.sin(1.0))  # (h=1, w=0): second half carries h


def test_product_refuses_cpu_tensors():
    import torch

    from paper_2501_05460_b200 import kernels
    with pytest.raises(ValueError):
        kernels.linear(torch.zeros(4, 8, dtype=torch.bfloat16), torch.zeros(8, 8, dtype=torch.bfloat16))


def test_llm_configs_match_reference_catalog():
    """The prefill consumer's LLM shapes agree with the reference catalog (models.cfg): layers,
    KV heads, head dim, hidden -> the same KV bytes per token the P->D handoff moves."""
    from paper_2501_05460_b200.prefill import INTERNLM25_7B, QWEN2_7B
    for cfg in (QWEN2_7B, INTERNLM25_7B):
        g = cfg.geometry
        assert (cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.hidden) == (g.num_layers, g.kv_heads, g.head_dim,
                                                                         g.hidden_dim)
        assert cfg.q_heads * cfg.head_dim == cfg.hidden
        assert 2 * cfg.layers * cfg.kv_heads * cfg.head_dim * 2 == g.kv_bytes_per_token()
    assert QWEN2_7B.geometry.kv_bytes_per_token() == 57344 and INTERNLM25_7B.geometry.kv_bytes_per_token() == 131072
