"""Out-of-bounds write guard (compute-sanitizer is closed on this GPU pool): every libepd
kernel writes its output into the middle of a larger buffer whose head and tail guard
bands hold a canary pattern; the bands must come back untouched, at ragged shapes that
exercise the tail paths (partial M / N tiles, half-width tiles, straddling attention
items, odd record counts)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes of canary on each side


def _guarded(shape, dtype, device):
    """(full byte buffer, view of `shape` in its middle); the guard bands hold 0xA5."""
    n = torch.empty(shape, dtype=dtype).numel() * torch.tensor([], dtype=dtype).element_size()
    raw = torch.full((GUARD + n + GUARD,), 0xA5, dtype=torch.uint8, device=device)
    view = raw[GUARD:GUARD + n].view(dtype).view(shape)
    return raw, view


def _intact(raw):
    head, tail = raw[:GUARD], raw[-GUARD:]
    return bool((head == 0xA5).all()) and bool((tail == 0xA5).all())


def _bf(*s, device="cuda"):
    return (torch.randn(*s, device=device) * 0.1).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(130, 200, 64), (1000, 1152, 1152), (257, 4304, 128), (3000, 328, 72)])
@pytest.mark.parametrize("act", ["none", "gelu_erf"])
def test_gemm_rows_and_acc_stay_in_bounds(cuda, M, N, K, act):
    from paper_2501_05460_b200 import kernels
    a, w, b = _bf(M, K), _bf(N, K), _bf(N)
    raw, out = _guarded((M, N), torch.bfloat16, cuda)
    kernels.linear(a, w, bias=b, act=act, out=out)
    rawf, h = _guarded((M, N), torch.float32, cuda)
    h.zero_()
    kernels.linear_acc(a, w, h, bias=b)
    torch.cuda.synchronize()
    assert _intact(raw) and _intact(rawf)
    ref = a.float() @ w.float().t() + b.float()
    assert ((h - ref).abs().max() / ref.abs().max()) < 1e-2


def test_swiglu_and_attention_stay_in_bounds(cuda):
    from paper_2501_05460_b200 import kernels
    M, F, K = 700, 512, 256
    w = kernels.swiglu_interleave(_bf(F, K), _bf(F, K))
    raw, out = _guarded((M, F), torch.bfloat16, cuda)
    kernels.linear(_bf(M, K), w, act="swiglu", out=out)
    for B, H, T, dv, causal in [(3, 4, 1025, 64, False), (2, 5, 1024, 72, False), (1, 8, 333, 128, True)]:
        qkv = _bf(B * T, 3 * H * dv)
        rawa, o = _guarded((B * T, H * dv), torch.bfloat16, cuda)
        kernels.attention(qkv[:, :H * dv], qkv[:, H * dv:2 * H * dv], qkv[:, 2 * H * dv:], B, H, T, T, dv,
                          dv ** -0.5, out=o, causal=causal)
        torch.cuda.synchronize()
        assert _intact(rawa), (B, H, T, dv)
    assert _intact(raw)


def test_norms_patchify_records_stay_in_bounds(cuda):
    from paper_2501_05460_b200 import kernels
    from paper_2501_05460_b200._lib import call
    import ctypes as C
    g1, b1 = torch.ones(1152, dtype=torch.bfloat16, device=cuda), torch.zeros(1152, dtype=torch.bfloat16, device=cuda)
    raw, out = _guarded((77, 1152), torch.bfloat16, cuda)
    kernels.layernorm_f32(torch.randn(77, 1152, device=cuda), g1, b1, 1e-6, out=out)
    tiles = torch.randint(0, 256, (3, 448, 448, 3), dtype=torch.uint8, device=cuda)
    rawp, xp = _guarded((3 * 1024, 640), torch.bfloat16, cuda)
    kernels.patchify(tiles, 14, 640, (0.5, 0.5, 0.5), (0.5, 0.5, 0.5), out=xp)
    src = torch.randn(9, 48, device=cuda)
    rawr, dst = _guarded((9, 48), torch.float32, cuda)
    idx = torch.tensor([8, 0, 3, 1, 7, 2, 6, 5, 4], dtype=torch.int32, device=cuda)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    call("epd_scatter_records", C.c_void_p(src.data_ptr()), C.c_void_p(idx.data_ptr()), 9, 48 * 4,
         C.c_void_p(dst.data_ptr()), s)
    torch.cuda.synchronize()
    assert _intact(raw) and _intact(rawp) and _intact(rawr)
    assert torch.equal(dst[idx.long()], src)


def test_encoder_output_and_cache_plan_stay_in_bounds(cuda):
    from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM
    from paper_2501_05460_b200.encoder import VisionEncoder
    from paper_2501_05460_b200.mmcache import MMTokenCache
    from paper_2501_05460_b200.stage import tiles_for_request
    for cfg, n in [(SIGLIP_MINICPM.with_layers(2), 3), (INTERNVIT_300M.with_layers(2), 5)]:
        enc = VisionEncoder(cfg, cuda, max_tiles=4)
        raw, out = _guarded((n, cfg.out_tokens, cfg.out_dim), torch.bfloat16, cuda)
        enc.encode(tiles_for_request(n, cfg, seed=3).to(cuda), out)
        torch.cuda.synchronize()
        assert _intact(raw), cfg.name
    cache = MMTokenCache(16, 4, 8, cuda, secret=0)
    for step in range(20):
        recs = torch.randint(0, 256, (11, 64), dtype=torch.uint8, device=cuda)
        recs[5:] = recs[:6].clone()
        cache.plan(cache.hash(recs))
    cache.check()
