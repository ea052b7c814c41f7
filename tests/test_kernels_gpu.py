"""Per-kernel parity on the B200: each sm_100a kernel (called through the C ABI)
against a plain PyTorch fp32 reference of the same op on the same bf16 inputs.

Metric (BASELINE.json north_star): max|y - y_ref| / max|y_ref| <= 1e-2 for bf16.
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-2


def relerr(y, ref):
    y = y.float()
    ref = ref.float()
    return ((y - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


def _bf(*shape, scale=1.0, gen=None, device="cuda"):
    return (torch.randn(*shape, generator=gen, device=device) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K,bn", [
    (256, 256, 128, 0), (1000, 1152, 1152, 128), (1000, 1152, 1152, 192), (1000, 1152, 1152, 256),
    (384, 4304, 1152, 0), (256, 1152, 4304, 0), (4, 64, 64, 0), (16, 8, 8, 0), (10240, 3840, 1152, 0),
])
def test_linear_plain(cuda, M, N, K, bn):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N + K)
    a = _bf(M, K, gen=g)
    w = _bf(N, K, scale=K ** -0.5, gen=g)
    y = kernels.linear(a, w, bn=bn)
    torch.cuda.synchronize()
    ref = a.float() @ w.float().t()
    assert relerr(y, ref) <= TOL


@pytest.mark.parametrize("act", ["none", "gelu_tanh", "gelu_erf"])
def test_linear_epilogue(cuda, act):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(11)
    M, N, K, T = 2048, 1152, 640, 1024
    a = _bf(M, K, gen=g)
    w = _bf(N, K, scale=K ** -0.5, gen=g)
    b = _bf(N, gen=g)
    r = _bf(T, N, gen=g)
    ls = _bf(N, scale=0.1, gen=g)
    y = kernels.linear(a, w, bias=b, act=act, resid=r, r_mod=T, lscale=ls)
    torch.cuda.synchronize()
    x = a.float() @ w.float().t() + b.float()
    if act == "gelu_tanh":
        x = torch.nn.functional.gelu(x, approximate="tanh")
    elif act == "gelu_erf":
        x = torch.nn.functional.gelu(x)
    ref = r.float().repeat(M // T, 1) + ls.float() * x
    assert relerr(y, ref) <= TOL


def test_linear_inplace_residual(cuda):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(5)
    M, N, K = 1024, 1152, 1152
    a = _bf(M, K, gen=g)
    w = _bf(N, K, scale=K ** -0.5, gen=g)
    h = _bf(M, N, gen=g)
    ref = h.float() + a.float() @ w.float().t()
    kernels.linear(a, w, resid=h, out=h)
    torch.cuda.synchronize()
    assert relerr(h, ref) <= TOL


@pytest.mark.parametrize("M,N,K,bn,ls", [(2048, 1152, 1152, 0, True), (1000, 1152, 4304, 256, False),
                                          (4, 64, 64, 0, True)])
def test_linear_acc_f32(cuda, M, N, K, bn, ls):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    a = _bf(M, K, gen=g)
    w = _bf(N, K, scale=K ** -0.5, gen=g)
    b = _bf(N, gen=g)
    s = _bf(N, scale=0.1, gen=g) if ls else None
    h = torch.randn(M, N, generator=g, device=cuda)
    ref = h.clone() + (a.float() @ w.float().t() + b.float()) * (s.float() if ls else 1.0)
    kernels.linear_acc(a, w, h, bias=b, lscale=s, bn=bn)
    torch.cuda.synchronize()
    assert relerr(h, ref) <= 2e-3


def _attn_ref(q, k, v, B, H, Tq, Tk, Dv, hs, q_shared, scale):
    """fp32 reference on the row-major layout (head h = columns [h*hs, h*hs + Dv))."""
    def heads(x, T, nb):
        return x.float().reshape(nb, T, -1)[..., :H * hs].reshape(nb, T, H, hs)[..., :Dv].permute(0, 2, 1, 3)
    qf = heads(q, Tq, 1 if q_shared else B)
    if q_shared:
        qf = qf.expand(B, H, Tq, Dv)
    kf, vf = heads(k, Tk, B), heads(v, Tk, B)
    p = torch.softmax(qf @ kf.transpose(-1, -2) * scale, dim=-1)
    return (p @ vf).permute(0, 2, 1, 3).reshape(B * Tq, H * Dv)


@pytest.mark.parametrize("B,H,Tq,Tk,Dv,hs,q_shared,qscale", [
    (2, 16, 1024, 1024, 72, 72, False, 1.0),   # SigLIP: packed 72-wide heads (Dp 80 reads the next head)
    (2, 16, 1024, 1024, 72, 80, False, 1.0),   # padded 80-wide heads
    (1, 16, 1025, 1025, 64, 64, False, 1.0),   # InternViT (CLS -> ragged last key block, rows cross images)
    (2, 28, 64, 1024, 128, 128, True, 1.0),    # MiniCPM resampler cross-attention (shared queries)
    (1, 1, 4, 16, 8, 8, True, 1.0),            # tiny
    (3, 2, 300, 200, 64, 64, False, 1.0),
    (1, 4, 256, 1024, 72, 72, False, 6.0),     # peaked scores: exercises the lazy O rescale
])
def test_attention(cuda, B, H, Tq, Tk, Dv, hs, q_shared, qscale):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(B * 100 + H + Tq + Tk + hs)
    # Q, K, V as column sections of one fused projection matrix, as the encoder lays them out
    qkv = _bf(B * max(Tq, Tk), 3 * H * hs, gen=g)
    q = (_bf(Tq, H * hs, scale=qscale, gen=g) if q_shared else qkv[:B * Tq, :H * hs] * qscale)
    k = qkv[:B * Tk, H * hs:2 * H * hs]
    v = qkv[:B * Tk, 2 * H * hs:]
    scale = 1.0 / math.sqrt(Dv)
    y = kernels.attention(q, k, v, B, H, Tq, Tk, Dv, scale, head_stride=hs, q_shared=q_shared)
    torch.cuda.synchronize()
    assert relerr(y, _attn_ref(q, k, v, B, H, Tq, Tk, Dv, hs, q_shared, scale)) <= TOL


def test_attention_rejects_bad_layouts(cuda):
    from paper_2501_05460_b200 import kernels
    x = torch.zeros(128, 64, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ValueError):
        kernels.attention(x, x, x, 1, 1, 128, 128, 64, 0.125, head_stride=32)  # head_stride < Dv
    with pytest.raises(ValueError):
        kernels.attention(x.t(), x, x, 1, 1, 64, 128, 64, 0.125)                # not row-major


@pytest.mark.parametrize("rows,D", [(1000, 1152), (64, 3584), (8, 4096), (5, 8)])
def test_layernorm(cuda, rows, D):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(rows + D)
    x = _bf(rows, D, scale=3.0, gen=g) + 1.5
    gm = _bf(D, gen=g)
    bt = _bf(D, gen=g)
    y = kernels.layernorm(x, gm, bt, 1e-6)
    torch.cuda.synchronize()
    ref = torch.nn.functional.layer_norm(x.float(), (D,), gm.float(), bt.float(), 1e-6)
    assert relerr(y, ref) <= TOL


@pytest.mark.parametrize("rows,D", [(10240, 1152), (12300, 1024), (7, 4096), (3, 8)])
def test_layernorm_f32_input(cuda, rows, D):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(rows * 3 + D)
    x = torch.randn(rows, D, device=cuda, generator=g) * 4.0 + 2.5
    gm = _bf(D, gen=g)
    bt = _bf(D, gen=g)
    y = kernels.layernorm_f32(x, gm, bt, 1e-6)
    torch.cuda.synchronize()
    ref = torch.nn.functional.layer_norm(x, (D,), gm.float(), bt.float(), 1e-6)
    assert relerr(y, ref) <= TOL


def test_patchify(cuda):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(3)
    n, S, p = 3, 448, 14
    tiles = torch.randint(0, 256, (n, S, S, 3), dtype=torch.uint8, device=cuda, generator=g)
    mean, std = (0.5, 0.4, 0.3), (0.5, 0.6, 0.7)
    y = kernels.patchify(tiles, p, 640, mean, std)
    torch.cuda.synchronize()
    x = tiles.float() / 255.0
    x = (x - torch.tensor(mean, device=cuda)) / torch.tensor(std, device=cuda)
    x = x.permute(0, 3, 1, 2)  # n C S S
    cols = torch.nn.functional.unfold(x, kernel_size=p, stride=p)  # n, C*p*p, L  (c, ky, kx)
    ref = cols.transpose(1, 2).reshape(n * (S // p) ** 2, 3 * p * p)
    assert relerr(y[:, :588], ref) <= 4e-3
    assert y[:, 588:].abs().max().item() == 0


@pytest.mark.parametrize("M,T,H,Dp,dh,trans", [
    (2048, 1024, 16, 80, 72, (False, False, True)),   # SigLIP QKV
    (2050, 1025, 16, 64, 64, (False, False, True)),   # InternViT (images straddle M tiles)
    (64, 64, 28, 128, 128, (False,)),                 # resampler query projection
    (2048, 1024, 28, 128, 128, (False, True)),        # resampler K / V^T
    (4, 4, 1, 64, 8, (False,)),                       # tiny
])
def test_linear_heads(cuda, M, T, H, Dp, dh, trans):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(M + T + H)
    S = len(trans)
    K = 256
    a = _bf(M, K, gen=g)
    w = torch.zeros(S * H * Dp, K, dtype=torch.bfloat16, device=cuda)
    b = torch.zeros(S * H * Dp, dtype=torch.bfloat16, device=cuda)
    for s in range(S):
        for h in range(H):
            base = (s * H + h) * Dp
            w[base:base + dh] = _bf(dh, K, scale=K ** -0.5, gen=g)
            b[base:base + dh] = _bf(dh, gen=g)
    pos = _bf(T, S * H * Dp, gen=g)
    outs = kernels.linear_heads(a, w, H, Dp, T, S, trans=trans, bias=b, resid=pos, r_mod=T)
    torch.cuda.synchronize()
    full = a.float() @ w.float().t() + b.float() + pos.float().repeat(M // T, 1)
    nb = M // T
    for s in range(S):
        ref = full[:, s * H * Dp:(s + 1) * H * Dp].reshape(nb, T, H, Dp).permute(0, 2, 1, 3).reshape(nb * H, T, Dp)
        got = outs[s][..., :T].transpose(1, 2) if trans[s] else outs[s]
        assert relerr(got, ref) <= TOL, s


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"])
def cta_group(request, cuda):
    from paper_2501_05460_b200._lib import call
    call("epd_set_gemm_cta_group", request.param)
    yield request.param
    call("epd_set_gemm_cta_group", 0)


@pytest.mark.parametrize("M,N,K,bn", [(1000, 1152, 1152, 256), (2048, 3840, 1152, 0), (4096, 4304, 1152, 192),
                                      (2304, 1152, 4304, 0), (300, 512, 64, 256)])
def test_linear_cta_groups(cuda, cta_group, M, N, K, bn):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(M + N + K + cta_group)
    a = _bf(M, K, gen=g)
    w = _bf(N, K, scale=K ** -0.5, gen=g)
    b = _bf(N, gen=g)
    y = kernels.linear(a, w, bias=b, act="gelu_tanh", bn=bn)
    h = torch.randn(M, N, generator=g, device=cuda)
    ref_h = h.clone() + a.float() @ w.float().t()
    kernels.linear_acc(a, w, h, bn=bn)
    torch.cuda.synchronize()
    ref = torch.nn.functional.gelu(a.float() @ w.float().t() + b.float(), approximate="tanh")
    assert relerr(y, ref) <= TOL
    assert relerr(h, ref_h) <= 2e-3


def test_linear_heads_cta_pairs(cuda, cta_group):
    from paper_2501_05460_b200 import kernels
    g = torch.Generator(device=cuda).manual_seed(77)
    M, T, H, Dp, K = 3075, 1025, 16, 64, 256  # InternViT-like: images straddle 256-row pair tiles
    a = _bf(M, K, gen=g)
    w = _bf(3 * H * Dp, K, scale=K ** -0.5, gen=g)
    outs = kernels.linear_heads(a, w, H, Dp, T, 3, trans=(False, False, False))
    torch.cuda.synchronize()
    full = a.float() @ w.float().t()
    nb = M // T
    for s in range(3):
        ref = full[:, s * H * Dp:(s + 1) * H * Dp].reshape(nb, T, H, Dp).permute(0, 2, 1, 3).reshape(nb * H, T, Dp)
        assert relerr(outs[s], ref) <= TOL
