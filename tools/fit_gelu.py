#!/usr/bin/env python
"""Fit the GELU epilogue polynomials (csrc/gemm.cu gelu_poly): for z = min(|x|, 8),
phi(-z) = 2^-F(z) with F a degree-8 polynomial in v = z/4 - 1, so GELU(x) = x * phi(x) costs
one MUFU ex2 and stays relative-accurate on the negative tail (no 1 + tanh cancellation).
GELU-tanh uses the exact sigma(2u) form instead (ex2 + rcp on the MUFU, emulated below).
Prints the fp32 coefficients (highest power first) and the fp32-emulated accuracy."""
import numpy as np
import torch
from scipy.special import log_ndtr, ndtr

ZMAX, DEG = 8.0, 8
LOG2E = 1 / np.log(2)
K0, K1 = np.sqrt(2 / np.pi), 0.044715


def F_erf(z):  # -log2 Phi(-z)
    return -log_ndtr(-z) * LOG2E


def exact_phi(kind, x):
    if kind == "erf":
        return ndtr(x)
    from scipy.special import expit
    return expit(2 * K0 * (x + K1 * x ** 3))  # 0.5 (1 + tanh u) without cancellation


def fit(Fz):
    k = np.arange(4000)
    v = np.cos(np.pi * (k + 0.5) / 4000)
    c = np.polynomial.chebyshev.chebfit(v, Fz((v + 1) * ZMAX / 2), DEG)
    return np.polynomial.chebyshev.cheb2poly(c).astype(np.float32)[::-1]  # highest power first


def emulate(p, x):
    z = np.minimum(np.abs(x), np.float32(ZMAX))
    v = (z * np.float32(2 / ZMAX) - np.float32(1)).astype(np.float32)
    acc = np.full_like(v, p[0])
    for c in p[1:]:
        acc = (acc * v + c).astype(np.float32)
    q = np.exp2(-acc.astype(np.float64)).astype(np.float32)
    return (x * np.where(x >= 0, np.float32(1) - q, q)).astype(np.float32)


if __name__ == "__main__":
    x = np.linspace(-ZMAX, ZMAX, 800001).astype(np.float32)
    for kind, Fz in (("erf", F_erf),):
        p = fit(Fz)
        g = emulate(p, x)
        ex = x.astype(np.float64) * exact_phi(kind, x.astype(np.float64))
        m = np.abs(ex) > 1e-30
        rel = np.abs(g[m] - ex[m]) / np.abs(ex[m])
        mis = (torch.from_numpy(g).bfloat16() != torch.from_numpy(ex.astype(np.float32)).bfloat16()).float().mean()
        print(f"{kind}: max rel err {rel.max():.2e}, bf16 outputs differing from exact {float(mis):.5f}")
        print("  {" + ", ".join(f"{c:.9e}f" for c in p) + "}")


def emulate_tanh_rcp(x):
    """fp32 emulation of gemm.cu gelu_tanh_chunk (ex2 + reciprocal, both MUFU; emulated as
    correctly rounded, the hardware approximations are within ~2 ulp)."""
    f = np.float32
    z = np.abs(x)
    a = (z * (f(-0.10294324159622192) * (z * z) + f(-2.302208185195923))).astype(np.float32)
    e = np.exp2(a.astype(np.float64)).astype(np.float32)
    y = (f(1) + e).astype(np.float32)
    yy = (y * np.roll(y, 1)).astype(np.float32)  # the pair product (neighbours stand in for the pair)
    r = ((f(1) / yy).astype(np.float32) * np.roll(y, 1)).astype(np.float32)
    return (x * np.where(x >= 0, r, e * r)).astype(np.float32)


if __name__ == "__main__":
    g = emulate_tanh_rcp(x)
    ex = x.astype(np.float64) * exact_phi("tanh", x.astype(np.float64))
    m = np.abs(ex) > 1e-30
    mis = (torch.from_numpy(g).bfloat16() != torch.from_numpy(ex.astype(np.float32)).bfloat16()).float().mean()
    print(f"tanh (ex2 + rcp): max rel err {(np.abs(g[m] - ex[m]) / np.abs(ex[m])).max():.2e}, "
          f"bf16 outputs differing {float(mis):.5f}")
