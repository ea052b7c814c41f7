"""Torch-tensor front ends for the kernel-level C-ABI ops (libepd.so).

PyTorch supplies device memory and the current stream; all arithmetic runs in
the sm_100a kernels. Every function requires CUDA tensors and fails loudly
otherwise -- there is no CPU path.
"""
from __future__ import annotations

import torch

from ._lib import call

ACT = {"none": 0, "gelu_tanh": 1, "gelu_erf": 2, "swiglu": 3}


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _need_cuda(*ts: torch.Tensor | None) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libepd ops take CUDA tensors only (no CPU fallback)")


def linear(a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, act: str = "none",
           resid: torch.Tensor | None = None, r_mod: int = 0, lscale: torch.Tensor | None = None,
           out: torch.Tensor | None = None, bn: int = 0) -> torch.Tensor:
    """out = act(a @ w.T + bias); if resid: out = resid[row % r_mod] + lscale * out (bf16).

    act="swiglu": w's rows alternate 32-row gate / up groups (see swiglu_interleave); out has
    N/2 columns, out[:, 32g + j] = silu(gate) * up of group g."""
    _need_cuda(a, w, bias, resid, lscale, out)
    M, K = a.shape
    N = w.shape[0]
    if out is None:
        out = torch.empty(M, N // 2 if act == "swiglu" else N, dtype=torch.bfloat16, device=a.device)
    call("epd_linear_bf16", a.data_ptr(), a.stride(0), w.data_ptr(), w.stride(0), M, N, K, _ptr(bias),
         ACT[act], _ptr(resid), resid.stride(0) if resid is not None else 0, r_mod, _ptr(lscale),
         out.data_ptr(), out.stride(0), bn, _stream(a))
    return out


def linear_acc(a: torch.Tensor, w: torch.Tensor, h: torch.Tensor, bias: torch.Tensor | None = None,
               lscale: torch.Tensor | None = None, bn: int = 0, max_split: int = 0) -> torch.Tensor:
    """h (fp32, in place) += lscale * (a @ w.T + bias). ``max_split`` > 1 lets the GEMM split
    K (deterministic order, not batch invariant; for the LLM prefill)."""
    _need_cuda(a, w, h, bias, lscale)
    if h.dtype != torch.float32:
        raise ValueError("h must be fp32")
    M, K = a.shape
    N = w.shape[0]
    call("epd_linear_acc_f32_split", a.data_ptr(), a.stride(0), w.data_ptr(), w.stride(0), M, N, K, _ptr(bias),
         _ptr(lscale), h.data_ptr(), h.stride(0), bn, max_split, _stream(a))
    return h


def linear_heads(a: torch.Tensor, w: torch.Tensor, H: int, Dp: int, T: int, sections: int,
                 trans=(False, False, True), bias: torch.Tensor | None = None,
                 resid: torch.Tensor | None = None, r_mod: int = 0):
    """Project a [M, K] -> per-head Q/K [nb*H, T, Dp] / keys-major V^T [nb*H, Dp, Tpad] tensors."""
    _need_cuda(a, w, bias, resid)
    M, K = a.shape
    N = w.shape[0]
    nb = -(-M // T)
    Tpad = (T + 7) // 8 * 8
    outs = []
    for s in range(sections):
        shape = (nb * H, Dp, Tpad) if trans[s] else (nb * H, T, Dp)
        outs.append(torch.zeros(shape, dtype=torch.bfloat16, device=a.device))
    ptrs = [o.data_ptr() for o in outs] + [None] * (3 - sections)
    mask = sum(1 << s for s in range(sections) if trans[s])
    call("epd_linear_heads_bf16", a.data_ptr(), a.stride(0), w.data_ptr(), w.stride(0), M, N, K, _ptr(bias),
         _ptr(resid), resid.stride(0) if resid is not None else 0, r_mod, H, Dp, T, Tpad, H * Dp, ptrs[0], ptrs[1],
         ptrs[2], mask, _stream(a))
    return outs


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, B: int, H: int, Tq: int, Tk: int,
              Dv: int, scale: float, head_stride: int | None = None, q_shared: bool = False,
              out: torch.Tensor | None = None, kv_heads: int | None = None, causal: bool = False) -> torch.Tensor:
    """Fused MHA / GQA read in place from row-major projections.

    q: [B*Tq (or Tq if q_shared), >= H*head_stride] (a column slice of a wider matrix is fine),
    k, v: [B*Tk, ...] with ``kv_heads`` heads (query head h uses K/V head h // (H // kv_heads));
    head h occupies columns [h*head_stride, h*head_stride + Dv). ``causal``: query t sees keys
    <= t + (Tk - Tq). Returns out [B*Tq, H*Dv].
    """
    _need_cuda(q, k, v, out)
    hs = head_stride or Dv
    Dp = 64 if Dv <= 64 else (80 if Dv <= 80 else 128)
    for t in (q, k, v):
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError("q, k, v must be 2-D row-major (unit column stride)")
    if out is None:
        out = torch.empty(B * Tq, H * Dv, dtype=torch.bfloat16, device=q.device)
    flags = (1 if q_shared else 0) | (2 if causal else 0)
    call("epd_attention_bf16", q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(), v.stride(0),
         out.data_ptr(), out.stride(0), B, H, kv_heads or 0, Tq, Tk, Dp, Dv, hs, flags, float(scale), _stream(q))
    return out


def layernorm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float,
              out: torch.Tensor | None = None) -> torch.Tensor:
    _need_cuda(x, gamma, beta, out)
    rows, D = x.shape
    if out is None:
        out = torch.empty_like(x)
    call("epd_layernorm_bf16", x.data_ptr(), x.stride(0), out.data_ptr(), out.stride(0), gamma.data_ptr(),
         beta.data_ptr(), rows, D, float(eps), _stream(x))
    return out


def layernorm_f32(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """fp32 rows -> LayerNorm -> bf16 rows (the residual-stream normalisation)."""
    _need_cuda(x, gamma, beta, out)
    if x.dtype != torch.float32:
        raise ValueError("layernorm_f32 takes fp32 rows")
    rows, D = x.shape
    if out is None:
        out = torch.empty(rows, D, dtype=torch.bfloat16, device=x.device)
    call("epd_layernorm_f32_bf16", x.data_ptr(), x.stride(0), out.data_ptr(), out.stride(0), gamma.data_ptr(),
         beta.data_ptr(), rows, D, float(eps), _stream(x))
    return out


def patchify(tiles: torch.Tensor, patch: int, kpad: int, mean, std, row_offset: int = 0,
             rows_per_tile: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """uint8 [n,S,S,C] -> bf16 [n*rows_per_tile, kpad] normalised im2col rows."""
    _need_cuda(tiles)
    import ctypes
    n, S, _, Cc = tiles.shape
    npatch = (S // patch) ** 2
    rpt = rows_per_tile or npatch + row_offset
    if out is None:
        out = torch.zeros(n * rpt, kpad, dtype=torch.bfloat16, device=tiles.device)
    if out.shape != (n * rpt, kpad) or out.dtype != torch.bfloat16 or not out.is_contiguous():
        raise ValueError(f"out must be contiguous bf16 [{n * rpt}, {kpad}]")
    m = (ctypes.c_float * 3)(*mean)
    s = (ctypes.c_float * 3)(*std)
    call("epd_patchify_u8", tiles.data_ptr(), n, S, Cc, patch, kpad, row_offset, rpt,
         ctypes.cast(m, ctypes.c_void_p), ctypes.cast(s, ctypes.c_void_p), out.data_ptr(), _stream(tiles))
    return out


# ---- prefill consumer (llm.cu)

def swiglu_interleave(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """[F, K] gate and up rows -> [2F, K] in the 32-row alternating layout act="swiglu" reads."""
    F, K = gate.shape
    if F % 32 or up.shape != gate.shape:
        raise ValueError("gate/up must be equal [F, K] with F % 32 == 0")
    return torch.stack([gate.view(F // 32, 32, K), up.view(F // 32, 32, K)], 1).reshape(2 * F, K)


def rmsnorm_f32(x: torch.Tensor, gamma: torch.Tensor, eps: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """fp32 rows -> RMSNorm(gamma) -> bf16 rows."""
    _need_cuda(x, gamma, out)
    rows, D = x.shape
    if out is None:
        out = torch.empty(rows, D, dtype=torch.bfloat16, device=x.device)
    call("epd_rmsnorm_f32_bf16", x.data_ptr(), x.stride(0), out.data_ptr(), out.stride(0), gamma.data_ptr(), rows, D,
         float(eps), _stream(x))
    return out


def rope_(x: torch.Tensor, col0: int, nheads: int, head_dim: int, theta: float, pos0: int = 0,
          table: torch.Tensor | None = None) -> torch.Tensor:
    """In-place rotary embedding (rotate-half) on heads [0, nheads) starting at column col0.
    ``table``: optional rope_table(...) for the same rows / head_dim / pos0 / theta."""
    _need_cuda(x, table)
    call("epd_rope_bf16", x.data_ptr(), x.stride(0), x.shape[0], col0, nheads, head_dim, pos0, float(theta),
         _ptr(table), _stream(x))
    return x


def rope_table(rows: int, head_dim: int, theta: float, pos0: int = 0, device=None) -> torch.Tensor:
    """fp32 [rows, head_dim/2, 2] (cos, sin) table for rope_."""
    t = torch.empty(rows, head_dim // 2, 2, dtype=torch.float32, device=device)
    call("epd_rope_table", t.data_ptr(), rows, head_dim, pos0, float(theta), _stream(t))
    return t


def silu_mul(gu: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """[rows, 2F] (gate | up) -> silu(gate) * up [rows, F]."""
    _need_cuda(gu, out)
    rows, F2 = gu.shape
    if out is None:
        out = torch.empty(rows, F2 // 2, dtype=torch.bfloat16, device=gu.device)
    call("epd_silu_mul_bf16", gu.data_ptr(), gu.stride(0), out.data_ptr(), out.stride(0), rows, F2 // 2, _stream(gu))
    return out


def kv_write_paged(k: torch.Tensor, v_off: int, row_elems: int, block_ids: torch.Tensor, block_size: int,
                   pool: torch.Tensor, layer: int) -> None:
    """Rows of K (k) and V (k + v_off columns) into the paged pool [2L][blocks][block_size*row_elems]."""
    _need_cuda(k, block_ids, pool)
    call("epd_kv_write_paged", k.data_ptr(), k.stride(0), v_off, k.shape[0], row_elems, block_ids.data_ptr(),
         block_size, pool.data_ptr(), pool.shape[1] * pool.shape[2], 2 * layer, _stream(k))


def gather_rows_f32(src: torch.Tensor, index: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[r] = float(src[index[r]])."""
    _need_cuda(src, index, out)
    call("epd_gather_rows_f32", src.data_ptr(), src.stride(0), index.data_ptr(), index.numel(), out.shape[1],
         out.data_ptr(), out.stride(0), _stream(src))
    return out


def argmax(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    _need_cuda(x, out)
    if out is None:
        out = torch.empty(1, dtype=torch.int32, device=x.device)
    call("epd_argmax_bf16", x.data_ptr(), x.numel(), out.data_ptr(), _stream(x))
    return out
