"""Encode worker: the B200 vision encoder behind the reference's encode interface.

Reference seam: ``engine._Sim._start_encode`` charges each IRP worker
``costs.encode_latency(params, patches_on_worker, tp_width=1, batch_size=n)``
seconds (engine.py:603-609, costs.py:78-90). :class:`VisionEncoder` does the
real work for a worker's tiles on its GPU; :meth:`VisionEncoder.encode_latency`
keeps that signature so measured B200 latencies can be fed back through
``costs.calibrate`` (costs.py:146-176).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import EncoderDesc, call, lib
from .configs import SEED, EncoderConfig
from .weights import canonical_weights as _canonical
from .weights import init_weights


def _desc(cfg: EncoderConfig, max_tiles: int) -> EncoderDesc:
    d = EncoderDesc()
    d.family = cfg.family
    d.image_size = cfg.image_size
    d.patch_size = cfg.patch_size
    d.channels = cfg.channels
    d.hidden = cfg.hidden
    d.layers = cfg.layers
    d.heads = cfg.heads
    d.mlp = cfg.mlp
    d.out_tokens = cfg.out_tokens
    d.out_dim = cfg.out_dim
    d.out_heads = cfg.out_heads
    d.max_tiles = max_tiles
    d.ln_eps = cfg.ln_eps
    for i in range(3):
        d.mean[i] = cfg.mean[i]
        d.std[i] = cfg.std[i]
    return d


class EncoderSchema:
    """Host-only handle: create the C encoder object to read its weight schema."""

    def __init__(self, cfg: EncoderConfig, max_tiles: int = 1, device: int = 0):
        self.cfg = cfg
        self._h = C.c_void_p()
        desc = _desc(cfg, max_tiles)
        call("epd_encoder_create", C.byref(desc), device, C.byref(self._h))

    def schema(self) -> list[tuple[str, tuple[int, ...]]]:
        L = lib()
        out = []
        shape = (C.c_int64 * 4)()
        for i in range(L.epd_encoder_num_weights(self._h)):
            name = C.c_char_p()
            nd = C.c_int32()
            call("epd_encoder_weight_info", self._h, i, C.byref(name), C.byref(nd), shape)
            out.append((name.value.decode(), tuple(int(shape[j]) for j in range(nd.value))))
        return out

    def flops_per_tile(self) -> float:
        return float(lib().epd_encoder_flops_per_tile(self._h))

    def launches(self, n: int) -> int:
        return int(lib().epd_encoder_launches(self._h, n))

    def close(self) -> None:
        if self._h:
            lib().epd_encoder_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def canonical_weights(cfg: EncoderConfig, seed: int = SEED) -> dict[str, torch.Tensor]:
    """The fp32 canonical weights both the GPU path and the CPU oracle use (schema from
    weights.weight_schema, which tests/test_abi_cpu.py pins to the C library's)."""
    return _canonical(cfg, seed)


class VisionEncoder(EncoderSchema):
    """One GPU's encoder: bf16 weights + workspace owned by libepd.

    ``encode(tiles)`` maps device uint8 tiles [n, S, S, C] to MM tokens
    [n, out_tokens, out_dim] (bf16) in tile order. With ``check_fp32=True`` the
    library also keeps fp32 weight images and ``encode_f32(tiles)`` runs the same
    pipeline in fp32 on CUDA cores (the north star's 1e-4 check mode).
    """

    def __init__(self, cfg: EncoderConfig, device: torch.device | int = 0, max_tiles: int = 16,
                 weights: dict[str, torch.Tensor] | None = None, seed: int = SEED,
                 check_fp32: bool = False):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("VisionEncoder runs on a CUDA device only (no CPU fallback)")
        super().__init__(cfg, max_tiles, self.device.index or 0)
        self.max_tiles = max_tiles
        sch = self.schema()
        if weights is None:
            weights = init_weights(sch, cfg, seed)
        for i, (name, shape) in enumerate(sch):
            t = weights[name].detach().to("cpu", torch.float32).contiguous()
            if tuple(t.shape) != shape:
                raise ValueError(f"weight {name}: shape {tuple(t.shape)} != {shape}")
            call("epd_encoder_set_weight", self._h, i, C.c_void_p(t.data_ptr()), t.numel())
        self.check_fp32 = check_fp32
        if check_fp32:
            call("epd_encoder_enable_fp32_check", self._h)
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            call("epd_encoder_finalize", self._h, C.c_void_p(stream.cuda_stream))

    def _check_io(self, tiles: torch.Tensor, out: torch.Tensor | None, dtype: torch.dtype) -> torch.Tensor:
        if tiles.device != self.device or tiles.dtype != torch.uint8:
            raise ValueError("tiles must be uint8 on the encoder's device")
        c = self.cfg
        if tuple(tiles.shape[1:]) != (c.image_size, c.image_size, c.channels):
            raise ValueError(f"tiles must be [n, {c.image_size}, {c.image_size}, {c.channels}]")
        if out is None:
            out = torch.empty(tiles.shape[0], c.out_tokens, c.out_dim, dtype=dtype, device=self.device)
        if out.dtype != dtype or tuple(out.shape) != (tiles.shape[0], c.out_tokens, c.out_dim):
            raise ValueError(f"out must be {dtype} [n, {c.out_tokens}, {c.out_dim}]")
        if not tiles.is_contiguous() or not out.is_contiguous():
            raise ValueError("tiles and out must be contiguous")
        return out

    def encode(self, tiles: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = self._check_io(tiles, out, torch.bfloat16)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        call("epd_encode_tiles", self._h, C.c_void_p(tiles.data_ptr()), tiles.shape[0],
             C.c_void_p(out.data_ptr()), C.c_void_p(stream))
        return out

    def encode_f32(self, tiles: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if not self.check_fp32:
            raise RuntimeError("encode_f32 needs VisionEncoder(check_fp32=True)")
        out = self._check_io(tiles, out, torch.float32)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        call("epd_encode_tiles_f32", self._h, C.c_void_p(tiles.data_ptr()), tiles.shape[0],
             C.c_void_p(out.data_ptr()), C.c_void_p(stream))
        return out

    # -- reference-shaped latency provider ------------------------------------------
    def encode_latency(self, params, patches_on_worker: int, tp_width: int = 1, batch_size: int = 1,
                       repeats: int = 3) -> float:
        """Measured seconds for ``patches_on_worker`` tiles, with costs.encode_latency's
        signature and edge rules (costs.py:78-90): negative -> ValueError, empty batch -> 0."""
        if patches_on_worker < 0:
            raise ValueError("patch count must be non-negative")
        if batch_size == 0 or patches_on_worker == 0:
            return 0.0
        n = patches_on_worker
        c = self.cfg
        tiles = torch.randint(0, 256, (n, c.image_size, c.image_size, c.channels), dtype=torch.uint8,
                              device=self.device)
        out = torch.empty(n, c.out_tokens, c.out_dim, dtype=torch.bfloat16, device=self.device)
        self.encode(tiles, out)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(self.device)
        s.record()
        for _ in range(repeats):
            self.encode(tiles, out)
        e.record()
        torch.cuda.synchronize(self.device)
        return s.elapsed_time(e) / repeats / 1e3


__all__ = ["VisionEncoder", "EncoderSchema", "canonical_weights", "_lib"]
