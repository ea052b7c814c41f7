"""ctypes binding of ``libepd.so`` (the C ABI declared in ``include/epd.h``).

The product path has no CPU fallback: if the library is missing or fails to
load, :func:`lib` raises. Status codes map onto the exception classes the
reference raises for the same condition (see ``include/epd.h``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("EPD_LIB_PATH") or Path(__file__).resolve().parent / "libepd.so")

EPD_OK = 0
EPD_ERR_VALUE = 1
EPD_ERR_RUNTIME = 2
EPD_ERR_CAPACITY = 4
EPD_ERR_CUDA = 5
EPD_ERR_UNSUPPORTED = 6

FAMILY_SIGLIP_RESAMPLER = 1
FAMILY_INTERNVIT_MLP = 2


class CapacityExceeded(Exception):
    """Mirror of ``disaggsim.simconfig.CapacityExceeded`` (simconfig.py:19-20)."""


class EncoderDesc(C.Structure):
    _fields_ = [
        ("family", C.c_int32), ("image_size", C.c_int32), ("patch_size", C.c_int32),
        ("channels", C.c_int32), ("hidden", C.c_int32), ("layers", C.c_int32),
        ("heads", C.c_int32), ("mlp", C.c_int32), ("out_tokens", C.c_int32),
        ("out_dim", C.c_int32), ("out_heads", C.c_int32), ("max_tiles", C.c_int32),
        ("ln_eps", C.c_float), ("mean", C.c_float * 3), ("std", C.c_float * 3),
    ]


_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64

# name -> (restype, argtypes)
_SIGS = {
    "epd_abi_version": (_i32, []),
    "epd_last_error": (C.c_char_p, []),
    "epd_irp_shard": (_i32, [_i64, _i32, C.POINTER(_i64)]),
    "epd_irp_ranges": (_i32, [_i64, _i32, C.POINTER(_i64), C.POINTER(_i64)]),
    "epd_encoder_create": (_i32, [C.POINTER(EncoderDesc), _i32, C.POINTER(_vp)]),
    "epd_encoder_destroy": (None, [_vp]),
    "epd_encoder_num_weights": (_i32, [_vp]),
    "epd_encoder_weight_info": (_i32, [_vp, _i32, C.POINTER(C.c_char_p), C.POINTER(_i32), C.POINTER(_i64)]),
    "epd_encoder_set_weight": (_i32, [_vp, _i32, _vp, _i64]),
    "epd_encoder_finalize": (_i32, [_vp, _vp]),
    "epd_encode_tiles": (_i32, [_vp, _vp, _i32, _vp, _vp]),
    "epd_encoder_enable_fp32_check": (_i32, [_vp]),
    "epd_encode_tiles_f32": (_i32, [_vp, _vp, _i32, _vp, _vp]),
    "epd_encoder_flops_per_tile": (C.c_double, [_vp]),
    "epd_encoder_launches": (_i32, [_vp, _i32]),
    "epd_encoder_set_graphs": (_i32, [_vp, _i32]),
    "epd_encoder_profile": (_i32, [_vp, _i32]),
    "epd_encoder_profile_read": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32]),
    "epd_encoder_profile_launches": (_i32, [_vp, _vp, _vp, _vp, _i32]),
    "epd_hash_records": (_i32, [_vp, _i32, _i64, _i64, _vp, _vp, _vp]),
    "epd_hash_records_keyed": (_i32, [_vp, _i32, _i64, _i64, C.c_uint64, C.c_uint64, _vp, _vp, _vp]),
    "epd_mmcache_plan": (_i32, [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "epd_mmcache_create": (_i32, [_i64, _i32, C.POINTER(_vp)]),
    "epd_mmcache_destroy": (None, [_vp]),
    "epd_mmcache_lookup": (_i32, [_vp, _vp, _i32, _vp, _vp, _vp]),
    "epd_mmcache_insert": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "epd_mmcache_erase": (_i32, [_vp, _vp, _i32, _vp]),
    "epd_mmcache_clear": (_i32, [_vp, _vp]),
    "epd_mmcache_check": (_i32, [_vp, _vp]),
    "epd_gather_records": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp]),
    "epd_scatter_records": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp]),
    "epd_timestamp": (_i32, [_vp, _vp]),
    "epd_comm_version": (_i32, [C.POINTER(_i32)]),
    "epd_comm_unique_id": (_i32, [_vp]),
    "epd_comm_init": (_i32, [_vp, _i32, _i32, _i32, C.POINTER(_vp)]),
    "epd_comm_destroy": (None, [_vp]),
    "epd_gather_tokens": (_i32, [_vp, _vp, _i64, _i64, _vp, _i32, _vp]),
    "epd_comm_send": (_i32, [_vp, _vp, _i64, _i32, _vp]),
    "epd_comm_recv": (_i32, [_vp, _vp, _i64, _i32, _vp]),
    "epd_comm_group_start": (_i32, []),
    "epd_comm_group_end": (_i32, []),
    "epd_kv_handoff_send": (_i32, [_vp, _vp, _i32, _i64, _i64, _vp, _i32, _vp, _i32, _vp]),
    "epd_kv_handoff_recv": (_i32, [_vp, _vp, _i32, _i64, _i64, _vp, _i32, _vp, _i32, _vp]),
    "epd_peer_alloc": (_i32, [_i64, C.POINTER(_vp)]),
    "epd_peer_free": (_i32, [_vp]),
    "epd_peer_export": (_i32, [_vp, _vp]),
    "epd_peer_open": (_i32, [_vp, C.POINTER(_vp)]),
    "epd_peer_close": (_i32, [_vp]),
    "epd_peer_put": (_i32, [_vp, _vp, _i64, _vp, C.c_uint32, _vp]),
    "epd_peer_signal": (_i32, [_vp, C.c_uint32, _vp]),
    "epd_stream_wait_geq": (_i32, [_vp, C.c_uint32, _vp]),
    "epd_kv_move": (_i32, [_vp, _i64, _vp, _i64, _i32, _i64, _vp, _vp, _i32, _vp]),
    "epd_kv_pack": (_i32, [_vp, _i32, _i64, _i64, _vp, _i32, _vp, _vp]),
    "epd_kv_unpack": (_i32, [_vp, _i32, _i64, _i64, _vp, _i32, _vp, _vp]),
    "epd_linear_bf16": (_i32, [_vp, _i32, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _i32, _vp,
                               _vp, _i32, _i32, _vp]),
    "epd_set_gemm_cta_group": (_i32, [_i32]),
    "epd_linear_acc_f32": (_i32, [_vp, _i32, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _i32, _vp]),
    "epd_linear_acc_f32_split": (_i32, [_vp, _i32, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _i32, _i32, _vp]),
    "epd_linear_heads_bf16": (_i32, [_vp, _i32, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _i32, _i32, _i32,
                                     _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "epd_attention_bf16": (_i32, [_vp, _i32, _vp, _i32, _vp, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                  _i32, _i32, _i32, C.c_float, _vp]),
    "epd_layernorm_bf16": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _i32, _i32, C.c_float, _vp]),
    "epd_layernorm_f32_bf16": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _i32, _i32, C.c_float, _vp]),
    "epd_rmsnorm_f32_bf16": (_i32, [_vp, _i32, _vp, _i32, _vp, _i32, _i32, C.c_float, _vp]),
    "epd_rope_bf16": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, C.c_float, _vp, _vp]),
    "epd_rope_table": (_i32, [_vp, _i32, _i32, _i32, C.c_float, _vp]),
    "epd_silu_mul_bf16": (_i32, [_vp, _i32, _vp, _i32, _i32, _i32, _vp]),
    "epd_kv_write_paged": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i64, _i32, _vp]),
    "epd_gather_rows_f32": (_i32, [_vp, _i32, _vp, _i32, _i32, _vp, _i32, _vp]),
    "epd_argmax_bf16": (_i32, [_vp, _i32, _vp, _vp]),
    "epd_blocks_init": (_i32, [_vp, _vp, _i32, _vp]),
    "epd_blocks_alloc": (_i32, [_vp, _vp, _i32, _vp, _vp]),
    "epd_blocks_free": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "epd_tile_image": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "epd_patchify_u8": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load libepd.so once; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -m paper_2501_05460_b200.build` "
                        "(there is no CPU fallback for the encode path)")
                h = C.CDLL(str(LIB_PATH))
                for name, (res, args) in _SIGS.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                if h.epd_abi_version() != 1:
                    raise RuntimeError("libepd ABI version mismatch")
                _lib = h
    return _lib


def check(status: int) -> None:
    """Raise the reference-equivalent exception for a non-zero status."""
    if status == EPD_OK:
        return
    msg = (lib().epd_last_error() or b"").decode(errors="replace")
    if status in (EPD_ERR_VALUE, EPD_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if status == EPD_ERR_CAPACITY:
        raise CapacityExceeded(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
