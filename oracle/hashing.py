"""Content-hash oracle (numpy) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Specification of the MM-cache key (the reference has no content cache --
SURVEY.md 0.4, parity unpinned by the reference). For a record of L bytes
(L % 8 == 0), with little-endian u64 words w_i and all arithmetic mod 2^64:

    x_i  = w_i ^ (i * 0x9E3779B97F4A7C15 + (0x243F6A8885A308D3 ^ s0))
    a_i  = fmix64(x_i),   b_i = fmix64(a_i + (0x632BE59BD9B4E019 ^ s1))
    key0 = fmix64((sum_i a_i) ^ L ^ s1),  key1 = fmix64((sum_i b_i) + L * 0xD6E8FEB86659FD93 + s0)
    key0 = 1 if key0 == 0

(s0, s1) is the cache's secret; (0, 0) is the known-answer mode the KATs pin.

fmix64 is the MurmurHash3 64-bit finalizer. The sums commute, so the GPU's
parallel reduction order cannot change the key (bit-exact).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
SEED = np.uint64(0x243F6A8885A308D3)
LANE_B = np.uint64(0x632BE59BD9B4E019)
LEN_MUL = np.uint64(0xD6E8FEB86659FD93)
C1 = np.uint64(0xFF51AFD7ED558CCD)
C2 = np.uint64(0xC4CEB53FE5D4A1A3)
S33 = np.uint64(33)


def fmix64(k: np.ndarray) -> np.ndarray:
    k = np.asarray(k, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        k ^= k >> S33
        k *= C1
        k ^= k >> S33
        k *= C2
        k ^= k >> S33
    return k


def content_hash(record, secret: tuple[int, int] = (0, 0)) -> tuple[int, int]:
    """(key0, key1) of one record (bytes-like or uint8 array) under ``secret`` = (s0, s1)."""
    buf = np.ascontiguousarray(np.frombuffer(bytes(record) if not isinstance(record, np.ndarray) else
                                             record.tobytes(), dtype=np.uint8))
    L = buf.size
    if L % 8:
        raise ValueError("record length must be a multiple of 8 bytes")
    w = buf.view("<u8").astype(np.uint64)
    i = np.arange(w.size, dtype=np.uint64)
    s0, s1 = np.uint64(secret[0]), np.uint64(secret[1])
    with np.errstate(over="ignore"):
        x = w ^ (i * GOLDEN + (SEED ^ s0))
        a = fmix64(x)
        b = fmix64(a + (LANE_B ^ s1))
        sa = np.uint64(a.sum(dtype=np.uint64))
        sb = np.uint64(b.sum(dtype=np.uint64))
        k0 = int(fmix64(np.array([sa ^ np.uint64(L) ^ s1]))[0])
        k1 = int(fmix64(np.array([sb + np.uint64(L) * LEN_MUL + s0]))[0])
    if k0 == 0:
        k0 = 1
    return k0, k1


def hash_tiles(tiles, secret: tuple[int, int] = (0, 0)) -> list[tuple[int, int]]:
    """Keys of each tile of a uint8 array [n, ...] (one record per tile)."""
    arr = np.asarray(tiles)
    return [content_hash(arr[i], secret) for i in range(arr.shape[0])]
