"""Content-addressed multimodal-token cache on the GPU.

Stands behind the encode instance's ``BlockManager(CacheKind.MM)``
(engine.py:155-157, blocks.py:14-61) and adds what the reference's staging
buffer lacks: tiles whose content was already encoded are served from HBM and
skip the encoder entirely.

Everything runs on the device (libepd):

* the content hash of each tile (``epd_hash_records_keyed``, K11), keyed with a per-process
  random secret so an uploaded tile cannot be crafted offline to collide with a popular
  image (``secret=0`` is the known-answer mode the KATs pin);
* the request plan (``epd_mmcache_plan``, K12): hash-table lookups, hit / miss / dup
  classification in tile order, LRU refresh and eviction of entries the request does not
  reference, LIFO entry ids for the misses and their insertion -- one CTA, the behaviour
  specified by oracle/mmcache.py and checked tile for tile by tests/test_mmcache_gpu.py.

The host reads back one 20-byte count record per request (how many tiles to encode); the
tile lists themselves stay on the device and drive the gather of miss tiles, the scatter of
their tokens into ``store`` and the packing of the request.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import CapacityExceeded, call, lib

HIT, MISS, DUP = "hit", "miss", "dup"
_KINDS = (HIT, MISS, DUP)


def _s(dev: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def hash_tiles(tiles: torch.Tensor, keys: torch.Tensor | None = None, scratch: torch.Tensor | None = None,
               secret: tuple[int, int] = (0, 0)) -> torch.Tensor:
    """Device content keys [n, 2] (int64 storage of u64) of uint8 tiles [n, ...]."""
    if not tiles.is_cuda or tiles.dtype != torch.uint8 or not tiles.is_contiguous():
        raise ValueError("tiles must be a contiguous uint8 CUDA tensor")
    n = tiles.shape[0]
    rec = tiles[0].numel() if n else 0
    if keys is None:
        keys = torch.empty(n, 2, dtype=torch.int64, device=tiles.device)
    if scratch is None:
        scratch = torch.empty(max(n, 1), 2, dtype=torch.int64, device=tiles.device)
    call("epd_hash_records_keyed", C.c_void_p(tiles.data_ptr()), n, rec, rec, C.c_uint64(secret[0]),
         C.c_uint64(secret[1]), C.c_void_p(keys.data_ptr()), C.c_void_p(scratch.data_ptr()), _s(tiles.device))
    return keys


@dataclass
class CachePlan:
    """One request's plan; the tensors live on the device."""

    n: int
    entries: torch.Tensor       # int32 [n]: entry holding each tile's tokens
    kinds_dev: torch.Tensor     # int32 [n]: 0 hit / 1 miss / 2 dup
    miss_tiles: torch.Tensor    # int32 [n_miss]: tiles to encode (first occurrences), tile order
    miss_entries: torch.Tensor  # int32 [n_miss]: the entries they are written to
    victim_keys_dev: torch.Tensor  # int64 [n_victims, 2]: keys evicted, eviction order
    n_miss: int
    n_hit: int
    n_dup: int
    n_victims: int

    @property
    def kinds(self) -> list[str]:
        """Per-tile classification (reads the device tensor back)."""
        return [_KINDS[k] for k in self.kinds_dev.cpu().tolist()]

    @property
    def victims(self) -> list[tuple[int, int]]:
        v = self.victim_keys_dev.cpu().numpy().view(np.uint64)
        return [(int(a), int(b)) for a, b in v]

    @property
    def counts(self) -> dict:
        return {HIT: self.n_hit, MISS: self.n_miss, DUP: self.n_dup}


class MMTokenCache:
    """``capacity`` entries of one tile's MM tokens each. ``secret``: None = a random
    per-process key (serving), 0 = the unkeyed known-answer mode, or an int / (s0, s1)."""

    def __init__(self, capacity: int, tokens_per_tile: int, hidden: int, device: torch.device | int = 0,
                 secret=None):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        if secret is None:
            s = os.environ.get("EPD_CACHE_SECRET")
            secret = int(s, 0) if s else struct.unpack("<QQ", os.urandom(16))
        if isinstance(secret, int):
            secret = (secret & (2 ** 64 - 1), (secret >> 64) & (2 ** 64 - 1))
        self.secret = (int(secret[0]), int(secret[1]))
        self._h = C.c_void_p()
        call("epd_mmcache_create", int(capacity), self.device.index or 0, C.byref(self._h))
        self.store = torch.empty(capacity, tokens_per_tile, hidden, dtype=torch.bfloat16, device=self.device)
        self._counts_host = torch.zeros(5, dtype=torch.int32).pin_memory()
        self._counts_ready = torch.cuda.Event()
        self._live = 0
        self.stats = {"hit": 0, "miss": 0, "dup": 0, "evicted": 0}

    def close(self) -> None:
        if self._h:
            lib().epd_mmcache_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self) -> int:
        return self._live

    def hash(self, tiles: torch.Tensor) -> torch.Tensor:
        """Keyed content keys of this cache's tiles."""
        return hash_tiles(tiles, secret=self.secret)

    def clear(self) -> None:
        call("epd_mmcache_clear", self._h, _s(self.device))
        self._live = 0

    def plan(self, keys_dev: torch.Tensor) -> CachePlan:
        """Classify a request's tiles, evict and assign entries -- all on the device; the host
        waits only for the 20-byte count record."""
        n = keys_dev.shape[0]
        dev = self.device
        entries = torch.empty(n, dtype=torch.int32, device=dev)
        kinds = torch.empty(n, dtype=torch.int32, device=dev)
        miss_tiles = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        miss_entries = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        victims = torch.empty(max(n, 1), 2, dtype=torch.int64, device=dev)
        counts = torch.empty(5, dtype=torch.int32, device=dev)
        call("epd_mmcache_plan", self._h, C.c_void_p(keys_dev.data_ptr()), n, C.c_void_p(entries.data_ptr()),
             C.c_void_p(kinds.data_ptr()), C.c_void_p(miss_tiles.data_ptr()), C.c_void_p(miss_entries.data_ptr()),
             C.c_void_p(victims.data_ptr()), C.c_void_p(counts.data_ptr()), _s(dev))
        self._counts_host.copy_(counts, non_blocking=True)
        self._counts_ready.record(torch.cuda.current_stream(dev))
        self._counts_ready.synchronize()
        m, hits, dups, nv, status = (int(x) for x in self._counts_host.tolist())
        if status:
            raise CapacityExceeded(f"a request of {n} tiles has more distinct tiles than the cache holds "
                                   f"({self.capacity})")
        self._live += m - nv
        self.stats["hit"] += hits
        self.stats["miss"] += m
        self.stats["dup"] += dups
        self.stats["evicted"] += nv
        return CachePlan(n, entries, kinds, miss_tiles[:m], miss_entries[:m], victims[:nv], m, hits, dups, nv)

    def check(self) -> None:
        call("epd_mmcache_check", self._h, _s(self.device))
