"""Content-addressed multimodal-token cache on the GPU.

Stands behind the encode instance's ``BlockManager(CacheKind.MM)``
(engine.py:155-157, blocks.py:14-61) and adds what the reference's staging
buffer lacks: tiles whose content was already encoded are served from HBM and
skip the encoder entirely.

Device side (libepd): the content hash of each tile (``epd_hash_records``,
K11) and an open-addressing hash table from key to entry id
(``epd_mmcache_*``, K12); entry e's MM tokens live in ``store[e]``.
Host side: entry ids come from a :class:`~.blockpool.BlockManager`-style LIFO
stack and eviction is least-recently-used over keys the current request does
not reference -- the behaviour specified by oracle/mmcache.py and checked
tile-for-tile by tests/test_mmcache_gpu.py.
"""
from __future__ import annotations

import ctypes as C
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import CapacityExceeded, call, lib

HIT, MISS, DUP = "hit", "miss", "dup"


def _s(dev: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def hash_tiles(tiles: torch.Tensor, keys: torch.Tensor | None = None,
               scratch: torch.Tensor | None = None) -> torch.Tensor:
    """Device content keys [n, 2] (int64 storage of u64) of uint8 tiles [n, ...]."""
    if not tiles.is_cuda or tiles.dtype != torch.uint8 or not tiles.is_contiguous():
        raise ValueError("tiles must be a contiguous uint8 CUDA tensor")
    n = tiles.shape[0]
    rec = tiles[0].numel() if n else 0
    if keys is None:
        keys = torch.empty(n, 2, dtype=torch.int64, device=tiles.device)
    if scratch is None:
        scratch = torch.empty(max(n, 1), 2, dtype=torch.int64, device=tiles.device)
    call("epd_hash_records", C.c_void_p(tiles.data_ptr()), n, rec, rec, C.c_void_p(keys.data_ptr()),
         C.c_void_p(scratch.data_ptr()), _s(tiles.device))
    return keys


@dataclass
class CachePlan:
    kinds: list            # per tile: HIT / MISS / DUP
    entries: np.ndarray    # per tile: entry id holding its tokens (int32)
    miss_tiles: np.ndarray  # tile indices to encode (first occurrences of uncached keys), tile order
    miss_entries: np.ndarray  # entry ids they are written to
    victims: list          # keys evicted to make room


class MMTokenCache:
    def __init__(self, capacity: int, tokens_per_tile: int, hidden: int, device: torch.device | int = 0):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        self._h = C.c_void_p()
        call("epd_mmcache_create", int(capacity), self.device.index or 0, C.byref(self._h))
        self.store = torch.empty(capacity, tokens_per_tile, hidden, dtype=torch.bfloat16, device=self.device)
        self._free = list(range(capacity - 1, -1, -1))
        self._lru: OrderedDict = OrderedDict()  # key -> entry, oldest first
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
        return len(self._lru)

    # ---------------------------------------------------------------- device ops
    def lookup(self, keys: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        n = keys.shape[0]
        entry = torch.empty(n, dtype=torch.int32, device=self.device)
        dup = torch.empty(n, dtype=torch.int32, device=self.device)
        call("epd_mmcache_lookup", self._h, C.c_void_p(keys.data_ptr()), n, C.c_void_p(entry.data_ptr()),
             C.c_void_p(dup.data_ptr()), _s(self.device))
        return entry, dup

    def _insert(self, keys: torch.Tensor, entries: torch.Tensor) -> None:
        call("epd_mmcache_insert", self._h, C.c_void_p(keys.data_ptr()), C.c_void_p(entries.data_ptr()),
             keys.shape[0], _s(self.device))

    def _erase(self, keys: torch.Tensor) -> None:
        call("epd_mmcache_erase", self._h, C.c_void_p(keys.data_ptr()), keys.shape[0], _s(self.device))

    def clear(self) -> None:
        call("epd_mmcache_clear", self._h, _s(self.device))
        self._free = list(range(self.capacity - 1, -1, -1))
        self._lru.clear()

    # ---------------------------------------------------------------- request flow
    def plan(self, keys_dev: torch.Tensor) -> CachePlan:
        """Classify a request's tiles (device lookup), evict and assign entries.

        One small device->host read (keys, lookup, in-batch duplicates) per request.
        """
        n = keys_dev.shape[0]
        entry_d, dup_d = self.lookup(keys_dev)
        packed = torch.cat([keys_dev.view(torch.int32).reshape(n, 4), entry_d.view(n, 1), dup_d.view(n, 1)], 1)
        host = packed.cpu().numpy()
        keys = [tuple(int(x) for x in row) for row in host[:, :4].view(np.uint64).reshape(n, 2)]
        looked = host[:, 4]
        dup = host[:, 5]
        distinct = list(dict.fromkeys(keys))
        if len(distinct) > self.capacity:
            raise CapacityExceeded(f"{len(distinct)} distinct tiles > cache capacity {self.capacity}")
        # device table is authoritative for hits; the host LRU must agree
        hit_keys = []
        for i, k in enumerate(keys):
            if looked[i] >= 0:
                if self._lru.get(k) != int(looked[i]):
                    raise RuntimeError("device MM-cache table and host LRU disagree")
                hit_keys.append(k)
        for k in dict.fromkeys(hit_keys):
            self._lru.move_to_end(k)
        pinned = set(hit_keys)
        first_miss = [i for i in range(n) if looked[i] < 0 and dup[i] < 0]
        victims = []
        while len(self._free) < len(first_miss):
            victim = next(k for k in self._lru if k not in pinned)
            victims.append(victim)
            self._free.append(self._lru.pop(victim))
        miss_entries = []
        for i in first_miss:
            e = self._free.pop()
            self._lru[keys[i]] = e
            miss_entries.append(e)
        new = dict(zip(first_miss, miss_entries))
        kinds, entries = [], np.empty(n, dtype=np.int32)
        for i in range(n):
            if looked[i] >= 0:
                kinds.append(HIT)
                entries[i] = looked[i]
            elif dup[i] < 0:
                kinds.append(MISS)
                entries[i] = new[i]
            else:
                kinds.append(DUP)
                entries[i] = new[int(dup[i])]
        if victims:
            vk = torch.tensor(np.array(victims, dtype=np.uint64).view(np.int64), device=self.device)
            self._erase(vk)
        if first_miss:
            idx = torch.tensor(first_miss, dtype=torch.int64, device=self.device)
            self._insert(keys_dev.index_select(0, idx).contiguous(),
                         torch.tensor(miss_entries, dtype=torch.int32, device=self.device))
        for k in kinds:
            self.stats[k] += 1
        self.stats["evicted"] += len(victims)
        return CachePlan(kinds, entries, np.array(first_miss, dtype=np.int64),
                         np.array(miss_entries, dtype=np.int32), victims)

    def check(self) -> None:
        call("epd_mmcache_check", self._h, _s(self.device))
