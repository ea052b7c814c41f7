"""MM-token cache behaviour oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Specification of the content-addressed multimodal-token cache (no reference
counterpart beyond BlockManager's id discipline, blocks.py:14-61 -- parity
unpinned by the reference):

* capacity C entries (one entry = one tile's MM tokens); entry ids come from a
  LIFO free stack initialised like BlockManager (first allocations get 0,1,2...,
  freed ids are reused first);
* per request, tiles are classified in tile order: ``hit`` (key cached),
  ``miss`` (first occurrence of an uncached key -- will be encoded) or ``dup``
  (repeat of an earlier miss in the same request -- reuses that tile's entry);
* eviction is least-recently-used over keys not referenced by the current
  request; a hit refreshes recency; new keys are inserted in tile order;
* a request whose distinct keys exceed C raises CapacityExceeded.
"""
from __future__ import annotations

from collections import OrderedDict


class CapacityExceeded(Exception):
    pass


class MMCacheOracle:
    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        self._free = list(range(capacity - 1, -1, -1))
        self._map: OrderedDict = OrderedDict()  # key -> entry, LRU order (oldest first)

    def __len__(self) -> int:
        return len(self._map)

    def process(self, keys: list) -> list[tuple[str, int]]:
        """Classify one request's tile keys; returns [(kind, entry)] in tile order."""
        keys = [tuple(k) for k in keys]
        distinct = list(dict.fromkeys(keys))
        if len(distinct) > self.capacity:
            raise CapacityExceeded(f"{len(distinct)} distinct tiles > cache capacity {self.capacity}")
        hits = [k for k in distinct if k in self._map]
        misses = [k for k in distinct if k not in self._map]
        for k in hits:  # refresh recency in tile order
            self._map.move_to_end(k)
        pinned = set(hits)
        victims = []
        while len(self._free) < len(misses):
            for k in self._map:
                if k not in pinned:
                    victims.append(k)
                    break
            else:  # pragma: no cover - excluded by the capacity check
                raise CapacityExceeded("no evictable entry")
            self._free.append(self._map.pop(victims[-1]))
        new = {}
        for k in misses:
            e = self._free.pop()
            new[k] = e
            self._map[k] = e
        out = []
        seen = set()
        for k in keys:
            if k in new:
                out.append(("dup" if k in seen else "miss", new[k]))
                seen.add(k)
            else:
                out.append(("hit", self._map[k]))
        self.last_victims = victims
        return out
