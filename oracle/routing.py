"""Routing / accounting oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain-Python restatement of the reference's encode-path control logic, pinned
against golden vectors generated from the reference itself
(tests/golden/make_golden.py -> tests/golden/reference_golden.json).
Citations are relative to /root/reference/pkg/src/disaggsim/.
"""
from __future__ import annotations

import math


def irp_shard(patches: int, width: int) -> list[int]:
    """engine.py:55-62: balanced partition, remainder to the lowest workers."""
    if width < 1:
        raise ValueError("shard width must be >= 1")
    if patches < 0:
        raise ValueError("patch count must be non-negative")
    base, rem = divmod(patches, width)
    return [base + 1] * rem + [base] * (width - rem)


def shard_ranges(patches: int, width: int) -> list[tuple[int, int]]:
    """Worker k's contiguous tile range [first, first+count) in request tile order
    (implied by the shard order of engine.py:589-602)."""
    out, acc = [], 0
    for c in irp_shard(patches, width):
        out.append((acc, c))
        acc += c
    return out


def plan_batch(patches_per_request: list[int], width: int):
    """engine.py:583-602 (_start_encode): per request, the non-empty shards
    [(worker, tiles)] (text-only -> [(0, 0)]); per worker, its tile load and
    the number of requests it serves. Every request restarts at worker 0."""
    worker_load = [0] * width
    worker_reqs = [0] * width
    shards = []
    for p in patches_per_request:
        if p == 0:
            s = [(0, 0)]
        else:
            s = [(k, c) for k, c in enumerate(irp_shard(p, width)) if c > 0]
        shards.append(s)
        for k, c in s:
            worker_load[k] += c
            worker_reqs[k] += 1
    return shards, worker_load, worker_reqs


def ep_bytes(tiles: int, tokens_per_patch: int, mm_bytes_per_token: int) -> int:
    """engine.py:524: EP-migration bytes of one shard (post-projector tokens)."""
    return tiles * tokens_per_patch * mm_bytes_per_token


def pd_bytes(total_tokens: int, kv_bytes_per_token: int) -> int:
    """engine.py:553-554: PD-migration bytes of one request."""
    return total_tokens * kv_bytes_per_token


def kv_bytes_per_token(num_layers, kv_heads, head_dim, bytes_per_param=2) -> int:
    """models.py:128-130."""
    return 2 * num_layers * kv_heads * head_dim * bytes_per_param


def mm_bytes_per_token(hidden_dim, bytes_per_param=2) -> int:
    """models.py:133-135."""
    return hidden_dim * bytes_per_param


def tokens_for_request(patch_table: dict, tokens_per_patch: int, images, prompt_tokens: int):
    """models.py:146-155 (KeyError on unknown resolution, as UnknownResolution is a KeyError)."""
    mm = sum(patch_table[tuple(r)] * tokens_per_patch for r in images)
    return mm, mm + prompt_tokens


class BlockManager:
    """blocks.py:14-61: whole-block reservation with a LIFO free stack."""

    def __init__(self, block_size: int, total_blocks: int):
        if block_size < 1:
            raise ValueError("block_size must be >= 1")
        if total_blocks < 0:
            raise ValueError("total_blocks must be >= 0")
        self.block_size = block_size
        self.total_blocks = total_blocks
        self._free = list(range(total_blocks - 1, -1, -1))
        self.allocated: dict[int, list[int]] = {}

    def blocks_needed(self, tokens: int) -> int:
        return math.ceil(tokens / self.block_size) if tokens > 0 else 0

    @property
    def free_blocks(self) -> int:
        return len(self._free)

    @property
    def used_blocks(self) -> int:
        return self.total_blocks - len(self._free)

    def can_allocate(self, tokens: int) -> bool:
        return self.blocks_needed(tokens) <= len(self._free)

    def allocate(self, rid: int, tokens: int) -> list[int]:
        if rid in self.allocated:
            raise RuntimeError("already holds blocks")
        need = self.blocks_needed(tokens)
        if need > len(self._free):
            raise RuntimeError("overcommitted")
        blocks = [self._free.pop() for _ in range(need)]
        self.allocated[rid] = blocks
        return blocks

    def free(self, rid: int) -> None:
        try:
            blocks = self.allocated.pop(rid)
        except KeyError:
            raise RuntimeError("holds no blocks") from None
        self._free.extend(reversed(blocks))


def percentile(values, q: float) -> float:
    """metrics.py:103-108: nearest rank with Python's (banker's) round."""
    ordered = sorted(values)
    if not ordered:
        return 0.0
    idx = min(len(ordered) - 1, max(0, round(q * (len(ordered) - 1))))
    return ordered[idx]
