"""Prefill -> decode KV-block handoff (PD migration): one block-to-block kernel on a shared GPU, NCCL P2P across GPUs.

Reference seam (relative to /root/reference/pkg/src/disaggsim/):
``_try_reserve_decode`` reserves ``total_tokens + output_tokens`` KV tokens on
the decode instance (engine.py:542-552), schedules a transfer of
``total_tokens * kv_bytes_per_token`` bytes (engine.py:553-554) and
``_on_transfer_end("pd")`` frees the prefill-side blocks once it lands
(engine.py:436-439).

Here the KV cache is a real paged pool: ``2 * num_layers`` segments (K and V
per layer) of ``num_blocks`` blocks, each block = ``block_size`` tokens x
``kv_heads`` x ``head_dim`` bf16. Across GPUs the prefill rank packs the request's blocks
into one contiguous buffer (``epd_kv_pack``), sends it with NCCL P2P, and the
decode rank unpacks into the block ids its BlockManager reserved
(``epd_kv_unpack``). When prefill and decode share a GPU, one kernel moves every
block straight from the prefill pool into the decode pool (``epd_kv_move``: half the
HBM traffic of pack + unpack). Whole blocks move; the reference's byte count is the
token-exact figure and is reported alongside (``pd_bytes``).
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from ._lib import call
from .blockpool import BlockManager, CacheKind
from .routing import pd_bytes


class PagedKVCache:
    def __init__(self, num_layers: int, kv_heads: int, head_dim: int, block_size: int, num_blocks: int,
                 device: torch.device):
        self.num_layers, self.kv_heads, self.head_dim = num_layers, kv_heads, head_dim
        self.block_size, self.num_blocks = block_size, num_blocks
        self.device = torch.device(device)
        self.segments = 2 * num_layers
        self.block_elems = block_size * kv_heads * head_dim
        self.pool = torch.zeros(self.segments, num_blocks, self.block_elems, dtype=torch.bfloat16,
                                device=self.device)
        self.manager = BlockManager(CacheKind.KV, block_size, num_blocks)

    @property
    def block_bytes(self) -> int:
        return self.block_elems * 2

    @property
    def kv_bytes_per_token(self) -> int:  # models.py:128-130
        return 2 * self.num_layers * self.kv_heads * self.head_dim * 2

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def pack(self, block_ids: list[int], out: torch.Tensor | None = None) -> torch.Tensor:
        n = len(block_ids)
        if out is None:
            out = torch.empty(n, self.segments, self.block_elems, dtype=torch.bfloat16, device=self.device)
        ids = torch.tensor(block_ids, dtype=torch.int32, device=self.device)
        call("epd_kv_pack", C.c_void_p(self.pool.data_ptr()), self.segments, self.num_blocks * self.block_bytes,
             self.block_bytes, C.c_void_p(ids.data_ptr()), n, C.c_void_p(out.data_ptr()), self._stream())
        return out

    def move_to(self, dst: "PagedKVCache", src_ids: list[int], dst_ids: list[int]) -> None:
        """dst.pool[s][dst_ids[i]] = self.pool[s][src_ids[i]] for every segment (one kernel)."""
        if len(src_ids) != len(dst_ids):
            raise ValueError("move_to: src and dst block lists differ in length")
        if (dst.segments, dst.block_elems) != (self.segments, self.block_elems):
            raise ValueError("move_to: pools of different geometry")
        n = len(src_ids)
        ids = torch.tensor(list(src_ids) + list(dst_ids), dtype=torch.int32, device=self.device)
        call("epd_kv_move", C.c_void_p(self.pool.data_ptr()), self.num_blocks * self.block_bytes,
             C.c_void_p(dst.pool.data_ptr()), dst.num_blocks * dst.block_bytes, self.segments, self.block_bytes,
             C.c_void_p(ids.data_ptr()), C.c_void_p(ids.data_ptr() + 4 * n), n, self._stream())

    def unpack(self, packed: torch.Tensor, block_ids: list[int]) -> None:
        n = len(block_ids)
        ids = torch.tensor(block_ids, dtype=torch.int32, device=self.device)
        call("epd_kv_unpack", C.c_void_p(packed.data_ptr()), self.segments, self.num_blocks * self.block_bytes,
             self.block_bytes, C.c_void_p(ids.data_ptr()), n, C.c_void_p(self.pool.data_ptr()), self._stream())


def kv_handoff(rid: int, total_tokens: int, output_tokens: int, src: PagedKVCache | None, dst: PagedKVCache | None,
               src_rank: int, dst_rank: int, rank: int, group=None) -> dict:
    """Move request ``rid``'s KV blocks from the prefill rank to the decode rank.

    The prefill side must already hold ``src.manager.allocated[rid]``. The decode
    side reserves ``total_tokens + output_tokens`` (engine.py:543) and receives the
    first ``blocks_needed(total_tokens)`` of its blocks. The prefill blocks are
    freed after the send completes (engine.py:437). Returns byte accounting.
    """
    info = {"pd_bytes": None, "moved_bytes": 0, "dst_blocks": None}
    if rank == src_rank:
        src_ids = src.manager.allocated[rid]
        info["pd_bytes"] = pd_bytes(total_tokens, src.kv_bytes_per_token)
        info["moved_bytes"] = len(src_ids) * src.segments * src.block_bytes
        if dst_rank == src_rank:
            dst_ids = dst.manager.allocate(rid, total_tokens + output_tokens)
            src.move_to(dst, src_ids, dst_ids[:len(src_ids)])
            info["dst_blocks"] = dst_ids
        else:
            dist.send(src.pack(src_ids), dst_rank, group=group)
        src.manager.free(rid)
    elif rank == dst_rank:
        dst_ids = dst.manager.allocate(rid, total_tokens + output_tokens)
        nb = dst.manager.blocks_needed(total_tokens)
        buf = torch.empty(nb, dst.segments, dst.block_elems, dtype=torch.bfloat16, device=dst.device)
        dist.recv(buf, src_rank, group=group)
        dst.unpack(buf, dst_ids[:nb])
        info["dst_blocks"] = dst_ids
        info["moved_bytes"] = buf.numel() * 2
    return info
