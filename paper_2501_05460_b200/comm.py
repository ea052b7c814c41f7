"""NCCL communicator owned by libepd (``epd_comm_*`` in include/epd.h).

The stage handoff's NCCL legs -- the EP gather of MM tokens to the prefill rank and the
PD KV-block handoff -- are C-ABI calls, so a non-Python host binds the same entry points.
Python only creates the communicator: rank 0 makes the NCCL unique id and the host's
process group (gloo or NCCL) broadcasts it; ``epd_comm_init`` is then the collective.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from ._lib import call, lib

ID_BYTES = 128


def _s(dev: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


class NcclComm:
    """One rank's endpoint of an NCCL communicator over the process group's ranks."""

    def __init__(self, device: torch.device | int, rank: int | None = None, world: int | None = None, group=None,
                 uid: bytes | None = None):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        if uid is None:
            obj = [None]
            if self.rank == 0:
                buf = (C.c_uint8 * ID_BYTES)()
                call("epd_comm_unique_id", buf)
                obj = [bytes(buf)]
            if self.world > 1:
                dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            uid = obj[0]
        idbuf = (C.c_uint8 * ID_BYTES).from_buffer_copy(uid)
        self._h = C.c_void_p()
        call("epd_comm_init", idbuf, self.world, self.rank, self.device.index or 0, C.byref(self._h))

    def close(self) -> None:
        if self._h:
            lib().epd_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ EP gather
    def gather_tokens(self, shard: torch.Tensor | None, n_tiles: int, packed: torch.Tensor | None,
                      root: int = 0) -> None:
        """Every rank's IRP shard of an n-tile request (epd_irp_ranges) -> ``packed`` on
        ``root`` at its tile offset. ``shard`` / ``packed``: bf16 [tiles, tokens, hidden]."""
        ref = shard if shard is not None else packed
        tile_bytes = ref[0].numel() * ref.element_size() if ref is not None and ref.shape[0] else 1
        if packed is not None and packed.shape[0]:
            tile_bytes = packed[0].numel() * packed.element_size()
        call("epd_gather_tokens", self._h, C.c_void_p(shard.data_ptr() if shard is not None else None), n_tiles,
             tile_bytes, C.c_void_p(packed.data_ptr() if packed is not None else None), root, _s(self.device))

    # ------------------------------------------------------------------ raw P2P
    def send(self, t: torch.Tensor, peer: int) -> None:
        call("epd_comm_send", self._h, C.c_void_p(t.data_ptr()), t.numel() * t.element_size(), peer,
             _s(self.device))

    def recv(self, t: torch.Tensor, peer: int) -> None:
        call("epd_comm_recv", self._h, C.c_void_p(t.data_ptr()), t.numel() * t.element_size(), peer,
             _s(self.device))

    @staticmethod
    def group_start() -> None:
        call("epd_comm_group_start")

    @staticmethod
    def group_end() -> None:
        call("epd_comm_group_end")

    # ------------------------------------------------------------------ PD handoff
    def kv_send(self, cache, block_ids: torch.Tensor, staging: torch.Tensor, peer: int) -> None:
        call("epd_kv_handoff_send", self._h, C.c_void_p(cache.pool.data_ptr()), cache.segments,
             cache.num_blocks * cache.block_bytes, cache.block_bytes, C.c_void_p(block_ids.data_ptr()),
             block_ids.numel(), C.c_void_p(staging.data_ptr()), peer, _s(self.device))

    def kv_recv(self, cache, block_ids: torch.Tensor, staging: torch.Tensor, peer: int) -> None:
        call("epd_kv_handoff_recv", self._h, C.c_void_p(cache.pool.data_ptr()), cache.segments,
             cache.num_blocks * cache.block_bytes, cache.block_bytes, C.c_void_p(block_ids.data_ptr()),
             block_ids.numel(), C.c_void_p(staging.data_ptr()), peer, _s(self.device))
