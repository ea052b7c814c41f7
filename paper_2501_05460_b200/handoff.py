"""Prefill -> decode KV-block handoff (PD migration).

Reference seam (relative to /root/reference/pkg/src/disaggsim/):
``_try_reserve_decode`` (engine.py:542-555) reserves ``total_tokens + output_tokens`` KV
tokens on the decode instance -- or returns False, and ``_on_batch_end`` parks the request
in the ``pd_wait`` FIFO (engine.py:406-407), retried head-of-line by ``_retry_waits``
(engine.py:686-690) -- then schedules a transfer of ``total_tokens * kv_bytes_per_token``
bytes (engine.py:553-554); ``_on_transfer_end("pd")`` frees the prefill-side blocks once
it lands (engine.py:436-439).

Here the KV cache is a real paged pool: ``2 * num_layers`` segments (K and V per layer) of
``num_blocks`` blocks, each ``block_size`` tokens x ``kv_heads`` x ``head_dim`` bf16, written
by the prefill (prefill.py). :class:`KVHandoff` runs the reference's protocol between the
prefill and the decode rank, in the same order on both:

1. prefill -> decode: header (rid, total, output, n_blocks); the sender first checks
   ``n_blocks == blocks_needed(total_tokens)`` (blocks.py:24-26) -- a malformed handoff is
   announced (n_blocks = -1) and raised on both sides instead of hanging a transfer;
2. decode: ``can_allocate(total + output)`` -> ``allocate`` (LIFO ids, blocks.py:29-61) and
   reply (ok, reserved ids); not ok -> both sides return None and the caller parks the
   request in ``pd_wait`` (:meth:`KVHandoff.submit` / :meth:`KVHandoff.retry_waits`);
3. the blocks move, by transport:

   * ``local`` (prefill and decode share a GPU and a process): one block-to-block kernel
     (``epd_kv_move``);
   * ``nvlink-peer`` (default across processes): the decode pool is mapped into the prefill
     process (CUDA IPC); the decode stream releases the reserved blocks (a flag store after
     its earlier readers), the prefill stream waits for it, pushes every block into the
     decode pool with the same ``epd_kv_move`` kernel over NVLink and raises the decode
     rank's data flag; the decode stream waits on it. No staging buffer, no host sync;
   * ``nccl``: pack -> ncclSend -> ncclRecv -> unpack through the C ABI
     (``epd_kv_handoff_send/recv``, comm.py) -- the baseline.

4. the prefill blocks are freed (stream-ordered after the move).

Whole blocks move; the reference's token-exact byte count is reported beside it.
"""
from __future__ import annotations

import ctypes as C
import os
from collections import deque

import torch
import torch.distributed as dist

from ._lib import CapacityExceeded, call
from .blockpool import BlockManager, CacheKind
from .routing import pd_bytes

__all__ = ["PagedKVCache", "KVHandoff", "kv_handoff", "CapacityExceeded"]


class _Cai:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PagedKVCache:
    """Paged KV pool + its reference BlockManager. ``shareable=True`` allocates the pool with
    ``epd_peer_alloc`` so another process can map it (the nvlink-peer handoff target)."""

    def __init__(self, num_layers: int, kv_heads: int, head_dim: int, block_size: int, num_blocks: int,
                 device: torch.device, shareable: bool = False):
        self.num_layers, self.kv_heads, self.head_dim = num_layers, kv_heads, head_dim
        self.block_size, self.num_blocks = block_size, num_blocks
        self.device = torch.device(device)
        self.segments = 2 * num_layers
        self.block_elems = block_size * kv_heads * head_dim
        self._raw = None
        if shareable:
            nbytes = self.segments * num_blocks * self.block_elems * 2
            p = C.c_void_p()
            with torch.cuda.device(self.device):
                call("epd_peer_alloc", nbytes, C.byref(p))
            self._raw = p.value
            self.pool = torch.as_tensor(_Cai(self._raw, nbytes), device=self.device).view(torch.bfloat16).view(
                self.segments, num_blocks, self.block_elems)
        else:
            self.pool = torch.zeros(self.segments, num_blocks, self.block_elems, dtype=torch.bfloat16,
                                    device=self.device)
        self.manager = BlockManager(CacheKind.KV, block_size, num_blocks)

    def close(self) -> None:
        if self._raw is not None:
            torch.cuda.synchronize(self.device)
            self.pool = None
            call("epd_peer_free", C.c_void_p(self._raw))
            self._raw = None

    def export(self) -> bytes:
        if self._raw is None:
            raise RuntimeError("export needs PagedKVCache(shareable=True)")
        h = (C.c_uint8 * 64)()
        call("epd_peer_export", C.c_void_p(self._raw), h)
        return bytes(h)

    @property
    def block_bytes(self) -> int:
        return self.block_elems * 2

    @property
    def segment_stride(self) -> int:
        return self.num_blocks * self.block_bytes

    @property
    def kv_bytes_per_token(self) -> int:  # models.py:128-130
        return 2 * self.num_layers * self.kv_heads * self.head_dim * 2

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def blocks(self, block_ids) -> torch.Tensor:
        """[n, segments, block_elems] copy of the given blocks (tests / verification)."""
        ids = torch.as_tensor(list(block_ids), dtype=torch.int64, device=self.device)
        return self.pool.index_select(1, ids).transpose(0, 1).contiguous()

    def pack(self, block_ids: list[int], out: torch.Tensor | None = None) -> torch.Tensor:
        n = len(block_ids)
        if out is None:
            out = torch.empty(n, self.segments, self.block_elems, dtype=torch.bfloat16, device=self.device)
        ids = torch.tensor(block_ids, dtype=torch.int32, device=self.device)
        call("epd_kv_pack", C.c_void_p(self.pool.data_ptr()), self.segments, self.segment_stride,
             self.block_bytes, C.c_void_p(ids.data_ptr()), n, C.c_void_p(out.data_ptr()), self._stream())
        return out

    def move_to(self, dst: "PagedKVCache", src_ids: list[int], dst_ids: list[int], dst_ptr: int | None = None) -> None:
        """dst.pool[s][dst_ids[i]] = self.pool[s][src_ids[i]] for every segment (one kernel);
        ``dst_ptr`` overrides the destination base (a peer mapping of dst's pool)."""
        if len(src_ids) != len(dst_ids):
            raise ValueError("move_to: src and dst block lists differ in length")
        if (dst.segments, dst.block_elems) != (self.segments, self.block_elems):
            raise ValueError("move_to: pools of different geometry")
        n = len(src_ids)
        ids = torch.tensor(list(src_ids) + list(dst_ids), dtype=torch.int32, device=self.device)
        base = dst.pool.data_ptr() if dst_ptr is None else dst_ptr
        call("epd_kv_move", C.c_void_p(self.pool.data_ptr()), self.segment_stride, C.c_void_p(base),
             dst.segment_stride, self.segments, self.block_bytes, C.c_void_p(ids.data_ptr()),
             C.c_void_p(ids.data_ptr() + 4 * n), n, self._stream())

    def unpack(self, packed: torch.Tensor, block_ids: list[int]) -> None:
        n = len(block_ids)
        ids = torch.tensor(block_ids, dtype=torch.int32, device=self.device)
        call("epd_kv_unpack", C.c_void_p(packed.data_ptr()), self.segments, self.segment_stride,
             self.block_bytes, C.c_void_p(ids.data_ptr()), n, C.c_void_p(self.pool.data_ptr()), self._stream())


class _DistCtl:
    """Host control messages between the two handoff ranks (torch.distributed P2P objects)."""

    def __init__(self, group=None):
        self.group = group

    def send(self, obj, dst: int) -> None:
        dist.send_object_list([obj], dst=dst, group=self.group)

    def recv(self, src: int):
        box = [None]
        dist.recv_object_list(box, src=src, group=self.group)
        return box[0]


class KVHandoff:
    """One rank's endpoint of the prefill -> decode handoff (see the module docstring).

    Every rank of the pair calls :meth:`submit` / :meth:`try_reserve_decode` /
    :meth:`retry_waits` in the same order. ``src`` (prefill pool) lives on ``src_rank``,
    ``dst`` (decode pool; ``shareable=True`` for the nvlink-peer transport) on ``dst_rank``."""

    def __init__(self, rank: int, src_rank: int, dst_rank: int, src: PagedKVCache | None = None,
                 dst: PagedKVCache | None = None, transport: str | None = None, group=None, comm=None, ctl=None,
                 comm_ranks: tuple[int, int] | None = None):
        self.rank, self.src_rank, self.dst_rank = rank, src_rank, dst_rank
        # the prefill / decode ranks inside ``comm`` (nccl transport), when it spans a subgroup
        self.comm_src, self.comm_dst = comm_ranks if comm_ranks is not None else (src_rank, dst_rank)
        self.src, self.dst = src, dst
        self.is_src, self.is_dst = rank == src_rank, rank == dst_rank
        if self.is_src and src is None or self.is_dst and dst is None:
            raise ValueError("the prefill rank needs src and the decode rank needs dst")
        if transport is None:
            transport = "local" if src_rank == dst_rank else os.environ.get("EPD_KV", "nvlink-peer")
        if (transport == "local") != (src_rank == dst_rank):
            raise ValueError("transport 'local' is for a prefill and decode rank in one process")
        if transport not in ("local", "nvlink-peer", "nccl"):
            raise ValueError(f"unknown KV handoff transport {transport!r}")
        if transport == "nccl" and comm is None:
            raise ValueError("the nccl transport needs an NcclComm")
        self.transport, self.comm = transport, comm
        self.ctl = ctl if ctl is not None else _DistCtl(group)
        self.pd_wait: deque = deque()
        self.seq = 0
        self._owned, self._opened = [], []
        if transport == "nvlink-peer" and (self.is_src or self.is_dst):
            self._setup_peer()

    # ------------------------------------------------------------------ nvlink-peer setup
    def _flag(self) -> int:
        p = C.c_void_p()
        call("epd_peer_alloc", 4, C.byref(p))
        self._owned.append(p.value)
        return p.value

    @staticmethod
    def _export(ptr: int) -> bytes:
        h = (C.c_uint8 * 64)()
        call("epd_peer_export", C.c_void_p(ptr), h)
        return bytes(h)

    def _map(self, handle: bytes, ptr: int, pid: int) -> int:
        if pid == os.getpid():
            return ptr
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        p = C.c_void_p()
        call("epd_peer_open", buf, C.byref(p))
        self._opened.append(p.value)
        return p.value

    def _setup_peer(self) -> None:
        dev = (self.src if self.is_src else self.dst).device
        with torch.cuda.device(dev):
            if self.is_src:
                self._rel = self._flag()  # decode -> prefill: "reserved blocks may be overwritten"
                self.ctl.send({"pid": os.getpid(), "rel": (self._rel, self._export(self._rel))}, self.dst_rank)
                rec = self.ctl.recv(self.dst_rank)
                self._dst_pool = self._map(rec["pool"][1], rec["pool"][0], rec["pid"])
                self._dst_data = self._map(rec["data"][1], rec["data"][0], rec["pid"])
                seg, elems, stride = rec["geometry"]
                if (seg, elems) != (self.src.segments, self.src.block_elems):
                    raise ValueError(f"KV pools differ in geometry: {(seg, elems)} vs "
                                     f"{(self.src.segments, self.src.block_elems)}")
                self._dst_geom = _Geom(seg, elems, stride)
            else:
                self._data = self._flag()  # prefill -> decode: "blocks of handoff seq landed"
                rec = self.ctl.recv(self.src_rank)
                self._src_rel = self._map(rec["rel"][1], rec["rel"][0], rec["pid"])
                self.ctl.send({"pid": os.getpid(), "pool": (self.dst.pool.data_ptr(), self.dst.export()),
                               "data": (self._data, self._export(self._data)),
                               "geometry": (self.dst.segments, self.dst.block_elems, self.dst.segment_stride)},
                              self.src_rank)

    def close(self) -> None:
        if self._opened or self._owned:
            torch.cuda.synchronize()
            for p in self._opened:
                call("epd_peer_close", C.c_void_p(p))
            for p in self._owned:
                call("epd_peer_free", C.c_void_p(p))
            self._opened, self._owned = [], []

    # ------------------------------------------------------------------ protocol
    def submit(self, rid: int, total_tokens: int, output_tokens: int) -> dict | None:
        """_on_batch_end for a finished prefill (engine.py:405-407): try the handoff now, else
        park the request in ``pd_wait``. Returns the handoff info, or None when parked."""
        info = self.try_reserve_decode(rid, total_tokens, output_tokens)
        if info is None:
            self.pd_wait.append((rid, total_tokens, output_tokens))
        return info

    def retry_waits(self) -> list[dict]:
        """_retry_waits (engine.py:686-690): head-of-line, stop at the first that still fails."""
        done = []
        while self.pd_wait:
            info = self.try_reserve_decode(*self.pd_wait[0])
            if info is None:
                break
            self.pd_wait.popleft()
            done.append(info)
        return done

    def try_reserve_decode(self, rid: int, total_tokens: int, output_tokens: int) -> dict | None:
        """_try_reserve_decode (engine.py:542-555) + the transfer + _on_transfer_end("pd")."""
        need = total_tokens + output_tokens
        if self.transport == "local":
            src, dst = self.src, self.dst
            src_ids = self._check_src(rid, total_tokens)
            if not dst.manager.can_allocate(need):
                return None
            dst_ids = dst.manager.allocate(rid, need)
            src.move_to(dst, src_ids, dst_ids[:len(src_ids)])
            src.manager.free(rid)
            return self._info(rid, total_tokens, src_ids, dst_ids)
        if self.is_src:
            return self._src_side(rid, total_tokens, output_tokens)
        if self.is_dst:
            return self._dst_side(rid, total_tokens, output_tokens)
        return None

    def _check_src(self, rid: int, total_tokens: int) -> list[int]:
        src_ids = self.src.manager.allocated.get(rid)
        if src_ids is None:
            raise RuntimeError(f"request {rid} holds no prefill KV blocks")
        nb = self.src.manager.blocks_needed(total_tokens)
        if len(src_ids) != nb:
            raise ValueError(f"request {rid}: {len(src_ids)} prefill KV blocks, but {total_tokens} tokens need {nb}")
        return src_ids

    def _info(self, rid, total_tokens, src_ids, dst_ids) -> dict:
        cache = self.src if self.src is not None else self.dst
        nb = len(src_ids) if src_ids is not None else cache.manager.blocks_needed(total_tokens)
        return {"rid": rid, "seq": self.seq, "transport": self.transport,
                "pd_bytes": pd_bytes(total_tokens, cache.kv_bytes_per_token),
                "moved_bytes": nb * cache.segments * cache.block_bytes,
                "src_blocks": src_ids, "dst_blocks": dst_ids}

    def _src_side(self, rid, total_tokens, output_tokens):
        try:
            src_ids = self._check_src(rid, total_tokens)
        except (ValueError, RuntimeError):
            self.ctl.send({"rid": rid, "total": total_tokens, "output": output_tokens, "nb": -1}, self.dst_rank)
            raise
        nb = len(src_ids)
        self.ctl.send({"rid": rid, "total": total_tokens, "output": output_tokens, "nb": nb}, self.dst_rank)
        reply = self.ctl.recv(self.dst_rank)
        if not reply["ok"]:
            if reply.get("error"):
                raise ValueError(reply["error"])
            return None
        self.seq += 1
        dst_ids = reply["dst"]
        if self.transport == "nvlink-peer":
            raw = C.c_void_p(torch.cuda.current_stream(self.src.device).cuda_stream)
            call("epd_stream_wait_geq", C.c_void_p(self._rel), self.seq, raw)
            self.src.move_to(self._dst_geom, src_ids, dst_ids, dst_ptr=self._dst_pool)
            call("epd_peer_signal", C.c_void_p(self._dst_data), self.seq, raw)
        else:
            ids = torch.tensor(src_ids, dtype=torch.int32, device=self.src.device)
            staging = torch.empty(nb, self.src.segments, self.src.block_elems, dtype=torch.bfloat16,
                                  device=self.src.device)
            self.comm.kv_send(self.src, ids, staging, self.comm_dst)
        self.src.manager.free(rid)  # _on_transfer_end("pd"): later reuse is stream-ordered after the move
        return self._info(rid, total_tokens, src_ids, dst_ids)

    def _dst_side(self, rid, total_tokens, output_tokens):
        h = self.ctl.recv(self.src_rank)
        if h["rid"] != rid or h["total"] != total_tokens or h["output"] != output_tokens:
            raise RuntimeError(f"KV handoff out of step: prefill sent {h}, decode expects rid {rid}")
        if h["nb"] < 0:
            raise ValueError(f"request {rid}: the prefill rank's KV blocks do not match {total_tokens} tokens")
        nb = self.dst.manager.blocks_needed(total_tokens)
        if h["nb"] != nb:
            msg = f"request {rid}: prefill sends {h['nb']} KV blocks, decode expects {nb}"
            self.ctl.send({"ok": False, "error": msg}, self.src_rank)
            raise ValueError(msg)
        need = total_tokens + output_tokens
        if not self.dst.manager.can_allocate(need):
            self.ctl.send({"ok": False}, self.src_rank)
            return None
        dst_ids = self.dst.manager.allocate(rid, need)
        self.seq += 1
        if self.transport == "nvlink-peer":
            raw = C.c_void_p(torch.cuda.current_stream(self.dst.device).cuda_stream)
            # the reserved blocks may still be read by this stream's earlier work (a finished
            # request freed them): release them only after it
            call("epd_peer_signal", C.c_void_p(self._src_rel), self.seq, raw)
            self.ctl.send({"ok": True, "dst": dst_ids[:nb]}, self.src_rank)
            call("epd_stream_wait_geq", C.c_void_p(self._data), self.seq, raw)
        else:
            self.ctl.send({"ok": True, "dst": dst_ids[:nb]}, self.src_rank)
            ids = torch.tensor(dst_ids[:nb], dtype=torch.int32, device=self.dst.device)
            staging = torch.empty(nb, self.dst.segments, self.dst.block_elems, dtype=torch.bfloat16,
                                  device=self.dst.device)
            self.comm.kv_recv(self.dst, ids, staging, self.comm_src)
        return self._info(rid, total_tokens, None, dst_ids)


class _Geom:
    """Geometry of a decode pool that lives in another process (mapped over CUDA IPC)."""

    def __init__(self, segments: int, block_elems: int, segment_stride: int):
        self.segments, self.block_elems, self.segment_stride = segments, block_elems, segment_stride


def kv_handoff(rid: int, total_tokens: int, output_tokens: int, src: PagedKVCache | None, dst: PagedKVCache | None,
               src_rank: int, dst_rank: int, rank: int, group=None) -> dict:
    """One-shot handoff on a shared GPU (src_rank == dst_rank == rank); raises
    CapacityExceeded if the decode pool cannot take the request."""
    h = KVHandoff(rank, src_rank, dst_rank, src, dst, group=group)
    info = h.try_reserve_decode(rid, total_tokens, output_tokens)
    if info is None:
        raise CapacityExceeded(f"decode KV pool cannot reserve {total_tokens + output_tokens} tokens")
    return info
