"""EP gather over NVLink peer memory: the encode ranks store their shards of MM tokens
straight into the prefill rank's packed buffer (reference: engine._send_ready_shards /
_schedule_transfer, engine.py:511-526; arrival accounting _on_transfer_end("ep"),
engine.py:424-435 -- prefill starts only once every shard has landed).

Protocol (per request, sequence number ``seq`` = 1, 2, ... identical on every rank):

* The prefill rank owns ``SLOTS`` packed-token slots and one data flag per rank; every
  encode rank owns ``SLOTS`` release flags. All of it is exported with CUDA IPC once
  (:meth:`PeerGather.__init__`, one ``all_gather_object``) and mapped by the peers.
* Prefill rank, at the start of request ``seq``: its stream first waits for the
  slot's previous readback, then raises every encode rank's release flag
  ``rel[seq % SLOTS] = seq`` (a remote store ordered after all earlier work on its
  stream, i.e. after every consumer of request ``seq - SLOTS`` that used the slot).
* Encode rank k: its stream waits (locally) for ``rel[seq % SLOTS] >= seq``, stores
  its shard into the slot at its tile offset and raises ``data[k] = seq`` on the
  prefill rank.
* Prefill rank: its stream waits (locally) for ``data[k] >= seq`` of every rank with a
  non-empty shard; the packed buffer is then complete, in request order.

No host synchronisation, no collective launch and no spinning kernel: every wait is a
stream memory operation on the waiting rank's own memory, every signal a store over
NVLink. ``exchange`` is the only collective (setup time)."""
from __future__ import annotations

import ctypes as C
import os

import torch

from ._lib import call

SLOTS = 2


class _Cai:
    """__cuda_array_interface__ over a raw device allocation (uint8)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _alloc(nbytes: int) -> int:
    p = C.c_void_p()
    call("epd_peer_alloc", nbytes, C.byref(p))
    return p.value


def _export(ptr: int) -> bytes:
    h = (C.c_uint8 * 64)()
    call("epd_peer_export", C.c_void_p(ptr), h)
    return bytes(h)


def _open(handle: bytes) -> int:
    buf = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    call("epd_peer_open", buf, C.byref(p))
    return p.value


class PeerGather:
    """Shard -> prefill-rank transport over peer memory for one :class:`~.stage.EncodeStage`.

    ``exchange(record) -> list[record]`` gathers one picklable record per rank (rank
    order); with ``torch.distributed`` it is ``all_gather_object``. Ranks in the same
    process (a single-GPU loopback, used by the tests) share raw pointers instead of
    IPC handles."""

    def __init__(self, device, rank: int, world: int, sink: int, slot_bytes: int, exchange):
        self.device = torch.device(device)
        self.rank, self.world, self.sink = rank, world, sink
        self.slot_bytes = -(-slot_bytes // 256) * 256
        self.seq = 0
        self._owned: list[int] = []
        self._opened: list[int] = []
        with torch.cuda.device(self.device):
            # every rank takes part in exactly one exchange, even if its own setup failed, so
            # a local failure surfaces on all ranks instead of leaving peers in the collective
            rec = {"pid": os.getpid(), "rank": rank}
            try:
                rel = self._own(4 * SLOTS)
                rec["rel"] = (rel, _export(rel))
                if rank == sink:
                    slots = self._own(SLOTS * self.slot_bytes)
                    flags = self._own(4 * world)
                    rec["slots"] = (slots, _export(slots))
                    rec["data"] = (flags, _export(flags))
            except Exception as e:
                rec["error"] = f"{type(e).__name__}: {e}"
            recs = exchange(rec)
            if [r["rank"] for r in recs] != list(range(world)):
                self.close()
                raise RuntimeError("peer gather: exchange must return one record per rank in rank order")
            bad = [f"rank {r['rank']}: {r['error']}" for r in recs if "error" in r]
            if bad:
                self.close()
                raise RuntimeError("peer gather setup failed: " + "; ".join(bad))
            self.rel_local = rel
            # a failure to map a peer's buffer is local; EncodeStage.enable_peer_gather agrees
            # on the outcome with one all_reduce
            try:
                if rank == sink:
                    self.slots = slots
                    self.data_local = flags
                    self.rel_remote = {k: self._map(recs[k]["rel"], recs[k]["pid"])
                                       for k in range(world) if k != sink}
                    self._slot_u8 = torch.as_tensor(_Cai(slots, SLOTS * self.slot_bytes), device=self.device)
                    self._free = [None] * SLOTS  # per-slot event of its last readback
                else:
                    self.slots_remote = self._map(recs[sink]["slots"], recs[sink]["pid"])
                    self.data_remote = self._map(recs[sink]["data"], recs[sink]["pid"])
            except Exception:
                self.close()
                raise

    # ------------------------------------------------------------------ setup helpers
    def _own(self, nbytes: int) -> int:
        p = _alloc(nbytes)
        self._owned.append(p)
        return p

    def _map(self, entry, pid) -> int:
        ptr, handle = entry
        if pid == os.getpid():
            return ptr  # same process (loopback): the raw pointer is valid here
        p = _open(handle)
        self._opened.append(p)
        return p

    def close(self) -> None:
        if not (self._opened or self._owned):
            return
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            call("epd_peer_close", C.c_void_p(p))
        for p in self._owned:
            call("epd_peer_free", C.c_void_p(p))
        self._opened, self._owned = [], []

    # ------------------------------------------------------------------ per request
    def begin(self) -> int:
        """Start the next request (every rank, same order); returns its sequence number."""
        self.seq += 1
        return self.seq

    def packed(self, seq: int, n: int, tokens: int, hidden: int, stream) -> tuple[torch.Tensor, int]:
        """Prefill rank: the slot for request ``seq`` as a [n, tokens, hidden] bf16 tensor.
        The stream first waits for the slot's previous readback, then releases the slot to
        the encode ranks (see the module docstring)."""
        s = seq % SLOTS
        if n * tokens * hidden * 2 > self.slot_bytes:
            raise ValueError(f"peer gather: {n} tiles exceed the slot ({self.slot_bytes} bytes)")
        if self._free[s] is not None:
            stream.wait_event(self._free[s])
            self._free[s] = None
        raw = C.c_void_p(stream.cuda_stream)
        for k, rel in self.rel_remote.items():
            call("epd_peer_signal", C.c_void_p(rel + 4 * s), seq, raw)
        base = s * self.slot_bytes
        view = self._slot_u8[base:base + n * tokens * hidden * 2].view(torch.bfloat16).view(n, tokens, hidden)
        return view, s

    def set_free_event(self, s: int, ev) -> None:
        self._free[s] = ev

    def put(self, seq: int, local: torch.Tensor, first: int, stream) -> None:
        """Encode rank: after the slot is released, store ``local`` (this rank's shard,
        contiguous) at tile offset ``first`` of the prefill rank's slot, then raise this
        rank's data flag to ``seq``."""
        s = seq % SLOTS
        raw = C.c_void_p(stream.cuda_stream)
        call("epd_stream_wait_geq", C.c_void_p(self.rel_local + 4 * s), seq, raw)
        nbytes = local.numel() * local.element_size()
        off = s * self.slot_bytes + first * (nbytes // max(local.shape[0], 1))
        call("epd_peer_put", C.c_void_p(local.data_ptr()), C.c_void_p(self.slots_remote + off), nbytes,
             C.c_void_p(self.data_remote + 4 * self.rank), seq, raw)

    def put_many(self, seq: int, pieces, stream) -> None:
        """Encode rank: several pieces [(local view, tile offset)] of one exchange, then one
        flag (the batched path, EncodeStage.process_batch)."""
        s = seq % SLOTS
        raw = C.c_void_p(stream.cuda_stream)
        call("epd_stream_wait_geq", C.c_void_p(self.rel_local + 4 * s), seq, raw)
        for i, (local, first) in enumerate(pieces):
            local = local.contiguous()
            nbytes = local.numel() * local.element_size()
            off = s * self.slot_bytes + first * (nbytes // max(local.shape[0], 1))
            last = i == len(pieces) - 1
            call("epd_peer_put", C.c_void_p(local.data_ptr()), C.c_void_p(self.slots_remote + off), nbytes,
                 C.c_void_p(self.data_remote + 4 * self.rank if last else None), seq, raw)

    def wait(self, seq: int, ranges, stream) -> None:
        """Prefill rank: the stream waits until every other rank with a non-empty shard has
        landed its shard of request ``seq``."""
        raw = C.c_void_p(stream.cuda_stream)
        for k, (_, count) in enumerate(ranges):
            if k != self.sink and count > 0:
                call("epd_stream_wait_geq", C.c_void_p(self.data_local + 4 * k), seq, raw)
