"""Encode -> prefill serving runtime: multi-request encode batches, MM-block reservations on
both sides, the ep_wait FIFO and measured trace records.

This is the reference engine's encode branch with real work in place of modeled time
(citations relative to /root/reference/pkg/src/disaggsim/):

* ``_start_encode`` (engine.py:570-613): the encode instance takes the longest FCFS prefix
  of its queue (up to ``max_batch``) whose full ``mm_tokens`` fit its MM blocks
  (``form_batch`` + E-side ``mm.allocate``, engine.py:571-576); every request is sharded with
  ``irp_shard`` over the IRP width, restarting at worker 0 (engine.py:583-602), and each
  worker encodes all of its shards of the batch in ONE encoder call;
* ``_on_worker_done`` / ``_try_reserve_prefill`` (engine.py:369-383, 528-540): a finished
  request reserves its ``mm_tokens`` in the prefill instance's MM blocks; if they do not fit
  it joins ``ep_wait`` and its shards stay on the encode workers; ``_retry_waits``
  (engine.py:680-685) retries the head of ``ep_wait`` before new work;
* ``_send_ready_shards`` / ``_on_transfer_end("ep")`` (engine.py:424-435, 521-526): every
  worker stores its shards straight into the reserved prefill-side blocks (16-token records,
  over NVLink peer memory across GPUs); once all shards landed the E-side blocks are freed
  and the request queues for prefill;
* ``_on_batch_end`` (engine.py:385-407): prefill reads its MM tokens from those blocks
  (paged prefill), the first token ends it, and the P-side blocks are freed.

* ``_on_arrival`` / ``_admission_reason`` (engine.py:319-355): a request that can never fit
  (no tokens, longer than the model's context, more MM tokens than an encode instance's or
  the prefill instance's MM pool) raises :class:`CapacityExceeded`, or -- with
  ``admission_control`` -- is recorded as rejected with the reference's reason and dropped;

* ``assign_instance`` / ``_arrival_load`` (engine.py:65-78, 277-286): with several encode
  instances (the ranks split into equal groups, each one IRP instance), every arriving
  request goes to the instance the reference's policy picks -- round robin, or least
  loaded by outstanding tiles (queued + in flight), ties to the lowest id.

Ranks run in lockstep: rank 0 is the prefill instance and the coordinator (it owns the
queues and BlockManagers and broadcasts each round's commands); every rank is one IRP
encode worker of one encode instance. Times come from the GPUs' %globaltimer (``epd_timestamp``) and fill
``ShardRecord`` / ``RequestRecord`` (trace.py:18-53); :func:`check_causality` restates
``SimTrace._check_causality`` (trace.py:119-148) for the stages this path runs (decode is
out of scope, so token times are not checked).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from collections import deque
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from ._lib import CapacityExceeded, call
from .blockpool import BlockManager, CacheKind
from .routing import assign_instance, form_batch, plan_batch, shard_ranges


@dataclass
class ServeRequest:
    """workload.Request (workload.py:27) as the runtime needs it; ``tiles`` is every
    rank's host copy (uint8 [n, S, S, C], pinned)."""

    rid: int
    tiles: torch.Tensor
    prompt: torch.Tensor            # int32 [prompt_tokens]
    output_tokens: int = 1
    arrival: float = 0.0            # seconds after serve() starts (open-loop replay)


@dataclass
class ShardRecord:
    """trace.ShardRecord (trace.py:18-24); times in seconds on the trace clock."""

    worker: int
    patches: int
    start: float | None = None
    end: float | None = None
    transfer_end: float | None = None


@dataclass
class RequestRecord:
    """trace.RequestRecord (trace.py:27-53), the fields of the encode -> prefill path."""

    rid: int
    arrival: float
    prompt_tokens: int
    mm_tokens: int
    total_tokens: int
    output_tokens: int
    e_instance: int | None = 0
    p_instance: int | None = 0
    d_instance: int | None = None
    shards: list = field(default_factory=list)
    encode_start: float | None = None
    encode_end: float | None = None
    ep_transfer_end: float | None = None
    prefill_start: float | None = None
    prefill_end: float | None = None
    first_token_time: float | None = None
    pd_transfer_end: float | None = None
    completion_time: float | None = None
    first_token: int | None = None
    ep_waited: bool = False
    rejected: str | None = None     # admission: "empty" / "context" / "mm_capacity" / "kv_capacity"


class TraceInvariantError(ValueError):
    """trace.TraceInvariantError (trace.py:14-15)."""


def check_causality(r: RequestRecord) -> None:
    """SimTrace._check_causality (trace.py:119-148) without the decode token times; a rejected
    request has no times to order."""
    if r.rejected is not None:
        return
    def ordered(label, a, b):
        if a is not None and b is not None and a > b + 1e-12:
            raise TraceInvariantError(f"request {r.rid}: {label} out of order ({a} > {b})")

    ordered("arrival/encode", r.arrival, r.encode_start)
    ordered("encode start/end", r.encode_start, r.encode_end)
    for s in r.shards:
        ordered("shard start", r.encode_start, s.start)
        ordered("shard run", s.start, s.end)
        ordered("shard transfer", s.end, s.transfer_end)
        ordered("shard/ep-end", s.transfer_end, r.ep_transfer_end)
    ordered("encode/transfer", r.encode_end, r.ep_transfer_end)
    ordered("transfer/prefill", r.ep_transfer_end, r.prefill_start)
    ordered("prefill run", r.prefill_start, r.prefill_end)
    ordered("prefill/first token", r.prefill_end, r.first_token_time)
    ordered("first token/pd", r.first_token_time, r.pd_transfer_end)
    ordered("first token/completion", r.first_token_time, r.completion_time)


class _Stamps:
    """Device %globaltimer stamps (ns) in a small device buffer, read once at the end."""

    def __init__(self, device, cap: int = 1 << 14):
        self.buf = torch.zeros(cap, dtype=torch.int64, device=device)
        self.n = 0

    def mark(self, stream) -> int:
        if self.n >= self.buf.numel():
            raise RuntimeError("trace stamp buffer full")
        i = self.n
        self.n += 1
        call("epd_timestamp", C.c_void_p(self.buf.data_ptr() + 8 * i), C.c_void_p(stream.cuda_stream))
        return i

    def read(self) -> list[int]:
        return self.buf[:self.n].cpu().tolist()


def _peer_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    call("epd_peer_alloc", nbytes, C.byref(p))
    return p.value


def _peer_export(ptr: int) -> bytes:
    h = (C.c_uint8 * 64)()
    call("epd_peer_export", C.c_void_p(ptr), h)
    return bytes(h)


def _peer_open(handle: bytes) -> int:
    buf = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    call("epd_peer_open", buf, C.byref(p))
    return p.value


class _Cai:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class MMPool:
    """The prefill instance's MM blocks in HBM (BlockManager(MM), engine.py:155-157) and the
    path into them from every encode worker.

    Rank 0 owns ``[blocks * block_size, hidden]`` bf16 rows; with world > 1 the pool and one
    data flag per rank are exported over CUDA IPC, and every encode rank exports one release
    flag. A send round ``seq``: rank 0's stream releases the round's blocks to every encode
    rank (flag store after its earlier readers -- prefills of requests that freed them);
    encode rank k waits for it, scatters its 16-token records into the reserved blocks over
    NVLink and raises ``data[k] = seq``; rank 0's stream waits on the flags of the ranks that
    had records."""

    def __init__(self, device, rank: int, world: int, blocks: int, block_size: int, hidden: int, group=None):
        self.device, self.rank, self.world = torch.device(device), rank, world
        self.blocks, self.block_size, self.hidden = blocks, block_size, hidden
        self.rec_bytes = block_size * hidden * 2
        self.manager = BlockManager(CacheKind.MM, block_size, blocks) if rank == 0 else None
        self._owned, self._opened = [], []
        self.pool = None
        if world == 1:
            self.pool = torch.zeros(blocks * block_size, hidden, dtype=torch.bfloat16, device=self.device)
            self.base = self.pool.data_ptr()
            return
        with torch.cuda.device(self.device):
            rec = {"pid": os.getpid(), "rank": rank}
            rel = self._own(4)
            rec["rel"] = (rel, _peer_export(rel))
            if rank == 0:
                nbytes = blocks * self.rec_bytes
                pool = self._own(nbytes)
                data = self._own(4 * world)
                rec["pool"] = (pool, _peer_export(pool))
                rec["data"] = (data, _peer_export(data))
                self.pool = torch.as_tensor(_Cai(pool, nbytes), device=self.device).view(torch.bfloat16).view(
                    blocks * block_size, hidden)
            recs = [None] * world
            dist.all_gather_object(recs, rec, group=group)
            self.rel_local = rel
            if rank == 0:
                self.base = pool
                self.data_local = data
                self.rel_remote = {k: self._map(recs[k]["rel"], recs[k]["pid"]) for k in range(1, world)}
            else:
                self.base = self._map(recs[0]["pool"], recs[0]["pid"])
                self.data_remote = self._map(recs[0]["data"], recs[0]["pid"])

    def _own(self, nbytes: int) -> int:
        p = _peer_alloc(nbytes)
        self._owned.append(p)
        return p

    def _map(self, entry, pid) -> int:
        ptr, handle = entry
        if pid == os.getpid():
            return ptr
        p = _peer_open(handle)
        self._opened.append(p)
        return p

    def close(self) -> None:
        if self._owned or self._opened:
            torch.cuda.synchronize(self.device)
            self.pool = None
            for p in self._opened:
                call("epd_peer_close", C.c_void_p(p))
            for p in self._owned:
                call("epd_peer_free", C.c_void_p(p))
            self._owned, self._opened = [], []

    # ---------------------------------------------------------------- a send round
    def release(self, seq: int, stream) -> None:
        """rank 0: the round's blocks may be overwritten once this stream's earlier work is done."""
        raw = C.c_void_p(stream.cuda_stream)
        for k, rel in getattr(self, "rel_remote", {}).items():
            call("epd_peer_signal", C.c_void_p(rel), seq, raw)

    def put(self, seq: int, items, stream) -> None:
        """This rank's records of the round: items = [(src [r, block_size, hidden] bf16, ids int32 dev)]."""
        raw = C.c_void_p(stream.cuda_stream)
        if self.world > 1 and self.rank != 0:
            call("epd_stream_wait_geq", C.c_void_p(self.rel_local), seq, raw)
        for src, ids in items:
            call("epd_scatter_records", C.c_void_p(src.data_ptr()), C.c_void_p(ids.data_ptr()), ids.numel(),
                 self.rec_bytes, C.c_void_p(self.base), raw)
        if self.world > 1 and self.rank != 0:
            call("epd_peer_signal", C.c_void_p(self.data_remote + 4 * self.rank), seq, raw)

    def wait(self, seq: int, k: int, stream) -> None:
        """rank 0: the stream waits until rank k's records of round ``seq`` landed."""
        if k != 0:
            call("epd_stream_wait_geq", C.c_void_p(self.data_local + 4 * k), seq, C.c_void_p(stream.cuda_stream))


class EPDRuntime:
    """Lockstep encode -> prefill runtime over the ranks of an :class:`~.stage.EncodeStage`."""

    def __init__(self, stage, prefiller, max_batch: int = 4, e_mm_tokens: int = 48_000, p_mm_tokens: int = 48_000,
                 block_size: int = 16, group=None, instances: int = 1, policy: str = "round_robin",
                 pool=None, stamps=None, admission_control: bool = False, max_context_tokens: int | None = None):
        """``pool`` / ``stamps`` replace the device MM pool transport and the %globaltimer stamps
        (the gloo CPU tier injects host stand-ins; production uses MMPool and _Stamps)."""
        self.stage, self.pf = stage, prefiller
        self.cfg = stage.cfg
        self.rank, self.world, self.device = stage.rank, stage.world, stage.device
        self.group = group
        self.max_batch = max_batch
        self.block_size = block_size
        T = self.cfg.out_tokens
        if T % block_size:
            raise ValueError(f"tokens per tile ({T}) must be a multiple of the block size ({block_size})")
        self.bpt = T // block_size
        self.is_coord = self.rank == 0
        if self.is_coord and prefiller is None:
            raise ValueError("the prefill rank needs a Prefiller")
        if instances < 1 or self.world % instances:
            raise ValueError(f"{self.world} ranks do not split into {instances} equal encode instances")
        self.instances, self.policy = instances, policy
        self.width = self.world // instances            # IRP width of every encode instance
        self.inst, self.local = divmod(self.rank, self.width)
        # E-side MM blocks: each encode instance's reservation for a request's full mm_tokens
        self.e_mms = ([BlockManager(CacheKind.MM, block_size, -(-e_mm_tokens // block_size)) for _ in range(instances)]
                      if self.is_coord else None)
        nblocks = -(-p_mm_tokens // block_size)
        self.p = pool(self, nblocks) if pool is not None else MMPool(self.device, self.rank, self.world, nblocks,
                                                                     block_size, self.cfg.out_dim, group)
        self.stamps = stamps if stamps is not None else _Stamps(self.device)
        self.admission_control = admission_control
        if max_context_tokens is None and prefiller is not None:
            geo = getattr(getattr(prefiller, "cfg", None), "geometry", None)
            max_context_tokens = getattr(geo, "max_context_tokens", None)
        self.max_context = max_context_tokens
        self.seq = 0
        self.keep_mm = False  # tests: keep a copy of each request's MM tokens as prefill read them

    def close(self) -> None:
        self.p.close()

    # ---------------------------------------------------------------- collectives
    def _bcast(self, obj):
        if self.world == 1:
            return obj
        box = [obj]
        dist.broadcast_object_list(box, src=0, group=self.group)
        return box[0]

    # ---------------------------------------------------------------- serving
    def serve(self, requests: list[ServeRequest]) -> dict | None:
        """Serve a burst of requests (all arriving now), FCFS, to their first tokens. Every
        rank passes the same list. Returns (rank 0) the RequestRecords, the ep_wait history
        and the wall time; None elsewhere."""
        self._tiles = {r.rid: r.tiles for r in requests}
        try:
            return self._serve(requests)
        finally:
            self._tiles = {}

    def _sync(self) -> None:
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)

    def _serve(self, requests):
        s = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        T, D = self.cfg.out_tokens, self.cfg.out_dim
        reqs = {r.rid: r for r in requests}
        # trace clock: %globaltimer ns from a calibration stamp taken when the burst arrives
        self._sync()
        cal = self.stamps.mark(s)
        self._sync()
        held: dict[int, torch.Tensor] = {}      # rid -> this rank's encoded shard, not yet sent
        marks: dict = {}                         # ("start"|"end"|"xfer"|"ep"|"pre0"|"pre1", rid[, k]) -> slot
        if self.is_coord:
            # open-loop arrivals: a request joins its encode instance's queue once its arrival
            # time has passed; assign_instance on arrival (engine.py:270-283) with the instance
            # load = its outstanding tiles, queued and in flight (_arrival_load, engine.py:277-286)
            pending = deque(sorted(requests, key=lambda r: (r.arrival, r.rid)))
            open_loop = any(r.arrival > 0 for r in requests)
            queues = [deque() for _ in range(self.instances)]
            load = [0] * self.instances
            inst_of: dict[int, int] = {}
            rr = 0
            ep_wait: deque = deque()
            ready: deque = deque()
            recs: dict[int, RequestRecord] = {}
            p_blocks: dict[int, list[int]] = {}
            waited = []
            enc_done = None  # event after the coordinator's last encode (the instance is busy until then)

            def admit(now: float) -> None:
                nonlocal rr
                while pending and pending[0].arrival <= now:
                    r = pending.popleft()
                    mm = r.tiles.shape[0] * T
                    reason = self._admission_reason(mm, mm + int(r.prompt.numel()))
                    if reason is not None:
                        if not self.admission_control:
                            raise CapacityExceeded(f"request {r.rid} can never fit: {reason}")
                        recs[r.rid] = RequestRecord(r.rid, r.arrival, int(r.prompt.numel()), mm,
                                                    mm + int(r.prompt.numel()), r.output_tokens, e_instance=None,
                                                    p_instance=None, rejected=reason)
                        continue
                    iid, rr = assign_instance(self.policy, [(i, float(load[i])) for i in range(self.instances)], rr)
                    inst_of[r.rid] = iid
                    queues[iid].append(r.rid)
                    load[iid] += r.tiles.shape[0]
                    recs[r.rid] = RequestRecord(r.rid, r.arrival, int(r.prompt.numel()), mm,
                                                mm + int(r.prompt.numel()), r.output_tokens, e_instance=iid)
        first_tok, kept = {}, {}
        t_wall0 = time.perf_counter()
        while True:
            # ---- coordinator: _retry_waits first, then a new encode batch (engine.py:680-700)
            cmd = None
            if self.is_coord:
                try:
                    if open_loop:
                        # a new batch starts once the encode instance finished its previous one
                        # (engine.py: one running batch per instance); meanwhile requests arrive
                        if enc_done is not None:
                            enc_done.synchronize()
                        admit(time.perf_counter() - t_wall0)
                        if pending and not any(queues) and not ep_wait:
                            time.sleep(max(0.0, pending[0].arrival - (time.perf_counter() - t_wall0)))
                            admit(time.perf_counter() - t_wall0)
                    else:
                        admit(float("inf"))
                    pre = []
                    while ep_wait:
                        rid = ep_wait[0]
                        if not self.p.manager.can_allocate(recs[rid].mm_tokens):
                            break
                        ep_wait.popleft()
                        p_blocks[rid] = self.p.manager.allocate(rid, recs[rid].mm_tokens)
                        pre.append((rid, p_blocks[rid]))

                    batch = []
                    for iid, queue in enumerate(queues):  # every idle encode instance starts a batch
                        e_mm = self.e_mms[iid]

                        def fits(rid, e_mm=e_mm):
                            mm = recs[rid].mm_tokens
                            if not e_mm.can_allocate(mm):
                                return False
                            e_mm.allocate(rid, mm)
                            return True
                        b = form_batch(list(queue), self.max_batch, fits)
                        for _ in b:
                            queue.popleft()
                        batch += [(rid, reqs[rid].tiles.shape[0], iid) for rid in b]
                    done = not (any(queues) or ep_wait or batch or pre or pending)
                    if not done and not batch and not pre and not pending:
                        # nothing in flight and nothing can start (admission lets no such request in)
                        raise CapacityExceeded("the MM blocks cannot hold the head request (mm_capacity)")
                    cmd = {"pre": [(rid, blocks, inst_of[rid]) for rid, blocks in pre], "batch": batch, "done": done}
                except CapacityExceeded as e:  # every rank raises it (no rank left in a collective)
                    cmd = {"error": str(e)}
            cmd = self._bcast(cmd)
            if "error" in cmd:
                raise CapacityExceeded(cmd["error"])
            if cmd["done"]:
                break
            self._send(cmd["pre"], held, marks, s)
            if self.is_coord and cmd["batch"]:
                disp = self.stamps.mark(s)  # batch start: a text-only request's (empty) encode
                for rid, _, _ in cmd["batch"]:
                    marks[("disp", rid)] = disp
            self._encode(cmd["batch"], held, marks, s)
            if self.is_coord and open_loop and cmd["batch"] and s is not None:
                enc_done = torch.cuda.Event()
                enc_done.record(s)
            # ---- coordinator: _on_worker_done -> _try_reserve_prefill, else ep_wait (engine.py:369-383)
            post = None
            if self.is_coord:
                post = []
                for rid, _, iid in cmd["batch"]:
                    if self.p.manager.can_allocate(recs[rid].mm_tokens):
                        p_blocks[rid] = self.p.manager.allocate(rid, recs[rid].mm_tokens)
                        post.append((rid, p_blocks[rid], iid))
                    else:
                        ep_wait.append(rid)
                        recs[rid].ep_waited = True
                        waited.append(rid)
            post = self._bcast(post)
            self._send(post, held, marks, s)
            # ---- coordinator: every landed request -> prefill, first token, free P-side blocks
            if self.is_coord:
                for rid, _, iid in cmd["pre"] + post:
                    self.e_mms[iid].free(rid)      # _on_transfer_end("ep"): all shards landed
                    load[iid] -= reqs[rid].tiles.shape[0]
                    ready.append(rid)
                while ready:
                    rid = ready.popleft()
                    r = reqs[rid]
                    ids = torch.tensor(p_blocks[rid], dtype=torch.int64)
                    rows = (ids.view(-1, 1) * self.block_size + torch.arange(self.block_size)).view(-1).to(torch.int32)
                    if self.keep_mm:
                        kept[rid] = self.p.pool.index_select(0, rows.to(self.device).long()).view(-1, T, D)
                    marks[("pre0", rid)] = self.stamps.mark(s)
                    tok = self.pf.prefill(None, r.prompt, mm_pool=self.p.pool, mm_rows=rows)
                    marks[("pre1", rid)] = self.stamps.mark(s)
                    first_tok[rid] = tok.clone()
                    self.p.manager.free(rid)       # _on_batch_end: P-side MM blocks free
        self._sync()
        wall = time.perf_counter() - t_wall0
        st = self.stamps.read()
        mine = {k: st[v] for k, v in marks.items() if k[0] in ("start", "end")}
        allmarks = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(allmarks, mine, group=self.group)
        else:
            allmarks = [mine]
        if not self.is_coord:
            self.stamps.n = 0
            return None
        # ---- RequestRecords on the trace clock (seconds since the calibration stamp)
        base = st[cal]

        def sec(ns):
            return (ns - base) / 1e9
        for rid, rec in recs.items():
            if rec.rejected is not None:
                continue
            # arrivals are host seconds after the calibration stamp's completion, so they trail
            # the device clock slightly: arrival <= encode start holds by construction
            n = reqs[rid].tiles.shape[0]
            base_rank = rec.e_instance * self.width
            shards = []
            for k, (first, count) in enumerate(shard_ranges(n, self.width)):
                if count == 0:
                    continue
                m = allmarks[base_rank + k]
                shards.append(ShardRecord(k, count, sec(m[("start", rid)]), sec(m[("end", rid)]),
                                          sec(st[marks[("xfer", rid, base_rank + k)]])))
            rec.ep_transfer_end = sec(st[marks[("ep", rid)]])
            if not shards:
                # text-only request: one empty shard on worker 0 that starts with its batch and
                # "transfers" at once (engine.py:589-590: shards [(0, 0)], no EP bytes)
                t = sec(st[marks[("disp", rid)]])
                shards = [ShardRecord(0, 0, t, t, t)]
            rec.shards = shards
            rec.encode_start = min(x.start for x in shards)
            rec.encode_end = max(x.end for x in shards)
            rec.prefill_start = sec(st[marks[("pre0", rid)]])
            rec.prefill_end = rec.first_token_time = sec(st[marks[("pre1", rid)]])
            rec.first_token = int(first_tok[rid].item())
        self.stamps.n = 0
        return {"records": recs, "ep_wait": waited, "wall_s": wall, "mm": kept,
                "plans": plan_batch([reqs[r].tiles.shape[0] for r in reqs], self.width)[0]}

    def _admission_reason(self, mm_tokens: int, total_tokens: int) -> str | None:
        """_admission_reason (engine.py:319-344) for this path's pools: the encode instances'
        MM blocks and the prefill instance's MM blocks (its KV is the handoff's concern)."""
        if total_tokens == 0:
            return "empty"
        if self.max_context is not None and total_tokens > self.max_context:
            return "context"
        if self.e_mms[0].blocks_needed(mm_tokens) > self.e_mms[0].total_blocks:
            return "mm_capacity"
        if self.p.manager.blocks_needed(mm_tokens) > self.p.manager.total_blocks:
            return "kv_capacity"  # the reference's prefill-instance check (MM and KV together)
        return None

    # ---------------------------------------------------------------- per-rank work
    def _encode(self, batch, held, marks, s) -> None:
        """_start_encode on this worker: its shard of every request in the batch (restart at
        worker 0), uploaded into one buffer and encoded in one call."""
        if not batch:
            return
        parts = []
        for rid, n, iid in batch:
            if iid != self.inst:
                continue
            first, count = shard_ranges(n, self.width)[self.local]
            if count:
                parts.append((rid, first, count))
        if not parts:
            return
        total = sum(c for _, _, c in parts)
        reqs_tiles = self._tiles
        S, Cc = self.cfg.image_size, self.cfg.channels
        tiles = torch.empty(total, S, S, Cc, dtype=torch.uint8, device=self.device)
        o = 0
        for rid, first, count in parts:
            tiles[o:o + count].copy_(reqs_tiles[rid][first:first + count], non_blocking=True)
            o += count
        out = torch.empty(total, self.cfg.out_tokens, self.cfg.out_dim, dtype=torch.bfloat16, device=self.device)
        start = self.stamps.mark(s)
        self.stage.enc.encode(tiles, out)
        end = self.stamps.mark(s)
        o = 0
        for rid, first, count in parts:
            held[rid] = out[o:o + count]
            marks[("start", rid)] = start
            marks[("end", rid)] = end
            o += count

    def _send(self, sends, held, marks, s) -> None:
        """_send_ready_shards for a list of reserved requests: every rank stores its held
        shards into the requests' P-side blocks; rank 0 waits for all and stamps arrivals."""
        if not sends:
            return
        self.seq += 1
        if self.is_coord:
            self.p.release(self.seq, s)
        items = []
        has = [False] * self.world
        for rid, blocks, iid in sends:
            n = self._tiles[rid].shape[0]
            ranges = shard_ranges(n, self.width)
            for k, (first, count) in enumerate(ranges):
                if count:
                    has[iid * self.width + k] = True
            first, count = ranges[self.local] if iid == self.inst else (0, 0)
            if count:
                ids = torch.tensor(blocks[first * self.bpt:(first + count) * self.bpt], dtype=torch.int32).to(
                    self.device, non_blocking=True)
                src = held.pop(rid).reshape(count * self.bpt, self.block_size, self.cfg.out_dim)
                items.append((src, ids))
        self.p.put(self.seq, items, s)
        if self.is_coord:
            xfer = {}
            for k in range(self.world):
                if has[k]:
                    self.p.wait(self.seq, k, s)
                    xfer[k] = self.stamps.mark(s)
            ep = self.stamps.mark(s)
            for rid, blocks, iid in sends:
                n = self._tiles[rid].shape[0]
                for k, (first, count) in enumerate(shard_ranges(n, self.width)):
                    if count:
                        marks[("xfer", rid, iid * self.width + k)] = xfer[iid * self.width + k]
                marks[("ep", rid)] = ep

