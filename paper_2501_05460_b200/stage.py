"""Encode stage runtime: one request's tiles -> packed MM tokens on the prefill GPU.

Mirrors the encode branch of the reference engine, with real work in place of
modeled time (citations relative to /root/reference/pkg/src/disaggsim/):

1. ``_start_encode`` (engine.py:570-613): the request's tiles are partitioned
   with ``irp_shard`` over the IRP width = the encode ranks; rank k owns the
   contiguous range ``shard_ranges(n, w)[k]``; zero shards idle.
2. MM cache (blocks.py MM manager, engine.py:155-157 + the content cache the
   reference lacks): on the prefill rank the tiles are hashed and looked up;
   only first occurrences of uncached tiles are sharded and encoded.
3. ``_send_ready_shards`` / ``_on_transfer_end("ep")`` (engine.py:424-435,
   521-526): each rank's shard of post-projector tokens
   (``tiles * tokens_per_patch * mm_bytes_per_token`` bytes) goes to the
   prefill rank with NCCL point-to-point over NVLink, landing at its tile
   offset, so the packed buffer is in request order whatever the arrival
   order; prefill may start only once all shards landed.

Multi-GPU layout: one process per GPU (torchrun); ranks 0..w-1 are the encode
workers and rank ``prefill_rank`` (default 0) is also the prefill sink (at
w = 8 on an 8-GPU node the sink shares a GPU with encode worker 0 -- the
documented deviation from the reference's GPU budget rule, simconfig.py:86-88).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from .routing import ep_bytes, shard_ranges


# trace.ShardRecord (trace.py:18-24). The single-request path records worker and tiles; the
# serving runtime (runtime.EPDRuntime) also fills start / end / transfer_end from the GPUs'
# %globaltimer.
from .runtime import ShardRecord  # noqa: E402


@dataclass
class RequestResult:
    rid: int
    n_tiles: int
    encoded_tiles: int
    shards: list = field(default_factory=list)
    cache_counts: dict | None = None     # MM-token cache: {"hit", "miss", "dup"} tile counts
    plan: object | None = None           # the cache plan (device tensors; plan.kinds reads them back)
    ep_bytes: int = 0                    # bytes moved to the prefill rank (engine.py:524)
    tokens: torch.Tensor | None = None   # packed [n, tokens_per_tile, hidden] on the prefill rank
    readback: torch.cuda.Event | None = None  # set when tokens were copied into out_host


class EncodeStage:
    """Per-rank encode-stage executor.

    ``encoder`` must expose ``cfg`` (an EncoderConfig) and
    ``encode(tiles_dev, out)``; in production it is
    :class:`~.encoder.VisionEncoder` (sm_100a kernels). ``cache`` is an
    optional :class:`~.mmcache.MMTokenCache` living on the prefill rank; with
    world > 1 the encode ranks pass ``cached=True`` so they join its miss broadcast.
    """

    def __init__(self, encoder, device: torch.device, rank: int = 0, world: int = 1, prefill_rank: int = 0,
                 cache=None, group=None, cached: bool | None = None, comm=None):
        self.enc = encoder
        self.cfg = encoder.cfg
        self.device = torch.device(device)
        self.rank = rank
        self.world = world
        self.prefill_rank = prefill_rank
        self.cache = cache
        self.group = group
        # NCCL leg of the EP gather through the C ABI (comm.NcclComm -> epd_gather_tokens); without
        # it the fallback is torch.distributed's grouped P2P
        self.comm = comm
        if cache is not None and rank != prefill_rank:
            raise ValueError("the MM-token cache lives on the prefill rank")
        # Whether the prefill rank runs the MM-token cache: every rank must take the same
        # path (the cached one broadcasts the miss list first), so encode ranks are told.
        self.cached = (cache is not None) if cached is None else bool(cached)
        if self.cached and rank == prefill_rank and cache is None:
            raise ValueError("cached=True needs the cache object on the prefill rank")
        self._staging = None
        # Host I/O runs on its own streams so consecutive requests pipeline: request i+1's
        # H2D upload overlaps request i's encode, and request i's D2H readback overlaps
        # request i+1's encode (PCIe is full duplex; uploads and readbacks never queue
        # behind one another).
        self._up = torch.cuda.Stream(self.device) if self.device.type == "cuda" else None
        self._down = torch.cuda.Stream(self.device) if self.device.type == "cuda" else None
        # Double-buffered device rings for uploads and packed tokens (no per-request
        # allocation: caching-allocator churn across three streams can trigger synchronising
        # frees). A ring slot is reused two requests later, after the event that marks its
        # last consumer (the encode for inputs, the readback for packed tokens).
        self._rings: dict = {}
        # EP gather transport: NCCL grouped P2P by default; enable_peer_gather() switches the
        # no-cache path to stores over NVLink peer memory (peer.py)
        self._peer = None

    def enable_peer_gather(self, max_tiles: int, exchange=None) -> bool:
        """Collective over the stage's ranks: map the prefill rank's packed-token slots
        (room for ``max_tiles`` tiles) into every encode rank over CUDA IPC so shards are
        stored straight into them over NVLink (peer.py). Returns False, on every rank, if
        any rank could not set it up (the NCCL transport then stays in use)."""
        if self.world == 1 or self.device.type != "cuda":
            return False
        from .peer import PeerGather
        if exchange is None:
            def exchange(rec):
                out = [None] * self.world
                dist.all_gather_object(out, rec, group=self.group)
                return out
        slot_bytes = max_tiles * self.cfg.out_tokens * self.cfg.out_dim * 2
        err = None
        try:  # PeerGather runs exactly one exchange on every rank, failed or not
            peer = PeerGather(self.device, self.rank, self.world, self.prefill_rank, slot_bytes, exchange)
        except Exception as e:  # reported on every rank below
            peer, err = None, f"{type(e).__name__}: {e}"
        ok = torch.tensor([0 if peer is None else 1], dtype=torch.int32, device=self.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if int(ok.item()) == 1:
            self._peer = peer
            self._peer_tiles = max_tiles
            return True
        if peer is not None:
            peer.close()
        if err:
            import sys
            print(f"[rank {self.rank}] peer-memory gather unavailable ({err}); using NCCL P2P", file=sys.stderr)
        return False

    @property
    def transport(self) -> str:
        if self._peer is not None:
            return "nvlink-peer"
        if self.world == 1:
            return "local"
        return "nccl-capi" if self.comm is not None else "nccl-p2p"

    def close(self) -> None:
        if self._peer is not None:
            self._peer.close()
            self._peer = None

    def gather_only(self, local: torch.Tensor | None, n: int) -> torch.Tensor | None:
        """The EP exchange of one n-tile request on its own (bench: the gather's NVLink
        roofline): ``local`` is this rank's already-encoded shard; returns the packed
        buffer on the prefill rank."""
        ranges = shard_ranges(n, self.world)
        first, count = ranges[self.rank]
        ex = self._open_exchange(n, ring=False)
        if self.rank == self.prefill_rank and count > 0:
            ex["dest"][first:first + count].copy_(local)
        self._close_exchange(ex, local if count > 0 else None, ranges)
        return ex["dest"]

    # ------------------------------------------------------------------ helpers
    def _tokens_shape(self, n: int):
        return (n, self.cfg.out_tokens, self.cfg.out_dim)

    def _buffer(self, n: int) -> torch.Tensor:
        return torch.empty(self._tokens_shape(n), dtype=torch.bfloat16, device=self.device)

    def _slot(self, key, shape, dtype):
        # one ring per (use, shape); rings are never dropped (a dropped buffer may still be
        # read by queued work), so memory grows only with the number of distinct shapes
        key = (key, tuple(shape), dtype)
        r = self._rings.get(key)
        if r is None:
            r = {"bufs": [torch.empty(shape, dtype=dtype, device=self.device) for _ in range(2)],
                 "free": [None, None], "i": 0}
            self._rings[key] = r
        k = r["i"]
        r["i"] ^= 1
        return r, k

    def _upload(self, tiles_host: torch.Tensor, idx):
        """Pinned host tiles -> device on the upload stream (into a ring slot); the compute
        stream waits for it. Returns (tensor, release) -- call release() once the compute
        stream has queued the last read of the tensor."""
        if isinstance(idx, slice):
            host = tiles_host[idx]
        elif idx is None:
            host = tiles_host
        else:
            host = tiles_host.index_select(0, torch.as_tensor(idx, dtype=torch.int64))
        if self._up is None:
            return host.to(self.device, non_blocking=True), (lambda: None)
        compute = torch.cuda.current_stream(self.device)
        r, k = self._slot("in", host.shape, host.dtype)
        buf = r["bufs"][k]
        if r["free"][k] is not None:
            self._up.wait_event(r["free"][k])
        with torch.cuda.stream(self._up):
            buf.copy_(host, non_blocking=True)
        compute.wait_stream(self._up)

        def release():
            ev = torch.cuda.Event()
            ev.record(compute)
            r["free"][k] = ev
        return buf, release

    def _packed(self, n: int):
        """Packed-token buffer for n tiles from the ring (waits for its previous readback)."""
        if self._up is None:
            return self._buffer(n), None
        r, k = self._slot("out", self._tokens_shape(n), torch.bfloat16)
        if r["free"][k] is not None:
            torch.cuda.current_stream(self.device).wait_event(r["free"][k])
            r["free"][k] = None
        return r["bufs"][k], (lambda ev: r["free"].__setitem__(k, ev))

    def _readback(self, tokens: torch.Tensor, out_host: torch.Tensor, slot=None) -> torch.cuda.Event:
        """Packed tokens -> pinned host buffer on the download stream, after the compute
        stream's work so far; returns the event that marks the copy done."""
        compute = torch.cuda.current_stream(self.device)
        self._down.wait_stream(compute)
        with torch.cuda.stream(self._down):
            out_host.copy_(tokens, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._down)
        if slot is not None:
            slot(ev)  # the slot's next use waits for this readback
        else:
            tokens.record_stream(self._down)
        return ev

    def join(self) -> None:
        """Make the caller's stream wait for all host I/O issued so far."""
        if self._up is not None:
            compute = torch.cuda.current_stream(self.device)
            compute.wait_stream(self._up)
            compute.wait_stream(self._down)

    def _gather(self, local: torch.Tensor | None, dest: torch.Tensor | None, ranges) -> None:
        """Shards -> prefill rank at their unit offsets (grouped point-to-point)."""
        if self.world == 1:
            return
        if self.comm is not None:
            n = sum(c for _, c in ranges)
            self.comm.gather_tokens(local, n, dest, root=self.prefill_rank)
            return
        ops = []
        if self.rank == self.prefill_rank:
            for k, (first, count) in enumerate(ranges):
                if k != self.rank and count > 0:
                    ops.append(dist.P2POp(dist.irecv, dest[first:first + count], k, self.group))
        else:
            first, count = ranges[self.rank]
            if count > 0:
                ops.append(dist.P2POp(dist.isend, local, self.prefill_rank, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    # ------------------------------------------------------------------ request
    def process(self, tiles_host: torch.Tensor, rid: int = 0, tiles_dev: torch.Tensor | None = None,
                out_host: torch.Tensor | None = None) -> RequestResult:
        """Encode one request. ``tiles_host``: uint8 [n, S, S, C] (pinned for async copies);
        if ``tiles_dev`` (all tiles, already on this rank's device) is given, no H2D copy
        is made. Returns the packed tokens on the prefill rank; with ``out_host`` (pinned,
        [n, tokens, hidden] bf16) the prefill rank also reads them back asynchronously and
        ``result.readback`` is the event to wait on."""
        res = self._process(tiles_host, rid, tiles_dev)
        if out_host is not None and res.tokens is not None:
            slot = getattr(res, "_slot", None)
            res.readback = self._readback(res.tokens, out_host, slot) if self._down is not None else None
            if res.readback is None:
                out_host.copy_(res.tokens)
        return res

    def process_image(self, image_host: torch.Tensor, model: str, rid: int = 0,
                      out_host: torch.Tensor | None = None) -> RequestResult:
        """One request = one photo (uint8 HWC, pinned): upload it, cut the model's tiles on the
        GPU (tiler.py), then encode as :meth:`process`. Single-rank
        (the tiles are then sharded by process() when world > 1 via tiles_dev on each rank)."""
        from .tiler import plan, tile_image
        H, W, Cc = image_host.shape
        cols, rows, thumb, _ = plan(model, W, H)
        n = cols * rows + (1 if thumb else 0)
        img, release = self._upload(image_host[None], None)
        r, k = self._slot("tiles", (n, self.cfg.image_size, self.cfg.image_size, Cc), torch.uint8)
        tiles = tile_image(img[0], model, tile=self.cfg.image_size, out=r["bufs"][k])
        release()
        res = self.process(None, rid, tiles_dev=tiles, out_host=out_host)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        r["free"][k] = ev  # the tiles slot is reusable once this request's encode is queued
        return res

    def process_batch(self, tiles_host: list | None = None, tiles_dev: list | None = None,
                      out_host: torch.Tensor | None = None) -> RequestResult:
        """Encode a batch of requests (``_start_encode``, engine.py:583-602): every request is
        IRP-sharded over the ranks restarting at worker 0, each rank encodes all of its shards of
        the batch in ONE encoder call, and the shards land on the prefill rank in one exchange,
        packed request after request (request r at tile offset sum(n[:r])). Pass the requests'
        host tiles (pinned) or device tiles; every rank passes the same batch. Uncached path."""
        if self.cached:
            raise ValueError("process_batch runs the uncached path")
        src_list = tiles_dev if tiles_dev is not None else tiles_host
        ns = [t.shape[0] for t in src_list]
        offs = [sum(ns[:r]) for r in range(len(ns))]
        m = sum(ns)
        is_sink = self.rank == self.prefill_rank
        parts, senders = [], set()
        for r, n in enumerate(ns):
            for k, (first, count) in enumerate(shard_ranges(n, self.world)):
                if count:
                    senders.add(k)
                    if k == self.rank:
                        parts.append((r, first, count))
        mine = sum(c for _, _, c in parts)
        ex = self._open_exchange(m, ring=True)
        local = None
        if mine:
            S, Cc = self.cfg.image_size, self.cfg.channels
            if tiles_dev is not None and len(parts) == 1:
                r, first, count = parts[0]
                src, release = tiles_dev[r][first:first + count], None
            elif self._up is None:  # host-side stage (gloo CPU tier)
                src = torch.cat([src_list[r][first:first + count] for r, first, count in parts])
                release = None
            else:
                ring, k = self._slot("bin", (mine, S, S, Cc), torch.uint8)
                if ring["free"][k] is not None:  # the slot's previous encode has read it
                    torch.cuda.current_stream(self.device).wait_event(ring["free"][k])
                src = ring["bufs"][k]
                o = 0
                for r, first, count in parts:
                    src[o:o + count].copy_(src_list[r][first:first + count], non_blocking=True)
                    o += count

                def release(ring=ring, k=k):
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.current_stream(self.device))
                    ring["free"][k] = ev
            local = self._buffer(mine)
            self.enc.encode(src.contiguous(), local)
            if release is not None:
                release()
        pieces, o = [], 0
        for r, first, count in parts:
            pieces.append((local[o:o + count], offs[r] + first))
            o += count
        self._close_pieces(ex, pieces, senders, ns, offs)
        res = RequestResult(rid=0, n_tiles=m, encoded_tiles=mine)
        res._slot = ex["slot"]
        res.shards = [ShardRecord(k, c) for n in ns for k, (_, c) in enumerate(shard_ranges(n, self.world)) if c]
        tpp, bpt = self.cfg.out_tokens, self.cfg.out_dim * 2
        res.ep_bytes = sum(ep_bytes(c, tpp, bpt) for n in ns for k, (_, c) in enumerate(shard_ranges(n, self.world))
                           if k != self.prefill_rank)
        res.tokens = ex["dest"]
        if out_host is not None and res.tokens is not None:
            res.readback = self._readback(res.tokens, out_host, res._slot) if self._down is not None else None
            if res.readback is None:
                out_host.copy_(res.tokens)
        return res

    def _close_pieces(self, ex: dict, pieces, senders, ns, offs) -> None:
        """process_batch's exchange: this rank's pieces (local view, tile offset in the batch)
        reach the prefill rank; the prefill rank copies its own pieces in place."""
        peer, is_sink = ex["peer"], self.rank == self.prefill_rank
        s = torch.cuda.current_stream(self.device) if peer is not None else None
        if is_sink:
            for view, off in pieces:
                ex["dest"][off:off + view.shape[0]].copy_(view)
        if peer is not None:
            if is_sink:
                fake = [(0, 1 if k in senders else 0) for k in range(self.world)]
                peer.wait(ex["seq"], fake, s)
            elif pieces:
                peer.put_many(ex["seq"], pieces, s)
            return
        if self.world == 1:
            return
        if self.comm is not None:  # one C-ABI gather per request (contiguous shards)
            by_req = {}
            for view, off in pieces:
                r = max(i for i in range(len(offs)) if offs[i] <= off)
                by_req[r] = view
            for r, n in enumerate(ns):
                dest = ex["dest"][offs[r]:offs[r] + n] if is_sink else None
                self.comm.gather_tokens(None if is_sink else by_req.get(r), n, dest, root=self.prefill_rank)
            return
        ops = []
        if is_sink:
            for r, n in enumerate(ns):
                for k, (first, count) in enumerate(shard_ranges(n, self.world)):
                    if k != self.rank and count:
                        dst = ex["dest"][offs[r] + first:offs[r] + first + count]
                        ops.append(dist.P2POp(dist.irecv, dst, k, self.group))
        else:
            for view, _ in pieces:
                ops.append(dist.P2POp(dist.isend, view.contiguous(), self.prefill_rank, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def _open_exchange(self, m: int, ring: bool) -> dict:
        """Start the EP exchange of an m-tile request on every rank: picks the transport
        (the peer slots when they are up and hold m tiles, else the collective) and, on the
        prefill rank, the buffer the shards land in -- a peer slot, a ring slot (``ring``,
        read back by process()) or a fresh buffer."""
        is_sink = self.rank == self.prefill_rank
        peer = self._peer if (self._peer is not None and 0 < m <= self._peer_tiles) else None
        ex = {"peer": peer, "seq": None, "dest": None, "slot": None}
        if peer is not None:
            ex["seq"] = peer.begin()
            if is_sink:
                ex["dest"], ps = peer.packed(ex["seq"], m, self.cfg.out_tokens, self.cfg.out_dim,
                                             torch.cuda.current_stream(self.device))
                ex["slot"] = lambda ev, ps=ps: peer.set_free_event(ps, ev)
        elif is_sink and ring:
            ex["dest"], ex["slot"] = self._packed(m)
        elif is_sink and m:
            ex["dest"] = self._buffer(m)
        return ex

    def _close_exchange(self, ex: dict, local: torch.Tensor | None, ranges) -> None:
        """Finish the exchange: this rank's shard (already encoded into ``local``, which on the
        prefill rank is a view of the destination) reaches the prefill rank at its tile offset."""
        peer, is_sink = ex["peer"], self.rank == self.prefill_rank
        first, count = ranges[self.rank]
        if peer is None:
            self._gather(local, ex["dest"], ranges)
        elif is_sink:
            peer.wait(ex["seq"], ranges, torch.cuda.current_stream(self.device))  # every shard landed
        elif count > 0:
            peer.put(ex["seq"], local, first, torch.cuda.current_stream(self.device))  # NVLink stores + flag

    def _process(self, tiles_host, rid, tiles_dev) -> RequestResult:
        n = tiles_host.shape[0] if tiles_host is not None else tiles_dev.shape[0]
        is_sink = self.rank == self.prefill_rank
        res = RequestResult(rid=rid, n_tiles=n, encoded_tiles=0)
        tpp, bpt = self.cfg.out_tokens, self.cfg.out_dim * 2

        if not self.cached:
            ranges = shard_ranges(n, self.world)
            first, count = ranges[self.rank]
            ex = self._open_exchange(n, ring=True)
            packed = ex["dest"]
            local = None
            if count > 0:
                release = None
                if tiles_dev is not None:
                    src = tiles_dev[first:first + count]
                else:
                    src, release = self._upload(tiles_host, slice(first, first + count))
                local = packed[first:first + count] if is_sink else self._buffer(count)
                self.enc.encode(src.contiguous(), local)
                if release is not None:
                    release()
            self._close_exchange(ex, local, ranges)
            res._slot = ex["slot"]
            res.encoded_tiles = count
            res.shards = [ShardRecord(k, c) for k, (_, c) in enumerate(ranges) if c > 0]
            res.ep_bytes = sum(ep_bytes(c, tpp, bpt) for k, (_, c) in enumerate(ranges) if k != self.prefill_rank)
            res.tokens = packed
            return res

        # ---- cached path (cache on the prefill rank): the plan stays on the device; the
        # host learns only the miss count (the number of tiles to encode)
        plan = None
        release_all = release_mine = None
        miss_dev = None
        if is_sink:
            if tiles_dev is not None:
                all_dev = tiles_dev
            else:
                all_dev, release_all = self._upload(tiles_host, None)
            plan = self.cache.plan(self.cache.hash(all_dev.contiguous()))
            m = plan.n_miss
            miss_dev = plan.miss_tiles.long()
        if self.world > 1:
            on_dev = dist.get_backend(self.group) == "nccl"
            cnt = torch.tensor([0 if plan is None else m], dtype=torch.int64,
                               device=self.device if on_dev else "cpu")
            dist.broadcast(cnt, self.prefill_rank, group=self.group)
            m = int(cnt.item())
            if m:
                if is_sink:
                    midx = miss_dev if on_dev else miss_dev.cpu()
                else:
                    midx = torch.empty(m, dtype=torch.int64, device=self.device if on_dev else "cpu")
                dist.broadcast(midx, self.prefill_rank, group=self.group)
                miss_dev = midx.to(self.device)
        ranges = shard_ranges(m, self.world)
        first, count = ranges[self.rank]
        # every rank knows m, so every rank picks the same transport for this request
        ex = self._open_exchange(m, ring=False)
        staging = ex["dest"]
        local = None
        if count > 0:
            my = miss_dev[first:first + count]
            if is_sink:
                src = all_dev.index_select(0, my)
                local = staging[first:first + count]
            else:
                if tiles_dev is not None:
                    src = tiles_dev.index_select(0, my)
                else:
                    src, release_mine = self._upload(tiles_host, my.cpu())  # host tiles: index on the host
                local = self._buffer(count)
            self.enc.encode(src.contiguous(), local)
        for release in (release_all, release_mine):
            if release is not None:
                release()  # the compute stream has queued its last read of the uploaded tiles
        self._close_exchange(ex, local, ranges)
        res.encoded_tiles = count
        res.shards = [ShardRecord(k, c) for k, (_, c) in enumerate(ranges) if c > 0]
        res.ep_bytes = sum(ep_bytes(c, tpp, bpt) for k, (_, c) in enumerate(ranges) if k != self.prefill_rank)
        if is_sink:
            from ._lib import call
            import ctypes as C
            rec = tpp * bpt
            s = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
            if m:
                call("epd_scatter_records", C.c_void_p(staging.data_ptr()), C.c_void_p(plan.miss_entries.data_ptr()),
                     m, rec, C.c_void_p(self.cache.store.data_ptr()), s)
            packed = self._buffer(n)
            call("epd_gather_records", C.c_void_p(self.cache.store.data_ptr()), C.c_void_p(plan.entries.data_ptr()),
                 n, rec, C.c_void_p(packed.data_ptr()), s)
            res.plan = plan
            res.cache_counts = plan.counts
            res.tokens = packed
        return res


def tiles_for_request(n: int, cfg, seed: int, repeat_period: int | None = None) -> torch.Tensor:
    """Synthetic uint8 HWC tiles [n, S, S, C] (uniform 0..255, seeded). With
    ``repeat_period`` p, tile i repeats tile i - p (the C4 repeated-image workload)."""
    g = torch.Generator().manual_seed(seed)
    S, Cc = cfg.image_size, cfg.channels
    if repeat_period:
        base = torch.randint(0, 256, (repeat_period, S, S, Cc), dtype=torch.uint8, generator=g)
        reps = -(-n // repeat_period)
        return base.repeat(reps, 1, 1, 1)[:n].contiguous()
    return torch.randint(0, 256, (n, S, S, Cc), dtype=torch.uint8, generator=g)


def unit_order(n: int, world: int) -> np.ndarray:
    """Owner rank of each unit under shard_ranges (for tests/inspection)."""
    owner = np.empty(n, dtype=np.int64)
    for k, (f, c) in enumerate(shard_ranges(n, world)):
        owner[f:f + c] = k
    return owner
