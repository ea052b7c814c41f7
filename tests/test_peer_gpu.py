"""EP gather over peer memory (peer.py, csrc/peer.cu) on one B200, loopback: every "rank"
is an object in this process with its own CUDA stream, so the remote pointers are local
ones and no IPC mapping is involved (the multi-process IPC exchange runs in bench.py at
N > 1). What is checked here is the transport itself -- the 16 B put kernel, the release
/ data flags, the stream-memop waits and the slot reuse protocol -- and that the packed
buffer equals the NCCL path's (request order, bit-exact). No kernel spins: every wait is a
cuStreamWaitValue32 on the waiting object's own memory.

In one process, streams can share a hardware work queue, so a stream-memop wait can block
an unrelated stream queued behind it. Across processes (the deployment: one process per
GPU) a wait is only ever satisfied by another process; here every wait is enqueued after
the work that satisfies it, so the tests cannot deadlock on a shared queue."""
import threading

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(120, method="thread")]


def _loopback(world, slot_bytes, device):
    """One PeerGather per rank, constructed concurrently (the exchange is a rendezvous)."""
    from paper_2501_05460_b200.peer import PeerGather
    recs = [None] * world
    bar = threading.Barrier(world)
    out = [None] * world
    errs = []

    def make(rank):
        def exchange(rec):
            recs[rank] = rec
            bar.wait()
            return list(recs)
        try:
            out[rank] = PeerGather(device, rank, world, 0, slot_bytes, exchange)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            bar.abort()

    ts = [threading.Thread(target=make, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out


def test_peer_put_protocol_loopback(cuda):
    from paper_2501_05460_b200.routing import shard_ranges
    world, tokens, hidden = 3, 4, 64
    peers = _loopback(world, 16 * tokens * hidden * 2, cuda)
    streams = [torch.cuda.Stream(cuda) for _ in range(world)]
    g = torch.Generator(device=cuda).manual_seed(5)
    for req, n in enumerate([10, 7, 3, 16, 1, 12]):
        ranges = shard_ranges(n, world)
        data = torch.randn(n, tokens, hidden, device=cuda, generator=g).to(torch.bfloat16)
        torch.cuda.synchronize()
        seqs = [p.begin() for p in peers]
        assert len(set(seqs)) == 1
        seq = seqs[0]
        sink = peers[0]
        with torch.cuda.stream(streams[0]):
            packed, _ = sink.packed(seq, n, tokens, hidden, streams[0])
            f0, c0 = ranges[0]
            packed[f0:f0 + c0].copy_(data[f0:f0 + c0])  # the sink's own shard, in place
        for k in range(1, world):
            first, count = ranges[k]
            if count:
                with torch.cuda.stream(streams[k]):
                    local = data[first:first + count].clone()
                    peers[k].put(seq, local, first, streams[k])
        with torch.cuda.stream(streams[0]):
            sink.wait(seq, ranges, streams[0])
            got = packed.clone()
        torch.cuda.synchronize()
        assert torch.equal(got, data), (req, n)
    for p in peers:
        p.close()


def test_peer_slot_reuse_after_release(cuda):
    """Slot reuse: request 3 lands in request 1's slot only after the sink released it.
    The sink's stream is held back (~25 ms) before the release and reads the slot there:
    it still holds request 1's shard; after the release, request 3's."""
    world, tokens, hidden = 2, 4, 64
    peers = _loopback(world, 4 * tokens * hidden * 2, cuda)
    s0, s1 = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    n, ranges = 2, [(0, 1), (1, 1)]
    views, vals = {}, {}
    early = None
    for r in range(1, 4):  # request 1 -> slot 1, 2 -> slot 0, 3 -> slot 1 again
        seq = peers[0].begin()
        assert peers[1].begin() == seq
        with torch.cuda.stream(s0):
            if r == 3:
                torch.cuda._sleep(50_000_000)
                early = views[1][1].clone()  # slot 1 before request 3 is released into it
            packed, _ = peers[0].packed(seq, n, tokens, hidden, s0)  # release (enqueued first)
            views[r] = packed
        with torch.cuda.stream(s1):
            local = torch.full((1, tokens, hidden), float(10 * r), device=cuda, dtype=torch.bfloat16)
            peers[1].put(seq, local, 1, s1)
        with torch.cuda.stream(s0):
            packed[0].fill_(float(r))
            peers[0].wait(seq, ranges, s0)
            vals[r] = packed.clone()
    torch.cuda.synchronize()
    assert torch.all(early == 10.0)
    for r in range(1, 4):
        assert torch.all(vals[r][0] == float(r)) and torch.all(vals[r][1] == float(10 * r)), r
    for p in peers:
        p.close()


def test_stage_peer_gather_equals_direct_encode(cuda):
    """EncodeStage with the peer transport (3 loopback ranks, one encoder each): the
    prefill rank's packed tokens equal encoding every tile directly, bit for bit, across
    several requests (slot reuse)."""
    from paper_2501_05460_b200.configs import SEED, TINY_VIT
    from paper_2501_05460_b200.encoder import VisionEncoder
    from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request
    cfg, world = TINY_VIT, 3
    encs = [VisionEncoder(cfg, cuda, max_tiles=8) for _ in range(world)]  # same seeded weights
    peers = _loopback(world, 16 * cfg.out_tokens * cfg.out_dim * 2, cuda)
    stages = []
    for r in range(world):
        st = EncodeStage(encs[r], cuda, rank=r, world=world, prefill_rank=0)
        st._peer, st._peer_tiles = peers[r], 16
        stages.append(st)
    assert stages[0].transport == "nvlink-peer"
    # the prefill rank's wait is deferred until the encode ranks' puts are enqueued
    deferred = []
    real_wait = peers[0].wait
    peers[0].wait = lambda seq, ranges, stream: deferred.append((seq, ranges, stream))
    streams = [torch.cuda.Stream(cuda) for _ in range(world)]
    for req, n in enumerate([7, 4, 10, 2]):
        tiles = tiles_for_request(n, cfg, seed=SEED + req).to(cuda)
        direct = encs[0].encode(tiles)
        torch.cuda.synchronize()
        results = [None] * world
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                results[r] = stages[r].process(None, tiles_dev=tiles)
        seq, ranges, stream = deferred.pop()
        real_wait(seq, ranges, stream)
        with torch.cuda.stream(stream):
            got = results[0].tokens.clone()
        torch.cuda.synchronize()
        assert torch.equal(got, direct), (req, n)
        assert results[1].tokens is None
    for st in stages:
        st.close()


def _ipc_worker(rank, port, q):
    import os

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2501_05460_b200.peer import PeerGather
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)

        def exchange(rec):
            out = [None, None]
            dist.all_gather_object(out, rec)
            return out
        peer = PeerGather(dev, rank, 2, 0, 4 * 4 * 64 * 2, exchange)
        s = torch.cuda.current_stream(dev)
        seq = peer.begin()
        data = torch.arange(3 * 4 * 64, device=dev, dtype=torch.float32).view(3, 4, 64).to(torch.bfloat16)
        # every device-side wait below is already satisfied when it is enqueued (host barriers
        # order the two processes), so nothing on the GPU waits on the other process
        if rank == 0:
            packed, _ = peer.packed(seq, 3, 4, 64, s)  # release -> the producer's flag over IPC
            packed[0].copy_(data[0])
            torch.cuda.synchronize()
        dist.barrier()
        if rank == 1:
            peer.put(seq, data[1:3].contiguous(), 1, s)  # stores into rank 0's slot over IPC
            torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            peer.wait(seq, [(0, 1), (1, 2)], s)
            q.put(("ok", torch.equal(packed.cpu(), data.cpu())))
        else:
            q.put(("ok", True))
        dist.barrier()
        peer.close()
    except Exception as e:  # surfaced to the parent
        q.put(("err", f"rank {rank}: {type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


def test_peer_ipc_two_processes(cuda):
    """The IPC half of the transport: two processes on this GPU exchange handles
    (all_gather_object), map each other's buffers and move a shard plus both flags."""
    import socket

    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=100) for _ in range(2)]
    for p in procs:
        p.join(timeout=30)
    assert all(o == ("ok", True) for o in outs), outs


def test_peer_setup_failure_is_reported_on_every_rank(cuda):
    """A rank whose allocation fails still takes part in the one exchange, so every rank
    raises the same error instead of a peer waiting forever in the collective."""
    from paper_2501_05460_b200.peer import PeerGather
    world = 2
    recs = [None] * world
    bar = threading.Barrier(world)
    errs = [None] * world

    def make(rank):
        def exchange(rec):
            recs[rank] = rec
            bar.wait()
            return list(recs)
        try:
            # the prefill rank (0) asks for an impossible slot; rank 1's setup succeeds
            PeerGather(cuda, rank, world, 0, (1 << 50) if rank == 0 else 1024, exchange)
        except Exception as e:
            errs[rank] = e

    ts = [threading.Thread(target=make, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(isinstance(e, RuntimeError) and "rank 0" in str(e) for e in errs), errs
