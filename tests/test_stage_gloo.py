"""Multi-process CPU tier (gloo, world_size 2 and 3) for the IRP encode stage: tile
routing, the EP gather to the prefill rank in request order, and the byte
accounting -- with a deterministic stand-in encoder (the real one needs the B200;
its numerics are covered by tests/test_encoder_gpu.py)."""
import os
import socket
from dataclasses import dataclass

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_05460_b200.routing import shard_ranges


@dataclass(frozen=True)
class _Cfg:
    image_size: int = 8
    channels: int = 3
    out_tokens: int = 4
    out_dim: int = 8


class _StandInEncoder:
    """tokens[i, t, d] = mean(tile_i) + t + d/10 + rank*0 (rank-independent, tile-determined)."""

    cfg = _Cfg()

    def __init__(self):
        self.calls = []

    def encode(self, tiles, out):
        self.calls.append(tiles.shape[0])
        m = tiles.float().mean(dim=(1, 2, 3))
        t = torch.arange(4).view(1, 4, 1).float()
        d = torch.arange(8).view(1, 1, 8).float() / 10
        out.copy_((m.view(-1, 1, 1) + t + d).to(out.dtype))
        return out


def _expected(tiles):
    enc = _StandInEncoder()
    out = torch.empty(tiles.shape[0], 4, 8, dtype=torch.bfloat16)
    return enc.encode(tiles, out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_05460_b200.stage import EncodeStage
        g = torch.Generator().manual_seed(n)
        tiles = torch.randint(0, 256, (n, 8, 8, 3), dtype=torch.uint8, generator=g)
        enc = _StandInEncoder()
        st = EncodeStage(enc, torch.device("cpu"), rank=rank, world=world, prefill_rank=0)
        # the peer-memory transport needs CUDA IPC: a CPU stage keeps the collective path
        assert not st.enable_peer_gather(16) and st.transport == "nccl-p2p"
        res = st.process(tiles, rid=7)
        first, count = shard_ranges(n, world)[rank]
        out = {"rank": rank, "encoded": res.encoded_tiles, "calls": enc.calls[:],
               "shards": [(s.worker, s.patches) for s in res.shards], "ep_bytes": res.ep_bytes}
        # the exchange on its own (bench.py gather_bench): a pre-encoded shard -> packed buffer
        local = _expected(tiles[first:first + count]) if count else None
        gathered = st.gather_only(local, n)
        if rank == 0:
            # numpy arrays pickle by value (torch tensors would travel as shared-memory fds
            # that the parent can only open while this process is still alive)
            out["tokens"] = res.tokens.float().numpy()
            out["expected"] = _expected(tiles).float().numpy()
            out["gathered"] = gathered.float().numpy()
        q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 10), (3, 10), (2, 1), (3, 13)])
def test_irp_gather_request_order(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o["rank"])
    ranges = shard_ranges(n, world)
    for o in outs:
        assert o["encoded"] == ranges[o["rank"]][1]
        assert sum(o["calls"]) == ranges[o["rank"]][1]
        assert o["shards"] == [(k, c) for k, (_, c) in enumerate(ranges) if c > 0]
    # EP bytes: every non-prefill shard, tokens_per_tile * hidden * 2 bytes per tile (engine.py:524)
    assert outs[0]["ep_bytes"] == sum(c for k, (_, c) in enumerate(ranges) if k != 0) * 4 * 8 * 2
    assert (outs[0]["tokens"] == outs[0]["expected"]).all()
    assert (outs[0]["gathered"] == outs[0]["expected"]).all()


class _GlooComm:
    """Stand-in for comm.NcclComm.gather_tokens over gloo (the C ABI's epd_gather_tokens
    contract: rank k's shard of epd_irp_ranges(n, world) lands on the root at its offset)."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def gather_tokens(self, shard, n_tiles, packed, root=0):
        ranges = shard_ranges(n_tiles, self.world)
        if self.rank == root:
            for k, (first, count) in enumerate(ranges):
                if count and k != root:
                    buf = torch.empty_like(packed[first:first + count])
                    dist.recv(buf, k)
                    packed[first:first + count] = buf
        elif ranges[self.rank][1]:
            dist.send(shard.contiguous(), root)


def _batch_worker(rank, world, port, ns, use_comm, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_05460_b200.stage import EncodeStage
        batch = [torch.randint(0, 256, (n, 8, 8, 3), dtype=torch.uint8, generator=torch.Generator().manual_seed(i))
                 for i, n in enumerate(ns)]
        enc = _StandInEncoder()
        st = EncodeStage(enc, torch.device("cpu"), rank=rank, world=world, prefill_rank=0,
                         comm=_GlooComm(rank, world) if use_comm else None)
        res = st.process_batch(tiles_host=batch)
        mine = sum(shard_ranges(n, world)[rank][1] for n in ns)
        out = {"rank": rank, "calls": enc.calls[:], "mine": mine, "encoded": res.encoded_tiles}
        if rank == 0:
            out["tokens"] = res.tokens.float().numpy()
            out["expected"] = torch.cat([_expected(t) for t in batch]).float().numpy()
        q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,ns,use_comm", [(2, (10, 10), False), (3, (10, 13, 1), False), (3, (10, 10, 10), True),
                                               (2, (1, 5), True), (3, (4, 0, 2), False), (2, (0, 3, 0), True)])
def test_process_batch_gloo(world, ns, use_comm):
    """EncodeStage.process_batch: every request IRP-sharded over all ranks from worker 0, one
    encoder call per rank for all its shards, the batch packed request after request on the
    prefill rank -- torch P2P and the C-ABI gather contract (per request)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, ns, use_comm, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in range(world)], key=lambda o: o["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for o in outs:
        assert o["encoded"] == o["mine"]
        assert o["calls"] == ([o["mine"]] if o["mine"] else [])  # one encoder call per rank
    assert (outs[0]["tokens"] == outs[0]["expected"]).all()
