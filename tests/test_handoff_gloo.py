"""Multi-process CPU tier (gloo, world 2) for the prefill -> decode KV handoff protocol
(handoff.KVHandoff): reservation handshake, pd_wait deferral and head-of-line retry,
reference block ids and frees on both ranks, a mismatched block count raising on both ranks
(no hang), and the moved KV bit for bit -- the scenario of
tools/kv_handoff_check.py with a stand-in byte transport over gloo (the GPU transports run
in tests/test_kv_handoff_multiprocess_gpu.py)."""
import os
import socket
import sys
from pathlib import Path

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))


class _GlooComm:
    """Stand-in for comm.NcclComm's KV legs: pack/unpack with torch indexing, bytes over gloo."""

    def kv_send(self, cache, ids, staging, peer):
        staging.copy_(cache.pool[:, ids.long()].transpose(0, 1))
        dist.send(staging, peer)

    def kv_recv(self, cache, ids, staging, peer):
        dist.recv(staging, peer)
        cache.pool[:, ids.long()] = staging.transpose(0, 1)


def _fill(cache, rid, total, ids):
    g = torch.Generator().manual_seed(rid)
    for b in ids:
        cache.pool[:, b] = torch.randn(cache.segments, cache.block_elems, generator=g).to(torch.bfloat16)


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import kv_handoff_check as k
        from paper_2501_05460_b200.handoff import KVHandoff, PagedKVCache
        cpu = torch.device("cpu")
        src = PagedKVCache(k.LAYERS, k.KV_HEADS, k.HEAD_DIM, k.BLOCK, k.SRC_BLOCKS, cpu) if rank == 0 else None
        dst = PagedKVCache(k.LAYERS, k.KV_HEADS, k.HEAD_DIM, k.BLOCK, k.DST_BLOCKS, cpu) if rank == 1 else None
        h = KVHandoff(rank, 0, 1, src, dst, transport="nccl", comm=_GlooComm())
        errs = k.scenario(h, rank, _fill)
        q.put((rank, errs))
    except Exception as e:  # reported by the parent
        import traceback
        q.put((rank, [f"{type(e).__name__}: {e}\n{traceback.format_exc()}"]))
    finally:
        dist.destroy_process_group()


def test_kv_handoff_protocol_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == [] and res[1] == [], res
