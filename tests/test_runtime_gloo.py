"""Multi-process CPU tier (gloo, world 1 and 2) for the serving runtime's control logic
(runtime.EPDRuntime): batches (form_batch with the E-side reservation, IRP shards restarting
at worker 0, one encode call per worker), P-side reservations with the ep_wait FIFO, the
shards' 16-token records landing in the reserved blocks, encode-instance assignment, block
accounting and the records' causality -- with host stand-ins for the encoder, the prefill,
the device MM-pool transport and the GPU clock (the CUDA versions run in
tests/test_runtime_gpu.py)."""
import os
import socket
import time
from dataclasses import dataclass

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

TILES = [3, 1, 4, 0, 2, 5, 1, 2]  # request 3 is text-only (engine.py:589-590)
T, D, BS = 16, 8, 16  # tokens per tile (one 16-token block), token width, block size


@dataclass(frozen=True)
class _Cfg:
    image_size: int = 4
    channels: int = 3
    out_tokens: int = T
    out_dim: int = D


class _Encoder:
    """tokens[i, t, d] = mean(tile_i) + t / 16 + d / 100: tile-determined, rank-independent."""

    cfg = _Cfg()

    def __init__(self):
        self.calls = []

    def encode(self, tiles, out):
        self.calls.append(tiles.shape[0])
        m = tiles.float().mean(dim=(1, 2, 3)).view(-1, 1, 1)
        t = torch.arange(T).view(1, T, 1).float() / 16
        d = torch.arange(D).view(1, 1, D).float() / 100
        out.copy_((m + t + d).to(out.dtype))
        return out


class _Stage:
    def __init__(self, rank, world):
        self.enc, self.cfg = _Encoder(), _Cfg()
        self.rank, self.world, self.device = rank, world, torch.device("cpu")


class _Prefiller:
    """First "token" = a checksum of the MM rows it reads; the rows are kept for checking."""

    def __init__(self):
        self.seen = []

    def prefill(self, mm_tokens, prompt, mm_pool=None, mm_rows=None):
        x = mm_pool[mm_rows.long()].float()
        self.seen.append(x.clone())
        return torch.tensor([int(x.sum().item() * 1000) % 100003], dtype=torch.int32)


class _HostPool:
    """The MM-pool transport over gloo: encode ranks send (ids, records), rank 0 scatters."""

    def __init__(self, rt, nblocks):
        from paper_2501_05460_b200.blockpool import BlockManager, CacheKind
        self.rank = rt.rank
        self.manager = BlockManager(CacheKind.MM, BS, nblocks) if rt.rank == 0 else None
        self.pool = torch.zeros(nblocks * BS, D, dtype=torch.bfloat16) if rt.rank == 0 else None

    def release(self, seq, stream):
        pass

    def put(self, seq, items, stream):
        if self.rank == 0:
            for src, ids in items:
                self.pool.view(-1, BS, D)[ids.long()] = src
        elif items:  # rank 0 waits only for ranks that hold records this round
            n = torch.tensor([len(items)])
            dist.send(n, 0)
            for src, ids in items:
                dist.send(torch.tensor([ids.numel()]), 0)
                dist.send(ids.to(torch.int64), 0)
                dist.send(src.contiguous().view(torch.int16), 0)

    def wait(self, seq, k, stream):
        if k == 0:
            return
        n = torch.zeros(1, dtype=torch.int64)
        dist.recv(n, k)
        for _ in range(int(n)):
            c = torch.zeros(1, dtype=torch.int64)
            dist.recv(c, k)
            ids = torch.zeros(int(c), dtype=torch.int64)
            dist.recv(ids, k)
            rec = torch.zeros(int(c), BS, D, dtype=torch.int16)
            dist.recv(rec, k)
            self.pool.view(-1, BS, D)[ids] = rec.view(torch.bfloat16)

    def close(self):
        pass


class _Stamps:
    def __init__(self):
        self.t, self.n = [], 0

    def mark(self, stream):
        self.t.append(time.perf_counter_ns())
        self.n += 1
        return self.n - 1

    def read(self):
        return list(self.t[:self.n])


def _requests():
    from paper_2501_05460_b200.runtime import ServeRequest
    reqs = []
    for i, n in enumerate(TILES):
        g = torch.Generator().manual_seed(900 + i)
        tiles = torch.randint(0, 256, (n, 4, 4, 3), dtype=torch.uint8, generator=g)
        reqs.append(ServeRequest(i, tiles, torch.arange(3, dtype=torch.int32)))
    return reqs


def _run(rank, world, scenario):
    from paper_2501_05460_b200.routing import shard_ranges
    from paper_2501_05460_b200.runtime import EPDRuntime, check_causality
    kw = {"plain": {}, "pwait": {"p_mm_tokens": 6 * T}, "ewait": {"e_mm_tokens": 6 * T},
          "inst_rr": {"instances": world, "policy": "round_robin"},
          "inst_ll": {"instances": world, "policy": "least_loaded"}, "poisson": {},
          "admit": {"e_mm_tokens": 6 * T, "admission_control": True, "max_context_tokens": 150},
          "admit_raise": {"e_mm_tokens": 6 * T}}[scenario]
    stage, pf = _Stage(rank, world), (_Prefiller() if rank == 0 else None)
    rt = EPDRuntime(stage, pf, max_batch=3, block_size=BS, pool=_HostPool, stamps=_Stamps(), **kw)
    rt.keep_mm = True
    reqs = _requests()
    rejected = {}
    if scenario.startswith("admit"):
        # _admission_reason (engine.py:319-344): 7 tiles never fit a 6-tile encode pool; no
        # tokens at all is "empty"; 12 tiles x 16 + 3 prompt tokens exceed a 150-token context
        from paper_2501_05460_b200.runtime import ServeRequest
        extra = [(100, 7, 3, "mm_capacity"), (101, 0, 0, "empty")]
        if scenario == "admit":
            extra.append((102, 12, 3, "context"))
        for rid, n, np_, why in extra:
            g = torch.Generator().manual_seed(rid)
            tiles = torch.randint(0, 256, (n, 4, 4, 3), dtype=torch.uint8, generator=g)
            reqs.insert(2, ServeRequest(rid, tiles, torch.arange(np_, dtype=torch.int32)))
            rejected[rid] = why
        if scenario == "admit_raise":
            from paper_2501_05460_b200._lib import CapacityExceeded
            try:
                rt.serve(reqs)
            except CapacityExceeded as e:
                return ([] if "can never fit" in str(e) else [f"unexpected message {e}"]), stage.enc.calls
            return ["admission_control=False must raise CapacityExceeded on every rank"], stage.enc.calls
    if scenario == "poisson":  # open loop: generate_poisson arrivals at 150 requests/s
        from paper_2501_05460_b200.routing import poisson_arrivals
        for r, t in zip(reqs, poisson_arrivals(150.0, len(reqs), 3)):
            r.arrival = t
    out = rt.serve(reqs)
    errs = []
    if rank == 0:
        for rid, why in rejected.items():
            if out["records"][rid].rejected != why or out["records"][rid].shards:
                errs.append(f"request {rid}: rejected {out['records'][rid].rejected!r}, expected {why!r}")
        reqs = [r for r in reqs if r.rid not in rejected]
        for r in reqs:
            rec = out["records"][r.rid]
            want = _Encoder().encode(r.tiles, torch.empty(r.tiles.shape[0], T, D, dtype=torch.bfloat16))
            if not torch.equal(out["mm"][r.rid], want):
                errs.append(f"request {r.rid}: MM tokens in the P-side blocks differ")
            exp = [(k, c) for k, (_, c) in enumerate(shard_ranges(r.tiles.shape[0], rt.width)) if c] or [(0, 0)]
            if [(s.worker, s.patches) for s in rec.shards] != exp:
                errs.append(f"request {r.rid}: shards {rec.shards}")
            try:
                check_causality(rec)
            except ValueError as e:
                errs.append(str(e))
        if rt.p.manager.used_blocks or any(m.used_blocks for m in rt.e_mms):
            errs.append("MM blocks leaked")
        # P side holds 6 tiles: batch (0,1,2) -> 2 waits; (3,4,5) -> text-only 3 reserves 0
        # blocks, 5 waits; (6,7) -> 7 waits (_try_reserve_prefill, FIFO retries first)
        if scenario == "pwait" and out["ep_wait"] != [2, 5, 7]:
            errs.append(f"ep_wait history {out['ep_wait']}")
        if scenario != "pwait" and out["ep_wait"]:
            errs.append(f"unexpected ep_wait {out['ep_wait']}")
        if scenario == "poisson":
            for r in reqs:
                rec = out["records"][r.rid]
                if rec.arrival != r.arrival or rec.encode_start < r.arrival:
                    errs.append(f"request {r.rid}: arrival {rec.arrival} / encode start {rec.encode_start}")
        starts = {round(rec.encode_start, 9) for rec in out["records"].values() if rec.rejected is None}
        if scenario == "ewait" and len(starts) < 4 * rt.instances:
            errs.append(f"ewait: {len(starts)} batches")
        if scenario.startswith("inst"):
            from paper_2501_05460_b200.routing import assign_instance
            load, rr, want = [0] * world, 0, []
            for r in reqs:
                iid, rr = assign_instance(kw["policy"], [(i, float(load[i])) for i in range(world)], rr)
                want.append(iid)
                load[iid] += r.tiles.shape[0]
            if [out["records"][r.rid].e_instance for r in reqs] != want:
                errs.append(f"instances {[out['records'][r.rid].e_instance for r in reqs]} vs {want}")
    # every worker encoded its shards of a batch in one call
    return errs, stage.enc.calls


def _worker(rank, world, port, scenario, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(rank, world, scenario)))
    except Exception as e:
        import traceback
        q.put((rank, ([f"{type(e).__name__}: {e}\n{traceback.format_exc()}"], [])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,scenario", [(1, "plain"), (1, "pwait"), (2, "plain"), (2, "pwait"),
                                            (2, "ewait"), (2, "inst_rr"), (2, "inst_ll"), (1, "poisson"),
                                            (2, "poisson"), (2, "admit"), (2, "admit_raise")])
def test_runtime_control_logic_gloo(world, scenario):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, (errs, calls) in res.items():
        assert errs == [], (rank, errs)
        # batches of up to 3 requests: one encoder call per batch this worker has shards in
        assert len(calls) <= len(TILES)
