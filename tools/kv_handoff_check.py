"""Prefill -> decode KV handoff across two processes (handoff.KVHandoff), checked against the
reference's block semantics and bit for bit.

Rank 0 is the prefill instance, rank 1 the decode instance. The sequence follows
engine._on_batch_end / _try_reserve_decode / _retry_waits (engine.py:385-407, 542-555,
686-690): a request the decode pool cannot take is parked in pd_wait while a later, smaller
one still goes through; decode completions free blocks and the head of pd_wait retries.
Every id list on both sides equals the same operations on the reference BlockManager
restatement (oracle/routing.py, pinned to blocks.py by the golden tests), the prefill
blocks are freed after each handoff (engine.py:436-439), and the decode pool holds exactly
the prefill's KV. A handoff whose prefill block count does not match its tokens fails on
both ranks instead of hanging.

GPU mode (this file as a script; one GPU is enough): both processes on cuda:0, gloo for the
host control messages, the nvlink-peer transport (CUDA IPC mapping of the decode pool, the
block-move kernel, cross-process stream-memop flags), the prefill KV written by a real
TINY_LLM prefill. CPU mode (tests/test_handoff_gloo.py): the same scenario with a stand-in
transport over gloo.

usage: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/kv_handoff_check.py
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

LAYERS, KV_HEADS, HEAD_DIM, BLOCK = 2, 2, 64, 16
SRC_BLOCKS, DST_BLOCKS = 64, 24
# (rid, total_tokens, output_tokens): decode needs 8, 12, 17, 3 blocks of 24
REQUESTS = [(1, 100, 20), (2, 150, 30), (3, 60, 200), (4, 33, 1)]


def scenario(h, rank: int, fill) -> list[str]:
    """Run the handoff sequence on both ranks (h: KVHandoff); returns failure messages."""
    from oracle.routing import BlockManager as RefBM
    errs: list[str] = []
    ref_src = RefBM(BLOCK, SRC_BLOCKS)
    ref_dst = RefBM(BLOCK, DST_BLOCKS)
    sent = {}  # rid -> expected block contents (prefill rank)

    def expect(cond, msg):
        if not cond:
            errs.append(msg)

    def prefill(rid, total):
        if rank == 0:
            ids = h.src.manager.allocate(rid, total)
            expect(ids == ref_src.allocate(rid, total), f"prefill ids of {rid}")
            fill(h.src, rid, total, ids)
            sent[rid] = h.src.blocks(ids).cpu()

    def after(rid, total, out, info):
        if info is None:
            return
        nb = -(-total // BLOCK)
        if rank == 0:
            ref_src.free(rid)
            expect(rid not in h.src.manager.allocated, f"prefill blocks of {rid} not freed")
            expect(h.src.manager.free_blocks == ref_src.free_blocks, "prefill free count")
            dist.send(sent[rid].contiguous(), 1)
        else:
            ids = ref_dst.allocate(rid, total + out)
            expect(info["dst_blocks"] == ids, f"decode ids of {rid}: {info['dst_blocks']} vs {ids}")
            # contents (before a later request may reuse the blocks): exactly the prefill's KV
            exp = torch.empty(nb, 2 * LAYERS, BLOCK * KV_HEADS * HEAD_DIM, dtype=torch.bfloat16)
            dist.recv(exp, 0)
            have = h.dst.blocks(info["dst_blocks"][:nb]).cpu()
            expect(torch.equal(have, exp), f"decode KV of request {rid} differs from the prefill's")
            expect(exp.abs().sum() > 0, f"request {rid}: empty KV")
        expect(info["pd_bytes"] == total * 2 * LAYERS * KV_HEADS * HEAD_DIM * 2, "pd_bytes")
        expect(info["moved_bytes"] == nb * 2 * LAYERS * BLOCK * KV_HEADS * HEAD_DIM * 2, "moved_bytes")

    results = {}
    for rid, total, out in REQUESTS:
        prefill(rid, total)
        info = h.submit(rid, total, out)
        results[rid] = info
        after(rid, total, out, info)
    expect(results[1] and results[2] and results[4] and results[3] is None,
           f"deferral pattern {[results[r] is None for r in (1, 2, 3, 4)]}")
    expect([w[0] for w in h.pd_wait] == [3], f"pd_wait {list(h.pd_wait)}")

    def complete(rid):  # the decode instance finishes a request (engine.py:418-421)
        if rank == 1:
            h.dst.manager.free(rid)
            ref_dst.free(rid)

    complete(1)
    expect(h.retry_waits() == [], "request 3 must still wait (9 free blocks < 17)")
    complete(2)
    done = h.retry_waits()
    expect(len(done) == 1 and not h.pd_wait, "request 3 must go through after request 2 completes")
    if done:
        after(3, 60, 200, done[0])

    # malformed: the prefill rank holds 3 blocks but announces 100 tokens (7 blocks)
    if rank == 0:
        h.src.manager.allocate(5, 40)
    try:
        h.submit(5, 100, 1)
        errs.append("a mismatched block count must raise")
    except ValueError:
        pass
    if rank == 0:
        h.src.manager.free(5)
    return errs


def _fill_with_prefill(device):
    from paper_2501_05460_b200.prefill import TINY_LLM, Prefiller
    cfg = TINY_LLM
    assert (cfg.layers, cfg.kv_heads, cfg.head_dim) == (LAYERS, KV_HEADS, HEAD_DIM)
    pf = Prefiller(cfg, device, max_tokens=256, use_graphs=False)

    def fill(cache, rid, total, ids):
        g = torch.Generator().manual_seed(1000 + rid)
        text = torch.randint(0, cfg.vocab, (total,), dtype=torch.int32, generator=g).to(device)
        pf.prefill(None, text, kv=cache, block_ids=ids)
    return fill


def main() -> None:
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("KV_CHECK_TIMEOUT", "150")), exit=True)
    from paper_2501_05460_b200.handoff import KVHandoff, PagedKVCache
    transport = sys.argv[1] if len(sys.argv) > 1 else "nvlink-peer"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    assert world == 2
    # nvlink-peer runs both ranks on one GPU (IPC); nccl needs a GPU per rank
    dev = torch.device("cuda", rank if transport == "nccl" else 0)
    torch.cuda.set_device(dev)
    comm = None
    if transport == "nccl":
        from paper_2501_05460_b200.comm import NcclComm
        comm = NcclComm(dev)
    src = PagedKVCache(LAYERS, KV_HEADS, HEAD_DIM, BLOCK, SRC_BLOCKS, dev) if rank == 0 else None
    dst = PagedKVCache(LAYERS, KV_HEADS, HEAD_DIM, BLOCK, DST_BLOCKS, dev, shareable=True) if rank == 1 else None
    h = KVHandoff(rank, 0, 1, src, dst, transport=transport, comm=comm)
    errs = scenario(h, rank, _fill_with_prefill(dev) if rank == 0 else None)
    flag = torch.tensor([len(errs)])
    dist.all_reduce(flag)
    for e in errs:
        print(f"[rank {rank}] {e}", flush=True)
    h.close()
    if dst is not None:
        dst.close()
    if rank == 0:
        print(f"kv_handoff_check transport={transport}: {'OK' if int(flag) == 0 else f'{int(flag)} BAD'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(flag) == 0 else 1)


if __name__ == "__main__":
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    main()
