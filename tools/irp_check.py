"""Multi-process check of the IRP encode stage with the peer-memory gather, runnable on ONE
GPU: every rank is a process on the same device, the control plane is gloo, the data path
is the real one (CUDA IPC mappings between the processes, the put kernel, cross-process
stream-memop waits). Only NVLink itself is missing. The prefill rank checks that the packed
tokens of every request equal a direct single-process encode, bit for bit.

No kernel waits on another rank: the only cross-process waits are stream memory operations
(the mechanism CUDA IPC events use between processes on one GPU).

usage: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
           tools/irp_check.py [requests] [tiles] [cache]
With "cache" the prefill rank holds the MM-token cache (cleared per request, tile i + n/2
repeats tile i): misses are sharded over the ranks and land in the peer slot as staging.
With "batch" every step is a batch of `world` requests (EncodeStage.process_batch: each
request sharded over all ranks from worker 0, one encoder call per rank, one exchange); the
packed batch must equal the requests' direct encodes, request after request."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.configs import SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402
from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("IRP_CHECK_TIMEOUT", "150")), exit=True)
    reqs = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    use_cache = len(sys.argv) > 3 and sys.argv[3] == "cache"
    use_batch = len(sys.argv) > 3 and sys.argv[3] == "batch"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = SIGLIP_MINICPM.with_layers(4)
    enc = VisionEncoder(cfg, dev, max_tiles=n)
    cache = None
    if use_cache and rank == 0:
        from paper_2501_05460_b200.mmcache import MMTokenCache
        cache = MMTokenCache(capacity=4 * n, tokens_per_tile=cfg.out_tokens, hidden=cfg.out_dim, device=dev)
    stage = EncodeStage(enc, dev, rank=rank, world=world, prefill_rank=0, cache=cache, cached=use_cache)
    ok = stage.enable_peer_gather(max(n * (world if use_batch else 1), 16))
    assert ok and stage.transport == "nvlink-peer", "peer gather did not come up"
    requests = [tiles_for_request(n, cfg, seed=100 + i, repeat_period=(n // 2 if use_cache else None)).pin_memory()
                for i in range(4)]
    expected = None
    if rank == 0:
        expected = [enc.encode(t.to(dev)).clone() for t in requests]
        torch.cuda.synchronize()
    dist.barrier()
    bad = 0
    outs = []
    if use_batch:
        for i in range(reqs):
            batch = [requests[(i + r) % 4] for r in range(world)]
            res = stage.process_batch(tiles_host=batch)
            if rank == 0:
                want = torch.cat([expected[(i + r) % 4] for r in range(world)])
                if not torch.equal(res.tokens, want):
                    bad += 1
                    print(f"batch {i}: packed tokens differ", flush=True)
        out_host = torch.empty(n * world, cfg.out_tokens, cfg.out_dim, dtype=torch.bfloat16).pin_memory()
        res = stage.process_batch(tiles_host=requests[:world] if world <= 4 else [requests[r % 4] for r in range(world)],
                                  out_host=out_host if rank == 0 else None)
        stage.join()
        torch.cuda.synchronize()
        if rank == 0 and not torch.equal(out_host, torch.cat([expected[r % 4] for r in range(world)]).cpu()):
            bad += 1
            print("batch readback differs", flush=True)
        flag = torch.tensor([bad])
        dist.all_reduce(flag)
        transport = stage.transport
        stage.close()
        if rank == 0:
            print(f"irp_check world={world} tiles={n} batch requests={reqs + 1}: "
                  f"{'OK' if int(flag) == 0 else f'{int(flag)} BAD'} (transport {transport})", flush=True)
        dist.destroy_process_group()
        sys.exit(0 if int(flag) == 0 else 1)
    # pipelined: requests are issued back to back, slots reused every other request
    for i in range(reqs):
        if cache is not None:
            cache.clear()  # every request misses (and repeats within itself)
        res = stage.process(requests[i % 4])
        if rank == 0:
            outs.append((i, res.tokens.clone()))  # clone on the compute stream, before reuse
    torch.cuda.synchronize()
    if rank == 0:
        for i, tok in outs:
            if not torch.equal(tok, expected[i % 4]):
                bad += 1
                diff = (tok.float() - expected[i % 4].float()).abs().max().item()
                print(f"request {i}: packed tokens differ (max {diff:.3e})")
    # and one request at a time, with host readback through the prefill rank's slot
    out_host = torch.empty(n, cfg.out_tokens, cfg.out_dim, dtype=torch.bfloat16).pin_memory()
    for i in range(4):
        if cache is not None:
            cache.clear()
        res = stage.process(requests[i], out_host=out_host if rank == 0 else None)
        stage.join()
        torch.cuda.synchronize()
        if rank == 0 and not torch.equal(out_host, expected[i].cpu()):
            bad += 1
            print(f"readback {i}: differs")
    flag = torch.tensor([bad])
    dist.all_reduce(flag)
    dist.barrier()
    transport = stage.transport
    stage.close()
    if rank == 0:
        print(f"irp_check world={world} tiles={n}{' cache' if use_cache else ''} requests={reqs + 4}: "
              f"{'OK' if int(flag) == 0 else f'{int(flag)} BAD'} (transport {transport})", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(flag) == 0 else 1)


if __name__ == "__main__":
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    main()
