"""EPDRuntime end to end (runtime.py), world 1 or torchrun world 2/3 on one GPU.

Scenarios (every rank passes the same requests; rank 0 checks):
  plain   -- ample MM pools: every request's MM tokens, as the prefill read them from its
             P-side blocks, equal a direct encode bit for bit, its first token equals a direct
             prefill, the batches follow form_batch / plan_batch (restart at worker 0), every
             block is returned and the measured records satisfy the reference's causality rules;
  pwait   -- a prefill-side pool of 6 tiles: requests that do not fit wait in ep_wait (FIFO)
             while encoding continues; outputs stay exact;
  ewait   -- an encode-side pool of 6 tiles: batches stop at the first misfit (form_batch);
  inst_rr / inst_ll -- every rank its own encode instance (IRP width 1): requests assigned
             round robin / least loaded by outstanding tiles (assign_instance, engine.py:65-78).

usage: python tools/runtime_check.py [scenario]            (world 1)
       torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P tools/runtime_check.py [scenario]
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

TILES = [3, 1, 4, 0, 2, 5, 1, 2]  # request 3 is text-only (engine.py:589-590)


def main() -> None:
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("RUNTIME_CHECK_TIMEOUT", "200")), exit=True)
    from paper_2501_05460_b200.configs import SIGLIP_MINICPM
    from paper_2501_05460_b200.encoder import VisionEncoder
    from paper_2501_05460_b200.prefill import QWEN2_7B, LLMConfig, Prefiller
    from paper_2501_05460_b200.routing import shard_ranges
    from paper_2501_05460_b200.runtime import EPDRuntime, ServeRequest, check_causality
    from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request
    scenario = sys.argv[1] if len(sys.argv) > 1 else "plain"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = SIGLIP_MINICPM.with_layers(2)
    enc = VisionEncoder(cfg, dev, max_tiles=16)
    stage = EncodeStage(enc, dev, rank=rank, world=world)
    lcfg = LLMConfig("test-llm", 2, QWEN2_7B.hidden, 28, 4, 128, 1024, 1000, 1e6, 1e-6, True)
    pf = Prefiller(lcfg, dev, max_tokens=max(TILES) * cfg.out_tokens + 16) if rank == 0 else None
    T = cfg.out_tokens
    kw = {"plain": {}, "pwait": {"p_mm_tokens": 6 * T}, "ewait": {"e_mm_tokens": 6 * T},
          "inst_rr": {"instances": world, "policy": "round_robin"},
          "inst_ll": {"instances": world, "policy": "least_loaded"}}[scenario]
    rt = EPDRuntime(stage, pf, max_batch=3, **kw)
    rt.keep_mm = True
    reqs = []
    for i, n in enumerate(TILES):
        g = torch.Generator().manual_seed(500 + i)
        prompt = torch.randint(0, lcfg.vocab, (12,), dtype=torch.int32, generator=g).to(dev)
        reqs.append(ServeRequest(i, tiles_for_request(n, cfg, seed=900 + i).pin_memory(), prompt))
    out = rt.serve(reqs)
    out2 = rt.serve(reqs)  # a second burst reuses the freed blocks
    errs = []
    if rank == 0:
        for res in (out, out2):
            for r in reqs:
                rec = res["records"][r.rid]
                direct = enc.encode(r.tiles.to(dev))
                tok = pf.prefill(direct.view(-1, cfg.out_dim), r.prompt).clone()
                torch.cuda.synchronize()
                if not torch.equal(res["mm"][r.rid], direct):
                    errs.append(f"request {r.rid}: MM tokens in the P-side blocks differ from a direct encode")
                if rec.first_token != int(tok.item()):
                    errs.append(f"request {r.rid}: first token {rec.first_token} vs direct {int(tok.item())}")
                want = [(k, c) for k, (_, c) in enumerate(shard_ranges(r.tiles.shape[0], rt.width)) if c] or [(0, 0)]
                if [(s.worker, s.patches) for s in rec.shards] != want:
                    errs.append(f"request {r.rid}: shards {rec.shards} vs {want}")
                try:
                    check_causality(rec)
                except ValueError as e:
                    errs.append(str(e))
        if rt.p.manager.used_blocks or any(m.used_blocks for m in rt.e_mms):
            errs.append("MM blocks leaked")
        if scenario.startswith("inst"):
            from paper_2501_05460_b200.routing import assign_instance
            load, rr, want_inst = [0] * world, 0, []
            for r in reqs:
                iid, rr = assign_instance(kw["policy"], [(i, float(load[i])) for i in range(world)], rr)
                want_inst.append(iid)
                load[iid] += r.tiles.shape[0]
            got_inst = [out["records"][r.rid].e_instance for r in reqs]
            print(f"instances: {got_inst}", flush=True)
            if got_inst != want_inst or len(set(got_inst)) != world:
                errs.append(f"{scenario}: instances {got_inst}, expected {want_inst}")
        waited = out["ep_wait"]
        if scenario == "pwait":
            # P pool of 6 tiles, batches of 3 (tiles 3 1 4 | 0 2 5 | 1 2): r2 waits (3+1+4 > 6);
            # round 2 sends r2 first, then text-only r3 reserves 0 blocks, r4 fits and r5 waits
            # (each tries on its own, engine.py:381-383); round 3 sends r5, r6 fits, r7 waits
            # (engine.py:680-685)
            if waited != [2, 5, 7]:
                errs.append(f"pwait: ep_wait history {waited}, expected [2, 5, 7]")
        elif waited:
            errs.append(f"{scenario}: unexpected ep_wait {waited}")
        encs = sorted({round(r.encode_start, 9) for r in out["records"].values()})
        print(f"batches (distinct encode starts): {len(encs)}; ep_wait: {waited}", flush=True)
        if scenario == "ewait" and len(encs) < 4:
            errs.append("ewait: the E-side pool must split the burst into more batches")
    flag = torch.tensor([len(errs)])
    if world > 1:
        dist.all_reduce(flag)
    for e in errs:
        print(f"[rank {rank}] {e}", flush=True)
    rt.close()
    if rank == 0:
        print(f"runtime_check world={world} {scenario}: {'OK' if int(flag) == 0 else f'{int(flag)} BAD'}", flush=True)
    if world > 1:
        dist.destroy_process_group()
    sys.exit(0 if int(flag) == 0 else 1)


if __name__ == "__main__":
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    main()
