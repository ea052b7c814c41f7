"""Generate golden vectors by running the reference itself (disaggsim).

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json. Every vector is an output of the
reference's own functions (/root/reference/pkg/src/disaggsim), so the CPU
oracle and the product's host logic are pinned to the reference, not to a
restatement of it.
"""
from __future__ import annotations

import json
import random
import sys
from dataclasses import replace
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "reference_golden.json"


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    from disaggsim.blocks import BlockManager, CacheKind
    from disaggsim.costs import CostParams, transfer_latency, Channel
    from disaggsim.engine import assign_instance, form_batch, irp_shard, run_simulation
    from disaggsim.simconfig import SchedulePolicy
    from disaggsim.metrics import _percentile, ttft
    from disaggsim.models import (HardwareSpec, ModelSpec, StageRole, builtin_catalog, kv_bytes_per_token,
                                  mm_bytes_per_token, tokens_for_request)
    from disaggsim.simconfig import InstanceConfig, SystemConfig
    from disaggsim.workload import Request, Slo

    g: dict = {"source": "disaggsim @ /root/reference/pkg/src (imported, unmodified)"}

    # --- irp_shard (engine.py:55-62)
    shard = []
    for p in list(range(0, 41)) + [100, 200, 400, 401]:
        for w in range(1, 17):
            shard.append([p, w, irp_shard(p, w)])
    g["irp_shard"] = shard
    errs = []
    for p, w in [(10, 0), (-1, 4), (5, -3)]:
        try:
            irp_shard(p, w)
            errs.append([p, w, None])
        except ValueError:
            errs.append([p, w, "ValueError"])
    g["irp_shard_errors"] = errs

    # --- assign_instance (engine.py:65-78) and form_batch (engine.py:81-93)
    rng0 = random.Random(65)
    assign = []
    for _ in range(300):
        cands = [[i, rng0.choice([0.0, 1.0, 2.0, round(rng0.random(), 6)])]
                 for i in sorted(rng0.sample(range(10), rng0.randint(1, 6)))]
        ctr = rng0.randrange(0, 20)
        for pol in SchedulePolicy:
            assign.append([pol.value, cands, ctr, list(assign_instance(pol, [tuple(c) for c in cands], ctr))])
    g["assign_instance"] = assign
    batches = []
    for _ in range(100):
        q = list(range(rng0.randint(0, 8)))
        fit = {i: rng0.random() < 0.8 for i in q}
        mb = rng0.randint(1, 5)
        batches.append([q, mb, [fit[i] for i in q], form_batch(q, mb, lambda i: fit[i])])
    g["form_batch"] = batches

    # --- BlockManager op sequences (blocks.py:14-61)
    rng = random.Random(20260808)
    seqs = []
    for trial in range(12):
        block_size = rng.choice([1, 4, 16])
        total = rng.choice([0, 3, 10, 64, 3000])
        m = BlockManager(CacheKind.MM, block_size, total)
        ops, live = [], []
        for step in range(60):
            r = rng.random()
            if r < 0.55 or not live:
                rid = rng.randrange(0, 40)
                tokens = rng.choice([0, 1, 15, 16, 17, 33, 64, 640, 1302, rng.randrange(0, 200)])
                try:
                    ids = m.allocate(rid, tokens)
                    live.append(rid)
                    ops.append(["alloc", rid, tokens, ids, m.free_blocks, m.used_blocks])
                except RuntimeError:
                    ops.append(["alloc", rid, tokens, "RuntimeError", m.free_blocks, m.used_blocks])
            elif r < 0.9:
                rid = rng.choice(live)
                live.remove(rid)
                m.free(rid)
                ops.append(["free", rid, None, None, m.free_blocks, m.used_blocks])
            else:
                rid = rng.randrange(40, 50)
                try:
                    m.free(rid)
                    ops.append(["free", rid, None, None, m.free_blocks, m.used_blocks])
                except RuntimeError:
                    ops.append(["free", rid, None, "RuntimeError", m.free_blocks, m.used_blocks])
            tokens = rng.randrange(0, 300)
            ops.append(["can", None, tokens, m.can_allocate(tokens), m.blocks_needed(tokens), None])
        seqs.append({"block_size": block_size, "total": total, "ops": ops})
    g["block_manager"] = seqs

    # --- geometry (models.py:128-155, models.cfg)
    cat = builtin_catalog()
    geo = {}
    for name, model in cat.items():
        entry = {"kv_bytes_per_token": kv_bytes_per_token(model), "mm_bytes_per_token": mm_bytes_per_token(model),
                 "tokens_per_patch": model.tokens_per_patch, "hidden_dim": model.hidden_dim,
                 "patch_table": [[list(k), v] for k, v in sorted(model.patch_table.items())], "requests": []}
        for images in [[], [(4032, 3024)], [(4032, 3024)] * 2, [(313, 234), (787, 444)], [(4032, 3024)] * 40]:
            req = Request(id=0, arrival_time=0.0, prompt_tokens=22, images=tuple(images), output_tokens=8,
                          slo=Slo(1.0, 1.0))
            entry["requests"].append([[list(i) for i in images], 22, list(tokens_for_request(model, req))])
        geo[name] = entry
    g["geometry"] = geo

    # --- transfer byte counts / latency (costs.py:113-119; test_costs.py:96-101 style)
    hw = HardwareSpec(gpu_memory=80e9, intra_node_bandwidth=100e9, inter_node_bandwidth=25e9, num_gpus=8)
    g["transfer"] = [[nb, transfer_latency(nb, Channel.INTRA, hw)] for nb in [0, 1302 * 131072, 458752, 405.5e6]]

    # --- engine shard plans and EP/PD byte counts from full simulations
    toy = ModelSpec(name="toy", encoder_params=1_000_000, llm_params=4_000_000, num_layers=2, kv_heads=2,
                    head_dim=4, hidden_dim=8, tokens_per_patch=4, max_context_tokens=10_000,
                    patch_table={(100, 100): 6, (200, 200): 12, (64, 64): 4}, bytes_per_param=2)
    cost = CostParams(enc_base=0.2, enc_per_patch=0.1, prefill_base=0.1, prefill_per_token=0.01,
                      prefill_quad=1e-5, decode_base=0.05, decode_per_seq=0.01, decode_per_kv_token=0.0,
                      transfer_setup=0.0)
    sims = []
    for width in (1, 2, 3, 4, 8):
        for max_batch in (1, 3):
            hw2 = HardwareSpec(gpu_memory=1e9, intra_node_bandwidth=1e8, inter_node_bandwidth=5e7, num_gpus=16)
            cfg = SystemConfig(instances=(InstanceConfig(role=StageRole.ENCODE, tp=width, max_batch=max_batch),
                                          InstanceConfig(role=StageRole.PREFILL, max_batch=4),
                                          InstanceConfig(role=StageRole.DECODE, max_batch=8)),
                               hardware=hw2, model=toy, cost=cost)
            rng2 = random.Random(width * 10 + max_batch)
            reqs = []
            t = 0.0
            for rid in range(12):
                t += rng2.random() * 0.3
                k = rng2.choice([0, 1, 1, 2, 3])
                images = tuple(rng2.choice([(100, 100), (200, 200), (64, 64)]) for _ in range(k))
                reqs.append(Request(id=rid, arrival_time=t, prompt_tokens=rng2.randrange(1, 40), images=images,
                                    output_tokens=rng2.randrange(1, 6), slo=Slo(100.0, 10.0)))
            trace = run_simulation(cfg, reqs, seed=0)
            trace.validate()
            out = []
            for rid in sorted(trace.requests):
                rec = trace.requests[rid]
                out.append({"rid": rid, "images": [list(i) for i in reqs[rid].images],
                            "prompt": reqs[rid].prompt_tokens, "mm_tokens": rec.mm_tokens,
                            "total_tokens": rec.total_tokens,
                            "shards": [[s.worker, s.patches] for s in rec.shards],
                            "encode_start": rec.encode_start, "encode_end": rec.encode_end,
                            "ep_transfer_end": rec.ep_transfer_end, "first_token": rec.first_token_time,
                            "pd_transfer_end": rec.pd_transfer_end,
                            "ttft": ttft(trace, rid) if rec.completed else None})
            # batches: group requests by identical encode_start (one encode batch)
            sims.append({"width": width, "max_batch": max_batch, "requests": out})
    g["simulations"] = sims

    # --- PR1 oracle config: toy model, 1 request x 4 tiles (64x64 -> 4), 1E-1P-1D
    hw3 = HardwareSpec(gpu_memory=1e9, intra_node_bandwidth=1e8, inter_node_bandwidth=5e7, num_gpus=8)
    cfg3 = SystemConfig(instances=(InstanceConfig(role=StageRole.ENCODE), InstanceConfig(role=StageRole.PREFILL),
                                   InstanceConfig(role=StageRole.DECODE, max_batch=4)),
                        hardware=hw3, model=replace(toy, patch_table={(64, 64): 4}), cost=cost)
    tr = run_simulation(cfg3, [Request(id=0, arrival_time=0.0, prompt_tokens=10, images=((64, 64),),
                                       output_tokens=4, slo=Slo(100.0, 10.0))])
    rec = tr.requests[0]
    g["pr1"] = {"mm_tokens": rec.mm_tokens, "total_tokens": rec.total_tokens,
                "shards": [[s.worker, s.patches] for s in rec.shards], "encode_end": rec.encode_end,
                "ep_transfer_end": rec.ep_transfer_end, "first_token": rec.first_token_time,
                "pd_transfer_end": rec.pd_transfer_end, "completion": rec.completion_time}

    # --- percentile (metrics.py:103-108)
    pct = []
    rng4 = random.Random(7)
    for n in [0, 1, 2, 3, 4, 5, 10, 50, 99, 100, 101]:
        vals = [round(rng4.random() * 10, 6) for _ in range(n)]
        for q in (0.0, 0.25, 0.5, 0.9, 0.99, 1.0):
            pct.append([vals, q, _percentile(vals, q)])
    g["percentile"] = pct

    OUT.write_text(json.dumps(g, indent=None, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
