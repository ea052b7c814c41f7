"""Drop-in check inside the reference itself: the reference simulator's own engine
(disaggsim.engine.run_simulation) runs with the product's host pieces swapped in --
blockpool.BlockManager for blocks.BlockManager (engine.py:18, 155-161), routing.irp_shard
(engine.py:55-62, evaluated by the C ABI), routing.assign_instance (engine.py:65-78) and
routing.form_batch (engine.py:81-93) -- and every trace must be identical to the stock run.

Needs the reference checkout (build container only; skipped where it is absent)."""
import random
import sys
from dataclasses import asdict
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not (REF / "disaggsim").exists(), reason="reference checkout not present")


@pytest.fixture(scope="module")
def ds():
    sys.dont_write_bytecode = True
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import disaggsim.engine as engine
    import disaggsim.models as models
    import disaggsim.simconfig as simconfig
    import disaggsim.costs as costs
    import disaggsim.workload as workload
    return engine, models, simconfig, costs, workload


def _configs(ds):
    engine, models, sc, costs, wl = ds
    toy = models.ModelSpec(name="toy", encoder_params=1_000_000, llm_params=4_000_000, num_layers=2, kv_heads=2,
                           head_dim=4, hidden_dim=8, tokens_per_patch=4, max_context_tokens=10_000,
                           patch_table={(100, 100): 6, (200, 200): 12, (64, 64): 4}, bytes_per_param=2)
    cost = costs.CostParams(enc_base=0.2, enc_per_patch=0.1, prefill_base=0.1, prefill_per_token=0.01,
                            prefill_quad=1e-5, decode_base=0.05, decode_per_seq=0.01, decode_per_kv_token=0.0,
                            transfer_setup=0.0)
    hw = models.HardwareSpec(gpu_memory=1e9, intra_node_bandwidth=1e8, inter_node_bandwidth=5e7, num_gpus=32)
    out = []
    for width, n_e, policy, kv_frac in [(1, 1, "fcfs", None), (4, 1, "fcfs", None), (3, 2, "least_loaded", None),
                                         (2, 3, "round_robin", None), (8, 2, "least_loaded", 0.02)]:
        pol = sc.SchedulePolicy(policy)
        inst = [sc.InstanceConfig(role=models.StageRole.ENCODE, tp=width, max_batch=3, policy=pol)
                for _ in range(n_e)]
        inst += [sc.InstanceConfig(role=models.StageRole.PREFILL, max_batch=4, policy=pol) for _ in range(2)]
        inst += [sc.InstanceConfig(role=models.StageRole.DECODE, max_batch=8, policy=pol) for _ in range(2)]
        kw = {} if kv_frac is None else {"mm_cache_tokens": 64}  # tiny MM pools: ep_wait / deferrals
        cfg = sc.SystemConfig(instances=tuple(inst), hardware=hw, model=toy, cost=cost, **kw)
        rng = random.Random(width * 7 + n_e)
        reqs, t = [], 0.0
        for rid in range(40):
            t += rng.random() * 0.25
            k = rng.choice([0, 1, 1, 2, 3, 4])
            images = tuple(rng.choice([(100, 100), (200, 200), (64, 64)]) for _ in range(k))
            reqs.append(wl.Request(id=rid, arrival_time=t, prompt_tokens=rng.randrange(1, 40), images=images,
                                   output_tokens=rng.randrange(1, 6), slo=wl.Slo(100.0, 10.0)))
        out.append((cfg, reqs))
    return out


def _trace_dict(trace):
    return {rid: asdict(rec) for rid, rec in sorted(trace.requests.items())}


def test_reference_engine_with_product_pieces_is_identical(ds, monkeypatch):
    engine = ds[0]
    from paper_2501_05460_b200 import blockpool, routing
    stock = [_trace_dict(engine.run_simulation(cfg, reqs, seed=0)) for cfg, reqs in _configs(ds)]
    monkeypatch.setattr(engine, "BlockManager", blockpool.BlockManager)
    monkeypatch.setattr(engine, "irp_shard", routing.irp_shard)
    monkeypatch.setattr(engine, "assign_instance", routing.assign_instance)
    monkeypatch.setattr(engine, "form_batch", routing.form_batch)
    swapped = [_trace_dict(engine.run_simulation(cfg, reqs, seed=0)) for cfg, reqs in _configs(ds)]
    assert engine.BlockManager is blockpool.BlockManager
    for a, b in zip(stock, swapped):
        assert a == b
    # the workloads exercise multi-request batches, several E instances and IRP widths
    assert any(len(r["shards"]) > 1 for t in stock for r in t.values())
    assert {r["e_instance"] for t in stock for r in t.values()} >= {0, 1}


def test_assign_instance_matches_reference(ds):
    engine = ds[0]
    from paper_2501_05460_b200.routing import assign_instance
    import disaggsim.simconfig as sc
    rng = random.Random(3)
    for _ in range(500):
        cands = [(i, rng.choice([0.0, 1.0, 2.0, rng.random()])) for i in sorted(rng.sample(range(10), rng.randint(1, 6)))]
        ctr = rng.randrange(0, 20)
        for pol in sc.SchedulePolicy:
            assert assign_instance(pol, cands, ctr) == engine.assign_instance(pol, cands, ctr)
            assert assign_instance(pol.value, cands, ctr) == engine.assign_instance(pol, cands, ctr)
    with pytest.raises(ValueError):
        assign_instance("fcfs", [])


def test_poisson_arrivals_match_reference(ds):
    """routing.poisson_arrivals (the open-loop replay of EPDRuntime / bench c2p) reproduces
    workload.generate_poisson's arrival times exactly (workload.py:71-96)."""
    wl = ds[4]
    from paper_2501_05460_b200.routing import poisson_arrivals
    for rate, n, seed in [(0.125, 100, 20260808), (40.0, 64, 7), (3.0, 5, 0)]:
        import disaggsim.models as models
        spec = wl.WorkloadSpec(rate_lambda=rate, num_requests=n, seed=seed, prompt_tokens=22, output_tokens=8,
                               images_per_request=1, resolution=(4032, 3024))
        ref = [r.arrival_time for r in wl.generate_poisson(spec)]
        assert poisson_arrivals(rate, n, seed) == ref
