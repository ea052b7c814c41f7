"""CPU tier: the oracle AND the product's host logic against golden vectors produced
by running the reference itself (tests/golden/make_golden.py). Bit-exact."""
import json
from pathlib import Path

import pytest

import oracle.routing as orr
from paper_2501_05460_b200 import routing
from paper_2501_05460_b200.blockpool import BlockManager, CacheKind
from paper_2501_05460_b200.configs import INTERNVL2_8B, MINICPM_V26, UnknownResolution

G = json.loads((Path(__file__).parent / "golden" / "reference_golden.json").read_text())


@pytest.mark.parametrize("impl", [orr.irp_shard, routing.irp_shard], ids=["oracle", "product"])
def test_irp_shard_table(impl):
    for p, w, expect in G["irp_shard"]:
        assert impl(p, w) == expect, (p, w)


@pytest.mark.parametrize("impl", [orr.irp_shard, routing.irp_shard], ids=["oracle", "product"])
def test_irp_shard_errors(impl):
    for p, w, err in G["irp_shard_errors"]:
        if err is None:
            impl(p, w)
        else:
            with pytest.raises(ValueError):
                impl(p, w)


def test_shard_ranges_contiguous_in_request_order():
    for p, w, expect in G["irp_shard"]:
        rs = routing.shard_ranges(p, w)
        assert rs == orr.shard_ranges(p, w)
        assert [c for _, c in rs] == expect
        assert all(f == sum(expect[:k]) for k, (f, _) in enumerate(rs))


def _run_ops(m, ops):
    for kind, rid, tokens, result, free_after, used_after in ops:
        if kind == "alloc":
            if result == "RuntimeError":
                with pytest.raises(RuntimeError):
                    m.allocate(rid, tokens)
            else:
                assert m.allocate(rid, tokens) == result
        elif kind == "free":
            if result == "RuntimeError":
                with pytest.raises(RuntimeError):
                    m.free(rid)
            else:
                m.free(rid)
        else:  # can
            assert m.can_allocate(tokens) == result
            assert m.blocks_needed(tokens) == free_after
            continue
        assert m.free_blocks == free_after and m.used_blocks == used_after


@pytest.mark.parametrize("impl", ["oracle", "product"])
def test_block_manager_sequences(impl):
    for seq in G["block_manager"]:
        if impl == "oracle":
            m = orr.BlockManager(seq["block_size"], seq["total"])
        else:
            m = BlockManager(CacheKind.MM, seq["block_size"], seq["total"])
        _run_ops(m, seq["ops"])


def test_block_manager_geometry_errors():
    with pytest.raises(ValueError):
        BlockManager(CacheKind.KV, 0, 4)
    with pytest.raises(ValueError):
        BlockManager(CacheKind.KV, 16, -1)


@pytest.mark.parametrize("geo", [MINICPM_V26, INTERNVL2_8B], ids=lambda g: g.name)
def test_geometry_matches_reference_catalog(geo):
    ref = G["geometry"][geo.name]
    assert geo.kv_bytes_per_token() == ref["kv_bytes_per_token"]
    assert geo.mm_bytes_per_token() == ref["mm_bytes_per_token"]
    assert geo.tokens_per_patch == ref["tokens_per_patch"]
    assert sorted([list(k), v] for k, v in geo.patch_table.items()) == ref["patch_table"]
    for images, prompt, expect in ref["requests"]:
        assert list(geo.tokens_for_request([tuple(i) for i in images], prompt)) == expect
        assert list(orr.tokens_for_request(geo.patch_table, geo.tokens_per_patch, images, prompt)) == expect
    with pytest.raises(UnknownResolution):
        geo.tiles_for_image((1, 1))
    with pytest.raises(KeyError):
        geo.tiles_for_image((1, 1))


def test_engine_shard_plans_and_ep_bytes():
    """Shard plans of every encode batch in full reference simulations (multi-request
    batches included) == plan_batch; EP bytes == tiles * tokens_per_patch * mm_bpt."""
    table = {(100, 100): 6, (200, 200): 12, (64, 64): 4}
    checked = 0
    for sim in G["simulations"]:
        batches = {}
        for r in sim["requests"]:
            if r["encode_start"] is None:
                continue
            batches.setdefault(r["encode_start"], []).append(r)
        for start, reqs in sorted(batches.items()):
            reqs.sort(key=lambda r: r["rid"])
            patches = [sum(table[tuple(i)] for i in r["images"]) for r in reqs]
            for impl in (orr.plan_batch, routing.plan_batch):
                shards, load, nreq = impl(patches, sim["width"])
                assert [[list(s) for s in sh] for sh in shards] == [r["shards"] for r in reqs]
                assert sum(load) == sum(patches)
            for r, p in zip(reqs, patches):
                assert sum(s[1] * 4 for s in r["shards"]) == r["mm_tokens"]
                assert sum(routing.ep_bytes(s[1], 4, 16) for s in r["shards"]) == r["mm_tokens"] * 16
            checked += len(reqs)
    assert checked > 50


def test_pr1_config_plan():
    pr1 = G["pr1"]
    shards, _, _ = routing.plan_batch([4], 1)
    assert [list(s) for s in shards[0]] == pr1["shards"]
    assert pr1["mm_tokens"] == 16 and pr1["total_tokens"] == 26
    # EP bytes of the PR1 request (4 tiles x 4 tokens x 16 B) reproduce the reference's transfer time
    assert (pr1["ep_transfer_end"] - pr1["encode_end"]) == pytest.approx(routing.ep_bytes(4, 4, 16) / 1e8, abs=1e-12)
    assert (pr1["pd_transfer_end"] - pr1["first_token"]) == pytest.approx(routing.pd_bytes(26, 64) / 1e8, abs=1e-12)


def test_percentile():
    import bench
    for vals, q, expect in G["percentile"]:
        assert orr.percentile(vals, q) == expect
        assert bench._percentile(vals, q) == expect


def test_assign_instance_and_form_batch_golden():
    """engine.assign_instance / form_batch (engine.py:65-93) outputs recorded from the reference."""
    from paper_2501_05460_b200.routing import assign_instance, form_batch
    g = G
    assert len(g["assign_instance"]) == 900
    for pol, cands, ctr, out in g["assign_instance"]:
        assert list(assign_instance(pol, [tuple(c) for c in cands], ctr)) == out
    for q, mb, fit, out in g["form_batch"]:
        assert form_batch(q, mb, lambda i: fit[i]) == out
