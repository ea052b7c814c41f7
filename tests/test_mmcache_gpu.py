"""MM-token cache and KV handoff on the B200, bit-exact against the CPU oracles:
content keys (K11), hash-table hit/miss/dup classification, entry ids and evictions
(K12), the cached encode path (C4 shape, scaled), and the paged KV pack/unpack (C2)."""
import numpy as np
import pytest
import torch

from oracle.hashing import content_hash
from oracle.mmcache import MMCacheOracle

pytestmark = pytest.mark.gpu


def test_hash_kernel_matches_oracle(cuda):
    from paper_2501_05460_b200.mmcache import hash_tiles
    rng = np.random.default_rng(3)
    for shape in [(5, 448, 448, 3), (3, 56, 56, 3), (4, 8), (2, 64), (7, 4096)]:
        arr = rng.integers(0, 256, shape, dtype=np.uint8)
        if shape == (4, 8):
            arr[:] = 0
        keys = hash_tiles(torch.from_numpy(arr).to(cuda)).cpu().numpy().view(np.uint64)
        for i in range(shape[0]):
            assert tuple(int(k) for k in keys[i]) == content_hash(arr[i]), (shape, i)


def test_cache_sequence_matches_oracle(cuda):
    from paper_2501_05460_b200.mmcache import MMTokenCache
    rng = np.random.default_rng(11)
    pool = rng.integers(0, 256, (30, 8 * 8 * 3), dtype=np.uint8)  # 30 distinct records
    secret = (0x0123456789ABCDEF, 0xFEDCBA9876543210)
    cache = MMTokenCache(capacity=12, tokens_per_tile=4, hidden=8, device=cuda, secret=secret)
    oracle = MMCacheOracle(12)
    for step in range(400):
        n = int(rng.integers(1, 12))
        ids = rng.integers(0, 30 if step > 5 else 10, n)
        tiles = torch.from_numpy(pool[ids]).to(cuda)
        plan = cache.plan(cache.hash(tiles))
        expect = oracle.process([content_hash(pool[i], secret) for i in ids])
        got = list(zip(plan.kinds, [int(e) for e in plan.entries]))
        assert got == expect, step
        assert plan.victims == oracle.last_victims
        assert plan.miss_tiles.tolist() == [i for i, (k, _) in enumerate(expect) if k == "miss"]
        assert len(cache) == len(oracle)
    cache.check()


def test_cache_capacity_exceeded_leaves_state_untouched(cuda):
    """A request with more distinct tiles than entries raises CapacityExceeded (the oracle's
    rule) without touching the cache; the next requests classify as from that state."""
    from paper_2501_05460_b200._lib import CapacityExceeded as DevCapacityExceeded
    from paper_2501_05460_b200.mmcache import MMTokenCache
    from oracle.mmcache import CapacityExceeded
    rng = np.random.default_rng(5)
    pool = rng.integers(0, 256, (6, 8 * 8 * 3), dtype=np.uint8)
    cache = MMTokenCache(capacity=2, tokens_per_tile=4, hidden=8, device=cuda, secret=0)
    oracle = MMCacheOracle(2)
    for ids in ([0], [0, 1, 2], [1, 1, 0], [3, 4, 5], [2, 3], [2, 2, 2, 2]):
        tiles = torch.from_numpy(pool[ids]).to(cuda)
        keys = [content_hash(pool[i], (0, 0)) for i in ids]
        try:
            expect = oracle.process(keys)
        except CapacityExceeded:
            with pytest.raises(DevCapacityExceeded):
                cache.plan(cache.hash(tiles))
            assert len(cache) == len(oracle)
            continue
        plan = cache.plan(cache.hash(tiles))
        assert list(zip(plan.kinds, [int(e) for e in plan.entries])) == expect, ids
        assert plan.victims == oracle.last_victims
    cache.check()


def test_keyed_hash_matches_oracle_and_differs_per_secret(cuda):
    from paper_2501_05460_b200.mmcache import MMTokenCache, hash_tiles
    rng = np.random.default_rng(4)
    arr = rng.integers(0, 256, (3, 448, 448, 3), dtype=np.uint8)
    t = torch.from_numpy(arr).to(cuda)
    for secret in [(1, 2), (2 ** 64 - 1, 12345)]:
        keys = hash_tiles(t, secret=secret).cpu().numpy().view(np.uint64)
        for i in range(3):
            assert tuple(int(k) for k in keys[i]) == content_hash(arr[i], secret)
    a, b = MMTokenCache(4, 4, 8, cuda), MMTokenCache(4, 4, 8, cuda)
    assert a.secret != b.secret  # random per cache: keys cannot be precomputed offline
    assert not torch.equal(a.hash(t), b.hash(t))


def test_cache_churn_keeps_probe_chains_short(cuda):
    """Eviction churn: every request brings new tiles, so every plan evicts; the
    planner rebuilds the table once tombstones pass a quarter of the slots, and plans stay
    exact and fast after thousands of evictions."""
    import time
    from paper_2501_05460_b200.mmcache import MMTokenCache
    rng = np.random.default_rng(5)
    cache = MMTokenCache(capacity=64, tokens_per_tile=4, hidden=8, device=cuda, secret=0)
    oracle = MMCacheOracle(64)
    times = []
    for step in range(600):
        recs = rng.integers(0, 256, (16, 64), dtype=np.uint8)
        recs[:4] = np.frombuffer(np.uint64(step // 3).tobytes() * 8, dtype=np.uint8)  # a few repeats
        t = torch.from_numpy(recs).to(cuda)
        keys = cache.hash(t)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = cache.plan(keys)
        times.append(time.perf_counter() - t0)
        expect = oracle.process([content_hash(r) for r in recs])
        assert list(zip(plan.kinds, [int(e) for e in plan.entries])) == expect, step
    assert cache.stats["evicted"] > 4000
    early, late = sorted(times[20:120])[50], sorted(times[-100:])[50]
    print(f"plan p50: first {early * 1e6:.0f} us, last {late * 1e6:.0f} us")
    assert late < 2 * early + 50e-6
    cache.check()


def test_cached_stage_bit_exact(cuda):
    """C4 shape scaled down: 40 tiles with tile i+20 == tile i. First request: 20 misses
    + 20 in-batch dups; second: 40 hits. Packed tokens == encoding every tile directly."""
    from paper_2501_05460_b200.configs import SEED, TINY_VIT
    from paper_2501_05460_b200.encoder import VisionEncoder
    from paper_2501_05460_b200.mmcache import MMTokenCache
    from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request
    cfg = TINY_VIT
    enc = VisionEncoder(cfg, cuda, max_tiles=16)
    tiles = tiles_for_request(40, cfg, SEED, repeat_period=20)
    direct = enc.encode(tiles.to(cuda))
    cache = MMTokenCache(64, cfg.out_tokens, cfg.out_dim, cuda)
    st = EncodeStage(enc, cuda, cache=cache)
    r1 = st.process(tiles.pin_memory())
    assert r1.cache_counts == {"hit": 0, "miss": 20, "dup": 20} and r1.encoded_tiles == 20
    assert r1.plan.kinds == ["miss"] * 20 + ["dup"] * 20
    r2 = st.process(tiles.pin_memory())
    assert r2.plan.kinds == ["hit"] * 40 and r2.encoded_tiles == 0
    torch.cuda.synchronize()
    assert torch.equal(r1.tokens, direct)
    assert torch.equal(r2.tokens, direct)


@pytest.mark.parametrize("cached", [False, True])
def test_stage_text_only_request(cuda, cached):
    """A request with no images (engine.py:589-590: text-only) encodes nothing, returns an
    empty packed buffer, and leaves the stage (and its cache) usable for the next request."""
    from paper_2501_05460_b200.configs import SEED, TINY_VIT
    from paper_2501_05460_b200.encoder import VisionEncoder
    from paper_2501_05460_b200.mmcache import MMTokenCache
    from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request
    cfg = TINY_VIT
    enc = VisionEncoder(cfg, cuda, max_tiles=8)
    cache = MMTokenCache(16, cfg.out_tokens, cfg.out_dim, cuda) if cached else None
    st = EncodeStage(enc, cuda, cache=cache)
    empty = tiles_for_request(0, cfg, SEED)
    r0 = st.process(empty.pin_memory())
    assert r0.encoded_tiles == 0 and tuple(r0.tokens.shape) == (0, cfg.out_tokens, cfg.out_dim)
    tiles = tiles_for_request(5, cfg, SEED)
    r1 = st.process(tiles.pin_memory())
    r2 = st.process(None, tiles_dev=empty.to(cuda))
    torch.cuda.synchronize()
    assert r2.tokens.shape[0] == 0
    assert torch.equal(r1.tokens, enc.encode(tiles.to(cuda)))
    if cached:
        assert r0.cache_counts == {"hit": 0, "miss": 0, "dup": 0} and len(cache) == 5
        cache.check()


def test_kv_pack_unpack_and_local_handoff(cuda):
    from paper_2501_05460_b200.handoff import PagedKVCache, kv_handoff
    p = PagedKVCache(num_layers=4, kv_heads=2, head_dim=16, block_size=16, num_blocks=40, device=cuda)
    d = PagedKVCache(num_layers=4, kv_heads=2, head_dim=16, block_size=16, num_blocks=50, device=cuda)
    p.pool.copy_(torch.randn_like(p.pool, dtype=torch.float32).to(torch.bfloat16))
    d.manager.allocate(99, 100)  # decode side already busy: ids shift
    total, out_tok = 70, 5
    src_ids = p.manager.allocate(1, total)
    assert src_ids == [0, 1, 2, 3, 4]
    packed = p.pack(src_ids)
    assert torch.equal(packed, p.pool[:, src_ids].permute(1, 0, 2))
    expect = p.pool[:, src_ids].clone()
    info = kv_handoff(1, total, out_tok, p, d, 0, 0, rank=0)
    torch.cuda.synchronize()
    dst = info["dst_blocks"]
    assert len(dst) == d.manager.blocks_needed(total + out_tok)
    assert torch.equal(d.pool[:, dst[:5]], expect)
    assert info["pd_bytes"] == total * p.kv_bytes_per_token
    assert info["moved_bytes"] == 5 * 16 * p.kv_bytes_per_token
    assert 1 not in p.manager.allocated  # prefill side freed after the send (engine.py:437)


def test_cached_stage_bit_exact_siglip_c4_shape(cuda):
    """C4's structure at the real encoder (SigLIP-400M + resampler, 27 layers): 40 tiles, tile
    i + 20 repeating tile i. The cached path (device plan, keyed hash, miss gather, scatter into
    the store, packing) returns exactly the tokens of encoding every tile directly; a second
    request is served from the cache alone."""
    from paper_2501_05460_b200.configs import SEED, SIGLIP_MINICPM
    from paper_2501_05460_b200.encoder import VisionEncoder
    from paper_2501_05460_b200.mmcache import MMTokenCache
    from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request
    cfg = SIGLIP_MINICPM
    enc = VisionEncoder(cfg, cuda, max_tiles=20)
    tiles = tiles_for_request(40, cfg, SEED, repeat_period=20)
    direct = torch.cat([enc.encode(tiles[i:i + 20].to(cuda)) for i in (0, 20)])
    cache = MMTokenCache(64, cfg.out_tokens, cfg.out_dim, cuda)
    st = EncodeStage(enc, cuda, cache=cache)
    r1 = st.process(tiles.pin_memory())
    r2 = st.process(tiles.pin_memory())
    torch.cuda.synchronize()
    assert r1.cache_counts == {"hit": 0, "miss": 20, "dup": 20} and r2.cache_counts["hit"] == 40
    assert torch.equal(r1.tokens, direct) and torch.equal(r2.tokens, direct)
