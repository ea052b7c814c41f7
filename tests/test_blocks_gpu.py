"""Device-side block free list against the host BlockManager
(itself pinned to the reference's blocks.py by tests/golden): identical ids, free lists and
errors over random allocate/free sequences, and the prefill writing real K/V straight into
device-allocated blocks."""
import random

import pytest
import torch

from paper_2501_05460_b200.blockpool import BlockManager, CacheKind, DeviceBlockManager

pytestmark = pytest.mark.gpu


def test_device_ids_match_host_sequence(cuda):
    rng = random.Random(7)
    host = BlockManager(CacheKind.KV, 16, 300)
    dev = DeviceBlockManager(CacheKind.KV, 16, 300, device=cuda)
    live = []
    for step in range(400):
        if live and (rng.random() < 0.45 or host.free_blocks < 40):
            rid = live.pop(rng.randrange(len(live)))
            host.free(rid)
            dev.free(rid)
        else:
            tokens = rng.choice([0, 1, 15, 16, 17, 100, 400, 662])
            if not host.can_allocate(tokens):
                with pytest.raises(RuntimeError):
                    dev.allocate_device(step, tokens)
                continue
            a = host.allocate(step, tokens)
            b = dev.allocate_device(step, tokens)
            assert b.tolist() == a
            live.append(step)
        assert dev.free_blocks == host.free_blocks
    torch.cuda.synchronize()
    assert dev.device_free_list().tolist() == host.device_free_list().tolist()
    with pytest.raises(RuntimeError):
        dev.free(10_000)
    with pytest.raises(RuntimeError):
        dev.allocate_device(live[0], 16)  # double allocate


def test_prefill_writes_kv_into_device_blocks(cuda):
    from paper_2501_05460_b200.handoff import PagedKVCache
    from paper_2501_05460_b200.prefill import TINY_LLM, Prefiller
    cfg = TINY_LLM
    pf = Prefiller(cfg, cuda, max_tokens=128)
    kv_host = PagedKVCache(cfg.layers, cfg.kv_heads, cfg.head_dim, 16, 32, cuda)
    kv_dev = PagedKVCache(cfg.layers, cfg.kv_heads, cfg.head_dim, 16, 32, cuda)
    kv_dev.manager = DeviceBlockManager(CacheKind.KV, 16, 32, device=cuda)
    g = torch.Generator(device=cuda).manual_seed(1)
    mm = (torch.randn(50, cfg.hidden, generator=g, device=cuda) * 0.5).to(torch.bfloat16)
    ids = torch.randint(0, cfg.vocab, (9,), generator=g, device=cuda, dtype=torch.int32)
    kv_host.manager.allocate(0, 5)  # occupy a few ids first so the request gets 1.. not 0..
    kv_dev.manager.allocate_device(0, 5)
    b_host = kv_host.manager.allocate(1, 59)
    b_dev = kv_dev.manager.allocate_device(1, 59)  # device tensor, no host round trip
    pf.prefill(mm, ids, kv=kv_host, block_ids=b_host)
    pf.prefill(mm, ids, kv=kv_dev, block_ids=b_dev)
    torch.cuda.synchronize()
    assert b_dev.tolist() == b_host
    assert torch.equal(kv_host.pool, kv_dev.pool)
