"""CPU tier for the MM-token cache specification: content-key KATs, a pure-Python
restatement of the key for small records, and the cache-behaviour oracle."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.hashing import content_hash
from oracle.mmcache import CapacityExceeded, MMCacheOracle

KAT = json.loads((Path(__file__).parent / "golden" / "hash_kat.json").read_text())
M = (1 << 64) - 1


def _fmix(k):
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & M
    k ^= k >> 33
    k = (k * 0xC4CEB53FE5D4A1A3) & M
    k ^= k >> 33
    return k


def _py_hash(b: bytes):
    sa = sb = 0
    for i in range(len(b) // 8):
        w = int.from_bytes(b[8 * i:8 * i + 8], "little")
        a = _fmix(w ^ ((i * 0x9E3779B97F4A7C15 + 0x243F6A8885A308D3) & M))
        sa = (sa + a) & M
        sb = (sb + _fmix((a + 0x632BE59BD9B4E019) & M)) & M
    L = len(b)
    k0 = _fmix(sa ^ L)
    k1 = _fmix((sb + L * 0xD6E8FEB86659FD93) & M)
    return (k0 or 1), k1


def _kat_records():
    rng = np.random.default_rng(20260808)
    return {"zeros8": np.zeros(8, np.uint8), "ramp64": np.arange(64, dtype=np.uint8),
            "ones4096": np.full(4096, 255, np.uint8),
            "rand_tile_448": rng.integers(0, 256, 448 * 448 * 3, dtype=np.uint8),
            "rand_tile_56": rng.integers(0, 256, 56 * 56 * 3, dtype=np.uint8)}


def test_hash_known_answers():
    for name, rec in _kat_records().items():
        assert [str(k) for k in content_hash(rec)] == KAT[name]["key"], name


@pytest.mark.parametrize("n", [8, 16, 64, 1000, 4096])
def test_hash_numpy_equals_pure_python(n):
    rec = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
    assert content_hash(rec) == _py_hash(rec.tobytes())


def test_hash_sensitivity():
    rec = np.random.default_rng(1).integers(0, 256, 56 * 56 * 3, dtype=np.uint8)
    base = content_hash(rec)
    for pos in (0, 1, 4000, rec.size - 1):
        r2 = rec.copy()
        r2[pos] ^= 1
        assert content_hash(r2) != base
    # swapping two words changes the key (position-keyed)
    r3 = rec.copy().view("<u8")
    r3[[0, 1]] = r3[[1, 0]]
    if r3[0] != r3[1]:
        assert content_hash(r3.view(np.uint8)) != base
    with pytest.raises(ValueError):
        content_hash(np.zeros(12, np.uint8))


def test_cache_oracle_first_request_and_repeat():
    c = MMCacheOracle(8)
    ks = [(1, 1), (2, 2), (1, 1), (3, 3)]
    assert c.process(ks) == [("miss", 0), ("miss", 1), ("dup", 0), ("miss", 2)]
    assert c.process([(3, 3), (4, 4), (2, 2)]) == [("hit", 2), ("miss", 3), ("hit", 1)]
    assert len(c) == 4


def test_cache_oracle_lru_eviction_and_lifo_ids():
    c = MMCacheOracle(3)
    c.process([(1, 0), (2, 0), (3, 0)])          # entries 0,1,2
    c.process([(1, 0)])                          # refresh key 1 -> LRU order 2,3,1
    out = c.process([(4, 0), (5, 0)])            # evict 2 (entry 1) then 3 (entry 2)
    assert c.last_victims == [(2, 0), (3, 0)]
    # freed entries are reused LIFO: entry 2 was freed last -> handed out first
    assert out == [("miss", 2), ("miss", 1)]
    assert c.process([(1, 0), (4, 0), (5, 0)]) == [("hit", 0), ("hit", 2), ("hit", 1)]


def test_cache_oracle_pins_current_hits():
    c = MMCacheOracle(2)
    c.process([(1, 0), (2, 0)])
    out = c.process([(2, 0), (9, 0)])  # key 1 is the only evictable entry
    assert c.last_victims == [(1, 0)]
    assert out == [("hit", 1), ("miss", 0)]


def test_cache_oracle_capacity():
    c = MMCacheOracle(2)
    with pytest.raises(CapacityExceeded):
        c.process([(1, 0), (2, 0), (3, 0)])
    assert c.process([(1, 0), (1, 0), (2, 0)]) == [("miss", 0), ("dup", 0), ("miss", 1)]


def test_c4_workload_classification():
    """C4: 40 images x 10 tiles, image i+20 repeats image i -> 200 misses then 200 dups;
    a second identical request hits all 400."""
    keys = [(i % 200 + 1, 7) for i in range(400)]
    c = MMCacheOracle(750)
    first = c.process(keys)
    assert [k for k, _ in first].count("miss") == 200 and [k for k, _ in first].count("dup") == 200
    second = c.process(keys)
    assert all(k == "hit" for k, _ in second)
    assert [e for _, e in first] == [e for _, e in second]
