"""Known-answer vectors for the MM-cache content key (oracle/hashing.py spec).

    python tests/golden/make_hash_kat.py   -> tests/golden/hash_kat.json
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle.hashing import content_hash  # noqa: E402


def records():
    yield "zeros8", np.zeros(8, np.uint8)
    yield "ramp64", np.arange(64, dtype=np.uint8)
    yield "ones4096", np.full(4096, 255, np.uint8)
    rng = np.random.default_rng(20260808)
    yield "rand_tile_448", rng.integers(0, 256, 448 * 448 * 3, dtype=np.uint8)
    yield "rand_tile_56", rng.integers(0, 256, 56 * 56 * 3, dtype=np.uint8)


def main():
    out = {name: {"len": int(r.size), "seed_note": "numpy default_rng(20260808) draws in order",
                  "key": [str(k) for k in content_hash(r)]} for name, r in records()}
    p = Path(__file__).parent / "hash_kat.json"
    p.write_text(json.dumps(out, indent=1))
    print(p)


if __name__ == "__main__":
    main()
