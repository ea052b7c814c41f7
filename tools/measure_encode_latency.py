"""Measured B200 encode latency per worker (seconds for p tiles, one GPU), both encoders,
through VisionEncoder.encode_latency (the reference's costs.encode_latency signature).
Writes argv[1] (default profiles/r02/encode_latency_b200.json); tools/calibrate_reference.py fits the
reference's CostParams from it."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402

out = {"device": torch.cuda.get_device_name(0), "note": "seconds per encode call of p tiles on one GPU "
       "(tiles resident, CUDA graph path, mean of 5 calls after a warm-up call)", "models": {}}
for ref_name, cfg in [("minicpm-v-2.6", SIGLIP_MINICPM), ("internvl2-8b", INTERNVIT_300M)]:
    enc = VisionEncoder(cfg, 0, max_tiles=16)
    samples = []
    for p in list(range(1, 17)) + [20, 24, 32]:
        samples.append([p, enc.encode_latency(None, p, repeats=5)])
    out["models"][ref_name] = {"encoder": cfg.name, "samples": samples}
    enc.close()
    print(ref_name, [(p, round(s * 1e3, 3)) for p, s in samples])
path = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r02" / "encode_latency_b200.json"
path.write_text(json.dumps(out, indent=1))
print(path)
