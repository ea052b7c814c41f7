"""Diagnose host-side overhead of the e2e encode step (debug helper)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.configs import SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402
from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request  # noqa: E402

dev = torch.device("cuda", 0)
cfg = SIGLIP_MINICPM
enc = VisionEncoder(cfg, dev, max_tiles=10)
st = EncodeStage(enc, dev)
th = tiles_for_request(10, cfg, 1).pin_memory()
td = th.to(dev)
oh = torch.empty(10, 64, 3584, dtype=torch.bfloat16).pin_memory()
for _ in range(3):
    st.process(None, tiles_dev=td)
torch.cuda.synchronize()
for name, fn in [("resident", lambda: st.process(None, tiles_dev=td)),
                 ("h2d_only", lambda: th.to(dev, non_blocking=True)),
                 ("e2e", lambda: oh.copy_(st.process(th).tokens, non_blocking=True))]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host issue {1e3*(t1-t0)/10:.3f} ms/step, device {e0.elapsed_time(e1)/10:.3f} ms/step, wall {1e3*(t2-t0)/10:.3f}")
