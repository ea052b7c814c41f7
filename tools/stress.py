"""Stress loop for intermittent device faults: C5-shaped encode (InternViT, 12 tiles) and
InternLM2.5 prefill of the packed tokens, or the C2 pair (SigLIP + Qwen2), repeated with a
synchronize per iteration so a fault is attributed to its iteration and stage.

usage: python tools/stress.py [c5|c2] [iterations] [encode|prefill|both]
       python tools/stress.py attn [launches]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM  # noqa: E402
from paper_2501_05460_b200.encoder import VisionEncoder  # noqa: E402
from paper_2501_05460_b200.prefill import INTERNLM25_7B, QWEN2_7B, Prefiller  # noqa: E402
from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request  # noqa: E402


def attn_stress(iters):
    """Attention alone, both head dims, every item mix (1..12 images): repeated launches
    must agree bit for bit."""
    from paper_2501_05460_b200 import kernels
    dev = torch.device("cuda")
    bad = 0
    for (H, T, Dv) in [(16, 1024, 72), (16, 1025, 64)]:
        for B in (1, 2, 3, 5, 10, 12):
            g = torch.Generator(device=dev).manual_seed(B)
            qkv = torch.randn(B * T, 3 * H * Dv, device=dev, generator=g).to(torch.bfloat16)
            q, k, v = qkv[:, :H * Dv], qkv[:, H * Dv:2 * H * Dv], qkv[:, 2 * H * Dv:]
            ref = kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5).clone()
            out = torch.empty_like(ref)
            for i in range(iters):
                kernels.attention(q, k, v, B, H, T, T, Dv, Dv ** -0.5, out=out)
                if i % 10 == 9:
                    torch.cuda.synchronize()
                    if not torch.equal(out, ref):
                        bad += 1
                        print(f"MISMATCH dh={Dv} B={B} iter {i}", flush=True)
    torch.cuda.synchronize()
    print(f"attention: {iters} launches per case, {bad} mismatching checks", flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "attn":
        attn_stress(int(sys.argv[2]) if len(sys.argv) > 2 else 200)
        return
    wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    what = sys.argv[3] if len(sys.argv) > 3 else "both"
    cfg, lcfg, n = (INTERNVIT_300M, INTERNLM25_7B, 12) if wl == "c5" else (SIGLIP_MINICPM, QWEN2_7B, 10)
    dev = torch.device("cuda", 0)
    enc = VisionEncoder(cfg, dev, max_tiles=n)
    stage = EncodeStage(enc, dev)
    tiles = tiles_for_request(n, cfg, seed=20260808).pin_memory()
    T = n * cfg.out_tokens + 22
    pf = Prefiller(lcfg, dev, max_tokens=T) if what != "encode" else None
    prompt = torch.randint(0, lcfg.vocab, (22,), dtype=torch.int32).to(dev)
    res = stage.process(tiles)
    torch.cuda.synchronize()
    ref = res.tokens.clone()
    ref_tok = None
    mismatches = 0
    t0 = time.time()
    for i in range(iters):
        stage_name = "encode"
        try:
            if what != "prefill":
                res = stage.process(tiles)
                torch.cuda.synchronize()
                if not torch.equal(res.tokens, ref):  # a race shows up as run-to-run drift
                    mismatches += 1
                    print(f"MISMATCH at iteration {i}: max |diff| "
                          f"{(res.tokens.float() - ref.float()).abs().max().item():.3e}", flush=True)
            if pf is not None:
                stage_name = "prefill"
                tok = pf.prefill(res.tokens.view(-1, cfg.out_dim), prompt)
                torch.cuda.synchronize()
                t = int(tok.item())
                if ref_tok is None:
                    ref_tok = t
                elif t != ref_tok:
                    mismatches += 1
                    print(f"MISMATCH at iteration {i}: first token {t} != {ref_tok}", flush=True)
        except Exception as e:
            print(f"FAULT at iteration {i} in {stage_name}: {e}", flush=True)
            raise
    print(f"{wl} {what}: {iters} iterations, {mismatches} mismatches, {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
