#!/usr/bin/env python
"""Encode-stage hot-path benchmark (BASELINE.json metric: encoded image tiles/s and
p50 TTFT at 1/2/4/8 B200 vs the host-CPU reference).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2|c4|c5]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1; one process per GPU)

One step = one request through the encode stage: its tiles are IRP-sharded over the
N encode ranks (irp_shard, engine.py:55-62), encoded by the sm_100a kernels, and the
MM tokens are gathered (NCCL P2P) in request order onto the prefill rank (rank 0).
Default workload (c2): MiniCPM-V 2.6-shaped SigLIP-400M + resampler, 10 tiles of
448x448 per request, bf16, random-init weights, synthetic uint8 tiles.

Prints ONE JSON line on rank 0 (see the task contract): `value` = whole-job tiles/s
with tiles resident in HBM; `e2e` = same through the public API with host buffers
(pinned H2D of the tiles + D2H of the packed MM tokens inside the timed region, every
step; the stage pipelines its upload / readback streams across consecutive requests as
a serving loop would); `p50_ttft_ms` = encode-side TTFT measured per request with
nothing else in flight (tile upload -> MM tokens packed on the prefill GPU -> readback).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "encoded image tiles/sec & p50 TTFT at 1/2/4/8 B200 vs host-CPU reference"

# reference synthetic prefill calibration for MiniCPM-V 2.6 / InternVL2-8B (presets.py:53-61),
# used only for the labelled "modeled prefill" add-on to the measured encode-side TTFT.
PREFILL_COST = {"minicpm-v-2.6": (0.05, 2e-4, 1e-8), "internvl2-8b": (0.05, 8e-5, 1e-9)}
PROMPT_TOKENS = 22


def modeled_prefill_s(model: str, total_tokens: int) -> float:
    """costs.prefill_latency (costs.py:93-99) at tp = pp = 1."""
    b, a, q = PREFILL_COST[model]
    return b + a * total_tokens + q * total_tokens * total_tokens


def workload(name: str):
    from paper_2501_05460_b200.configs import INTERNVIT_300M, SIGLIP_MINICPM, TINY_VIT
    if name == "c1":
        return dict(cfg=TINY_VIT, tiles=4, repeat=None, cache=False,
                    desc="C1: PR1 oracle config, tiny ViT (4 tokens x 8 dims per tile), 1 request x 4 tiles")
    if name == "c2":
        return dict(cfg=SIGLIP_MINICPM, tiles=10, repeat=None, cache=False, llm="qwen2-7b", kv_handoff=True,
                    desc="C2: MiniCPM-V 2.6-shaped SigLIP-400M + resampler, 10 tiles (448x448) per request "
                         "(+ Qwen2-7B prefill, prefill->decode KV-block handoff of 662 tokens)")
    if name == "c2i":
        return dict(cfg=SIGLIP_MINICPM, tiles=10, repeat=None, cache=False, llm="qwen2-7b", image=(4032, 3024),
                    desc="C2 from pixels: one 4032x3024 photo per request, MiniCPM-V slicing on the GPU -> "
                         "10 tiles (448x448) -> SigLIP-400M + resampler")
    if name == "c2s":
        return dict(cfg=SIGLIP_MINICPM, tiles=10, repeat=None, cache=False, llm="qwen2-7b", serve=(8, 4),
                    desc="C2 served: bursts of 8 MiniCPM-V requests (10 tiles each) through EPDRuntime, encode "
                         "batches of up to 4 requests (form_batch + E/P-side MM reservations), shards stored into "
                         "the prefill instance's paged MM blocks, Qwen2-7B prefill to the first token")
    if name == "c2p":
        return dict(cfg=SIGLIP_MINICPM, tiles=10, repeat=None, cache=False, llm="qwen2-7b", serve=(64, 4),
                    poisson=40.0,
                    desc="C2 open loop: 64 MiniCPM-V requests (10 tiles each) arriving as workload.generate_poisson "
                         "at 40 requests/s (seed 20260808), served by EPDRuntime (batches of up to 4, Qwen2-7B "
                         "prefill to the first token)")
    if name == "c4":
        return dict(cfg=SIGLIP_MINICPM, tiles=400, repeat=200, cache=True, llm="qwen2-7b",
                    desc="C4: 40 images x 10 tiles per request, image i+20 repeats image i (MM-token cache)")
    if name == "c4w":
        return dict(cfg=SIGLIP_MINICPM, tiles=400, repeat=None, cache=True, llm="qwen2-7b", rotate=(100, 20),
                    desc="C4 warm: 40 images x 10 tiles per request; each request repeats the previous request's "
                         "last 20 images (cross-request MM-token cache hits) and brings 20 new ones (misses)")
    if name == "c5":
        # the catalog maps a 4032x3024 image to 13 InternVL2-8B tiles (models.cfg:28):
        # 12 dynamic tiles + the thumbnail
        return dict(cfg=INTERNVIT_300M, tiles=13, repeat=None, cache=False, kv_handoff=True, llm="internlm2.5-7b",
                    desc="C5: InternVL2-8B-shaped InternViT-300M + pixel shuffle + mlp1, 13 tiles per request "
                         "(12 dynamic + thumbnail, models.cfg:28), + prefill->decode KV-block handoff (3350 tokens)")
    raise SystemExit(f"unknown workload {name}")


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # In-process NVML (no fork/exec inside the timed region); nvidia-smi as fallback.
        nvml = None
        try:
            import pynvml as nvml
            nvml.nvmlInit()
            h = nvml.nvmlDeviceGetHandleByIndex(self.index)
            smax = nvml.nvmlDeviceGetMaxClockInfo(h, nvml.NVML_CLOCK_SM)
            bits = [nvml.nvmlClocksEventReasonHwSlowdown, nvml.nvmlClocksEventReasonHwThermalSlowdown,
                    nvml.nvmlClocksEventReasonSwThermalSlowdown, nvml.nvmlClocksEventReasonSwPowerCap]
        except Exception:
            nvml = None
        while not self._stop.is_set():
            try:
                if nvml is not None:
                    sm = nvml.nvmlDeviceGetClockInfo(h, nvml.NVML_CLOCK_SM)
                    reasons = nvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    flags = ["Active" if reasons & b else "Not Active" for b in bits]
                    self.samples.append([str(sm), str(smax), "0"] + flags)
                else:
                    out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05 if nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[3 + i]
                          and not s[3 + i].startswith("Not")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(gpus: int) -> None:
    """`python bench.py --gpus N` with N > 1 outside torchrun: re-exec under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1). Under torchrun
    (WORLD_SIZE set) this is a no-op. NCCL's INIT log is kept on stderr so the rank count
    of every communicator can be checked."""
    if gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if os.environ.get("EPD_BENCH_ONE_GPU") != "1" and torch.cuda.device_count() < gpus:
        raise SystemExit(f"--gpus {gpus} but only {torch.cuda.device_count()} CUDA device(s) are visible "
                         "(EPD_BENCH_ONE_GPU=1 runs every rank on cuda:0 as a functional check)")
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py")] + sys.argv[1:]
    sys.stdout.flush()
    os.execvpe(sys.executable, cmd, env)


def init_dist(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus and world != 1:
        raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={world}")
    if world > 1 and os.environ.get("EPD_BENCH_ONE_GPU") == "1":
        # functional check of the N > 1 path on one GPU (every rank on cuda:0, gloo control
        # plane, the peer-memory gather between processes); its timings mean nothing
        import torch.distributed as dist
        local = 0
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
        dist.barrier()
    elif world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # first collective on every rank: the NCCL communicator exists before any rank
        # issues a grouped P2P gather (ranks with an empty shard skip those calls)
        dist.barrier()
    return world, rank, local


def bench_config(wl, world: int) -> dict:
    """The workload description both arms print (identical for --impl ours / reference)."""
    cfg = wl["cfg"]
    reqs = world if (world > 1 and not wl["cache"] and not wl.get("image") and not wl.get("serve")) else 1
    return {"workload": wl["desc"], "encoder": cfg.name, "tiles_per_request": wl["tiles"],
            "requests_per_step": reqs,
            "irp_width": world, "prefill_rank": 0, "parallelism": f"irp{world}",
            "l2": "working set > L2 (0.97 GB bf16 weights + ~0.5 GB activations streamed per step)",
            "weights": "random-init N(0,0.02), seed 20260808"}


def reference_arm(args, wl, world, rank):
    """--impl reference: the reference's CPU path for the encode stage = the fp32 CPU
    oracle (the reference ships no encoder), on all host cores."""
    if rank != 0:
        return
    # host only: the weight schema comes from weights.weight_schema, so this arm never
    # loads libepd.so (tests/test_bench_cpu.py checks it)
    import oracle.encoders as oe
    from paper_2501_05460_b200.stage import tiles_for_request
    from paper_2501_05460_b200.weights import canonical_weights
    cfg = wl["cfg"]
    torch.set_num_threads(os.cpu_count())
    w = canonical_weights(cfg, 20260808)
    tiles = tiles_for_request(min(wl["tiles"], 16), cfg, seed=20260808)
    per_step = 1  # bounded sample: one tile of the request per step
    for i in range(args.warmup):
        oe.encode(cfg, w, tiles[i % tiles.shape[0]:i % tiles.shape[0] + per_step])
    t0 = time.perf_counter()
    for i in range(args.steps):
        j = (args.warmup + i) % tiles.shape[0]
        oe.encode(cfg, w, tiles[j:j + per_step])
    dt = time.perf_counter() - t0
    v = args.steps * per_step / dt
    line = {"metric": METRIC, "value": v, "unit": "tiles/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if (wl["cache"] or wl.get("image")) else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "impl": "reference", "config": bench_config(wl, world), "sample_tiles_per_step": per_step,
            "cpu_baseline": {"value": v, "unit": "tiles/s", "cores": torch.get_num_threads(), "kind": "port",
                             "sample": f"{per_step} tile of the {wl['tiles']}-tile request per step (bounded "
                                       "sample), fp32 PyTorch CPU oracle (oracle/encoders.py)"},
            "e2e": {"value": v, "unit": "tiles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the measured LLM prefill (encode-side TTFT only)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warm-up raised to the minimum of 3", file=sys.stderr)
        args.warmup = 3
    wl = workload(args.workload)
    spawn_ranks(args.gpus)
    world, rank, local = init_dist(args.gpus) if args.impl == "ours" else (
        int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0)
    if args.impl == "reference":
        reference_arm(args, wl, world, rank)
        return
    if wl.get("serve"):
        run_serve(args, wl, world, rank, local)
        return
    run_ours(args, wl, world, rank, local)


def run_serve(args, wl, world, rank, local):
    """One step = one burst of requests served to their first tokens by runtime.EPDRuntime
    (value = tiles of the burst / burst time, max over ranks; TTFT per request from the
    measured RequestRecords, first_token_time - arrival, p50 by the reference's rule)."""
    import torch.distributed as dist

    from paper_2501_05460_b200.encoder import VisionEncoder, canonical_weights
    from paper_2501_05460_b200.prefill import QWEN2_7B, Prefiller
    from paper_2501_05460_b200.runtime import EPDRuntime, ServeRequest, check_causality
    from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg, n = wl["cfg"], wl["tiles"]
    n_req, max_batch = wl["serve"]
    enc = VisionEncoder(cfg, dev, max_tiles=n * max_batch, weights=canonical_weights(cfg))
    stage = EncodeStage(enc, dev, rank=rank, world=world)
    T_pre = n * cfg.out_tokens + PROMPT_TOKENS
    pf = Prefiller(QWEN2_7B, dev, max_tokens=T_pre) if rank == 0 else None
    rt = EPDRuntime(stage, pf, max_batch=max_batch)
    reqs = []
    arrivals = [0.0] * n_req
    if wl.get("poisson"):
        from paper_2501_05460_b200.routing import poisson_arrivals
        arrivals = poisson_arrivals(wl["poisson"], n_req, 20260808)
    pool = [tiles_for_request(n, cfg, seed=20260808 + i).pin_memory() for i in range(min(n_req, 8))]
    for i in range(n_req):
        prompt = torch.randint(0, QWEN2_7B.vocab, (PROMPT_TOKENS,), dtype=torch.int32,
                               generator=torch.Generator().manual_seed(100 + i)).to(dev)
        reqs.append(ServeRequest(i, pool[i % len(pool)], prompt, arrival=arrivals[i]))
    for _ in range(args.warmup):
        rt.serve(reqs)
    torch.cuda.synchronize()
    ttft, walls = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = rt.serve(reqs)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            if world > 1:
                t = torch.tensor([ms], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            walls.append(ms)
            if rank == 0:
                for rec in out["records"].values():
                    check_causality(rec)
                    ttft.append((rec.first_token_time - rec.arrival) * 1e3)
    rt.close()
    if rank != 0:
        return
    total_ms = sum(walls)
    value = n_req * n * args.steps / (total_ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": "tiles/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": bench_config(wl, world) | {"requests_per_burst": n_req, "max_batch": max_batch},
            "p50_ttft_ms": _percentile(ttft, 0.5), "ttft_p90_ms": _percentile(ttft, 0.9), "ttft_n": len(ttft),
            "ttft_note": "per request: first_token_time - arrival from the measured RequestRecords (%globaltimer); "
                         + ("open-loop Poisson arrivals (routing.poisson_arrivals = workload.generate_poisson)"
                            if wl.get("poisson") else "all requests arriving at the burst start")
                         + "; includes queueing behind earlier batches and prefills",
            "ep_wait_per_burst": len(out["ep_wait"]), "clocks": clk.summary(),
            "roofline": None, "cpu_baseline": None,
            "e2e": {"value": value, "unit": "tiles/s", "h2d_bytes_per_step": n_req * n * cfg.tile_bytes,
                    "d2h_bytes_per_step": 4 * n_req}}
    print(json.dumps(line), flush=True)


def run_ours(args, wl, world, rank, local):
    import torch.distributed as dist

    from paper_2501_05460_b200 import _lib
    from paper_2501_05460_b200.encoder import VisionEncoder, canonical_weights
    from paper_2501_05460_b200.mmcache import MMTokenCache
    from paper_2501_05460_b200.stage import EncodeStage, tiles_for_request

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = wl["cfg"]
    n = wl["tiles"]
    weights = canonical_weights(cfg)
    # One request per GPU per step (weak scaling): at N > 1 the step is a batch of N requests,
    # each IRP-sharded over all N ranks restarting at worker 0 (engine.py:583-602); every rank
    # encodes all of its shards of the batch in one call (EncodeStage.process_batch). At N = 1
    # this is the single request of round 1. Cached and photo workloads stay one request.
    from paper_2501_05460_b200.routing import shard_ranges as _sr
    batched = world > 1 and not wl["cache"] and not wl.get("image")
    reqs = world if batched else 1
    per_rank = max(sum(_sr(n, world)[k][1] for _ in range(reqs)) for k in range(world)) if batched else n
    max_tiles = 32 if per_rank > 32 else max(1, per_rank)
    enc = VisionEncoder(cfg, dev, max_tiles=max_tiles, weights=weights)
    cache = None
    if wl["cache"] and rank == 0:
        cache = MMTokenCache(capacity=max(n, 750), tokens_per_tile=cfg.out_tokens, hidden=cfg.out_dim, device=dev)
    comm = None
    if world > 1 and os.environ.get("EPD_GATHER", "peer") == "nccl":
        from paper_2501_05460_b200.comm import NcclComm
        comm = NcclComm(dev)  # the EP gather's NCCL leg through the C ABI (epd_gather_tokens)
    stage = EncodeStage(enc, dev, rank=rank, world=world, prefill_rank=0, cache=cache, cached=wl["cache"],
                        comm=comm)
    if world > 1 and os.environ.get("EPD_GATHER", "peer") != "nccl":
        stage.enable_peer_gather(max(n * reqs, 16))  # shards stored into the prefill GPU over NVLink

    rot = wl.get("rotate")
    if rot:
        # a pool of P images (+ the first 2 rq-image windows again, same content) so request k is the
        # contiguous window [rq*k mod P, rq*k mod P + 2 rq) of images: half of it is the previous
        # request's second half (cache hits), half is new (last seen P/rq requests ago: evicted)
        P, rq = rot
        per = n // (2 * rq)  # tiles per image
        pool = tiles_for_request(P * per, cfg, seed=20260808)
        tiles_pool = torch.cat([pool, pool[:2 * rq * per]]).pin_memory()
        pool_dev = tiles_pool.to(dev)
        step_no = [0]

        def window():
            o = (step_no[0] * rq % P) * per
            step_no[0] += 1
            return slice(o, o + n)
        tiles_host = tiles_pool[:n]
    else:
        tiles_host = tiles_for_request(n, cfg, seed=20260808, repeat_period=wl["repeat"]).pin_memory()
    image_host = None
    if wl.get("image"):
        # one synthetic photo per request; the stage tiles it on the GPU (tiler.py)
        iw, ih = wl["image"]
        g = torch.Generator().manual_seed(20260808)
        image_host = torch.randint(0, 256, (ih, iw, cfg.channels), dtype=torch.uint8, generator=g).pin_memory()
    tiles_dev = tiles_host.to(dev)
    out_host = torch.empty(n * reqs, cfg.out_tokens, cfg.out_dim, dtype=torch.bfloat16).pin_memory()
    if batched:
        batch_host = [tiles_host] + [tiles_for_request(n, cfg, seed=20260808 + r).pin_memory() for r in range(1, reqs)]
        batch_dev = [t.to(dev) for t in batch_host]

    def barrier():
        if world > 1:
            dist.barrier()

    def reset_cache():
        # C4: every request starts cold (its hits are in-request duplicates); C4 warm keeps the
        # cache across requests, so the previous request's images hit
        if cache is not None and not rot:
            cache.clear()

    def step_resident():
        reset_cache()
        if rot:
            return stage.process(None, tiles_dev=pool_dev[window()])
        if batched:
            return stage.process_batch(tiles_dev=batch_dev)
        return stage.process(None, tiles_dev=tiles_dev)

    def step_e2e():
        # pinned H2D of the request's tiles -> encode -> D2H of the packed tokens; the stage
        # pipelines its host I/O streams across consecutive requests
        reset_cache()
        if image_host is not None:
            return stage.process_image(image_host, cfg.geometry.name, out_host=out_host if rank == 0 else None)
        if rot:
            return stage.process(tiles_pool[window()], out_host=out_host if rank == 0 else None)
        if batched:
            return stage.process_batch(tiles_host=batch_host, out_host=out_host if rank == 0 else None)
        return stage.process(tiles_host, out_host=out_host if rank == 0 else None)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier()
        torch.cuda.synchronize()
        t_all0 = torch.cuda.Event(enable_timing=True)
        t_all1 = torch.cuda.Event(enable_timing=True)
        t_all0.record()
        last = None
        for i in range(k):
            evs[i][0].record()
            last = fn()
            evs[i][1].record()
        stage.join()  # the timed region ends after the last readback
        t_all1.record()
        torch.cuda.synchronize()
        barrier()
        total_ms = max_over_ranks(t_all0.elapsed_time(t_all1))
        per = [max_over_ranks(a.elapsed_time(b)) for a, b in evs]
        return total_ms, per, last

    for _ in range(args.warmup):
        step_resident()
        step_e2e()
    torch.cuda.synchronize()

    def latencies(fn, k):
        """Per-request latency with nothing else in flight (upload -> encode -> readback
        inside each request's events), max over ranks."""
        out = []
        for _ in range(k):
            barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            stage.join()
            b.record()
            torch.cuda.synchronize()
            out.append(max_over_ranks(a.elapsed_time(b)))
        return out

    with ClockSampler(local) as clk:
        total_ms, per_ms, last = timed(step_resident, args.steps)
        e2e_ms, _, last_e2e = timed(step_e2e, args.steps)
    e2e_per = latencies(step_e2e, max(50, args.steps))  # p50 TTFT over >= 50 requests

    # Full TTFT: the prefill rank runs the model's LLM prefill on
    # [MM tokens | prompt] and reads back the first token, so TTFT = tile upload -> encode ->
    # gather -> prefill -> first token on the host.
    prefill = None
    pf = prompt_ids = mm_last = None
    if wl.get("llm") and not args.no_prefill:
        from paper_2501_05460_b200.prefill import INTERNLM25_7B, QWEN2_7B, Prefiller
        lcfg = {"qwen2-7b": QWEN2_7B, "internlm2.5-7b": INTERNLM25_7B}[wl["llm"]]
        T_pre = n * cfg.out_tokens + PROMPT_TOKENS
        pf = Prefiller(lcfg, dev, max_tokens=T_pre) if rank == 0 else None
        prompt = torch.randint(0, lcfg.vocab, (PROMPT_TOKENS,), dtype=torch.int32,
                               generator=torch.Generator().manual_seed(20260808)).to(dev)
        tok_host = torch.empty(1, dtype=torch.int32).pin_memory()
        prompt_ids = prompt

        def step_ttft():
            reset_cache()  # every TTFT request starts cold, like the e2e loop (C4 warm: steady state)
            res = (stage.process_image(image_host, cfg.geometry.name) if image_host is not None
                   else stage.process(tiles_pool[window()] if rot else tiles_host))
            if pf is not None:
                tok = pf.prefill(res.tokens.view(-1, cfg.out_dim), prompt)
                tok_host.copy_(tok, non_blocking=True)
            return res

        def step_prefill_only():
            if pf is not None:
                pf.prefill(last.tokens[:n].reshape(-1, cfg.out_dim), prompt)

        for _ in range(3):
            mm_last = step_ttft().tokens
        if mm_last is not None:
            mm_last = mm_last.view(-1, cfg.out_dim).clone()
        torch.cuda.synchronize()
        ttft_full = latencies(step_ttft, max(50, args.steps))
        pre_only = latencies(step_prefill_only, 20)
        prefill = {"model": lcfg.name, "tokens": T_pre, "mm_tokens": n * cfg.out_tokens, "prompt_tokens": PROMPT_TOKENS,
                   "p50_ttft_ms": _percentile(ttft_full, 0.5), "ttft_n": len(ttft_full),
                   "ttft_p90_ms": _percentile(ttft_full, 0.9),
                   "prefill_p50_ms": _percentile(pre_only, 0.5),
                   "prefill_tflops": lcfg.flops(T_pre) / (_percentile(pre_only, 0.5) / 1e3) / 1e12,
                   "weights": "random-init N(0,0.02) bf16 of the public LLM geometry (catalog models.cfg layers / "
                              "KV heads / head dim / hidden + model card FFN / vocab)"}

    # profiled pass (same workload, after the timed region): per-kernel-class device times
    _lib.call("epd_encoder_profile", enc._h, 1)
    prof_steps = 2
    for _ in range(prof_steps):
        # ~30 ms of device sleep first: the step's eager launches and their events queue up
        # behind it, so each event pair brackets kernel time only, not host launch gaps
        torch.cuda._sleep(60_000_000)
        step_resident()
    torch.cuda.synchronize()
    import ctypes as C
    nc = 5
    ms = (C.c_double * nc)()
    fl = (C.c_double * nc)()
    by = (C.c_double * nc)()
    cnt = (C.c_int64 * nc)()
    _lib.call("epd_encoder_profile_read", enc._h, ms, fl, by, cnt, nc)
    _lib.call("epd_encoder_profile", enc._h, 0)

    kv = (kv_handoff_bench(wl, cfg, n, world, rank, dev, args, pf=pf, mm=mm_last, prompt=prompt_ids)
          if wl.get("kv_handoff") else None)
    gather = gather_bench(stage, cfg, n, world, rank, dev, args) if not wl["cache"] else None

    encoded_tiles = n * reqs  # tiles that complete the step's requests (cache hits count as served)
    value = encoded_tiles * args.steps / (total_ms / 1e3)
    e2e_value = encoded_tiles * args.steps / (e2e_ms / 1e3)
    p50_ttft = _percentile(e2e_per, 0.5)
    p50_resident = _percentile(per_ms, 0.5)
    if rank != 0:
        return

    enc_share = 1.0
    if cache is not None and last is not None and last.cache_counts is not None:
        enc_share = last.cache_counts["miss"] / n
    peaks, peak_src = measured_peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    gemm_tflops = fl[1] / (ms[1] / 1e3) / 1e12 if ms[1] > 0 else None
    flops_tile = enc.flops_per_tile()
    classes = ["patchify", "gemm", "attention", "layernorm", "other"]
    kernels = {classes[c]: {"ms_per_step": ms[c] / prof_steps, "launches_per_step": cnt[c] / prof_steps,
                            "share": ms[c] / max(sum(ms), 1e-9),
                            "tflops": (fl[c] / (ms[c] / 1e3) / 1e12) if ms[c] > 0 and fl[c] > 0 else None,
                            "gbs": (by[c] / (ms[c] / 1e3) / 1e9) if ms[c] > 0 and by[c] > 0 else None}
               for c in range(nc) if cnt[c]}
    traffic = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        traffic = json.loads(tj.read_text()).get(wl["cfg"].name, {}).get("gemm_dram_bytes_per_launch")

    my_tiles = (sum(stage_tiles_per_rank(n, world, rank) for _ in range(reqs)) if batched
                else stage_tiles_per_rank(n, world, rank))
    launches_per_step = enc.launches(my_tiles) + (2 if cache is not None else 0)
    if stage.transport == "nvlink-peer":
        launches_per_step += world - 1  # the prefill rank's release-flag stores (peer.py)
    model = cfg.geometry.name
    total_tokens = n * cfg.out_tokens + PROMPT_TOKENS
    prefill_ms = modeled_prefill_s(model, total_tokens) * 1e3 if model in PREFILL_COST else None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, weights, tiles_host)

    line = {
        "metric": METRIC, "value": value, "unit": "tiles/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if (wl["cache"] or wl.get("image")) else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": bench_config(wl, world), "ep_transport": stage.transport,
        "p50_ttft_ms": prefill["p50_ttft_ms"] if prefill else p50_ttft,
        "p50_ttft_ms_encode_side": p50_ttft,
        "p50_ttft_ms_resident": p50_resident,
        "ttft_ms_dist": {"n": len(e2e_per), "p90": _percentile(e2e_per, 0.9), "max": max(e2e_per),
                         "mean": sum(e2e_per) / len(e2e_per), "resident_max": max(per_ms)},
        "prefill": prefill,
        "p50_ttft_ms_encode_side_plus_modeled_prefill": (p50_ttft + prefill_ms) if prefill_ms is not None else None,
        "ttft_note": "p50_ttft_ms = full TTFT measured on B200 per isolated request, p50 over >= 50: H2D of the "
                     "request's tiles -> encode -> MM tokens packed on the prefill GPU -> LLM prefill of "
                     "[MM tokens | prompt] -> first token read back (see 'prefill'). p50_ttft_ms_encode_side stops at "
                     "the packed MM tokens (+ their D2H). The 'modeled prefill' variant adds the reference's "
                     "costs.prefill_latency with SYNTHETIC_COSTS (presets.py:53-61) instead.",
        "e2e": {"value": e2e_value, "unit": "tiles/s",
                "h2d_bytes_per_step": int(image_host.numel() * world if image_host is not None
                                          else n * reqs * cfg.tile_bytes),  # summed over ranks
                "d2h_bytes_per_step": int(out_host.numel() * 2)},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMM (all encoder GEMM launches, profiled pass)",
                     "achieved": gemm_tflops, "peak": peak, "unit": "TFLOP/s",
                     "frac": (gemm_tflops / peak) if gemm_tflops else None, "traffic": traffic,
                     "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
                     # encoder FLOPs actually executed: cache hits and in-batch duplicates
                     # are served without encoding, so only the misses count here
                     "encoder_achieved": value * enc_share * flops_tile / world / 1e12,
                     "encoder_frac": value * enc_share * flops_tile / world / 1e12 / peak,
                     "flops_per_tile": flops_tile},
        "kernels": kernels,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if wl.get("kv_handoff"):
        line["kv_handoff"] = kv
    if gather is not None:
        line["gather"] = gather
    if cache is not None and last is not None and last.cache_counts is not None:
        line["cache"] = {"hits": last.cache_counts["hit"], "misses": last.cache_counts["miss"],
                         "dups": last.cache_counts["dup"], "plan": "device (epd_mmcache_plan), keyed hash",
                         "host_reads_per_request": "20-byte miss count"}
    print(json.dumps(line), flush=True)


def kv_handoff_bench(wl, cfg, n, world, rank, dev, args, pf=None, mm=None, prompt=None):
    """Prefill -> decode KV-block handoff of one request (engine.py:542-555, 436-439) through
    handoff.KVHandoff: the prefill rank (0) holds the request's paged KV, written by the real
    LLM prefill of the request when it ran (``pf``), and the decode rank (the last rank; the
    same GPU at N = 1) reserves total + output tokens and receives it: one block-move kernel
    on a shared GPU, the same kernel pushing into the decode pool over NVLink across GPUs
    (EPD_KV=nccl: pack -> ncclSend/Recv -> unpack through the C ABI)."""
    from paper_2501_05460_b200.handoff import KVHandoff, PagedKVCache
    geo = cfg.geometry
    total = n * geo.tokens_per_patch + PROMPT_TOKENS
    out_tokens = 64
    p_rank, d_rank = 0, world - 1
    nblk = -(-(total + out_tokens) // 16) + 4
    transport = "local" if world == 1 else os.environ.get("EPD_KV", "nvlink-peer")
    grp = None
    if transport == "nccl" and world > 2:
        import torch.distributed as dist
        grp = dist.new_group([p_rank, d_rank])  # collective over the world: before the early return
    if rank not in (p_rank, d_rank):
        return None
    comm = None
    if transport == "nccl":
        from paper_2501_05460_b200.comm import NcclComm
        comm = NcclComm(dev, rank=0 if rank == p_rank else 1, world=2, group=grp)
    src = PagedKVCache(geo.num_layers, geo.kv_heads, geo.head_dim, 16, nblk, dev) if rank == p_rank else None
    dst = (PagedKVCache(geo.num_layers, geo.kv_heads, geo.head_dim, 16, nblk, dev, shareable=transport != "local")
           if rank == d_rank else None)
    h = KVHandoff(rank, p_rank, d_rank, src, dst, transport=transport, comm=comm, comm_ranks=(0, 1))
    kv_source = "zeros"
    if src is not None and pf is not None:
        # the request's real KV: the LLM prefill writes every layer's post-RoPE K/V into the
        # blocks; LIFO reuse hands the same ids back to every later allocation of this size
        ids = src.manager.allocate(-1, total)
        pf.prefill(mm, prompt, kv=src, block_ids=ids)
        src.manager.free(-1)
        kv_source = f"prefill ({pf.cfg.name})"

    def one(rid):
        if src is not None:
            src.manager.allocate(rid, total)
        info = h.try_reserve_decode(rid, total, out_tokens)
        if info is None:
            raise RuntimeError("decode pool could not reserve the request")
        if dst is not None:
            dst.manager.free(rid)
        return info

    for i in range(args.warmup):
        one(10_000 + i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        info = one(20_000 + i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    verified = None
    if world == 1:
        verified = bool(torch.equal(dst.blocks(info["dst_blocks"][:len(info["src_blocks"])]),
                                    src.blocks(info["src_blocks"])))
    h.close()
    if rank != 0:
        return None
    moved = info["moved_bytes"]
    paths = {"local": "epd_kv_move: one block-to-block kernel (same GPU)",
             "nvlink-peer": "epd_kv_move into the decode pool mapped over CUDA IPC (NVLink stores) + stream-memop flags",
             "nccl": "epd_kv_handoff_send/recv: pack -> ncclSend/Recv -> unpack (C ABI)"}
    return {"tokens": total, "pd_bytes": total * geo.kv_bytes_per_token(), "moved_bytes_per_request": moved,
            "ms_per_request": ms, "GBps": moved / (ms / 1e3) / 1e9, "transport": transport,
            "path": paths[transport], "kv_source": kv_source, "bit_exact": verified,
            "note": "whole 16-token blocks move; pd_bytes is the reference's token-exact count (engine.py:553-554); "
                    "each step includes the reservation handshake"}


NVLINK_GBPS = 900.0  # NVLink 5 per GPU per direction (nominal; MEASURED_PEAKS.json has no NVLink figure)


def gather_bench(stage, cfg, n, world, rank, dev, args):
    """The EP exchange alone (engine.py:521-526 bytes): every encode rank's shard of
    post-projector MM tokens -> the prefill rank at its tile offset (EncodeStage.gather_only:
    NVLink peer-memory stores, or NCCL grouped P2P with EPD_GATHER=nccl), timed on the
    device over K requests, max over ranks. Roofline: bytes into the prefill GPU / time
    against the NVLink ingress bandwidth."""
    import torch.distributed as dist

    from paper_2501_05460_b200.routing import ep_bytes, shard_ranges
    ranges = shard_ranges(n, world)
    tpp, bpt = cfg.out_tokens, cfg.out_dim * 2
    into_sink = sum(ep_bytes(c, tpp, bpt) for k, (_, c) in enumerate(ranges) if k != 0)
    if world == 1:
        return {"bytes_per_request": 0, "note": "single GPU: the shard is written in place into the packed buffer"}
    first, count = ranges[rank]
    local = torch.randn(max(count, 1), cfg.out_tokens, cfg.out_dim, device=dev).to(torch.bfloat16)[:count]
    for _ in range(args.warmup):
        stage.gather_only(local if count else None, n)
    torch.cuda.synchronize()
    ts = []
    for _ in range(max(args.steps, 20)):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        stage.gather_only(local if count else None, n)
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ts.append(float(t.item()))
    ms = _percentile(ts, 0.5)
    gbs = into_sink / (ms / 1e3) / 1e9
    return {"bytes_per_request": into_sink, "p50_ms": ms, "GBps": gbs, "peak_GBps": NVLINK_GBPS,
            "frac": gbs / NVLINK_GBPS, "peak_source": "nominal NVLink 5 ingress per GPU",
            "path": ("16 B stores into the prefill GPU's packed slot over NVLink peer memory (CUDA IPC) + "
                     "per-rank sequence flags, stream-memop waits (peer.py)") if stage.transport == "nvlink-peer"
            else "NCCL grouped P2P (batch_isend_irecv) into the prefill rank at tile offsets",
            "transport": stage.transport}


def stage_tiles_per_rank(n: int, world: int, rank: int) -> int:
    from paper_2501_05460_b200.routing import shard_ranges
    return shard_ranges(n, world)[rank][1]


def _percentile(values, q):
    """metrics._percentile (metrics.py:103-108): nearest rank, banker's round."""
    o = sorted(values)
    if not o:
        return 0.0
    return o[min(len(o) - 1, max(0, round(q * (len(o) - 1))))]


def cpu_baseline(cfg, weights, tiles_host):
    """fp32 CPU oracle on the host cores: 1 warm-up tile + 3 timed tiles (bounded sample,
    SURVEY.md 8(d))."""
    import oracle.encoders as oe
    torch.set_num_threads(os.cpu_count())
    t = tiles_host[:4].clone()
    oe.encode(cfg, weights, t[:1])
    t0 = time.perf_counter()
    oe.encode(cfg, weights, t[1:4])
    dt = time.perf_counter() - t0
    return {"value": 3 / dt, "unit": "tiles/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": "3 tiles of the request (after 1 warm-up tile), fp32 PyTorch CPU oracle "
                      "(oracle/encoders.py), rank 0"}


if __name__ == "__main__":
    main()
