"""Intra-request parallelism (IRP) routing on the host.

Mirrors the reference's encode-side routing so tile partitioning is bit-exact:

* :func:`irp_shard` -- engine.irp_shard (engine.py:55-62), evaluated by the C ABI
  (``epd_irp_shard``) so the Python host and any C/C++ caller share one routine;
* :func:`shard_ranges` -- worker k's contiguous tile range in request order
  (the order engine._start_encode assigns shards, engine.py:589-602);
* :func:`plan_batch` -- the multi-request batch plan of engine._start_encode
  (engine.py:583-602): zero shards dropped, text-only requests -> [(0, 0)],
  every request restarts at worker 0;
* :func:`assign_instance` -- engine.assign_instance (engine.py:65-78): which encode /
  prefill / decode instance takes a request (round-robin counter or least-loaded);
* :func:`form_batch` -- engine.form_batch (engine.py:81-93): the longest FCFS prefix that
  fits (the first misfit stops the batch);
* :func:`ep_bytes` / :func:`pd_bytes` -- EP/PD migration byte counts
  (engine.py:524, 553-554).
"""
from __future__ import annotations

import ctypes as C

from ._lib import call


def irp_shard(patches: int, width: int) -> list[int]:
    if not isinstance(width, int) or width < 1:
        raise ValueError("shard width must be >= 1")
    counts = (C.c_int64 * width)()
    call("epd_irp_shard", int(patches), int(width), counts)
    return [int(c) for c in counts]


def shard_ranges(patches: int, width: int) -> list[tuple[int, int]]:
    """[(first_tile, n_tiles)] per worker 0..width-1."""
    if not isinstance(width, int) or width < 1:
        raise ValueError("shard width must be >= 1")
    first = (C.c_int64 * width)()
    counts = (C.c_int64 * width)()
    call("epd_irp_ranges", int(patches), int(width), first, counts)
    return [(int(first[k]), int(counts[k])) for k in range(width)]


def plan_batch(patches_per_request: list[int], width: int):
    """(shards per request [(worker, tiles)], worker tile load, worker request count)."""
    worker_load = [0] * width
    worker_reqs = [0] * width
    shards = []
    for p in patches_per_request:
        s = [(0, 0)] if p == 0 else [(k, c) for k, c in enumerate(irp_shard(p, width)) if c > 0]
        shards.append(s)
        for k, c in s:
            worker_load[k] += c
            worker_reqs[k] += 1
    return shards, worker_load, worker_reqs


def _policy_name(policy) -> str:
    return getattr(policy, "value", policy)


def assign_instance(policy, candidates, rr_counter: int = 0) -> tuple[int, int]:
    """(instance id, next round-robin counter) from ordered (id, load) candidates.

    ``policy``: "fcfs" / "round_robin" / "least_loaded" or the reference's SchedulePolicy.
    Least-loaded takes the minimum load, ties to the lowest id, and leaves the counter;
    any other policy cycles through the candidates with the counter (engine.py:65-78)."""
    if not candidates:
        raise ValueError("no candidate instances")
    if _policy_name(policy) == "least_loaded":
        iid, _ = min(candidates, key=lambda pair: (pair[1], pair[0]))
        return iid, rr_counter
    iid, _ = candidates[rr_counter % len(candidates)]
    return iid, rr_counter + 1


def form_batch(queue, max_batch: int, fits) -> list:
    """Longest FCFS prefix of ``queue`` (up to ``max_batch``) whose members fit; ``fits`` is
    called once per accepted head and may commit reservations (engine.py:81-93)."""
    batch = []
    for item in queue:
        if len(batch) >= max_batch or not fits(item):
            break
        batch.append(item)
    return batch


def poisson_arrivals(rate: float, n: int, seed: int) -> list[float]:
    """Arrival times of workload.generate_poisson (workload.py:71-96): the cumulative sum of
    ``n`` seeded exponential gaps with mean 1 / rate (numpy PCG64 ``default_rng(seed)``)."""
    import numpy as np
    if rate <= 0 or n < 1:
        raise ValueError("rate must be positive and n >= 1")
    gaps = np.random.default_rng(seed).exponential(1.0 / rate, size=n)
    return [float(t) for t in np.cumsum(gaps)]


def ep_bytes(tiles: int, tokens_per_patch: int, mm_bytes_per_token: int) -> int:
    return tiles * tokens_per_patch * mm_bytes_per_token


def pd_bytes(total_tokens: int, kv_bytes_per_token: int) -> int:
    return total_tokens * kv_bytes_per_token
