"""Scheduler-throughput benchmark (mirrors batchsym/scalebench.py).

The reference drives one scheduler shard per worker process with a
synthetic saturated stream -- model ids round-robin, a fixed virtual gap at
80% of the shard's staggered capacity (scalebench.py:49-85) -- and reports
requests pushed per wall second.  Here the same stream is generated up
front and every worker's shard becomes one sub-cluster of a single engine
call (independent sub-clusters, simulator shards), so ``workers`` scales the
work handed to the GPU in one launch sequence.  Because the engine consumes
whole streams, the duration is met by growing the stream geometrically until
one call takes at least ``duration_s / 4`` of wall time (or the request cap
is reached); the last call is the measurement.  Each shard's schedule is
the reference's run_stream on the same stream (tests/test_scalebench.py).

``mode="step"`` drives the engine the way the reference's ``_shard_loop``
drives its Engine (scalebench.py:67-84): arrivals are generated and fed
chunk by chunk through the step API (Engine.step, sym_step), each step
processing every event up to the next chunk's first tick, with the
scheduler state resident on the device between steps, until
``duration_s`` of wall time has passed.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .profile import LatencyProfile, ModelSpec
from .scheduler import PolicyConfig
from .units import ms_to_ns

BENCH_ALPHA_MS = 1.0
BENCH_BETA_MS = 5.0
BENCH_SLO_MS = 25.0
BENCH_MAX_BATCH = 32
MAX_REQUESTS = 1 << 27


@dataclass(frozen=True)
class BenchPoint:
    workers: int
    gpus: int
    models: int
    requests: int
    elapsed_s: float

    @property
    def throughput_rps(self) -> float:
        return self.requests / self.elapsed_s if self.elapsed_s > 0 else 0.0

    @property
    def cost_per_decision_us(self) -> float:
        return 1e6 * self.elapsed_s / self.requests if self.requests else 0.0


def shard_models(n_models: int) -> list[ModelSpec]:
    profile = LatencyProfile.linear(BENCH_ALPHA_MS, BENCH_BETA_MS, max_batch=BENCH_MAX_BATCH)
    slo = ms_to_ns(BENCH_SLO_MS)
    return [ModelSpec(i, f"bench{i}", profile, slo) for i in range(n_models)]


def shard_gap_ns(n_gpus: int) -> int:
    """Virtual arrival gap: ~80% of the staggered capacity at batch 16
    (scalebench.py:58-62)."""
    profile = LatencyProfile.linear(BENCH_ALPHA_MS, BENCH_BETA_MS, max_batch=BENCH_MAX_BATCH)
    bs = 16
    cap_rps = n_gpus * bs * 1e9 / profile.latency(bs)
    return max(1, int(1e9 / (0.8 * cap_rps)))


def shard_stream(n: int, n_models: int, n_gpus: int) -> tuple[np.ndarray, np.ndarray]:
    """The first n arrivals of one shard's stream: request k (0-based)
    arrives at k*gap for model k mod n_models (scalebench.py:67-80)."""
    k = np.arange(n, dtype=np.int64)
    return k * shard_gap_ns(n_gpus), k % n_models


def _workers_stream(n: int, workers: int, n_models: int, n_gpus: int):
    """`workers` copies of the shard stream, model ids offset per shard,
    merged in tick order (shard order within a tick)."""
    ticks, midx = shard_stream(n, n_models, n_gpus)
    t = np.repeat(ticks, workers)
    m = (np.tile(np.arange(workers, dtype=np.int64) * n_models, n)
         + np.repeat(midx, workers))
    return t, m


def _engine(workers: int, n_models: int, n_gpus: int, device: int):
    from .simulator import Engine
    models = [ModelSpec(w * n_models + m.model_id, f"w{w}_{m.name}", m.profile, m.slo_ns)
              for w in range(workers) for m in shard_models(n_models)]
    shards = None
    if workers > 1:
        shards = (np.repeat(np.arange(workers), n_models), [n_gpus] * workers)
    return Engine(models, n_gpus * workers, PolicyConfig("deferred"), shards=shards,
                  device=device)


STEP_CHUNK = 1 << 16  # arrivals per shard per step


def _run_steps(workers: int, n_models: int, n_gpus: int, duration_s: float, device: int,
               chunk: int = STEP_CHUNK) -> tuple[int, float]:
    """The reference's saturated loop through the step API: chunk k holds
    the shard requests [k*chunk, (k+1)*chunk) of every worker; the step
    processes every event up to the next chunk's first tick."""
    eng = _engine(workers, n_models, n_gpus, device)
    gap = shard_gap_ns(n_gpus)
    try:
        eng.reset_steps()
        n = 0
        t0 = time.perf_counter()
        deadline = t0 + duration_s
        while True:
            k = np.arange(n, n + chunk, dtype=np.int64)
            t = np.repeat(k * gap, workers)
            m = (np.tile(np.arange(workers, dtype=np.int64) * n_models, chunk)
                 + np.repeat(k % n_models, workers))
            n += chunk
            eng.step(t, m, n * gap)
            if time.perf_counter() >= deadline or n * workers * 2 > MAX_REQUESTS:
                break
        return n * workers, time.perf_counter() - t0
    finally:
        eng.close()


def _run(workers: int, n_models: int, n_gpus: int, n: int, device: int) -> float:
    eng = _engine(workers, n_models, n_gpus, device)
    try:
        t, m = _workers_stream(n, workers, n_models, n_gpus)
        eng.run_stream(t, m, 1.0)  # warm: buffers sized, kernels loaded
        t0 = time.perf_counter()
        eng.run_stream(t, m, 1.0)
        return time.perf_counter() - t0
    finally:
        eng.close()


def _measure(workers: int, n_models: int, n_gpus: int, duration_s: float,
             device: int, mode: str = "whole") -> tuple[int, float]:
    if mode == "step":
        return _run_steps(workers, n_models, n_gpus, duration_s, device)
    if mode != "whole":
        raise ValueError(f"unknown mode {mode!r}")
    n = 1 << 14
    while True:
        el = _run(workers, n_models, n_gpus, n, device)
        if el >= duration_s / 4 or n * workers * 2 > MAX_REQUESTS:
            return n * workers, el
        n *= 2


def bench_workers(workers: int, total_models: int, total_gpus: int, duration_s: float,
                  device: int = 0, mode: str = "whole") -> BenchPoint:
    """Aggregate throughput with the model set sharded `workers` ways
    (scalebench.py:92-118)."""
    if workers == 0:
        return BenchPoint(0, total_gpus, total_models, 0, duration_s)
    n_models = max(1, total_models // workers)
    n_gpus = max(1, total_gpus // workers)
    n, el = _measure(workers, n_models, n_gpus, duration_s, device, mode)
    return BenchPoint(workers, total_gpus, total_models, n, el)


def bench_gpu_scaling(gpu_counts: list[int], duration_s: float, n_models: int = 32,
                      device: int = 0, mode: str = "whole") -> list[BenchPoint]:
    """Per-decision cost versus the GPU count of one shard (scalebench.py:121-129)."""
    points = []
    for g in gpu_counts:
        n, el = _measure(1, n_models, g, duration_s, device, mode)
        points.append(BenchPoint(1, g, n_models, n, el))
    return points


def scale_bench(worker_counts: list[int], gpu_counts: list[int], duration_s: float,
                total_models: int = 64, total_gpus: int = 128, device: int = 0,
                mode: str = "whole") -> dict:
    """Both dimensions: {'workers': [...], 'gpus': [...]} (scalebench.py:132-139).
    mode: "whole" (one engine call per measurement) or "step" (the
    reference's step loop through Engine.step)."""
    return {"workers": [bench_workers(w, total_models, total_gpus, duration_s, device, mode)
                        for w in worker_counts],
            "gpus": bench_gpu_scaling(gpu_counts, duration_s, device=device, mode=mode)}
