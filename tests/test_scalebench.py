"""Scheduler-throughput benchmark (reference scalebench.py): the package's
restated shard stream equals the reference loop's, and running it through
the engine (one shard, or several workers as sub-clusters of one call)
reproduces the reference loop's schedule
(tests/golden/make_golden.py:scalebench_cases)."""
from __future__ import annotations

import numpy as np
import pytest

import digest as D
from conftest import oracle_args
from paper_2308_07470_b200 import scalebench as SB
from paper_2308_07470_b200.scheduler import PolicyConfig

KEYS = ["8x16", "32x4", "1x1", "64x128"]
OUT = ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome")


def _g(golden, key):
    g = golden["scalebench"][key]
    return g, g["n_models"], g["n_gpus"], g["keep"]


@pytest.mark.parametrize("key", KEYS)
def test_stream_and_schedule_oracle(key, golden):
    from oracle import oracle
    g, M, G, keep = _g(golden, key)
    ticks, midx = SB.shard_stream(2 * keep, M, G)
    assert D.trace_digest(ticks[:keep], midx[:keep]) == g["stream"]
    o = oracle.run(arr_ticks=ticks, arr_midx=midx,
                   **oracle_args(SB.shard_models(M), G, PolicyConfig("deferred")))
    assert D.requests_digest(*[o[k][:keep] for k in OUT]) == g["requests"]


def test_bench_point_properties():
    p = SB.BenchPoint(2, 128, 64, 1000, 0.5)
    assert p.throughput_rps == 2000.0 and p.cost_per_decision_us == 500.0
    z = SB.BenchPoint(0, 128, 64, 0, 0.0)
    assert z.throughput_rps == 0.0 and z.cost_per_decision_us == 0.0
    assert SB.bench_workers(0, 64, 128, 1.0).requests == 0


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_schedule_engine(key, golden):
    from paper_2308_07470_b200.simulator import Engine
    g, M, G, keep = _g(golden, key)
    ticks, midx = SB.shard_stream(2 * keep, M, G)
    res = Engine(SB.shard_models(M), G, PolicyConfig("deferred")).run_stream(ticks, midx, 1.0)
    assert D.requests_digest(*[getattr(res, k)[:keep] for k in OUT]) == g["requests"]


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [2, 8])
def test_workers_as_subclusters(workers, golden):
    """`workers` shards in one engine call: every shard's schedule is the
    single-shard reference schedule."""
    from paper_2308_07470_b200.simulator import Engine
    from paper_2308_07470_b200.profile import ModelSpec
    g, M, G, keep = _g(golden, "8x16")
    t, m = SB._workers_stream(2 * keep, workers, M, G)
    models = [ModelSpec(w * M + x.model_id, f"w{w}_{x.name}", x.profile, x.slo_ns)
              for w in range(workers) for x in SB.shard_models(M)]
    eng = Engine(models, G * workers, PolicyConfig("deferred"),
                 shards=(np.repeat(np.arange(workers), M), [G] * workers))
    res = eng.run_stream(t, m, 1.0)
    for w in range(workers):
        sel = np.nonzero(m // M == w)[0][:keep]
        assert D.requests_digest(*[getattr(res, k)[sel] for k in OUT]) == g["requests"]


@pytest.mark.gpu
def test_scale_bench_runs():
    r = SB.scale_bench([1, 2], [4], 0.05, total_models=16, total_gpus=32)
    assert [p.workers for p in r["workers"]] == [1, 2]
    assert all(p.requests > 0 and p.elapsed_s > 0 for p in r["workers"] + r["gpus"])


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_schedule_engine_stepped(key, golden):
    """The reference loop's granularity through the step API (scalebench.py:
    67-84): chunks of arrivals, each step up to the next chunk's first
    tick, state on the device between steps -- the reference schedule."""
    from paper_2308_07470_b200.simulator import Engine
    g, M, G, keep = _g(golden, key)
    ticks, midx = SB.shard_stream(2 * keep, M, G)
    eng = Engine(SB.shard_models(M), G, PolicyConfig("deferred"))
    chunk = max(1, keep // 7)
    for lo in range(0, len(ticks), chunk):
        hi = min(len(ticks), lo + chunk)
        eng.step(ticks[lo:hi], midx[lo:hi], int(ticks[hi]) if hi < len(ticks) else eng.DRAIN)
    res = eng.step_result(1.0)
    assert D.requests_digest(*[getattr(res, k)[:keep] for k in OUT]) == g["requests"]
    eng.close()


@pytest.mark.gpu
def test_scale_bench_step_mode_runs():
    r = SB.scale_bench([1, 2], [4], 0.05, total_models=16, total_gpus=32, mode="step")
    assert [p.workers for p in r["workers"]] == [1, 2]
    assert all(p.requests > 0 and p.elapsed_s > 0 for p in r["workers"] + r["gpus"])
