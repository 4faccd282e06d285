"""compute_stats with the device reductions (sym_window_stats, SURVEY §8f
row 2) equals the host computation field for field: counts, goodput, bad
rate, per-GPU idle fractions, per-model p99 (nearest rank, drops as +inf),
largest queueing delay, batch histograms and median batch -- on bundled,
jittered (LATE outcomes), overloaded and sharded runs."""
from __future__ import annotations

import pytest

import cases

pytestmark = pytest.mark.gpu

BUNDLED = [c for c in cases.bundled() if c[0].endswith(("/base", "/eager", "/timeout30"))]
JIT = list(cases.jitter())
STRESS = list(cases.stress(60))[::3]


def _check(eng, res, dur, warm, cool):
    from paper_2308_07470_b200.metrics import compute_stats
    host = compute_stats(res, warm, cool, dur)
    dev = compute_stats(res, warm, cool, dur, engine=eng)
    assert dev == host


@pytest.mark.parametrize("case", BUNDLED + STRESS, ids=[c[0] for c in BUNDLED + STRESS])
def test_device_stats_equal_host(case):
    from paper_2308_07470_b200.simulator import Engine
    key, models, gpus, policy, ticks, midx, (dur, warm, cool) = case
    eng = Engine(models, gpus, policy)
    res = eng.run_stream(ticks, midx, dur)
    _check(eng, res, dur, warm, cool)
    _check(eng, res, dur, 0.0, 0.0)
    eng.close()


@pytest.mark.parametrize("case", JIT, ids=[c[0] for c in JIT])
def test_device_stats_equal_host_jittered(case):
    from paper_2308_07470_b200.simulator import Engine
    key, models, gpus, policy, ticks, midx, (dur, warm, cool), net, seed = case
    eng = Engine(models, gpus, policy, net, seed=seed)
    res = eng.run_stream(ticks, midx, dur)
    _check(eng, res, dur, warm, cool)
    eng.close()


def test_device_stats_sharded_c4():
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.simulator import Engine
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(1.0)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 1.0, 42)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
    res = eng.run_stream(ticks, midx, 1.0)
    _check(eng, res, 1.0, 0.1, 0.1)
    eng.close()


def test_auto_device_stats_for_large_runs():
    """The package's own callers reduce a large fresh result on the device
    (_fresh_stats); plain compute_stats reduces the result's arrays, so an
    edited result gets the host answer for the edit; a stale result never
    reaches the device -- same numbers whenever the arrays are unedited."""
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.metrics import _fresh_stats, compute_stats
    from paper_2308_07470_b200.simulator import Engine
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(1.0)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 1.0, 42)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
    res = eng.run_stream(ticks, midx, 1.0)
    assert res.n_requests >= 200_000 and res.device_engine() is eng
    dev = _fresh_stats(sc, res)
    host = compute_stats(res, 0.1, 0.1, 1.0)
    assert dev == host == compute_stats(res, 0.1, 0.1, 1.0, engine=eng)
    edited = res.req_outcome.copy()
    res.req_outcome[: len(edited) // 2] = 2  # the caller edits the result
    assert compute_stats(res, 0.1, 0.1, 1.0).dropped > host.dropped
    res.req_outcome[:] = edited
    res2 = eng.run_stream(ticks[: len(ticks) // 2], midx[: len(midx) // 2], 1.0)
    assert res.device_engine() is None and res2.device_engine() is eng  # res is stale now
    assert _fresh_stats(sc, res) == host
    eng.close()
    assert res2.device_engine() is None
