"""Pin the C oracle (and this package's trace generator and compute_stats)
against fixtures produced by the Python reference (tests/golden)."""
import pytest

import cases
import digest as D
from conftest import oracle_args
from oracle import oracle
from resultcheck import (check_against_golden, check_stats, oracle_gpu_logs,
                         oracle_result, oracle_trace)

ALL = list(cases.bundled()) + list(cases.stress()) + list(cases.config_cases())


@pytest.mark.parametrize("case", ALL, ids=[c[0] for c in ALL])
def test_oracle_matches_reference(case, golden):
    key, models, gpus, policy, ticks, midx, (dur, warm, cool) = case
    g = golden[key]
    assert D.trace_digest(ticks, midx) == g["trace_in"], "arrival stream differs"
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, record_trace=True, check_invariants=len(ticks) < 50_000,
                   **oracle_args(models, gpus, policy))
    counters = {k: o[k] for k in ("drops", "completions", "late", "ops", "evictions",
                                   "registrations", "handler_ops_max")}
    check_against_golden(g, o["req_dispatch"], o["req_start"], o["req_finish"],
                         o["req_batch"], o["req_outcome"], oracle_gpu_logs(o, gpus),
                         counters, trace=oracle_trace(o))
    check_stats(oracle_result(o, models, gpus, ticks, midx, dur), g, dur, warm, cool)


def test_c4_full_stream_digest(golden):
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(0.1)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 0.1, 42)
    assert D.trace_digest(ticks, midx) == golden["C4/trace_in@0.1"]


def test_autoscale_series_c5(golden):
    """C5 active-GPU series from the oracle run, with the
    package's epoch reductions, equals the reference's compute_stats +
    autoscale_advice per epoch."""
    import numpy as np
    from conftest import oracle_args
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.metrics import autoscale_series
    from paper_2308_07470_b200.workload import generate_arrivals
    from resultcheck import oracle_result
    sc = configs.c5(0.6)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 0.6, 42)
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(list(sc.models), 4096, sc.policy))
    res = oracle_result(o, list(sc.models), 4096, ticks, midx, 0.6)
    assert autoscale_series(res, 0.025, 0.6) == golden["C5/autoscale_series@0.6"]


JIT = list(cases.jitter())


@pytest.mark.parametrize("case", JIT, ids=[c[0] for c in JIT])
def test_oracle_jitter_matches_reference(case, golden):
    """Jittered network: histogram delays drawn per dispatch from the
    engine's numpy Philox substream (network.py:69-77, scheduler.py:198-200);
    starts shift, GPUs serialise (simulator.py:54-62), LATE outcomes appear."""
    from paper_2308_07470_b200.network import jitter_tables
    key, models, gpus, policy, ticks, midx, (dur, warm, cool), net, seed = case
    g = golden[key]
    assert D.trace_digest(ticks, midx) == g["trace_in"]
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, record_trace=True,
                   net=jitter_tables(net, seed), **oracle_args(models, gpus, policy))
    counters = {k: o[k] for k in ("drops", "completions", "late", "ops", "evictions",
                                   "registrations", "handler_ops_max")}
    check_against_golden(g, o["req_dispatch"], o["req_start"], o["req_finish"],
                         o["req_batch"], o["req_outcome"], oracle_gpu_logs(o, gpus),
                         counters, trace=oracle_trace(o))
    check_stats(oracle_result(o, models, gpus, ticks, midx, dur), g, dur, warm, cool)


def test_philox_stream_matches_numpy():
    """The oracle/engine Philox4x64-10 restatement equals numpy's stream."""
    import numpy as np
    from paper_2308_07470_b200.network import DelayDist, NetworkModel, jitter_tables
    from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
    from paper_2308_07470_b200.scheduler import PolicyConfig
    vals = [1000, 7000, 50000, 200000]
    w = [0.4, 0.3, 0.2, 0.1]
    net = NetworkModel(DelayDist.histogram(vals, w), DelayDist.constant(0))
    t = jitter_tables(net, 7)
    # 300 singleton dispatches on one model / many GPUs: start - emitted = draw
    m = [ModelSpec(0, "m", LatencyProfile.linear(0.0, 1.0, 1), 10_000_000)]
    ticks = np.arange(300, dtype=np.int64) * 5_000_000
    o = oracle.run(arr_ticks=ticks, arr_midx=np.zeros(300, np.int64), net=t,
                   **oracle_args(m, 4, PolicyConfig("eager", d_ctrl_ns=0)))
    g = np.random.Generator(np.random.Philox(key=t.key))
    want = [int(g.choice(np.asarray(vals), p=np.asarray(w) / sum(w))) for _ in range(300)]
    got = list(o["ord_start"] - o["ord_emitted"])
    assert got == want
