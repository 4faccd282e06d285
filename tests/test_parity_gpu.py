"""GPU parity: the CUDA engine against the reference fixtures (tests/golden)
and against the C oracle on the same inputs.  Bit-exact for every
per-request decision, batch composition, GPU assignment and counter."""
import numpy as np
import pytest

import cases
import digest as D
from conftest import oracle_args
from oracle import oracle
from resultcheck import check_against_golden, check_stats

pytestmark = pytest.mark.gpu

SMALL = list(cases.bundled()) + list(cases.stress())
CONFIGS = list(cases.config_cases())


def _engine(models, gpus, policy, **kw):
    from paper_2308_07470_b200 import Engine
    return Engine(models, gpus, policy, **kw)


def _run(case, **kw):
    key, models, gpus, policy, ticks, midx, _ = case
    eng = _engine(models, gpus, policy, **kw)
    res = eng.run_stream(ticks, midx, 1.0)
    return eng, res


def _counters(eng, res):
    return {"drops": res.drops, "completions": res.completions, "late": res.late,
            "ops": eng.rank.ops, "evictions": eng.rank.evictions,
            "registrations": eng.rank.registrations,
            "handler_ops_max": eng.handler_ops_max}


@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
def test_engine_trace_parity(case, golden):
    """record_trace: exact reference event trace (serial-scan path)."""
    eng, res = _run(case, record_trace=True, check_invariants=True)
    g = golden[case[0]]
    check_against_golden(g, res.req_dispatch, res.req_start, res.req_finish, res.req_batch,
                         res.req_outcome, res.gpu_logs, _counters(eng, res), trace=res.trace)
    eng.close()


@pytest.mark.parametrize("use_fast", [True, False], ids=["fast", "chain"])
@pytest.mark.parametrize("case", SMALL + CONFIGS, ids=[c[0] for c in SMALL + CONFIGS])
def test_engine_default_path_parity(case, use_fast, golden):
    """Default path (fresh-start pre-scan + parallel validated fast path, with
    the chain as fallback) and the chain alone, vs the reference digests and
    the oracle's arrays, plus compute_stats on the engine's RunResult."""
    key, models, gpus, policy, ticks, midx, (dur, warm, cool) = case
    eng = _engine(models, gpus, policy, use_fast=use_fast)
    res = eng.run_stream(ticks, midx, dur)
    g = golden[key]
    check_against_golden(g, res.req_dispatch, res.req_start, res.req_finish, res.req_batch,
                         res.req_outcome, res.gpu_logs, _counters(eng, res))
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
        np.testing.assert_array_equal(getattr(res, k), o[k], err_msg=k)
    check_stats(res, g, dur, warm, cool)
    if use_fast and key[:2] in ("C1", "C2", "C3", "C4", "C5") and "/base" in key:
        assert eng.stats["fast_shards"] == 1, "underload config must take the fast path"
    if not use_fast:
        assert eng.stats["fast_shards"] == 0
    eng.close()


def test_c4_sharded_single_call(golden):
    """All 8 C4 sub-clusters in ONE engine call equal the per-shard
    reference runs."""
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.simulator import Engine
    from paper_2308_07470_b200.workload import generate_arrivals
    dur = cases.GOLDEN_DURATIONS["C4"]
    sc = configs.c4(dur)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
    res = eng.run_stream(ticks, midx, dur)
    assert eng.stats["fast_shards"] == 8
    for s, (ms, g, ids) in enumerate(configs.shard_scenarios(sc)):
        sel = (midx >= ids[0]) & (midx <= ids[-1])
        gk = golden[f"C4s{s}/base@{dur}"]
        assert D.requests_digest(res.req_dispatch[sel], res.req_start[sel], res.req_finish[sel],
                                 res.req_batch[sel], res.req_outcome[sel]) == gk["requests"]
        logs = [[(a, b, m - ids[0], z) for a, b, m, z in res.gpu_logs[gg]]
                for gg in range(1024 * s, 1024 * (s + 1))]
        assert D.gpu_logs_digest(logs) == gk["gpu_logs"]
    eng.close()


def test_device_resident_entry_matches_host_entry():
    import torch
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.simulator import Engine
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c3(0.25)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 0.25, 42)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
    host = eng.run_stream(ticks, midx, 0.25)
    t = torch.from_numpy(ticks).cuda()
    m = torch.from_numpy(midx.astype(np.int32)).cuda()
    out, cnt = eng.run_device(t, m)
    n = len(ticks)
    for k, ref in (("dispatch", host.req_dispatch), ("start", host.req_start),
                   ("finish", host.req_finish), ("batch", host.req_batch),
                   ("outcome", host.req_outcome)):
        np.testing.assert_array_equal(out[k][:n].cpu().numpy(), ref, err_msg=k)
    assert cnt["n_batches"] == len(host.batches)
    eng.close()


def test_edge_cases():
    from paper_2308_07470_b200 import Engine, PolicyConfig, ProtocolError
    from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
    from paper_2308_07470_b200.units import ms_to_ns
    unit = [ModelSpec(0, "m0", LatencyProfile.linear(1.0, 5.0, 16), ms_to_ns(12.0)),
            ModelSpec(1, "m1", LatencyProfile.linear(0.5, 2.0, 1), ms_to_ns(9.0))]
    pol = PolicyConfig("deferred")

    def both(ticks, midx, gpus=1, models=unit, policy=pol):
        ticks = np.asarray(ticks, np.int64)
        midx = np.asarray(midx, np.int64)
        res = Engine(models, gpus, policy).run_stream(ticks, midx, 1.0)
        o = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
        for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
            np.testing.assert_array_equal(getattr(res, k), o[k], err_msg=k)
        return res

    res = both([], [])  # empty stream
    assert res.n_requests == 0 and len(res.batches) == 0
    both([0], [0])  # a single request
    both([5] * 40, [0, 1] * 20)  # one tick, max_batch 1 on m1
    both([5] * 40, [0] * 40, gpus=3, policy=PolicyConfig("eager"))
    tiny = [ModelSpec(0, "t", LatencyProfile.linear(1.0, 5.0, 8), ms_to_ns(6.0) + 1)]
    r = both(np.arange(0, 100) * 1000, [0] * 100, models=tiny,
             policy=PolicyConfig("deferred", d_ctrl_ns=10, d_data_ns=1))
    assert r.drops == 100  # d_ctrl + d_data + l(1) > SLO: everything dropped
    with pytest.raises(ProtocolError):
        Engine(unit, 1, pol).run_stream(np.array([0, 1]), np.array([0, 2]), 1.0)
    # many models, almost all idle; a large GPU pool with one request
    many = [ModelSpec(i, f"m{i}", LatencyProfile.linear(0.25 + 0.01 * (i % 7), 1.0 + i % 5, 256),
                      ms_to_ns(20.0 + i % 13)) for i in range(1000)]
    both([0, 0, 3, 1_000_000], [999, 0, 500, 999], gpus=8192, models=many)
    # one tick, full max_batch batches across several models and GPUs, each policy
    burst_t = [7_000] * 3000
    burst_m = [(k * 7) % 5 for k in range(3000)]
    for pk in ("deferred", "eager", "timeout"):
        kw = {"timeout_slo_frac": 0.3} if pk == "timeout" else {}
        both(burst_t, burst_m, gpus=4, models=many[:5], policy=PolicyConfig(pk, **kw))


def test_goodput_search_known_answers(golden):
    """goodput_search (a caller of run_scenario) on the engine reproduces the
    reference's probes and results bit for bit (Table 2 scenarios)."""
    from paper_2308_07470_b200 import goodput_search, load_scenario
    for name, want in golden["known_answers"]["goodput_search"].items():
        res = goodput_search(load_scenario(name))
        assert res.rate_rps == want["rate_rps"]
        assert [list(p) for p in res.probes] == [list(p) for p in want["probes"]]


def test_window_counts_and_autoscale_on_device(golden):
    """sym_window_counts (device reductions) equals the host reductions, and
    the C5 active-GPU series from the engine's result equals the reference."""
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.metrics import autoscale_series
    from paper_2308_07470_b200.parallel import window_counts_host
    from paper_2308_07470_b200.simulator import Engine
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c5(0.6)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 0.6, 42)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
    res = eng.run_stream(ticks, midx, 0.6)
    assert autoscale_series(res, 0.025, 0.6) == golden["C5/autoscale_series@0.6"]
    assert autoscale_series(res, 0.025, 0.6, engine=eng) == golden["C5/autoscale_series@0.6"]
    for lo, hi in ((0, 600_000_000), (60_000_000, 540_000_000), (1234567, 7654321)):
        dev = eng.window_counts(lo, hi)
        b = res.batches
        host = window_counts_host(res.req_model, res.req_arrival, res.req_outcome, b["gpu"],
                                  b["start"], b["finish"], len(sc.models), sc.gpu_count, lo, hi)
        for k in host:
            np.testing.assert_array_equal(dev[k], host[k], err_msg=k)
    eng.close()


JIT = list(cases.jitter())


@pytest.mark.parametrize("use_fast", [True, False], ids=["fast", "chain"])
@pytest.mark.parametrize("case", JIT, ids=[c[0] for c in JIT])
def test_engine_jitter_parity(case, use_fast, golden):
    """Jittered network on the device: per-dispatch Philox draws and the
    per-GPU serialisation reproduce the reference (starts, finishes, LATE
    outcomes, gpu_logs, trace) exactly."""
    from paper_2308_07470_b200.network import jitter_tables
    key, models, gpus, policy, ticks, midx, (dur, warm, cool), net, seed = case
    eng = _engine(models, gpus, policy, network=net, seed=seed, use_fast=use_fast,
                  record_trace=not use_fast)
    res = eng.run_stream(ticks, midx, dur)
    g = golden[key]
    check_against_golden(g, res.req_dispatch, res.req_start, res.req_finish, res.req_batch,
                         res.req_outcome, res.gpu_logs, _counters(eng, res),
                         trace=None if use_fast else res.trace)
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, net=jitter_tables(net, seed),
                   **oracle_args(models, gpus, policy))
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
        np.testing.assert_array_equal(getattr(res, k), o[k], err_msg=k)
    check_stats(res, g, dur, warm, cool)
    eng.close()
