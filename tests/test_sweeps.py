"""Grid sweeps (reference sweeps.py:67-142): rows equal
the reference's exactly (tests/golden/make_golden.py:sweep_cases).  The CPU
test drives the package's sweep/bisection logic over the oracle; the GPU
test runs every probe on the engine, serially and with concurrent searches."""
from __future__ import annotations

import pytest

from paper_2308_07470_b200 import metrics, sweeps
from paper_2308_07470_b200.scenario import load_scenario

CASES = [
    ("beta_ratio", "table2_resnet50", [1.0, 6.0], ["deferred", "eager"], None),
    ("timeout", "fig4b_timeout_sweep", [10.0, 60.0], None, None),
    ("offered_load", "table2_resnet50", [0.5, 1.25], None, 5000.0),
    ("slo", "table2_inceptionresnet", [40.0, 90.0], ["deferred", "timeout:30"], None),
]


def _check(rows, want):
    assert len(rows) == len(want)
    for r, w in zip(rows, want):
        assert r == w


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}/{c[1]}" for c in CASES])
def test_sweep_rows_oracle(case, golden, monkeypatch):
    from resultcheck import oracle_run_scenario
    monkeypatch.setattr(metrics, "run_scenario", oracle_run_scenario)
    monkeypatch.setattr(metrics, "BATCH_PROBES", False)
    monkeypatch.setattr(sweeps, "run_scenario", oracle_run_scenario)
    dim, name, grid, pols, peak = case
    rows = sweeps.run_sweep(dim, load_scenario(name), grid, pols, peak)
    _check(rows, golden["sweeps"][f"{dim}/{name}"])


def test_unknown_sweep_and_policy():
    sc = load_scenario("table2_resnet50")
    with pytest.raises(ValueError):
        sweeps.run_sweep("nope", sc, [1.0])
    with pytest.raises(ValueError):
        sweeps._policy(sc.policy, "greedy")


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [1, 4])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}/{c[1]}" for c in CASES])
def test_sweep_rows_engine(case, workers, golden):
    dim, name, grid, pols, peak = case
    rows = sweeps.run_sweep(dim, load_scenario(name), grid, pols, peak, workers=workers)
    _check(rows, golden["sweeps"][f"{dim}/{name}"])


@pytest.mark.parametrize("speculate", [1, 2, 3, 5])
def test_speculative_search_equals_sequential(speculate, golden, monkeypatch):
    """Concurrent speculative bisection walks the sequential path: same
    rate, same recorded probes (metrics.py:229-256 known answers)."""
    from resultcheck import oracle_run_scenario
    monkeypatch.setattr(metrics, "run_scenario", oracle_run_scenario)
    monkeypatch.setattr(metrics, "BATCH_PROBES", False)
    for name, want in golden["known_answers"]["goodput_search"].items():
        res = metrics.goodput_search(load_scenario(name), speculate=speculate)
        assert res.rate_rps == want["rate_rps"]
        assert [list(p) for p in res.probes] == [list(p) for p in want["probes"]]


def test_speculative_search_respects_max_iters(monkeypatch):
    from resultcheck import oracle_run_scenario
    monkeypatch.setattr(metrics, "run_scenario", oracle_run_scenario)
    monkeypatch.setattr(metrics, "BATCH_PROBES", False)
    sc = load_scenario("table2_inceptionresnet")
    for it in (1, 2, 4):
        a = metrics.goodput_search(sc, max_iters=it, keep_stats=True)
        b = metrics.goodput_search(sc, max_iters=it, keep_stats=True, speculate=3)
        assert a.rate_rps == b.rate_rps and a.probes == b.probes
        assert (a.stats_at_rate is None) == (b.stats_at_rate is None)
        if a.stats_at_rate is not None:
            assert a.stats_at_rate.goodput_rps == b.stats_at_rate.goodput_rps


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES[:2], ids=[f"{c[0]}/{c[1]}" for c in CASES[:2]])
def test_sweep_rows_engine_speculative(case, golden):
    dim, name, grid, pols, peak = case
    rows = sweeps.run_sweep(dim, load_scenario(name), grid, pols, peak, workers=4,
                            speculate=3)
    _check(rows, golden["sweeps"][f"{dim}/{name}"])


@pytest.mark.gpu
@pytest.mark.parametrize("speculate", [2, 3])
def test_batched_speculative_search_on_engine(speculate, golden):
    """Speculative rounds as sub-clusters of one engine call reproduce the
    sequential search exactly (rate and recorded probes)."""
    for name, want in golden["known_answers"]["goodput_search"].items():
        res = metrics.goodput_search(load_scenario(name), speculate=speculate, keep_stats=True)
        assert res.rate_rps == want["rate_rps"]
        assert [list(p) for p in res.probes] == [list(p) for p in want["probes"]]
        seq = metrics.goodput_search(load_scenario(name), keep_stats=True)
        assert res.stats_at_rate == seq.stats_at_rate


@pytest.mark.gpu
def test_probe_batch_equals_single_probes():
    sc = load_scenario("fig4b_timeout_zoo")
    rates = [sc.workload.rate_rps * f for f in (0.5, 0.9, 1.3, 2.0)] if hasattr(
        sc.workload, "rate_rps") else None
    if rates is None:
        pytest.skip("scenario has no scalar rate")
    batched = metrics.probe_batch(sc, rates)
    for r, (ok, st) in zip(rates, batched):
        ok1, st1 = metrics.probe_feasible(sc, r)
        assert ok == ok1 and st == st1
