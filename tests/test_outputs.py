"""Result files: the package's writers produce the
reference's summary.json / requests.csv / trace.csv / batch_hist.csv /
latency.csv / utilization.csv byte for byte (digests from
tests/golden/make_golden.py:output_cases, reference outputs.py)."""
from __future__ import annotations

import os

import pytest

import cases
import digest as D
from conftest import oracle_args
from resultcheck import oracle_result, oracle_trace
from paper_2308_07470_b200 import outputs as O
from paper_2308_07470_b200.metrics import compute_stats
from paper_2308_07470_b200.network import jitter_tables

OUT = list(cases.outputs())
FILES = ("summary.json", "requests.csv", "trace.csv", "batch_hist.csv", "latency.csv",
         "utilization.csv")


def _texts(res, st, g, device=None):
    return {
        "summary.json": O.summary_json(st, g["scenario"], g["seed"], g["extra"]),
        "requests.csv": O.requests_csv(res, device),
        "trace.csv": O.trace_csv(res),
        "batch_hist.csv": O.batch_hist_csv(st),
        "latency.csv": O.latency_csv(res, device),
        "utilization.csv": O.utilization_csv(res, st),
    }


def _check(texts, g):
    for name in FILES:
        assert len(texts[name]) == g["bytes"][name], name
        assert D.text_digest(texts[name]) == g["digests"][name], name


@pytest.mark.parametrize("case", OUT, ids=[c[0] for c in OUT])
def test_writers_match_reference_oracle(case, golden):
    """Oracle-scheduled run -> package writers == reference file bytes."""
    from oracle import oracle
    key, sc, ticks, midx = case
    g = golden[key]
    models = list(sc.models)
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, record_trace=True,
                   net=jitter_tables(sc.network, sc.seed),
                   **oracle_args(models, sc.gpu_count, sc.policy))
    res = oracle_result(o, models, sc.gpu_count, ticks, midx, sc.duration_s)
    res.trace = oracle_trace(o)
    st = compute_stats(res, sc.warmup_s, sc.cooldown_s, sc.duration_s)
    _check(_texts(res, st, g, device=None), g)


def test_write_run_outputs_atomic(tmp_path):
    from oracle import oracle
    key, sc, ticks, midx = OUT[0]
    models = list(sc.models)
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, record_trace=True,
                   **oracle_args(models, sc.gpu_count, sc.policy))
    res = oracle_result(o, models, sc.gpu_count, ticks, midx, sc.duration_s)
    res.trace = oracle_trace(o)
    st = compute_stats(res, sc.warmup_s, sc.cooldown_s, sc.duration_s)
    paths = O.write_run_outputs(str(tmp_path / "run"), sc.name, sc.seed, res, st, device=None)
    assert [os.path.basename(p) for p in paths] == list(FILES)
    assert not [f for f in os.listdir(tmp_path / "run") if f.startswith(".tmp-")]
    again = O.write_run_outputs(str(tmp_path / "run"), sc.name, sc.seed, res, st, device=None)
    assert again == paths


def test_sweep_rows_csv_format():
    rows = [dict(dimension="slo", value=25, policy="deferred", goodput_rps=1234.56789,
                 bad_rate=0.0123456789, idle_fraction=0.5, median_batch_size=7)]
    assert O.sweep_rows_csv(rows) == (O.SWEEP_HEADER + "\n"
                                      "slo,25,deferred,1234.568,0.012346,0.500000,7.0\n")


@pytest.mark.gpu
@pytest.mark.parametrize("case", OUT, ids=[c[0] for c in OUT])
def test_writers_match_reference_engine(case, golden):
    """CUDA-engine run -> package writers == reference file bytes."""
    from paper_2308_07470_b200.simulator import Engine
    key, sc, ticks, midx = case
    g = golden[key]
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, sc.network, seed=sc.seed,
                 record_trace=True)
    res = eng.run_stream(ticks, midx, sc.duration_s)
    st = compute_stats(res, sc.warmup_s, sc.cooldown_s, sc.duration_s)
    _check(_texts(res, st, g, device=0), g)
    _check(_texts(res, st, g, device=None), g)


def _synthetic(n, seed=0, names=None):
    import numpy as np
    from paper_2308_07470_b200.simulator import RunResult
    rng = np.random.default_rng(seed)
    names = names or [f"m{i}" for i in range(7)]
    arr = np.sort(rng.integers(0, 10**12, n))
    big = np.iinfo(np.int64)
    return RunResult(
        model_names=names, gpu_count=4, duration_ns=10**12,
        req_model=rng.integers(0, len(names), n), req_arrival=arr, req_deadline=arr,
        req_dispatch=np.where(rng.random(n) < 0.01, -1, arr + 7),
        req_start=rng.choice([big.min, big.max, -5, 0, 10**18], n) if seed else arr + 100,
        req_finish=arr + rng.integers(-10**9, 10**13, n),
        req_batch=rng.integers(-2, 10**6, n), req_outcome=rng.integers(-1, 3, n))


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed", [(0, 0), (1, 0), (255, 0), (256, 0), (257, 1),
                                    (100_003, 1), (3_000_001, 0)])
def test_gpu_rows_equal_host_rows(n, seed):
    """GPU rendering == host rendering on raw columns: ragged block tails,
    negative and extreme int64 values, unfinished (-1) outcomes."""
    res = _synthetic(n, seed)
    assert O.requests_csv(res, 0) == O.requests_csv(res, None)
    assert O.latency_csv(res, 0) == O.latency_csv(res, None)


@pytest.mark.gpu
def test_gpu_rows_unicode_and_long_names():
    names = ["résnet-50_α", "x" * 300, "", "bert,base"]
    res = _synthetic(5000, 2, names)
    assert O.requests_csv(res, 0) == O.requests_csv(res, None)
    assert O.latency_csv(res, 0) == O.latency_csv(res, None)


@pytest.mark.gpu
def test_gpu_rows_reject_bad_ids():
    res = _synthetic(1000, 0)
    res.req_model[500] = 7
    with pytest.raises(ValueError):
        O.requests_csv(res, 0)
    res = _synthetic(1000, 0)
    res.req_outcome[3] = 5
    with pytest.raises(ValueError):
        O.latency_csv(res, 0)
