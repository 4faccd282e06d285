"""Compare scheduler outputs against golden digests / each other."""
from __future__ import annotations

import numpy as np

import digest as D
from paper_2308_07470_b200 import _native
from paper_2308_07470_b200.metrics import compute_stats
from paper_2308_07470_b200.simulator import RunResult
from paper_2308_07470_b200.units import s_to_ns

TRACE_NAMES = ("dispatch", "drop", "shrink")


def oracle_trace(o):
    tr = o["trace"]
    out = []
    for i in range(len(tr["t"])):
        rids = tuple(int(x) for x in tr["rids"][tr["rid_off"][i]:tr["rid_off"][i + 1]])
        out.append((int(tr["t"][i]), TRACE_NAMES[tr["kind"][i]], int(tr["model"][i]),
                    int(tr["gpu"][i]), int(tr["size"][i]), int(tr["start"][i]),
                    int(tr["finish"][i]), rids))
    return out


def oracle_gpu_logs(o, gpus):
    logs = [[] for _ in range(gpus)]
    for g, s, f, m, b in zip(o["ord_gpu"], o["ord_start"], o["ord_finish"], o["ord_model"],
                             o["ord_size"]):
        logs[int(g)].append((int(s), int(f), int(m), int(b)))
    return logs


def oracle_result(o, models, gpus, ticks, midx, duration_s) -> RunResult:
    """RunResult view of an oracle run (for compute_stats)."""
    nb = len(o["ord_gpu"])
    b = np.zeros(nb, dtype=_native.BATCH_DTYPE)
    for k_src, k_dst in (("ord_gpu", "gpu"), ("ord_start", "start"), ("ord_finish", "finish"),
                         ("ord_model", "model"), ("ord_size", "size"),
                         ("ord_emitted", "emitted")):
        b[k_dst] = o[k_src]
    slo = np.array([m.slo_ns for m in models], np.int64)
    return RunResult(model_names=[m.name for m in models], gpu_count=gpus,
                     duration_ns=s_to_ns(duration_s), req_model=np.asarray(midx, np.int64),
                     req_arrival=np.asarray(ticks, np.int64),
                     req_deadline=np.asarray(ticks, np.int64) + slo[np.asarray(midx)],
                     req_dispatch=o["req_dispatch"], req_start=o["req_start"],
                     req_finish=o["req_finish"], req_batch=o["req_batch"],
                     req_outcome=o["req_outcome"], drops=o["drops"],
                     completions=o["completions"], late=o["late"], batches=b)


def check_stats(res: RunResult, g: dict, dur, warm, cool):
    st = compute_stats(res, warm, cool, dur)
    gs = g["stats"]
    assert st.goodput_rps == gs["goodput_rps"]
    assert st.bad_rate == gs["bad_rate"]
    assert st.mean_idle_fraction == gs["mean_idle_fraction"]
    assert D._h(np.asarray(st.gpu_idle_fraction).view(np.int64)) == gs["idle_digest"]
    assert [m.p99_latency_ns for m in st.models] == gs["p99"]
    assert [m.median_batch for m in st.models] == gs["median_batch"]
    assert [m.max_queueing_delay_ns for m in st.models] == gs["max_qd"]
    assert D._h([x for m in st.models for kv in sorted(m.batch_hist.items())
                 for x in kv]) == gs["hist_digest"]


def check_against_golden(g: dict, dispatch, start, finish, batch, outcome, gpu_logs,
                         counters: dict, trace=None):
    assert D.requests_digest(dispatch, start, finish, batch, outcome) == g["requests"]
    assert D.gpu_logs_digest(gpu_logs) == g["gpu_logs"]
    for k, v in counters.items():
        assert v == g[k], f"{k}: {v} != golden {g[k]}"
    if trace is not None:
        assert D.event_trace_digest(trace) == g["events"]


def oracle_run_scenario(scenario, record_trace=False, check_invariants=False):
    """run_scenario on the CPU oracle (test infrastructure: lets the CPU
    suite exercise the host callers -- goodput_search, sweeps -- whose GPU
    runs go through the engine)."""
    from conftest import oracle_args
    from oracle import oracle
    from paper_2308_07470_b200.network import jitter_tables
    from paper_2308_07470_b200.workload import generate_arrivals
    assert scenario.shards is None
    models = list(scenario.models)
    ticks, midx = generate_arrivals(scenario.workload, [m.name for m in models],
                                    scenario.duration_s, scenario.seed)
    o = oracle.run(arr_ticks=ticks, arr_midx=midx, record_trace=record_trace,
                   net=jitter_tables(scenario.network, scenario.seed),
                   **oracle_args(models, scenario.gpu_count, scenario.policy))
    res = oracle_result(o, models, scenario.gpu_count, ticks, midx, scenario.duration_s)
    if record_trace:
        res.trace = oracle_trace(o)
    return res
