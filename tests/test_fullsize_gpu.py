"""BASELINE.json's configurations at FULL size (C4: 1000 models x 8192 GPUs,
60 s, ~72M requests; C3: 100 models x 1024 GPUs, 60 s Gamma-bursty, ~18M).

Two kinds of evidence at the size the benchmark runs:
* bit-exact parity with the CPU oracle on sampled C4 sub-clusters at their
  full 60 s length (~9M requests each), and
* size-independent properties of the whole run: every request resolved
  exactly once, service within its deadline, per-GPU busy intervals that
  never overlap, per-model FIFO service, batch sizes summing to the served
  count and within max_batch, l(b)-consistent finish times.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import oracle_args

pytestmark = pytest.mark.gpu


def _workload(name, dur):
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.CONFIGS[name](dur)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
    return sc, ticks, midx


def _check_properties(sc, res, ticks, midx):
    models = list(sc.models)
    n = len(ticks)
    stride = max(m.profile.max_batch for m in models)
    lat = np.stack([m.profile.table_array(stride) for m in models])
    slo = np.array([m.slo_ns for m in models], np.int64)
    mb = np.array([m.profile.max_batch for m in models], np.int64)
    o = res.req_outcome
    assert set(np.unique(o).tolist()) <= {0, 2}  # no jitter: completed or dropped
    dropped = o == 2
    assert int(dropped.sum()) == res.drops
    served = ~dropped
    assert np.all(res.req_dispatch[dropped] == -1)
    np.testing.assert_array_equal(res.req_arrival, ticks)
    np.testing.assert_array_equal(res.req_model, midx)
    np.testing.assert_array_equal(res.req_deadline, ticks + slo[midx])
    d, st, fi, b = (res.req_dispatch[served], res.req_start[served], res.req_finish[served],
                    res.req_batch[served])
    m = midx[served]
    assert np.all(d >= ticks[served]) and np.all(st >= d)
    assert np.all((b >= 1) & (b <= mb[m]))
    np.testing.assert_array_equal(fi, st + lat[m, b - 1])
    assert np.all(fi <= ticks[served] + slo[m])  # completed means on time
    # batches: sizes, per-GPU non-overlap
    bt = res.batches
    assert int(bt["size"].astype(np.int64).sum()) == int(served.sum())
    order = np.lexsort((bt["start"], bt["gpu"]))
    g, s, f = bt["gpu"][order], bt["start"][order], bt["finish"][order]
    same = g[1:] == g[:-1]
    assert np.all(s[1:][same] >= f[:-1][same]), "a GPU runs two batches at once"
    # per-model FIFO: dispatch non-decreasing in stream order within a model
    idx = np.nonzero(served)[0]
    order = np.lexsort((idx, midx[idx]))
    mm, dd = midx[idx][order], res.req_dispatch[idx][order]
    same = mm[1:] == mm[:-1]
    assert np.all(dd[1:][same] >= dd[:-1][same]), "a model served out of order"


def test_c4_full_size_properties_and_sampled_parity():
    from oracle import oracle
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.simulator import Engine
    sc, ticks, midx = _workload("C4", 60.0)
    assert len(ticks) > 70_000_000
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
    res = eng.run_stream(ticks, midx, 60.0)
    assert eng.stats["fast_shards"] == 8
    _check_properties(sc, res, ticks, midx)
    # bit-exact against the oracle on two full-length sub-clusters
    for s in (0, 7):
        ms, gpus, ids = configs.shard_scenarios(sc)[s]
        sel = np.nonzero((midx >= ids[0]) & (midx <= ids[-1]))[0]
        ref = oracle.run(arr_ticks=ticks[sel], arr_midx=midx[sel] - ids[0],
                         **oracle_args(list(ms), gpus, sc.policy))
        for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
            np.testing.assert_array_equal(getattr(res, k)[sel], ref[k], err_msg=f"{k} shard {s}")
    eng.close()


def test_c3_full_size_properties():
    from paper_2308_07470_b200.simulator import Engine
    sc, ticks, midx = _workload("C3", 60.0)
    assert len(ticks) > 15_000_000
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
    res = eng.run_stream(ticks, midx, 60.0)
    assert eng.stats["fast_shards"] == 1
    _check_properties(sc, res, ticks, midx)
    eng.close()
