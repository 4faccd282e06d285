"""BASELINE.json's configurations at FULL size (60 s traces: C2 2.4M
requests, C3 18M Gamma-bursty, C4 72M over 8 sub-clusters of 1000 models x
8192 GPUs, C5 20M diurnal).

Two kinds of evidence at the size the benchmark runs:
* bit-exact parity with the CPU oracle on EVERY config at its full length --
  all five per-request arrays, every batch record (GPU, model, size, start,
  finish, dispatch time) in emission order, and the drop count; C4 on all
  eight sub-clusters of one engine call; the eager, timeout-30 % and
  network-delay variants at full C3 and full C4-sub-cluster length;
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


def _compare_shard(res, sel, model_base, gpu_base, ref, tag):
    """Engine result restricted to one sub-cluster vs its oracle run."""
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
        got = getattr(res, k)[sel]
        if not np.array_equal(got, ref[k]):
            bad = int(np.nonzero(got != ref[k])[0][0])
            raise AssertionError(f"{tag}: {k} differs first at request {bad}: "
                                 f"{int(got[bad])} vs {int(ref[k][bad])}")
    b = res.batches
    mine = (b["gpu"] >= gpu_base) & (b["gpu"] < gpu_base + ref["n_gpus"])
    bb = b[mine]
    assert len(bb) == len(ref["ord_gpu"]), f"{tag}: batch count"
    np.testing.assert_array_equal(bb["gpu"] - gpu_base, ref["ord_gpu"], err_msg=f"{tag} gpu")
    np.testing.assert_array_equal(bb["model"] - model_base, ref["ord_model"],
                                  err_msg=f"{tag} model")
    np.testing.assert_array_equal(bb["size"], ref["ord_size"], err_msg=f"{tag} size")
    np.testing.assert_array_equal(bb["start"], ref["ord_start"], err_msg=f"{tag} start")
    np.testing.assert_array_equal(bb["finish"], ref["ord_finish"], err_msg=f"{tag} finish")
    np.testing.assert_array_equal(bb["emitted"], ref["ord_emitted"], err_msg=f"{tag} emitted")
    assert int(np.count_nonzero(res.req_outcome[sel] == 2)) == ref["drops"], f"{tag}: drops"


def _full_parity(name, variant, subclusters=None):
    """One engine call over the config (or the listed C4 sub-clusters) at
    60 s, every sub-cluster checked against its own oracle run."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.simulator import Engine
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.CONFIGS[name](60.0, variant)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 60.0, 42)
    parts = configs.shard_scenarios(sc)
    if subclusters is not None:  # a subset of C4's sub-clusters, renumbered
        from dataclasses import replace
        ids = [i for s in subclusters for i in parts[s][2]]
        new = np.full(len(sc.models), -1, np.int64)
        new[ids] = np.arange(len(ids))
        keep = new[midx] >= 0
        ticks, midx = ticks[keep], new[midx[keep]]
        models = [replace(sc.models[i], model_id=k) for k, i in enumerate(ids)]
        som = [j for j, s in enumerate(subclusters) for _ in parts[s][2]]
        gps = [parts[s][1] for s in subclusters]
        parts = [(tuple(parts[s][0]), parts[s][1],
                  list(range(sum(len(parts[t][2]) for t in subclusters[:j]),
                             sum(len(parts[t][2]) for t in subclusters[:j + 1]))))
                 for j, s in enumerate(subclusters)]
        shards = (som, gps) if len(subclusters) > 1 else None
        gpus = sum(gps)
    else:
        models, shards, gpus = list(sc.models), sc.shards, sc.gpu_count
    eng = Engine(models, gpus, sc.policy, shards=shards)
    res = eng.run_stream(ticks, midx, 60.0)
    _check_properties_any(models, res, ticks, midx)

    def one(part):
        ms, g, ids = part
        sel = np.nonzero((midx >= ids[0]) & (midx <= ids[-1]))[0]
        ref = oracle.run(arr_ticks=ticks[sel], arr_midx=midx[sel] - ids[0],
                         **oracle_args(list(ms), g, sc.policy))
        ref["n_gpus"] = g
        return sel, ids[0], ref
    with ThreadPoolExecutor(len(parts)) as ex:
        refs = list(ex.map(one, parts))
    gbase = 0
    for j, (sel, mbase, ref) in enumerate(refs):
        _compare_shard(res, sel, mbase, gbase, ref, f"{name}/{variant}/sub-cluster {j}")
        gbase += ref["n_gpus"]
    stats = dict(eng.stats)
    eng.close()
    return res, stats


def _check_properties_any(models, res, ticks, midx):
    """The size-independent properties for any policy (LATE never occurs
    without jitter; drops are allowed)."""
    o = res.req_outcome
    assert set(np.unique(o).tolist()) <= {0, 2}
    served = o != 2
    assert int(np.count_nonzero(~served)) == res.drops
    slo = np.array([m.slo_ns for m in models], np.int64)
    np.testing.assert_array_equal(res.req_deadline, ticks + slo[midx])
    assert np.all(res.req_finish[served] <= res.req_deadline[served])
    assert int(res.batches["size"].astype(np.int64).sum()) == int(served.sum())


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_full_length_parity(name):
    """C2, C3 and C5 at their full 60 s, bit-exact against the oracle."""
    _, stats = _full_parity(name, "deferred")
    assert stats["fast_shards"] == 1


def test_c4_full_length_parity_all_subclusters():
    """All of C4 (72M requests, 8 sub-clusters in one call) at 60 s: every
    sub-cluster bit-exact against its own oracle run."""
    res, stats = _full_parity("C4", "deferred")
    assert len(res.req_outcome) > 70_000_000 and stats["fast_shards"] == 8


@pytest.mark.parametrize("variant", ["timeout30", "delay", "eager"])
def test_c3_full_length_variants(variant):
    """The policy and network variants at full C3 length (18M Gamma-bursty
    requests)."""
    _full_parity("C3", variant)


@pytest.mark.parametrize("variant", ["timeout30", "delay", "eager"])
def test_c4_subcluster_full_length_variants(variant):
    """The variants at full C4-sub-cluster length (9M requests, 125 models x
    1024 GPUs), sub-clusters 0 and 5 in one call."""
    _full_parity("C4", variant, subclusters=[0, 5])
