"""The step API (sym_step / Engine.step): a stepped run, fed in chunks with
state carried on the device between calls, equals one whole run over the
concatenated stream bit for bit -- per-request arrays, batch records, drop
counts and the reference's op counters -- for every policy and gather,
overload and same-tick bursts included, whatever the chunking: chunks split
inside a same-tick run (until_tick = that tick), single-arrival chunks,
empty chunks, until_tick between arrivals.  The reference's own step API is
scalebench._shard_loop (scalebench.py:67-84)."""
import numpy as np
import pytest

import cases
from conftest import oracle_args
from oracle import oracle

pytestmark = pytest.mark.gpu

SMALL = list(cases.bundled()) + list(cases.stress(30))
DRAIN = (1 << 63) - 1


def _chunks(ticks, rng, mode):
    """Chunk boundaries and until_ticks.  mode: random cut points with
    until = the next arrival's tick (splits same-tick runs whenever the cut
    falls inside one); 'gaps' = until strictly between arrivals where
    possible; 'same_tick' = every cut inside a run of equal ticks."""
    n = len(ticks)
    if n == 0:
        return [(0, 0, DRAIN)]
    if mode == "same_tick":
        cuts = [i for i in range(1, n) if ticks[i] == ticks[i - 1]]
        cuts = sorted(rng.choice(cuts, size=min(len(cuts), 40), replace=False)) if cuts else []
    else:
        k = int(rng.integers(1, min(n, 60) + 1))
        cuts = sorted(set(rng.integers(1, n, size=k).tolist())) if n > 1 else []
    out, lo = [], 0
    for c in list(cuts) + [n]:
        if c == n:
            out.append((lo, n, DRAIN))
            break
        nxt = int(ticks[c])
        until = nxt
        if mode == "gaps" and nxt > ticks[c - 1]:
            until = int(rng.integers(int(ticks[c - 1]), nxt))
        out.append((lo, c, until))
        lo = c
    return out


def _stepped(eng, ticks, midx, chunks, dur, empty_steps=False):
    eng.reset_steps()
    prev = None
    for lo, hi, until in chunks:
        if empty_steps and prev is not None and until != DRAIN:
            eng.step(ticks[:0], midx[:0], prev)  # an empty step at the same until
        eng.step(ticks[lo:hi], midx[lo:hi], until)
        prev = until
    return eng.step_result(dur, drain=False)


def _check_equal(res, ref, tag):
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
        got = getattr(res, k)
        assert np.array_equal(got, ref[k]), f"{tag}: {k} differs at {np.nonzero(got != ref[k])[0][:5]}"
    b = res.batches
    o = ref
    order_ok = (np.array_equal(b["gpu"], o["ord_gpu"]) and np.array_equal(b["model"], o["ord_model"])
                and np.array_equal(b["size"], o["ord_size"])
                and np.array_equal(b["start"], o["ord_start"])
                and np.array_equal(b["finish"], o["ord_finish"])
                and np.array_equal(b["emitted"], o["ord_emitted"]))
    assert order_ok, f"{tag}: batch records differ"
    assert res.drops == o["drops"] and res.completions == o["completions"], tag


@pytest.mark.parametrize("mode", ["next_tick", "gaps", "same_tick"])
@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
def test_stepped_equals_whole_run(case, mode):
    from paper_2308_07470_b200 import Engine
    key, models, gpus, policy, ticks, midx, (dur, _, _) = case
    rng = np.random.default_rng(abs(hash((key, mode))) % (1 << 32))
    ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    eng = Engine(models, gpus, policy)
    res = _stepped(eng, ticks, midx, _chunks(ticks, rng, mode), dur, empty_steps=mode == "gaps")
    _check_equal(res, ref, f"{key}/{mode}")
    assert eng.rank.ops == ref["ops"] and eng.rank.registrations == ref["registrations"]
    assert eng.rank.evictions == ref["evictions"]
    assert eng.handler_ops_max == ref["handler_ops_max"]
    eng.close()


def test_single_arrival_steps():
    """The reference's own granularity: one arrival per step, until = the
    next arrival's tick (scalebench.py:70-82)."""
    from paper_2308_07470_b200 import Engine
    key, models, gpus, policy, ticks, midx, (dur, _, _) = next(
        c for c in cases.bundled() if c[0] == "fig6_stagger/base")
    ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    eng = Engine(models, gpus, policy)
    chunks = [(i, i + 1, int(ticks[i + 1]) if i + 1 < len(ticks) else DRAIN)
              for i in range(len(ticks))]
    _check_equal(_stepped(eng, ticks, midx, chunks, dur), ref, key)
    eng.close()


def test_mid_run_state_is_a_prefix_of_the_final_one():
    """After a partial step every decided field already has its final value
    and every undecided request reads -1, as in the reference mid-run: a
    request's outcome resolves at its completion tick."""
    from paper_2308_07470_b200 import Engine
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c2(1.0)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 1.0, 42)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
    final = eng.run_stream(ticks, midx, 1.0)
    half = len(ticks) // 2
    until = int(ticks[half])
    eng.step(ticks[:half], midx[:half], until)
    mid = eng.step_result(1.0, drain=False)
    assert len(mid.req_outcome) == half
    done = mid.req_dispatch >= 0
    assert done.any() and not done.all()
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch"):
        np.testing.assert_array_equal(getattr(mid, k)[done], getattr(final, k)[:half][done])
    assert np.all(mid.req_dispatch[done] <= until)
    completed = mid.req_outcome == 0
    assert np.all(mid.req_finish[completed] <= until)
    assert np.all(mid.req_outcome[done & ~completed] == -1)
    eng.step(ticks[half:], midx[half:], DRAIN)
    res = eng.step_result(1.0)
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
        np.testing.assert_array_equal(getattr(res, k), getattr(final, k))
    eng.close()


def test_multi_subcluster_stepped_run():
    """Several sub-clusters stepped in one engine (C4 at 0.5 s, 8 shards):
    equal to the whole run, batch records in sub-cluster order."""
    from paper_2308_07470_b200 import Engine
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(0.5)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 0.5, 42)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
    whole = eng.run_stream(ticks, midx, 0.5)
    rng = np.random.default_rng(7)
    res = _stepped(eng, ticks, midx, _chunks(ticks, rng, "next_tick"), 0.5)
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
        np.testing.assert_array_equal(getattr(res, k), getattr(whole, k))
    for f in ("gpu", "model", "size", "start", "finish", "emitted", "first_index"):
        np.testing.assert_array_equal(res.batches[f], whole.batches[f])
    eng.close()


def test_step_errors():
    from paper_2308_07470_b200 import Engine, PolicyConfig
    from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
    from paper_2308_07470_b200.scheduler import ProtocolError
    m = [ModelSpec(0, "m", LatencyProfile.linear(1.0, 5.0, 8), 50_000_000)]
    eng = Engine(m, 2, PolicyConfig("deferred"))
    eng.step(np.array([10, 20]), np.array([0, 0]), 30)
    with pytest.raises(ValueError):      # arrival before the previous until
        eng.step(np.array([25]), np.array([0]), 40)
    with pytest.raises(ValueError):      # until before the chunk's last arrival
        eng.step(np.array([35, 50]), np.array([0, 0]), 45)
    with pytest.raises(ProtocolError):   # unknown model; the state is untouched
        eng.step(np.array([35]), np.array([3]), 40)
    eng.step(np.array([35]), np.array([0]), DRAIN)
    res = eng.step_result(1.0)
    assert res.n_requests == 3 and set(res.req_outcome.tolist()) <= {0, 2}
    eng.close()


def test_slo_beyond_32_bits():
    """SLOs beyond 2^32 ns (4.3 s) keep every tick int64 end to end (finish -
    arrival above 2^32): same results as the oracle."""
    from paper_2308_07470_b200 import Engine, PolicyConfig
    from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
    from paper_2308_07470_b200.workload import WorkloadSpec, generate_arrivals
    for slo_ms in (50.0, 9000.0):
        models = [ModelSpec(i, f"m{i}", LatencyProfile.linear(1.0 + i, 5.0, 32),
                            int(slo_ms * 1e6)) for i in range(3)]
        ticks, midx = generate_arrivals(WorkloadSpec("poisson", 3000.0),
                                        [m.name for m in models], 20.0, 3)
        ref = oracle.run(arr_ticks=ticks, arr_midx=midx,
                         **oracle_args(models, 4, PolicyConfig("deferred")))
        eng = Engine(models, 4, PolicyConfig("deferred"))
        res = eng.run_stream(ticks, midx, 20.0)
        for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
            np.testing.assert_array_equal(getattr(res, k), ref[k], err_msg=f"{slo_ms} {k}")
        if slo_ms > 5000:
            assert int((res.req_finish - res.req_arrival).max()) > (1 << 32)
        eng.close()
