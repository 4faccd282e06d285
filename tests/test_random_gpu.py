"""Randomised parity beyond the golden set: 1000 further stress cases
(tests/stress_cases.py generator, seeds 1000..1999 -- same-tick bursts,
table profiles, max_batch caps, network delays, every policy and gather
mode, deep overload) run through the CUDA engine on both paths and compared
element-wise with the CPU oracle run on the box, plus the reference's op
counters."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import oracle_args
from stress_cases import make_case

pytestmark = pytest.mark.gpu
SEEDS = list(range(1000, 2000))
OUT = ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome")


def _case(seed):
    from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
    from paper_2308_07470_b200.scheduler import PolicyConfig
    c = make_case(seed)
    models = [ModelSpec(i, f"m{i}", LatencyProfile(p["kind"], p["max_batch"], 0, 0,
                                                    tuple(p["lat"])), p["slo"])
              for i, p in enumerate(c["models"])]
    return models, c["gpus"], PolicyConfig(**c["policy"]), c["ticks"], c["midx"]


@pytest.mark.parametrize("chunk", range(20))
def test_random_cases_engine_equals_oracle(chunk):
    from oracle import oracle
    from paper_2308_07470_b200.simulator import Engine
    for seed in SEEDS[chunk::20]:
        models, gpus, policy, ticks, midx = _case(seed)
        ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
        for use_fast in (True, False):
            eng = Engine(models, gpus, policy, use_fast=use_fast)
            res = eng.run_stream(ticks, midx, 1.0)
            for k in OUT:
                np.testing.assert_array_equal(getattr(res, k), ref[k],
                                              err_msg=f"seed {seed} fast={use_fast} {k}")
            assert res.drops == ref["drops"]
            assert (eng.rank.ops, eng.rank.evictions, eng.rank.registrations,
                    eng.handler_ops_max) == (ref["ops"], ref["evictions"],
                                             ref["registrations"], ref["handler_ops_max"]), seed
            eng.close()


JSEEDS = list(range(3000, 3200))


@pytest.mark.parametrize("chunk", range(8))
def test_random_jittered_cases_engine_equals_oracle(chunk):
    """The same generator with a random histogram network: per-dispatch
    Philox draws, GPU serialisation and LATE outcomes (network.py:69-77,
    simulator.py:54-62); planning bounds from the histograms' percentiles."""
    import random
    from dataclasses import replace
    from oracle import oracle
    from paper_2308_07470_b200.network import DelayDist, NetworkModel, jitter_tables
    from paper_2308_07470_b200.simulator import Engine
    for seed in JSEEDS[chunk::8]:
        models, gpus, policy, ticks, midx = _case(seed)
        rng = random.Random(seed)

        def dist():
            if rng.random() < 0.3:
                return DelayDist.constant(rng.choice([0, 5_000, 300_000]))
            k = rng.randint(1, 4)
            return DelayDist.histogram([rng.randint(0, 3_000_000) for _ in range(k)],
                                       [rng.uniform(0.01, 1.0) for _ in range(k)],
                                       rng.choice([0.5, 0.7, 0.9]))
        net = NetworkModel(dist(), dist())
        if net.jitterless:
            net = NetworkModel(DelayDist.histogram([0, 50_000, 2_000_000], [0.7, 0.2, 0.1]),
                               net.d_data)
        policy = replace(policy, d_ctrl_ns=net.plan_ctrl_ns, d_data_ns=net.plan_data_ns)
        ref = oracle.run(arr_ticks=ticks, arr_midx=midx, net=jitter_tables(net, seed),
                         **oracle_args(models, gpus, policy))
        for use_fast in (True, False):
            eng = Engine(models, gpus, policy, net, seed=seed, use_fast=use_fast)
            res = eng.run_stream(ticks, midx, 1.0)
            for k in OUT:
                np.testing.assert_array_equal(getattr(res, k), ref[k],
                                              err_msg=f"seed {seed} fast={use_fast} {k}")
            assert res.late == ref["late"] and res.drops == ref["drops"], seed
            eng.close()


@pytest.mark.parametrize("combo", range(40))
def test_random_subclusters_in_one_call(combo):
    """2-5 random cases as independent sub-clusters of ONE engine call (one
    policy): each sub-cluster's results equal its own oracle run, whatever
    the interleaving of the merged stream."""
    import random
    from oracle import oracle
    from paper_2308_07470_b200.profile import ModelSpec
    from paper_2308_07470_b200.simulator import Engine
    rng = random.Random(combo)
    parts = [_case(5000 + 10 * combo + k) for k in range(rng.randint(2, 5))]
    policy = parts[0][2]
    models, som, gps, ticks, midx = [], [], [], [], []
    for s, (ms, g, _, t, m) in enumerate(parts):
        base = len(models)
        models += [ModelSpec(base + x.model_id, f"s{s}_{x.name}", x.profile, x.slo_ns) for x in ms]
        som += [s] * len(ms)
        gps.append(g)
        ticks.append(np.asarray(t, np.int64))
        midx.append(np.asarray(m, np.int64) + base)
    t_all, m_all = np.concatenate(ticks), np.concatenate(midx)
    order = np.argsort(t_all, kind="stable")
    t_all, m_all = t_all[order], m_all[order]
    eng = Engine(models, sum(gps), policy, shards=(som, gps))
    res = eng.run_stream(t_all, m_all, 1.0)
    lo = 0
    for s, (ms, g, _, _, _) in enumerate(parts):
        sel = np.nonzero((m_all >= lo) & (m_all < lo + len(ms)))[0]
        ref = oracle.run(arr_ticks=t_all[sel], arr_midx=m_all[sel] - lo,
                         **oracle_args(list(ms), g, policy))
        for k in OUT:
            np.testing.assert_array_equal(getattr(res, k)[sel], ref[k],
                                          err_msg=f"combo {combo} shard {s} {k}")
        lo += len(ms)
    eng.close()


@pytest.mark.parametrize("combo", range(20))
def test_random_jittered_subclusters_in_one_call(combo):
    """Sub-clusters of one call under a histogram network: sub-cluster s
    draws its k-th dispatch delay from the engine's Philox stream exactly as
    a separate reference Engine with the same seed would."""
    import random
    from dataclasses import replace
    from oracle import oracle
    from paper_2308_07470_b200.network import DelayDist, NetworkModel, jitter_tables
    from paper_2308_07470_b200.profile import ModelSpec
    from paper_2308_07470_b200.simulator import Engine
    rng = random.Random(900 + combo)
    parts = [_case(7000 + 10 * combo + k) for k in range(rng.randint(2, 4))]
    net = NetworkModel(DelayDist.histogram([0, rng.randint(1, 400_000), 2_000_000],
                                           [0.6, 0.3, 0.1], 0.7),
                       DelayDist.histogram([0, 3_000, 50_000], [0.5, 0.4, 0.1]))
    policy = replace(parts[0][2], d_ctrl_ns=net.plan_ctrl_ns, d_data_ns=net.plan_data_ns)
    seed = 11 + combo
    models, som, gps, ticks, midx = [], [], [], [], []
    for s, (ms, g, _, t, m) in enumerate(parts):
        base = len(models)
        models += [ModelSpec(base + x.model_id, f"s{s}_{x.name}", x.profile, x.slo_ns) for x in ms]
        som += [s] * len(ms)
        gps.append(g)
        ticks.append(np.asarray(t, np.int64))
        midx.append(np.asarray(m, np.int64) + base)
    t_all, m_all = np.concatenate(ticks), np.concatenate(midx)
    order = np.argsort(t_all, kind="stable")
    t_all, m_all = t_all[order], m_all[order]
    eng = Engine(models, sum(gps), policy, net, seed=seed, shards=(som, gps))
    res = eng.run_stream(t_all, m_all, 1.0)
    lo = 0
    for s, (ms, g, _, _, _) in enumerate(parts):
        sel = np.nonzero((m_all >= lo) & (m_all < lo + len(ms)))[0]
        ref = oracle.run(arr_ticks=t_all[sel], arr_midx=m_all[sel] - lo,
                         net=jitter_tables(net, seed), **oracle_args(list(ms), g, policy))
        for k in OUT:
            np.testing.assert_array_equal(getattr(res, k)[sel], ref[k],
                                          err_msg=f"combo {combo} shard {s} {k}")
        lo += len(ms)
    eng.close()
