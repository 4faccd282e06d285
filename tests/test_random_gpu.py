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
