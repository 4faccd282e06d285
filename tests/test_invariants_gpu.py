"""Per-event invariant mode (Engine(check_invariants=True), the reference's
_verify after every event, simulator.py:224-225,276-305): the device chain
checks conservation, the GPU state machine, the registered-candidate indices
and candidate feasibility after every event; clean runs equal the oracle,
and an injected break raises InvariantViolation."""
import numpy as np
import pytest

import cases
from conftest import oracle_args
from oracle import oracle

pytestmark = pytest.mark.gpu

SMALL = list(cases.bundled()) + list(cases.stress(30))


@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
def test_checked_runs_equal_oracle(case):
    from paper_2308_07470_b200 import Engine
    key, models, gpus, policy, ticks, midx, (dur, _, _) = case
    eng = Engine(models, gpus, policy, check_invariants=True)
    res = eng.run_stream(ticks, midx, dur)
    ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
        np.testing.assert_array_equal(getattr(res, k), ref[k], err_msg=k)
    assert eng.stats["fast_shards"] == 0  # every event went through the checked chain
    eng.close()


@pytest.mark.parametrize("key", ["fig6_stagger/base", "table2_resnet50/eager",
                                 "fig4b_timeout_zoo/timeout30"])
def test_injected_break_raises(key):
    from paper_2308_07470_b200 import Engine
    from paper_2308_07470_b200.simulator import InvariantViolation
    key, models, gpus, policy, ticks, midx, (dur, _, _) = next(
        c for c in cases.bundled() if c[0] == key)
    eng = Engine(models, gpus, policy, check_invariants=True)
    eng._inject_fault = True
    with pytest.raises(InvariantViolation, match="after chain event 10"):
        eng.run_stream(ticks, midx, dur)
    eng._inject_fault = False
    eng.run_stream(ticks, midx, dur)  # the engine is usable afterwards
    eng.close()


def test_checked_stepped_run():
    from paper_2308_07470_b200 import Engine
    key, models, gpus, policy, ticks, midx, (dur, _, _) = next(
        c for c in cases.bundled() if c[0] == "table2_resnet50/eager")
    eng = Engine(models, gpus, policy, check_invariants=True)
    half = len(ticks) // 2
    eng.step(ticks[:half], midx[:half], int(ticks[half]))
    eng.step(ticks[half:], midx[half:], eng.DRAIN)
    res = eng.step_result(dur)
    ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    np.testing.assert_array_equal(res.req_outcome, ref["req_outcome"])
    eng.close()
