"""Small engine workload that runs every kernel family once -- the parallel
path (one and several sub-clusters), the chain (eager overload, trace,
invariant mode), the step API, jitter, window statistics, batch records, GPU
text formatting and the partitioner -- each engine result checked against
the oracle.  Run under guard mode (SYM_GUARD=1, tests/test_guard_gpu.py) it
is the engine's memcheck/initcheck; compute-sanitizer itself is closed on the
GPU pool (profiles/r02_sanitizer_memcheck.log)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import cases  # noqa: E402
from conftest import oracle_args  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

want = {"fig6_stagger/base", "table2_resnet50/eager", "fig4b_timeout_zoo/timeout30",
        "stress/3", "stress/17"}
KEYS = ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome")


def same(res, ref, tag):
    for k in KEYS:
        assert np.array_equal(getattr(res, k), ref[k]), (tag, k)


n_ok = 0
for c in list(cases.bundled()) + list(cases.stress(20)):
    if c[0] not in want:
        continue
    key, models, gpus, policy, ticks, midx, (dur, w, cd) = c
    ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    for kw in (dict(), dict(use_fast=False), dict(record_trace=True),
               dict(check_invariants=True)):
        eng = Engine(models, gpus, policy, **kw)
        res = eng.run_stream(ticks, midx, dur)
        same(res, ref, (key, kw))
        eng.window_stats(0, int(dur * 1e9))
        eng.close()
        n_ok += 1
    eng = Engine(models, gpus, policy)
    half = len(ticks) // 2
    eng.step(ticks[:half], midx[:half], int(ticks[half]) if half < len(ticks) else eng.DRAIN)
    eng.step(ticks[half:], midx[half:], eng.DRAIN)
    res = eng.step_result(dur)
    same(res, ref, (key, "step"))
    eng.close()
    n_ok += 1
sc = configs.c4(0.02)
ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], 0.02, 42)
eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
res = eng.run_stream(ticks, midx, 0.02)
eng.window_stats(0, 20_000_000)
eng.close()
for s_, (ms, gpus, ids) in enumerate(configs.shard_scenarios(sc)):
    sel = np.nonzero((midx >= ids[0]) & (midx <= ids[-1]))[0]
    ref = oracle.run(arr_ticks=ticks[sel], arr_midx=midx[sel] - ids[0],
                     **oracle_args(list(ms), gpus, sc.policy))
    for k in KEYS:
        assert np.array_equal(getattr(res, k)[sel], ref[k]), ("c4", s_, k)
n_ok += 1
for c in cases.jitter():
    key, models, gpus, policy, ticks, midx, (dur, w, cd), net, seed = c
    eng = Engine(models, gpus, policy, net, seed=seed)
    eng.run_stream(ticks, midx, dur)
    eng.close()
    n_ok += 1
    break
from paper_2308_07470_b200 import outputs as O  # noqa: E402
sc6 = next(o for o in cases.outputs())
key, scn, ticks, midx = sc6
eng = Engine(list(scn.models), scn.gpu_count, scn.policy)
res = eng.run_stream(ticks, midx, scn.duration_s)
assert O.requests_csv(res, 0) == O.requests_csv(res, None)
eng.close()
from paper_2308_07470_b200 import partitioner as PT  # noqa: E402
PT.brute_force(PT.random_instance(8, 3, 0))
PT.solve(PT.random_instance(40, 4, 1), time_budget_s=0.2, seed=0)
print(f"sanitize workload ok: {n_ok} engine runs")
