"""Multi-rank host logic of the sharded path on CPU (gloo, world sizes 2 and 8):
sub-cluster assignment, per-rank integer summaries, the single all-reduce,
and the cluster statistics rebuilt from it -- checked against
compute_stats on the whole run.  Each rank resolves its sub-clusters with
the CPU oracle (test infrastructure), standing in for its GPU."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_07470_b200 import configs
from paper_2308_07470_b200.parallel import (SummaryLayout, assign, cluster_stats,
                                            reduce_summaries, window_counts_host)

DUR = 0.05


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_runs(sc, ticks, midx, shards):
    from conftest import oracle_args
    from oracle import oracle
    out = []
    for s, (ms, g, ids) in enumerate(configs.shard_scenarios(sc)):
        if s not in shards:
            continue
        sel = (midx >= ids[0]) & (midx <= ids[-1])
        o = oracle.run(arr_ticks=ticks[sel], arr_midx=midx[sel] - ids[0],
                       **oracle_args(list(ms), g, sc.policy))
        out.append((s, ids, g, sel, o))
    return out


def _rank(rank, world, port, q):
    import sys
    sys.path[:0] = [os.path.dirname(__file__), os.path.dirname(os.path.dirname(__file__))]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(DUR)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], DUR, 42)
    layout = SummaryLayout(len(sc.models), sc.gpu_count)
    lo, hi = int(0.1 * DUR * 1e9), int(0.9 * DUR * 1e9)
    vec = layout.empty()
    for s, ids, g, sel, o in _shard_runs(sc, ticks, midx, assign(8, world)[rank]):
        cnt = window_counts_host(midx[sel] - ids[0], ticks[sel], o["req_outcome"], o["ord_gpu"],
                                 o["ord_start"], o["ord_finish"], len(ids), g, lo, hi)
        layout.put(vec, ids, np.arange(1024 * s, 1024 * (s + 1)), cnt)
    vec = reduce_summaries(vec)
    q.put((rank, cluster_stats(vec, layout, lo, hi)))
    dist.destroy_process_group()


def test_assignment_is_fixed_by_scenario():
    assert assign(8, 1) == [list(range(8))]
    assert assign(8, 2) == [[0, 2, 4, 6], [1, 3, 5, 7]]
    assert sorted(sum(assign(8, 4), [])) == list(range(8))
    assert assign(8, 8) == [[s] for s in range(8)]  # C4 on 8 B200s: one sub-cluster each


@pytest.mark.parametrize("world", [2, 8])
def test_gloo_summary_matches_whole_run_stats(world):
    """world ranks (gloo, one process each; 8 = C4 on a full box) reduce
    their sub-clusters' summaries into the whole run's statistics."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(got[r] == got[0] for r in range(world))  # every rank sees the same view
    # whole run, single process: compute_stats on the concatenated results
    from paper_2308_07470_b200.metrics import compute_stats
    from paper_2308_07470_b200.simulator import RunResult
    from paper_2308_07470_b200.workload import generate_arrivals
    from paper_2308_07470_b200 import _native
    sc = configs.c4(DUR)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], DUR, 42)
    n = len(ticks)
    arrs = {k: np.full(n, -1, np.int64) for k in ("dispatch", "start", "finish", "batch", "outcome")}
    recs = []
    for s, ids, g, sel, o in _shard_runs(sc, ticks, midx, set(range(8))):
        for k in arrs:
            arrs[k][sel] = o["req_" + k]
        b = np.zeros(len(o["ord_gpu"]), dtype=_native.BATCH_DTYPE)
        b["gpu"], b["start"], b["finish"] = o["ord_gpu"] + 1024 * s, o["ord_start"], o["ord_finish"]
        b["model"], b["size"] = o["ord_model"] + ids[0], o["ord_size"]
        recs.append(b)
    res = RunResult([m.name for m in sc.models], sc.gpu_count, int(DUR * 1e9), req_model=midx,
                    req_arrival=ticks, req_deadline=ticks, req_dispatch=arrs["dispatch"],
                    req_start=arrs["start"], req_finish=arrs["finish"], req_batch=arrs["batch"],
                    req_outcome=arrs["outcome"], batches=np.concatenate(recs))
    st = compute_stats(res, 0.1 * DUR, 0.1 * DUR, DUR)
    c = got[0]
    assert c["arrivals"] == st.arrivals and c["completed"] == st.completed
    assert c["goodput_rps"] == st.goodput_rps
    assert c["bad_rate"] == st.bad_rate
    assert c["mean_idle_fraction"] == st.mean_idle_fraction
