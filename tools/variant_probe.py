"""Device time and path of the policy / network variants at a given length
of C3 and of C4 sub-clusters 0 and 5, next to the C oracle's time (dev
tool: sizes the full-length parity tests)."""
import sys
import time
from dataclasses import replace

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import oracle  # noqa: E402
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402
from conftest import oracle_args  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
for name in ("C3", "C4"):
    for variant in ("timeout30", "delay", "eager"):
        sc = configs.CONFIGS[name](dur, variant)
        ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
        models, gpus = list(sc.models), sc.gpu_count
        if name == "C4":
            ms, g, ids = configs.shard_scenarios(sc)[0]
            keep = (midx >= ids[0]) & (midx <= ids[-1])
            ticks, midx = ticks[keep], midx[keep] - ids[0]
            models, gpus = list(ms), g
        eng = Engine(models, gpus, sc.policy)
        t0 = time.perf_counter()
        res = eng.run_stream(ticks, midx, dur)
        wall = time.perf_counter() - t0
        st = eng.stats
        t0 = time.perf_counter()
        ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, sc.policy))
        t_or = time.perf_counter() - t0
        ok = all(np.array_equal(getattr(res, k), ref[k]) for k in
                 ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"))
        print(f"{name}/{variant} {dur:g}s n={len(ticks)} fast={st['fast_shards']} "
              f"fail={hex(st['fast_fail_mask'])} chain_events={st['chain_events']} "
              f"dev_ms={st['ms_total']:.1f} chain_ms={st['ms_chain']:.1f} wall={wall:.2f}s "
              f"oracle={t_or:.2f}s drops={res.drops} parity={ok}", flush=True)
        eng.close()
