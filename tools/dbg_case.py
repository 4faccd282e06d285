"""Debug: one golden case through the engine (fast / chain, trace on/off)
vs the oracle; prints the first differences (dev tool)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import cases  # noqa: E402
from conftest import oracle_args  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

want = sys.argv[1:] or ["fig4b_timeout_zoo/base"]
for c in list(cases.bundled()) + list(cases.stress()) + list(cases.config_cases()):
    if not any(w == c[0] or (w.endswith("*") and c[0].startswith(w[:-1])) for w in want):
        continue
    key, models, gpus, policy, ticks, midx, _ = c
    ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    for kw in (dict(), dict(use_fast=False), dict(record_trace=True), dict(use_fresh=False)):
        eng = Engine(models, gpus, policy, **kw)
        res = eng.run_stream(ticks, midx, 1.0)
        bad = []
        for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome"):
            d = np.nonzero(getattr(res, k) != ref[k])[0]
            if len(d):
                bad.append(f"{k}@{d[:4].tolist()} got {getattr(res, k)[d[:4]].tolist()} "
                           f"want {ref[k][d[:4]].tolist()}")
        print(key, kw, "fast", eng.stats.get("fast_shards"), "OK" if not bad else "DIFF",
              "; ".join(bad), flush=True)
        eng.close()
