"""Wall time of the golden sweeps on the engine, serial vs concurrent
searches, and a reference-shaped scale_bench run."""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2308_07470_b200 import scalebench as SB, sweeps  # noqa: E402
from paper_2308_07470_b200.scenario import load_scenario  # noqa: E402

CASES = [
    ("beta_ratio", "table2_resnet50", [1.0, 6.0], ["deferred", "eager"], None),
    ("timeout", "fig4b_timeout_sweep", [10.0, 60.0], None, None),
    ("offered_load", "table2_resnet50", [0.5, 1.25], None, 5000.0),
    ("slo", "table2_inceptionresnet", [40.0, 90.0], ["deferred", "timeout:30"], None),
]

out = {}
sweeps.run_sweep("offered_load", load_scenario("table2_resnet50"), [0.5], None, 5000.0)  # warm
for workers, spec in ((1, 0), (4, 0), (1, 3), (4, 2), (4, 3), (8, 3)):
    t0 = time.perf_counter()
    for dim, name, grid, pols, peak in CASES:
        sweeps.run_sweep(dim, load_scenario(name), grid, pols, peak, workers=workers,
                         speculate=spec)
    out[f"sweeps_w{workers}_s{spec}_s"] = round(time.perf_counter() - t0, 3)
    print(json.dumps(out), flush=True)
r = SB.scale_bench([1, 8], [16, 1024], 1.0)
out["scale_bench"] = {k: [dict(workers=p.workers, gpus=p.gpus, models=p.models,
                                requests=p.requests, elapsed_s=round(p.elapsed_s, 4),
                                rps=round(p.throughput_rps)) for p in v]
                      for k, v in r.items()}
print(json.dumps(out))
