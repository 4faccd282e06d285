"""Quick device-timing probe of the engine on the benchmark configs (dev tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

for spec in sys.argv[1:]:
    name, dur = spec.split(":")[:2]
    fast = not spec.endswith(":chain")
    dur = float(dur)
    sc = configs.CONFIGS[name](dur)
    t0 = time.time()
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
    tg = time.time() - t0
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards, use_fast=fast)
    t = torch.from_numpy(ticks).cuda()
    m = torch.from_numpy(midx.astype(np.int32)).cuda()
    for rep in range(3):
        out, cnt = eng.run_device(t, m)
    n = len(ticks)
    print(f"{spec} n={n} gen={tg:.1f}s  " + "  ".join(
        f"{k}={v:.3f}" if isinstance(v, float) else f"{k}={v}" for k, v in cnt.items()),
        f"req/s(total)={n / (cnt['ms_total'] / 1e3):.3e}", flush=True)
    eng.close()
