"""Device-timing probe of saturated scalebench shards (dev tool):
phase times, counters and the top kernels."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2308_07470_b200 import scalebench as SB  # noqa: E402
from paper_2308_07470_b200.scheduler import PolicyConfig  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

for spec in sys.argv[1:]:
    M, G, n = (int(x) for x in spec.split("x"))
    ticks, midx = SB.shard_stream(n, M, G)
    eng = Engine(SB.shard_models(M), G, PolicyConfig("deferred"))
    t = torch.from_numpy(ticks).cuda()
    m = torch.from_numpy(midx.astype(np.int32)).cuda()
    for rep in range(2):
        out, cnt = eng.run_device(t, m)
    eng.kernel_times(reset=True)
    out, cnt = eng.run_device(t, m, kernel_times=True)
    kt = eng.kernel_times()
    top = sorted(kt.items(), key=lambda kv: -kv[1][1])[:8]
    print(f"{spec}: " + "  ".join(
        f"{k}={v:.3f}" if isinstance(v, float) else f"{k}={v}" for k, v in cnt.items()),
        f"req/s={n / (cnt['ms_total'] / 1e3):.3e}", flush=True)
    print("   top:", ", ".join(f"{k}:{v[0]}x{v[1]:.3f}ms" for k, v in top), flush=True)
    eng.close()
