"""A few device-resident steps of bench.py's workload for ncu captures (dev
tool): python tools/bench_step.py [steps] [sub|full] [ktimes]
  sub  = C4 sub-cluster 0 (one engine shard, 9.0M requests: the N=8 rank)
  full = all of C4 (8 shards, 72M requests: the N=1 bench)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_workload  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "sub"
subs = [0] if mode == "sub" else list(range(8))
sc, models, gpus, shards, ticks, midx, _ = build_workload(60.0, subs)
eng = Engine(models, gpus, sc.policy, shards=shards)
t = torch.from_numpy(ticks).cuda()
m = torch.from_numpy(midx.astype(np.int32)).cuda()
for _ in range(steps):
    out, cnt = eng.run_device(t, m)
torch.cuda.synchronize()
print(mode, len(ticks), cnt["ms_total"], cnt["fast_shards"])
if "ktimes" in sys.argv:
    eng.kernel_times(reset=True)
    reps = 10
    tot = 0.0
    for _ in range(reps):
        out, cnt = eng.run_device(t, m, kernel_times=True)
        tot += cnt["ms_total"]
    kt = eng.kernel_times()
    ksum = sum(v[1] for v in kt.values()) / reps
    print(f"ms_total {tot / reps:.3f}  kernel sum {ksum:.3f}  launches/step "
          f"{sum(v[0] for v in kt.values()) / reps:.0f}")
    for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:20s} {v[0] / reps:5.1f} x {v[1] / v[0] * 1e3:9.1f} us")
