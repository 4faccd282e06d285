"""A few device-resident steps of bench.py's workload (C4 sub-cluster 0)
for ncu captures (dev tool): python tools/bench_step.py [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_workload  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sc, ms, gpus, ticks, midx = build_workload(60.0, 0)
eng = Engine(ms, gpus, sc.policy)
t = torch.from_numpy(ticks).cuda()
m = torch.from_numpy(midx.astype(np.int32)).cuda()
for _ in range(steps):
    out, cnt = eng.run_device(t, m)
torch.cuda.synchronize()
print(len(ticks), cnt["ms_total"])
if len(sys.argv) > 2 and sys.argv[2] == "ktimes":
    eng.kernel_times(reset=True)
    reps = 20
    tot = 0.0
    for _ in range(reps):
        out, cnt = eng.run_device(t, m, kernel_times=True)
        tot += cnt["ms_total"]
    kt = eng.kernel_times()
    ksum = sum(v[1] for v in kt.values()) / reps
    print(f"ms_total {tot / reps:.3f}  kernel sum {ksum:.3f}  launches/step "
          f"{sum(v[0] for v in kt.values()) / reps:.0f}")
    for _ in range(3):
        out, cnt = eng.run_device(t, m)
        print("plain ms_total", round(cnt["ms_total"], 3), {k: round(v, 3) for k, v in cnt.items() if k.startswith("ms_")})
