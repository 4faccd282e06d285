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
