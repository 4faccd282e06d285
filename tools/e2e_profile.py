"""Break down Engine.run_stream wall time on the bench workload (dev tool)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

sc, ms, gpus, ticks, midx = bench.build_workload(60.0, 0)
eng = Engine(ms, gpus, sc.policy)
pin_t = torch.from_numpy(ticks).pin_memory().numpy()
pin_m = torch.from_numpy(midx).pin_memory().numpy()
for _ in range(2):
    eng.run_stream(pin_t, pin_m, 60.0)
t0 = time.perf_counter()
for _ in range(3):
    eng.run_stream(pin_t, pin_m, 60.0)
print("run_stream ms", (time.perf_counter() - t0) / 3 * 1e3, "engine ms_total", eng.stats["ms_total"])
pr = cProfile.Profile()
pr.enable()
eng.run_stream(pin_t, pin_m, 60.0)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
