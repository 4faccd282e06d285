"""Do independent engines overlap on the device?  Runs K overloaded
single-model runs in K threads and reports wall time and per-run device
times (dev tool)."""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, ".")
from paper_2308_07470_b200 import scenario as SCN  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

sc = SCN.load_scenario("table2_resnet50").with_rate(11678.8)
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402
ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], sc.duration_s, sc.seed)


FAST = "nofast" not in sys.argv


def one(_):
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, use_fast=FAST)
    t0 = time.perf_counter()
    eng.run_stream(ticks, midx, sc.duration_s)
    w = time.perf_counter() - t0
    eng.close()
    return w, eng.stats["ms_total"], eng.stats["ms_chain"]


one(0)
for k in (1, 2, 4, 8):
    t0 = time.perf_counter()
    with ThreadPoolExecutor(k) as ex:
        outs = list(ex.map(one, range(k)))
    print(k, "threads wall", round(time.perf_counter() - t0, 3),
          [(round(w, 3), round(a, 1), round(c, 1)) for w, a, c in outs], flush=True)
