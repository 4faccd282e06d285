"""One overloaded single-model run (the first goodput-search probe of
table2_resnet50): the sequential live-event chain dominates (dev tool)."""
import sys

sys.path.insert(0, ".")
from paper_2308_07470_b200 import scenario as SCN  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

rate = float(sys.argv[1]) if len(sys.argv) > 1 else 11678.8
sc = SCN.load_scenario("table2_resnet50").with_rate(rate)
eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
res = eng.run(sc.workload, sc.duration_s, sc.seed)
print(res.n_requests, res.drops, eng.stats)
