"""Per-probe cost of a goodput search on the engine (dev tool)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2308_07470_b200 import metrics, scenario as SCN  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402

orig_run = Engine.run_stream
log = []


def timed_run(self, t, m, d):
    t0 = time.perf_counter()
    r = orig_run(self, t, m, d)
    log.append((len(t), time.perf_counter() - t0, dict(self.stats)))
    return r


Engine.run_stream = timed_run
import time as _t
_t0 = _t.perf_counter()
SCN.run_scenario(SCN.load_scenario("fig6_stagger"))
print("first run (context + module load)", round(_t.perf_counter() - _t0, 3))
for name in sys.argv[1:]:
    log.clear()
    sc = SCN.load_scenario(name)
    t0 = time.perf_counter()
    res = metrics.goodput_search(sc)
    el = time.perf_counter() - t0
    print(name, "rate", res.rate_rps, "probes", len(res.probes), f"total {el:.3f}s")
    for (rate, ok), (n, w, c) in zip(res.probes, log):
        print(f"   rate={rate:10.1f} ok={ok} n={n} run={w*1e3:8.2f}ms",
              {k: c[k] for k in ("ms_total", "chain_events", "fast_shards", "ms_chain") if k in c})
