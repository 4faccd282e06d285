"""C5 (diurnal ramp, 500 models x 4096 GPUs) at full length: engine run time
and the per-epoch active-GPU series (autoscale_series) on the host arrays vs
the device window reductions (dev tool)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.metrics import autoscale_series  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
sc = configs.CONFIGS["C5"](dur)
t0 = time.perf_counter()
ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
tg = time.perf_counter() - t0
eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
eng.run_stream(ticks, midx, dur)
t0 = time.perf_counter()
res = eng.run_stream(ticks, midx, dur)
tr = time.perf_counter() - t0
t0 = time.perf_counter()
series = autoscale_series(res, dur / 24, dur)
ta = time.perf_counter() - t0
t0 = time.perf_counter()
series_dev = autoscale_series(res, dur / 24, dur, engine=eng)
td = time.perf_counter() - t0
assert series_dev == series
print(f"C5 {dur:g}s: n={len(ticks)} gen {tg:.1f}s run_stream {tr * 1e3:.1f} ms "
      f"(device {eng.stats['ms_total']:.1f} ms, fast shards {eng.stats['fast_shards']}) "
      f"autoscale_series host {ta:.2f}s device {td * 1e3:.1f} ms; active GPUs {series[0]} -> {max(series)} -> {series[-1]}")
