"""compute_stats on a large engine result (C4 at full length, 72M requests):
the host reduction vs the device reductions (sym_window_stats) (dev tool)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.metrics import compute_stats  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
dur = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
sc = configs.CONFIGS[name](dur)
ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
res = eng.run_stream(ticks, midx, dur)
compute_stats(res, 0.1 * dur, 0.1 * dur, dur, engine=eng)  # warm
t0 = time.perf_counter()
st_dev = compute_stats(res, 0.1 * dur, 0.1 * dur, dur, engine=eng)
el_dev = time.perf_counter() - t0
t0 = time.perf_counter()
st = compute_stats(res, 0.1 * dur, 0.1 * dur, dur)
el = time.perf_counter() - t0
assert st == st_dev
print(f"{name} {dur:g}s n={len(ticks)}: compute_stats host {el:.2f} s, device {el_dev * 1e3:.1f} ms "
      f"(identical); goodput {st.goodput_rps:.1f}, p99[0] {st.models[0].p99_latency_ns}")
