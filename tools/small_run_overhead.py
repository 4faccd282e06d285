"""Fixed cost of one Engine.run_stream call on a tiny stream (dev tool)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2308_07470_b200 import load_scenario  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

for name in ("fig6_stagger", "table2_resnet50"):
    sc = load_scenario(name)
    t, m = generate_arrivals(sc.workload, [x.name for x in sc.models], sc.duration_s, sc.seed)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
    for _ in range(3):
        eng.run_stream(t, m, sc.duration_s)
    reps = 50
    t0 = time.perf_counter()
    for _ in range(reps):
        eng.run_stream(t, m, sc.duration_s)
    el = (time.perf_counter() - t0) / reps
    print(f"{name}: n={len(t)} run_stream {el * 1e3:.2f} ms (device {eng.stats['ms_total']:.2f} ms, "
          f"launches {eng.stats['launches']})", flush=True)
