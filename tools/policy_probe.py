"""Which path do eager / timeout policies take on the benchmark configs
(dev tool): fast_shards, fail mask, device ms."""
import sys
from dataclasses import replace

sys.path.insert(0, ".")
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.scheduler import PolicyConfig  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

for name, dur in (("C1", 60.0), ("C2", 1.0), ("C3", 0.25), ("C4", 0.1)):
    sc = configs.CONFIGS[name](dur)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
    for pol in (sc.policy, PolicyConfig("eager"), PolicyConfig("timeout", timeout_slo_frac=0.3)):
        eng = Engine(list(sc.models), sc.gpu_count, pol, shards=sc.shards)
        eng.run_stream(ticks, midx, dur)
        st = eng.stats
        print(name, pol.kind, len(ticks), "fast", st["fast_shards"], "fail", hex(st["fast_fail_mask"]),
              "chain_events", st["chain_events"], "ms", round(st["ms_total"], 2),
              "ms_chain", round(st["ms_chain"], 2), flush=True)
        eng.close()
