"""A/B of the fresh-start adoption table on chain-bound runs (dev tool)."""
import sys

sys.path.insert(0, ".")
from paper_2308_07470_b200 import configs, scenario as SCN  # noqa: E402
from paper_2308_07470_b200.scheduler import PolicyConfig  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

cases = []
sc = SCN.load_scenario("table2_resnet50").with_rate(11678.8)
t, m = generate_arrivals(sc.workload, [x.name for x in sc.models], sc.duration_s, sc.seed)
cases.append(("table2 overload", list(sc.models), sc.gpu_count, sc.policy, t, m))
for name, dur in (("C1", 60.0), ("C2", 1.0), ("C4", 0.1)):
    c = configs.CONFIGS[name](dur)
    t, m = generate_arrivals(c.workload, [x.name for x in c.models], dur, 42)
    cases.append((f"{name} eager", list(c.models), c.gpu_count, PolicyConfig("eager"), t, m,
                  c.shards))
for name, dur in (("C1", 60.0), ("C4", 0.1)):  # underload forced onto the chain
    c = configs.CONFIGS[name](dur)
    t, m = generate_arrivals(c.workload, [x.name for x in c.models], dur, 42)
    cases.append((f"{name} deferred chain", list(c.models), c.gpu_count, c.policy, t, m,
                  c.shards, False))
for case in cases:
    label, models, gpus, pol, t, m = case[:6]
    shards = case[6] if len(case) > 6 else None
    fast = case[7] if len(case) > 7 else True
    row = [label]
    for fresh in (True, False):
        eng = Engine(models, gpus, pol, shards=shards, use_fresh=fresh, use_fast=fast)
        eng.run_stream(t, m, 1.0)
        eng.run_stream(t, m, 1.0)
        st = eng.stats
        row.append(f"fresh={fresh}: total {st['ms_total']:.1f} ms (fresh {st['ms_fresh']:.1f}, "
                   f"chain {st['ms_chain']:.1f}, adoptions {st['fresh_adoptions']})")
        eng.close()
    print(" | ".join(row), flush=True)
