"""Rebuild every golden case's inputs with this package's own host code
(no reference import), so the same cases drive the oracle (CPU tests) and
the CUDA engine (GPU tests)."""
from __future__ import annotations

import numpy as np

from paper_2308_07470_b200 import configs
from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
from paper_2308_07470_b200.scenario import BUNDLED_SCENARIOS, load_scenario
from paper_2308_07470_b200.scheduler import PolicyConfig
from paper_2308_07470_b200.workload import generate_arrivals
from stress_cases import make_case

VARIANTS = {
    "eager": dict(kind="eager"),
    "timeout30": dict(kind="timeout", timeout_slo_frac=0.3),
    "delay": dict(kind="deferred", d_ctrl_ns=30_000, d_data_ns=3_000),
}


def _policy(base, v):
    return base if v == "base" else PolicyConfig(**VARIANTS[v])


def bundled():
    """(key, models, gpus, policy, ticks, midx, (dur, warm, cool))"""
    for name in BUNDLED_SCENARIOS:
        sc = load_scenario(name)
        ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models],
                                        sc.duration_s, sc.seed)
        for v in ("base", "eager", "timeout30", "delay"):
            yield (f"{name}/{v}", list(sc.models), sc.gpu_count, _policy(sc.policy, v),
                   ticks, midx, (sc.duration_s, sc.warmup_s, sc.cooldown_s))


JITTER_NETS = {
    "J1": {"d_ctrl": {"kind": "histogram", "values_us": [5, 30, 120, 900],
                      "weights": [0.6, 0.3, 0.09, 0.01], "plan_percentile": 0.5},
           "d_data": {"kind": "histogram", "values_us": [1, 3, 10], "weights": [0.8, 0.15, 0.05]}},
    "J2": {"d_ctrl": {"kind": "histogram", "values_us": [0, 400, 1500],
                      "weights": [0.8, 0.15, 0.05], "plan_percentile": 0.7},
           "d_data": {"kind": "constant", "value_us": 0}},
    "J3": {"d_ctrl": {"kind": "constant", "value_us": 30},
           "d_data": {"kind": "histogram", "values_us": [0, 2, 50], "weights": [0.5, 0.4, 0.1],
                      "plan_percentile": 0.6}},
}
JITTER_CASES = [("table2_resnet50", "J1", None), ("fig6_stagger", "J2", None),
                ("fig4b_timeout_zoo", "J3", None), ("table2_resnet50", "J1", "eager"),
                ("fig2_flattop", "J2", None), ("table2_inceptionresnet", "J3", "timeout")]


def jitter():
    """(key, models, gpus, policy, ticks, midx, (dur, warm, cool), network, seed)"""
    import copy
    from paper_2308_07470_b200._bundled import BUNDLED
    from paper_2308_07470_b200.scenario import _bundled_trace_dir, scenario_from_dict
    for name, net, kind in JITTER_CASES:
        doc = copy.deepcopy(BUNDLED[name])
        doc["network"] = JITTER_NETS[net]
        if kind:
            doc.setdefault("policy", {})["kind"] = kind
            if kind == "timeout":
                doc["policy"]["timeout_slo_frac"] = 0.3
        sc = scenario_from_dict(doc, name=name, base_dir=_bundled_trace_dir())
        ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models],
                                        sc.duration_s, sc.seed)
        yield (f"jitter/{name}/{net}/{kind or 'base'}", list(sc.models), sc.gpu_count,
               sc.policy, ticks, midx, (sc.duration_s, sc.warmup_s, sc.cooldown_s),
               sc.network, sc.seed)


def stress(n=60):
    for seed in range(n):
        c = make_case(seed)
        models = [ModelSpec(i, f"m{i}", LatencyProfile(p["kind"], p["max_batch"], 0, 0,
                                                        tuple(p["lat"])), p["slo"])
                  for i, p in enumerate(c["models"])]
        yield (f"stress/{seed}", models, c["gpus"], PolicyConfig(**c["policy"]),
               c["ticks"], c["midx"], (1.0, 0.1, 0.1))


GOLDEN_DURATIONS = {"C1": 60.0, "C2": 1.0, "C3": 0.25, "C4": 0.1, "C5": 0.6}


def config_cases(names=("C1", "C2", "C3", "C4", "C5")):
    for name in names:
        dur = GOLDEN_DURATIONS[name]
        variants = ("base", "eager", "timeout30", "delay") if name in ("C1", "C2") else ("base",)
        for v in variants:
            sc = configs.CONFIGS[name](dur, "deferred" if v == "base" else v)
            ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
            if name == "C4":
                for s, (ms, g, ids) in enumerate(configs.shard_scenarios(sc)):
                    sel = (midx >= ids[0]) & (midx <= ids[-1])
                    yield (f"C4s{s}/{v}@{dur}", list(ms), g, sc.policy, ticks[sel],
                           midx[sel] - ids[0], (dur, 0.1 * dur, 0.1 * dur))
            else:
                yield (f"{name}/{v}@{dur}", list(sc.models), sc.gpu_count, sc.policy, ticks,
                       midx, (dur, 0.1 * dur, 0.1 * dur))


OUTPUT_CASES = ["fig6_stagger", "fig7_skip", "table2_inceptionresnet", "fig4b_timeout_zoo",
                "jitter/fig6_stagger/J2/base", "jitter/table2_inceptionresnet/J3/timeout"]


def outputs():
    """(key, scenario, ticks, midx) for the output-file golden cases
    (make_golden.output_cases)."""
    import copy
    from paper_2308_07470_b200._bundled import BUNDLED
    from paper_2308_07470_b200.scenario import _bundled_trace_dir, scenario_from_dict
    for case in OUTPUT_CASES:
        if case.startswith("jitter/"):
            _, name, net, kind = case.split("/")
            doc = copy.deepcopy(BUNDLED[name])
            doc["network"] = JITTER_NETS[net]
            if kind != "base":
                doc.setdefault("policy", {})["kind"] = kind
                if kind == "timeout":
                    doc["policy"]["timeout_slo_frac"] = 0.3
            sc = scenario_from_dict(doc, name=name, base_dir=_bundled_trace_dir())
        else:
            sc = load_scenario(case)
        ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models],
                                        sc.duration_s, sc.seed)
        yield f"outputs/{case}", sc, ticks, midx
