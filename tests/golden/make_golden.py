"""Regenerate tests/golden/golden.json from the Python REFERENCE.

Run in the build container only (it imports batchsym from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Every case records the digest of the input arrival stream, of the
reference's per-request arrays, gpu_logs and event trace, its counters and
its compute_stats summary.  The C oracle is pinned against these
(tests/test_oracle_golden.py) and the CUDA engine against the oracle and
these (tests/test_parity_gpu.py).
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
from batchsym import metrics as RM  # noqa: E402
from batchsym.network import NetworkModel  # noqa: E402
from batchsym.profile import LatencyProfile, ModelSpec  # noqa: E402
from batchsym.scenario import BUNDLED_SCENARIOS, load_scenario  # noqa: E402
from batchsym.scheduler import PolicyConfig  # noqa: E402
from batchsym.simulator import Engine  # noqa: E402
from batchsym.workload import WorkloadSpec, generate_arrivals  # noqa: E402

import digest as D  # noqa: E402

POLICIES = {
    "base": None,
    "eager": dict(kind="eager"),
    "timeout30": dict(kind="timeout", timeout_slo_frac=0.3),
    "delay": dict(kind="deferred", d_ctrl_ns=30_000, d_data_ns=3_000),
}


def policy_for(base, variant):
    if variant == "base":
        return base
    return PolicyConfig(**POLICIES[variant])


def run_case(models, gpus, policy, ticks, midx, duration_s, warm, cool, network=None, seed=0):
    network = network or NetworkModel.constant(policy.d_ctrl_ns, policy.d_data_ns)
    eng = Engine(list(models), gpus, policy, network, seed=seed, record_trace=True)
    t0 = time.time()
    res = eng.run_stream(ticks, midx, duration_s)
    el = time.time() - t0
    st = RM.compute_stats(res, warm, cool, duration_s)
    return {
        "n": int(len(ticks)),
        "trace_in": D.trace_digest(ticks, midx),
        "requests": D.requests_digest(res.req_dispatch, res.req_start, res.req_finish,
                                      res.req_batch, res.req_outcome),
        "gpu_logs": D.gpu_logs_digest(res.gpu_logs),
        "events": D.event_trace_digest(res.trace),
        "drops": int(res.drops), "completions": int(res.completions), "late": int(res.late),
        "ops": int(eng.rank.ops), "evictions": int(eng.rank.evictions),
        "registrations": int(eng.rank.registrations),
        "handler_ops_max": int(eng.handler_ops_max),
        "batches": int(sum(len(g) for g in res.gpu_logs)),
        "stats": {
            "goodput_rps": st.goodput_rps, "bad_rate": st.bad_rate,
            "mean_idle_fraction": st.mean_idle_fraction,
            "idle_digest": D._h(np.asarray(st.gpu_idle_fraction).view(np.int64)),
            "p99": [m.p99_latency_ns for m in st.models],
            "median_batch": [m.median_batch for m in st.models],
            "max_qd": [m.max_queueing_delay_ns for m in st.models],
            "hist_digest": D._h([x for m in st.models for kv in sorted(m.batch_hist.items())
                                 for x in kv]),
        },
        "ref_seconds": round(el, 3),
    }


def bundled_cases(out):
    for name in BUNDLED_SCENARIOS:
        sc = load_scenario(name)
        ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models],
                                        sc.duration_s, sc.seed)
        for v in POLICIES:
            pol = policy_for(sc.policy, v)
            out[f"{name}/{v}"] = run_case(sc.models, sc.gpu_count, pol, ticks, midx,
                                          sc.duration_s, sc.warmup_s, sc.cooldown_s)
            print(name, v, out[f"{name}/{v}"]["ref_seconds"], flush=True)


def zoo_models(n, slo=None):
    from batchsym.profile import load_model_zoo
    zoo = load_model_zoo("a100")
    return [ModelSpec(i, f"{zoo[i % len(zoo)].name}_{i}",
                      LatencyProfile.linear(zoo[i % len(zoo)].alpha_ms, zoo[i % len(zoo)].beta_ms),
                      int(round((zoo[i % len(zoo)].slo_ms if slo is None else slo(i)) * 1e6)))
            for i in range(n)]


def config_cases(out):
    """C1-C5 at reduced durations; C4 per sub-cluster."""
    import math
    c5_dur = 0.6
    segs = tuple((j * c5_dur / 24, 600_000.0 * (0.55 - 0.45 * math.cos(2 * math.pi * j / 24)))
                 for j in range(24))
    cfgs = {
        "C1": ([ModelSpec(0, "ResNet50", LatencyProfile.linear(1.053, 5.072), 50_000_000)], 8,
               WorkloadSpec("poisson", 2000.0), 60.0),
        "C2": (zoo_models(10, slo=lambda i: float(round(20 + 80 * i / 9))), 64,
               WorkloadSpec("poisson", 40_000.0), 1.0),
        "C3": (zoo_models(100), 1024, WorkloadSpec("gamma", 300_000.0, gamma_shape=1 / 16), 0.25),
        "C4": (zoo_models(1000), 8192, WorkloadSpec("poisson", 1_200_000.0), 0.1),
        "C5": (zoo_models(500), 4096, WorkloadSpec("piecewise", segments=segs), c5_dur),
    }
    for name, (models, gpus, wl, dur) in cfgs.items():
        ticks, midx = generate_arrivals(wl, [m.name for m in models], dur, 42)
        variants = ("base", "eager", "timeout30", "delay") if name in ("C1", "C2") else ("base",)
        for v in variants:
            pol = policy_for(PolicyConfig("deferred"), v)
            if name == "C4":
                for s in range(8):
                    ids = np.arange(125 * s, 125 * (s + 1))
                    sel = (midx >= ids[0]) & (midx <= ids[-1])
                    sm = [ModelSpec(k, models[i].name, models[i].profile, models[i].slo_ns)
                          for k, i in enumerate(ids)]
                    out[f"C4s{s}/{v}@{dur}"] = run_case(sm, 1024, pol, ticks[sel],
                                                        midx[sel] - ids[0], dur, 0.1 * dur,
                                                        0.1 * dur)
                    print(name, s, out[f"C4s{s}/{v}@{dur}"]["ref_seconds"], flush=True)
                out[f"C4/trace_in@{dur}"] = D.trace_digest(ticks, midx)
            else:
                out[f"{name}/{v}@{dur}"] = run_case(models, gpus, pol, ticks, midx, dur,
                                                    0.1 * dur, 0.1 * dur)
                print(name, v, out[f"{name}/{v}@{dur}"]["ref_seconds"], flush=True)


def known_answers(out):
    """Scalar known answers used by the host tests (reference functions)."""
    from batchsym import metrics as M
    from batchsym.profile import max_feasible_batch, schedulable_window
    r50 = LatencyProfile.linear(1.053, 5.072)
    irv2 = LatencyProfile.linear(5.090, 18.368)
    ka = {
        "window_r50_25ms_b7": list(vars(schedulable_window(r50, 25_000_000, 7)).values()),
        "mfb_r50_12.5": max_feasible_batch(r50, 12_500_000),
        "mfb_irv2_62.222": max_feasible_batch(irv2, 62_222_000),
        "analytic": {f"{n}/{mode}": [s.batch_size, s.throughput_rps]
                     for n, p, slo in (("r50", r50, 25_000_000), ("irv2", irv2, 70_000_000))
                     for mode in ("staggered", "no_coordination")
                     for s in [M.analytical_solution(p, slo, 8, mode)]},
        "autoscale": [[r, f, n, M.autoscale_advice(r, f, n)]
                      for r, f, n in ((0.0, 0.5, 100), (0.2, 0.0, 100), (0.009, 0.06, 7),
                                      (0.5, 0.9, 3), (0.0, 1.0, 4096), (0.02, 0.3, 242))],
    }
    gs = {}
    for name in ("table2_resnet50", "table2_inceptionresnet"):
        res = M.goodput_search(load_scenario(name))
        gs[name] = {"rate_rps": res.rate_rps, "probes": res.probes}
        print("goodput", name, res.rate_rps, flush=True)
    ka["goodput_search"] = gs
    out["known_answers"] = ka


def autoscale_cases(out):
    """C5 active-GPU series: reference compute_stats per 25 ms epoch of the
    0.6 s diurnal run + autoscale_advice."""
    import math
    dur = 0.6
    segs = tuple((j * dur / 24, 600_000.0 * (0.55 - 0.45 * math.cos(2 * math.pi * j / 24)))
                 for j in range(24))
    models = zoo_models(500)
    ticks, midx = generate_arrivals(WorkloadSpec("piecewise", segments=segs),
                                    [m.name for m in models], dur, 42)
    eng = Engine(models, 4096, PolicyConfig("deferred"), NetworkModel.zero())
    res = eng.run_stream(ticks, midx, dur)
    series = []
    for e in range(24):
        st = RM.compute_stats(res, e * dur / 24, dur - (e + 1) * dur / 24, dur)
        r = min(st.bad_rate, math.nextafter(1.0, 0.0))
        series.append(4096 + RM.autoscale_advice(r, st.mean_idle_fraction, 4096))
    out["C5/autoscale_series@0.6"] = series
    print("autoscale", series, flush=True)


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


def jitter_cases(out):
    """Jittered network (network.py:69-77): histogram delays sampled per
    dispatch from the engine's Philox substream; LATE outcomes appear."""
    import copy
    import os as _os
    from batchsym.scenario import scenario_from_dict
    import yaml
    root = "/root/reference/pkg/src/batchsym/scenarios"
    for name, net, kind in JITTER_CASES:
        doc = yaml.safe_load(open(_os.path.join(root, name + ".yaml")))
        doc = copy.deepcopy(doc)
        doc["network"] = JITTER_NETS[net]
        if kind:
            doc.setdefault("policy", {})["kind"] = kind
            if kind == "timeout":
                doc["policy"]["timeout_slo_frac"] = 0.3
        sc = scenario_from_dict(doc, name=name, base_dir=root)
        ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models],
                                        sc.duration_s, sc.seed)
        key = f"jitter/{name}/{net}/{kind or 'base'}"
        out[key] = run_case(sc.models, sc.gpu_count, sc.policy, ticks, midx, sc.duration_s,
                            sc.warmup_s, sc.cooldown_s, network=sc.network, seed=sc.seed)
        print(key, out[key]["late"], out[key]["drops"], flush=True)


OUTPUT_FILES = ("summary.json", "requests.csv", "trace.csv", "batch_hist.csv",
                "latency.csv", "utilization.csv")
OUTPUT_CASES = ["fig6_stagger", "fig7_skip", "table2_inceptionresnet", "fig4b_timeout_zoo",
                "jitter/fig6_stagger/J2/base", "jitter/table2_inceptionresnet/J3/timeout"]


def output_cases(out):
    """Exact bytes of the reference's six result files (outputs.py) for a
    few bundled and jittered runs, as digests of the file text."""
    import copy
    import yaml
    from batchsym import outputs as RO
    from batchsym.scenario import scenario_from_dict
    root = "/root/reference/pkg/src/batchsym/scenarios"
    for case in OUTPUT_CASES:
        if case.startswith("jitter/"):
            _, name, net, kind = case.split("/")
            doc = copy.deepcopy(yaml.safe_load(open(os.path.join(root, name + ".yaml"))))
            doc["network"] = JITTER_NETS[net]
            if kind != "base":
                doc.setdefault("policy", {})["kind"] = kind
                if kind == "timeout":
                    doc["policy"]["timeout_slo_frac"] = 0.3
            sc = scenario_from_dict(doc, name=name, base_dir=root)
        else:
            sc = load_scenario(case)
        ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models],
                                        sc.duration_s, sc.seed)
        eng = Engine(list(sc.models), sc.gpu_count, sc.policy, sc.network, seed=sc.seed,
                     record_trace=True)
        res = eng.run_stream(ticks, midx, sc.duration_s)
        st = RM.compute_stats(res, sc.warmup_s, sc.cooldown_s, sc.duration_s)
        extra = {"gpu_count": sc.gpu_count, "policy": sc.policy.kind}
        t0 = time.time()
        files = {
            "summary.json": RO.summary_json(st, sc.name, sc.seed, extra),
            "requests.csv": RO.requests_csv(res),
            "trace.csv": RO.trace_csv(res),
            "batch_hist.csv": RO.batch_hist_csv(st),
            "latency.csv": RO.latency_csv(res),
            "utilization.csv": RO.utilization_csv(res, st),
        }
        el = time.time() - t0
        out[f"outputs/{case}"] = {
            "scenario": sc.name, "seed": sc.seed, "extra": extra,
            "digests": {k: D.text_digest(v) for k, v in files.items()},
            "bytes": {k: len(v) for k, v in files.items()},
            "ref_seconds": round(el, 3),
        }
        print("outputs", case, round(el, 3), flush=True)


SWEEP_CASES = [
    ("beta_ratio", "table2_resnet50", [1.0, 6.0], ["deferred", "eager"], None),
    ("timeout", "fig4b_timeout_sweep", [10.0, 60.0], None, None),
    ("offered_load", "table2_resnet50", [0.5, 1.25], None, 5000.0),
    ("slo", "table2_inceptionresnet", [40.0, 90.0], ["deferred", "timeout:30"], None),
]


def sweep_cases(out):
    """Rows of the reference's grid sweeps (sweeps.py:67-142), each point a
    goodput search or fixed-rate run through run_scenario."""
    from batchsym import sweeps as RS
    rows = {}
    for dim, name, grid, pols, peak in SWEEP_CASES:
        t0 = time.time()
        rows[f"{dim}/{name}"] = RS.run_sweep(dim, load_scenario(name), grid, pols, peak)
        print("sweep", dim, name, round(time.time() - t0, 2), flush=True)
    out["sweeps"] = rows


SCALEBENCH_SHARDS = [(8, 16), (32, 4), (1, 1), (64, 128)]
SCALEBENCH_KEEP = 5000


def scalebench_cases(out):
    """The reference's wall-clock shard loop (scalebench.py:49-85), run for a
    short interval with its Engine captured: the digest of its arrival
    stream and of the first SCALEBENCH_KEEP requests' outcomes pin the
    package's restated stream and the equivalence of the step loop with
    run_stream on that stream."""
    from batchsym import scalebench as RSB
    keep = SCALEBENCH_KEEP
    cases = {}
    for n_models, n_gpus in SCALEBENCH_SHARDS:
        captured = []

        class Capture(RSB.Engine):
            def __init__(self, *a, **k):
                super().__init__(*a, **k)
                captured.append(self)
        orig = RSB.Engine
        RSB.Engine = Capture
        try:
            n = RSB._shard_loop(n_models, n_gpus, 0.5)
        finally:
            RSB.Engine = orig
        eng = captured[0]
        assert n >= 2 * keep, n
        cases[f"{n_models}x{n_gpus}"] = {
            "n_models": n_models, "n_gpus": n_gpus, "keep": keep,
            "stream": D.trace_digest(eng._arrival[:keep], eng._model_idx[:keep]),
            "requests": D.requests_digest(eng._dispatch[:keep], eng._start[:keep],
                                          eng._finish[:keep], eng._batch[:keep],
                                          eng._outcome[:keep]),
            "resolved": int(sum(1 for o in eng._outcome[:keep] if o >= 0)),
        }
        print("scalebench", n_models, n_gpus, n, flush=True)
    out["scalebench"] = cases


PART_BRUTE = [(8, 3, 0), (10, 2, 1), (12, 3, 2), (9, 4, 3), (13, 3, 4), (6, 10, 5), (20, 2, 6)]
PART_TEXT = """# l=3
# R_max=400
# S_max=
# w=0.05
# C_max=7.5
model,rate_rps,static_mem_mb,dynamic_mem_mb
resnet50,120.5,98,40
bert,80,420.25,120
gpt2,35.125,510,200
vgg16,60,530,90
mobilenet,220,17,8
"""


def _part_variants(P, seed):
    """The random instance plus capped / weighted / change-budget variants."""
    from dataclasses import replace as dreplace
    base = P.random_instance(*seed)
    m, l = base.n_models, base.subclusters
    rng = np.random.default_rng(seed[2] + 100)
    cur = tuple(int(v) for v in rng.integers(0, l, m))
    cost = tuple(tuple(round(float(c), 3) for c in row) for row in rng.uniform(0.5, 3.0, (m, l)))
    return {
        "plain": base,
        "tight": dreplace(base, rate_cap=base.rate_cap / 1.5 * 1.02, mem_cap=base.mem_cap / 1.4),
        "infeasible": dreplace(base, rate_cap=1.0),
        "weighted": dreplace(base, weight=0.125),
        "budget": dreplace(base, current=cur, change_cost=cost, change_budget=6.0 + seed[2]),
        "unit_budget": dreplace(base, current=cur, change_budget=4.0),
    }


def partition_cases(out):
    """Reference partitioner (partitioner.py): brute-force optima, the first
    minimum over the random baseline's first draws, the solver's objective at
    a 1 s budget (a quality bar), and a parsed problem file."""
    from batchsym import partitioner as P
    from batchsym.workload import substream
    brute, rnd = {}, {}
    for inst in PART_BRUTE:
        for name, prob in _part_variants(P, inst).items():
            t0 = time.time()
            r = P.brute_force(prob)
            ev = r.evaluation
            brute[f"{inst}/{name}"] = {"assignment": list(r.assignment), "objective": ev.objective,
                                       "feasible": ev.feasible, "change_cost": ev.change_cost,
                                       "seconds": round(time.time() - t0, 2)}
            rng = substream(inst[2], 1)
            best_key, best_k, rows = None, None, []
            for _ in range(4):
                rows += [[int(v) for v in row] for row in rng.integers(0, prob.subclusters,
                                                                       size=(256, prob.n_models))]
            for k, x in enumerate(rows):
                e = P.evaluate(prob, x)
                key = (0.0 if e.feasible else 1.0, e.objective)
                if best_key is None or key < best_key:
                    best_key, best_k = key, k
            rnd[f"{inst}/{name}"] = {"index": best_k, "assignment": rows[best_k],
                                     "objective": best_key[1], "feasible": best_key[0] == 0.0}
            print("partition", inst, name, brute[f"{inst}/{name}"]["seconds"], flush=True)
    solve = {}
    for inst in [(60, 8, 11), (200, 16, 12), (40, 4, 13)]:
        prob = P.random_instance(*inst)
        r = P.solve(prob, 1.0, inst[2])
        solve[str(inst)] = {"objective": r.evaluation.objective, "feasible": r.feasible,
                            "restarts": r.restarts}
        print("partition solve", inst, r.evaluation.objective, r.restarts, flush=True)
    pp = P.parse_problem(PART_TEXT)
    out["partition"] = {"brute": brute, "random_first": rnd, "solve_1s": solve,
                        "parsed": {"names": list(pp.names), "rates": list(pp.rates),
                                   "static": list(pp.static_mem), "dynamic": list(pp.dynamic_mem),
                                   "l": pp.subclusters, "rate_cap": pp.rate_cap,
                                   "mem_cap": str(pp.mem_cap), "weight": pp.weight,
                                   "change_budget": pp.change_budget,
                                   "csv": P.assignment_csv(pp, [0, 1, 2, 0, 1])}}


def stress_cases(out, n_cases=60):
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from stress_cases import make_case
    for seed in range(n_cases):
        c = make_case(seed)
        models = [ModelSpec(i, f"m{i}", LatencyProfile(p["kind"], p["max_batch"], 0, 0,
                                                        tuple(p["lat"])), p["slo"])
                  for i, p in enumerate(c["models"])]
        pol = PolicyConfig(**c["policy"])
        out[f"stress/{seed}"] = run_case(models, c["gpus"], pol, c["ticks"], c["midx"], 1.0,
                                         0.1, 0.1)


if __name__ == "__main__":
    if sys.argv[1:] in (["outputs"], ["sweeps"], ["scalebench"], ["partition"]):  # refresh one section only
        path = os.path.join(HERE, "golden.json")
        out = json.load(open(path))
        {"outputs": output_cases, "sweeps": sweep_cases,
         "scalebench": scalebench_cases, "partition": partition_cases}[sys.argv[1]](out)
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)
        sys.exit(0)
    out = {"generator": "tests/golden/make_golden.py", "reference": "batchsym 0.1.0",
           "numpy": np.__version__}
    known_answers(out)
    jitter_cases(out)
    autoscale_cases(out)
    bundled_cases(out)
    stress_cases(out)
    config_cases(out)
    output_cases(out)
    sweep_cases(out)
    scalebench_cases(out)
    partition_cases(out)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote golden.json")
