"""CPU-only tests: host-side API mirror (profile/window/zoo/policy/scenario/
metrics known answers from the reference) and the C-ABI library surface."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2308_07470_b200 import (PolicyConfig, analytical_solution, autoscale_advice,
                                   load_model_zoo, load_scenario, max_feasible_batch,
                                   schedulable_window)
from paper_2308_07470_b200.profile import (InvalidBatchSize, LatencyProfile, ModelSpec,
                                           ProfileError, exec_latency)
from paper_2308_07470_b200.scenario import ScenarioError, scenario_from_dict
from paper_2308_07470_b200.units import ms_to_ns

UNIT = LatencyProfile.linear(1.0, 5.0, max_batch=16)
R50 = LatencyProfile.linear(1.053, 5.072)
IRV2 = LatencyProfile.linear(5.090, 18.368)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_latency_values():  # reference test_profile.py:55-58
    assert exec_latency(UNIT, 4) == ms_to_ns(9.0)
    assert exec_latency(R50, 16) == ms_to_ns(21.920)
    assert exec_latency(LatencyProfile.linear(0.054, 10.546), 1) == ms_to_ns(10.600)
    with pytest.raises(InvalidBatchSize):
        exec_latency(UNIT, 0)
    with pytest.raises(InvalidBatchSize):
        exec_latency(UNIT, 17)


def test_windows(golden):  # reference test_profile.py:68-87
    w = schedulable_window(UNIT, ms_to_ns(12.0), 4)
    assert (w.frontrun, w.latest) == (ms_to_ns(2.0), ms_to_ns(3.0))
    flat = LatencyProfile.linear(0.0, 7.0, max_batch=8)
    w = schedulable_window(flat, ms_to_ns(20.0), 3)
    assert w.frontrun == w.latest == ms_to_ns(13.0)
    w = schedulable_window(R50, ms_to_ns(25.0), 7)
    assert [w.frontrun, w.latest] == golden["known_answers"]["window_r50_25ms_b7"]
    w = schedulable_window(UNIT, ms_to_ns(30.0), 16)
    assert w.frontrun == w.latest
    for b in range(1, 16):
        w = schedulable_window(UNIT, ms_to_ns(100.0), b)
        assert w.latest - w.frontrun == UNIT.alpha_ns


def test_max_feasible(golden):
    ka = golden["known_answers"]
    assert max_feasible_batch(UNIT, ms_to_ns(12.0)) == 7
    assert max_feasible_batch(R50, ms_to_ns(12.5)) == ka["mfb_r50_12.5"] == 7
    assert max_feasible_batch(IRV2, ms_to_ns(62.222)) == ka["mfb_irv2_62.222"] == 8
    assert max_feasible_batch(UNIT, ms_to_ns(5.0)) == 0
    slo = ms_to_ns(25.0)
    for o1 in range(0, 21, 3):
        for o2 in range(0, 21, 4):
            lo, hi = sorted((ms_to_ns(float(o1)), ms_to_ns(float(o2))))
            assert max_feasible_batch(R50, slo, hi) <= max_feasible_batch(R50, slo, lo)


def test_tables():  # reference test_profile.py:110-127
    prof = LatencyProfile.table({1: 5.0, 4: 8.0, 8: 12.0})
    assert all(a <= b for a, b in zip(prof.lat_ns, prof.lat_ns[1:]))
    with pytest.raises(ProfileError):
        LatencyProfile.table({1: 5.0, 4: 3.0})
    prof = LatencyProfile.table({1: 1.0, 5: 5.0})
    assert [prof.latency(b) for b in range(1, 6)] == [ms_to_ns(float(v)) for v in range(1, 6)]
    prof = LatencyProfile.table([2.0, 3.0, 4.5])
    assert prof.latency(2) == ms_to_ns(3.0) and prof.max_batch == 3
    prof = LatencyProfile.table({1: 1.0, 3: 2.0}, max_batch=6)
    assert prof.lat_ns == (1_000_000, 1_500_000, 2_000_000, 2_000_000, 2_000_000, 2_000_000)
    with pytest.raises(ProfileError):
        LatencyProfile.linear(-1.0, 5.0)
    with pytest.raises(ProfileError):
        LatencyProfile.linear(1.0, 0.0)
    with pytest.raises(ProfileError):
        ModelSpec(0, "bad", UNIT, ms_to_ns(5.0))


def test_zoos():
    ti, a100 = load_model_zoo("1080ti"), load_model_zoo("a100")
    assert len(ti) == 35 and len(a100) == 37
    r50 = next(z for z in ti if z.name == "ResNet50")
    assert (r50.alpha_ms, r50.beta_ms, r50.slo_ms) == (2.050, 5.378, 27)
    d121 = next(z for z in a100 if z.name == "DenseNet121")
    assert (d121.alpha_ms, d121.beta_ms, d121.slo_ms) == (0.054, 10.546, 21)


def test_policy_validation():
    for bad in (dict(kind="lazy"), dict(kind="deferred", timeout_ns=-1),
                dict(kind="deferred", d_ctrl_ns=-5), dict(kind="deferred", gather="x"),
                dict(kind="deferred", gather="drop_head", target_batch=0),
                dict(kind="timeout", timeout_slo_frac=-0.1)):
        with pytest.raises(ValueError):
            PolicyConfig(**bad)
    assert PolicyConfig("timeout", timeout_slo_frac=0.3).resolve_timeout_ns(50_000_000) == 15_000_000


def test_scenarios_load_and_validate():
    sc = load_scenario("fig6_stagger")
    assert sc.gpu_count == 3 and sc.models[0].profile.max_batch == 16
    assert load_scenario("fig4b_timeout_zoo").models[0].name == "DenseNet121"
    assert len(load_scenario("fig2_flattop").models) == 10
    with pytest.raises(ScenarioError) as ei:
        scenario_from_dict({"models": [{"name": "a"}], "gpus": 0, "workload": {},
                            "duration_s": 1.0, "seed": "x"})
    msg = str(ei.value)
    assert "missing" in msg and "gpus" in msg and "seed" in msg
    with pytest.raises(FileNotFoundError):
        load_scenario("/nonexistent.yaml")


def test_analytical_and_autoscale(golden):
    ka = golden["known_answers"]
    for key, (bs, tpt) in ka["analytic"].items():
        name, mode = key.split("/")
        prof, slo = (R50, ms_to_ns(25.0)) if name == "r50" else (IRV2, ms_to_ns(70.0))
        s = analytical_solution(prof, slo, 8, mode)
        assert (s.batch_size, s.throughput_rps) == (bs, tpt)
    for r, f, n, want in ka["autoscale"]:
        assert autoscale_advice(r, f, n) == want
    with pytest.raises(ValueError):
        autoscale_advice(1.0, 0.0, 4)


def _lib_path():
    import __graft_entry__ as g
    return g.build_engine()


def test_library_exports_every_header_symbol():
    """The C-ABI library loads on a CPU-only host and exports exactly what
    include/symphony_b200.h declares (no compute call without a GPU)."""
    lib = ctypes.CDLL(_lib_path())
    header = open(os.path.join(ROOT, "include", "symphony_b200.h")).read()
    decls = re.findall(r"^\s*(?:[\w\s\*]+?)\b(sym_\w+)\s*\(", header, re.M)
    assert set(decls) >= {"sym_create", "sym_run", "sym_run_device", "sym_destroy"}
    for name in decls:
        assert hasattr(lib, name), name
    lib.sym_version.restype = ctypes.c_int32
    assert lib.sym_version() >= 1


def test_engine_api_validates_before_device(monkeypatch):
    from paper_2308_07470_b200 import Engine
    from paper_2308_07470_b200.network import DelayDist, NetworkModel
    m = [ModelSpec(0, "m", UNIT, ms_to_ns(12.0))]
    with pytest.raises(ValueError):
        Engine(m, 0, PolicyConfig("deferred"))
    jitter = NetworkModel(DelayDist.histogram([0, 10], [1, 1]), DelayDist.constant(0))
    assert Engine(m, 1, PolicyConfig("deferred"), jitter)._jitter is not None
    with pytest.raises(ValueError):
        Engine(m * 1, 2, PolicyConfig("deferred"), shards=([0], [1, 1]))


def test_product_has_no_oracle_dependency():
    """The product package must never import the oracle (it is the checker)."""
    pkg = os.path.join(ROOT, "paper_2308_07470_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|symoracle|symo_", src, re.M), f
