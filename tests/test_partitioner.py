"""Sub-cluster partitioner (reference partitioner.py):
host evaluation and file formats against the reference's values, the GPU
brute force and random baseline bit-exact against the reference's results,
the GPU multi-start local search against the reference solver's 1 s
objective (tests/golden/make_golden.py:partition_cases)."""
from __future__ import annotations

import ast
import math
from dataclasses import replace

import numpy as np
import pytest

from paper_2308_07470_b200 import partitioner as P

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


def variants(inst):
    base = P.random_instance(*inst)
    m, l = base.n_models, base.subclusters
    rng = np.random.default_rng(inst[2] + 100)
    cur = tuple(int(v) for v in rng.integers(0, l, m))
    cost = tuple(tuple(round(float(c), 3) for c in row) for row in rng.uniform(0.5, 3.0, (m, l)))
    return {
        "plain": base,
        "tight": replace(base, rate_cap=base.rate_cap / 1.5 * 1.02, mem_cap=base.mem_cap / 1.4),
        "infeasible": replace(base, rate_cap=1.0),
        "weighted": replace(base, weight=0.125),
        "budget": replace(base, current=cur, change_cost=cost, change_budget=6.0 + inst[2]),
        "unit_budget": replace(base, current=cur, change_budget=4.0),
    }


CASES = [(inst, name) for inst in PART_BRUTE for name in variants(inst)]
IDS = [f"{i}/{n}" for i, n in CASES]


@pytest.mark.parametrize("inst,name", CASES, ids=IDS)
def test_evaluate_matches_reference(inst, name, golden):
    prob = variants(inst)[name]
    g = golden["partition"]["brute"][f"{inst}/{name}"]
    ev = P.evaluate(prob, g["assignment"])
    assert ev.objective == g["objective"] and ev.feasible == g["feasible"]
    assert ev.change_cost == g["change_cost"]
    r = golden["partition"]["random_first"][f"{inst}/{name}"]
    ev = P.evaluate(prob, r["assignment"])
    assert ev.objective == r["objective"] and ev.feasible == r["feasible"]


def test_parse_problem_and_assignment_csv(golden):
    g = golden["partition"]["parsed"]
    p = P.parse_problem(PART_TEXT)
    assert list(p.names) == g["names"] and list(p.rates) == g["rates"]
    assert list(p.static_mem) == g["static"] and list(p.dynamic_mem) == g["dynamic"]
    assert p.subclusters == g["l"] and p.rate_cap == g["rate_cap"]
    assert str(p.mem_cap) == g["mem_cap"] and p.weight == g["weight"]
    assert p.change_budget == g["change_budget"]
    assert P.assignment_csv(p, [0, 1, 2, 0, 1]) == g["csv"]


@pytest.mark.parametrize("text,err", [
    ("model,rate_rps,static_mem_mb,dynamic_mem_mb\na,1,2,3\n", "missing '# l='"),
    ("# l=2\nmodel,rate\na,1\n", "expected header"),
    ("# l=2\nmodel,rate_rps,static_mem_mb,dynamic_mem_mb\na,1,2\n", "expected 4 fields"),
    ("# l=2\nmodel,rate_rps,static_mem_mb,dynamic_mem_mb\na,x,2,3\n", "could not convert"),
])
def test_parse_problem_errors(text, err):
    with pytest.raises(P.PartitionError, match=err):
        P.parse_problem(text)


def test_problem_validation():
    with pytest.raises(P.PartitionError):
        P.PartitionProblem((), (), (), (), 2)
    with pytest.raises(P.PartitionError):
        P.PartitionProblem(("a",), (1.0,), (-1.0,), (0.0,), 2)
    with pytest.raises(P.PartitionError):
        P.PartitionProblem(("a",), (1.0,), (1.0,), (0.0,), 2, current=(2,))
    prob = P.random_instance(5, 2, 0)
    with pytest.raises(P.PartitionError):
        P.evaluate(prob, [0, 1, 2, 0, 1])
    with pytest.raises(P.PartitionError):
        P.brute_force(P.random_instance(23, 2, 0))
    with pytest.raises(P.PartitionError):
        P.solve(prob, 0.0, 1)
    a, b = P.imbalance_factor(prob, [0, 1, 0, 1, 0])
    assert a >= 0 and b >= 0


@pytest.mark.gpu
@pytest.mark.parametrize("inst,name", CASES, ids=IDS)
def test_brute_force_gpu_matches_reference(inst, name, golden):
    g = golden["partition"]["brute"][f"{inst}/{name}"]
    r = P.brute_force(variants(inst)[name])
    assert list(r.assignment) == g["assignment"]
    assert r.evaluation.objective == g["objective"] and r.feasible == g["feasible"]


@pytest.mark.gpu
@pytest.mark.parametrize("inst,name", CASES[::3], ids=IDS[::3])
def test_random_baseline_gpu_matches_reference(inst, name, golden):
    g = golden["partition"]["random_first"][f"{inst}/{name}"]
    r = P.random_solver(variants(inst)[name], 60.0, inst[2], max_draws=1024)
    assert r.restarts == 1024
    assert list(r.assignment) == g["assignment"] and r.evaluation.objective == g["objective"]


@pytest.mark.gpu
def test_evaluate_many_equals_host():
    prob = variants((12, 3, 2))["budget"]
    rows = np.random.default_rng(5).integers(0, 3, (3000, 12))
    obj, feas, best = P.evaluate_many(prob, rows)
    host = [P.evaluate(prob, r) for r in rows]
    assert obj.tolist() == [e.objective for e in host]
    assert feas.tolist() == [e.feasible for e in host]
    keys = [(0.0 if e.feasible else 1.0, e.objective) for e in host]
    assert best == min(range(len(keys)), key=lambda k: (keys[k], k))


@pytest.mark.gpu
@pytest.mark.parametrize("inst", [(10, 2, 1), (12, 3, 2), (9, 4, 3), (13, 3, 4)])
def test_solve_reaches_brute_force_optimum(inst, golden):
    for name in ("plain", "weighted", "budget"):
        g = golden["partition"]["brute"][f"{inst}/{name}"]
        r = P.solve(variants(inst)[name], 0.5, 7, max_launches=2)
        assert r.feasible == g["feasible"]
        assert r.evaluation.objective <= g["objective"] * (1 + 1e-12) + 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["(60, 8, 11)", "(200, 16, 12)", "(40, 4, 13)"])
def test_solve_beats_reference_budget(key, golden):
    """Same 1 s budget: the device's parallel restarts find an assignment
    at least as good as the reference solver's."""
    g = golden["partition"]["solve_1s"][key]
    r = P.solve(P.random_instance(*ast.literal_eval(key)), 1.0, 3)
    assert r.feasible and g["feasible"]
    assert r.evaluation.objective <= g["objective"] + 1e-9
    assert math.isfinite(r.evaluation.objective) and r.restarts >= P.RESTARTS_PER_LAUNCH
