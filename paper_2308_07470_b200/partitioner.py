"""Sub-cluster partitioning (mirrors batchsym/partitioner.py).

Spread models across dispatcher sub-clusters so per-sub-cluster request
rate and static memory stay close to their averages:

    minimize  max_j |rate_j - mean_rate|  +  w * max_j |mem_j - mean_mem|

subject to rate_j <= rate_cap, mem_j + max(dynamic peak) <= mem_cap and an
optional change budget against a current assignment (partitioner.py:1-18).
Its output picks the C4 sub-clusters.

The searches run on the GPU (csrc/partition.cu): ``brute_force`` scores all
l^m assignments at once and returns exactly the reference's optimum (same
double-precision operations, same first-in-product-order tie-break);
``random_solver`` draws the reference's numpy rows and scores them in
batches; ``solve`` runs thousands of independent greedy + local-search
restarts per launch under the wall-clock budget.  Problem I/O, ``evaluate``
and the imbalance factors are host code, identical to the reference.
"""
from __future__ import annotations

import csv
import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from .workload import substream

INF = float("inf")
RESTARTS_PER_LAUNCH = 1024
RANDOM_BATCHES_PER_LAUNCH = 64


class PartitionError(ValueError):
    pass


@dataclass(frozen=True)
class PartitionProblem:
    names: tuple[str, ...]
    rates: tuple[float, ...]
    static_mem: tuple[float, ...]
    dynamic_mem: tuple[float, ...]
    subclusters: int
    rate_cap: float = INF
    mem_cap: float = INF
    weight: float | None = None  # None -> mean_rate / mean_mem
    current: tuple[int, ...] | None = None
    change_cost: tuple[tuple[float, ...], ...] | None = None  # c[i][j]
    change_budget: float = INF

    def __post_init__(self) -> None:  # partitioner.py:52-69
        m = len(self.names)
        if m == 0:
            raise PartitionError("no models")
        for fld in (self.rates, self.static_mem, self.dynamic_mem):
            if len(fld) != m:
                raise PartitionError("per-model arrays must align")
            if any(v < 0 for v in fld):
                raise PartitionError("negative model quantity")
        if self.subclusters < 1:
            raise PartitionError("need at least one sub-cluster")
        if self.current is not None:
            if len(self.current) != m:
                raise PartitionError("current assignment length mismatch")
            if any(not 0 <= j < self.subclusters for j in self.current):
                raise PartitionError("current assignment out of range")
        if self.change_cost is not None and len(self.change_cost) != m:
            raise PartitionError("change cost matrix must be m x l")

    @property
    def n_models(self) -> int:
        return len(self.names)

    @property
    def mean_rate(self) -> float:
        return sum(self.rates) / self.subclusters

    @property
    def mean_mem(self) -> float:
        return sum(self.static_mem) / self.subclusters

    def effective_weight(self) -> float:
        if self.weight is not None:
            return self.weight
        return self.mean_rate / self.mean_mem if self.mean_mem > 0 else 1.0

    def cost_of(self, i: int, j: int) -> float:
        return 1.0 if self.change_cost is None else self.change_cost[i][j]

    def move_cost(self, i: int, j_from: int, j_to: int) -> float:
        """One unload plus one load (partitioner.py:95-99)."""
        if j_from == j_to:
            return 0.0
        return self.cost_of(i, j_from) + self.cost_of(i, j_to)


@dataclass(frozen=True)
class Evaluation:
    objective: float
    rate_dev: float
    mem_dev: float
    feasible: bool
    violations: tuple[str, ...]
    change_cost: float


def _sums(problem: PartitionProblem, x: np.ndarray):
    """Per-sub-cluster rate / static-memory sums and dynamic peaks.  np.add.at
    accumulates unbuffered in model order, the order the reference's loop
    adds in (partitioner.py:118-123), so the float sums are identical."""
    l = problem.subclusters
    rate, mem, peak = np.zeros(l), np.zeros(l), np.zeros(l)
    np.add.at(rate, x, np.asarray(problem.rates, np.float64))
    np.add.at(mem, x, np.asarray(problem.static_mem, np.float64))
    np.maximum.at(peak, x, np.asarray(problem.dynamic_mem, np.float64))
    return rate, mem, peak


def evaluate(problem: PartitionProblem, assignment) -> Evaluation:
    """Objective, deviations, cap/budget violations (partitioner.py:114-145)."""
    x = np.asarray(assignment, dtype=np.int64).reshape(-1)
    if len(x) != problem.n_models or (len(x) and (x.min() < 0 or x.max() >= problem.subclusters)):
        raise PartitionError("malformed assignment")
    rate, mem, peak = _sums(problem, x)
    d_rate = float(np.abs(rate - problem.mean_rate).max())
    d_mem = float(np.abs(mem - problem.mean_mem).max())
    bad = []
    for j, (r, s) in enumerate(zip(rate.tolist(), (mem + peak).tolist())):
        if r > problem.rate_cap:
            bad.append(f"subcluster {j}: rate {r:.3f} > cap {problem.rate_cap:.3f}")
        if s > problem.mem_cap:
            bad.append(f"subcluster {j}: memory {s:.3f} > cap {problem.mem_cap:.3f}")
    moved = 0.0
    if problem.current is not None:
        for i, (was, now) in enumerate(zip(problem.current, x.tolist())):
            moved += problem.move_cost(i, was, now)  # sequential, as the reference sums
        if moved > problem.change_budget:
            bad.append(f"change cost {moved:.3f} > budget {problem.change_budget:.3f}")
    return Evaluation(d_rate + problem.effective_weight() * d_mem, d_rate, d_mem, not bad,
                      tuple(bad), moved)


def imbalance_factor(problem: PartitionProblem, assignment) -> tuple[float, float]:
    """(max - min) / avg of the per-sub-cluster rate and static-memory sums
    (partitioner.py:148-163)."""
    rate, mem, _ = _sums(problem, np.asarray(assignment, dtype=np.int64).reshape(-1))
    factors = []
    for sums in (rate.tolist(), mem.tolist()):
        avg = sum(sums) / problem.subclusters
        if avg <= 0:
            raise PartitionError("imbalance factor undefined for zero average")
        factors.append((max(sums) - min(sums)) / avg)
    return factors[0], factors[1]


@dataclass
class SolveResult:
    assignment: tuple[int, ...]
    evaluation: Evaluation
    restarts: int = 0
    improvements: int = 0

    @property
    def feasible(self) -> bool:
        return self.evaluation.feasible


# -- device searches ------------------------------------------------------------

class _Device:
    """The problem as the C ABI's sym_part_problem (arrays kept alive)."""

    def __init__(self, problem: PartitionProblem, device: int):
        from . import _native
        self.lib = _native.load()
        self.device = device
        m, l = problem.n_models, problem.subclusters
        if l > 64:
            raise PartitionError("the device searches support at most 64 sub-clusters")
        self.keep = [np.ascontiguousarray(a, np.float64) for a in
                     (problem.rates, problem.static_mem, problem.dynamic_mem)]
        cur = cost = None
        if problem.current is not None:
            cur = np.ascontiguousarray(problem.current, np.int32)
            self.keep.append(cur)
        if problem.change_cost is not None:
            cost = np.ascontiguousarray(problem.change_cost, np.float64).reshape(m, l)
            self.keep.append(cost)
        dp = C.POINTER(C.c_double)
        self.p = _native.SymPartProblem(
            m, l, *[a.ctypes.data_as(dp) for a in self.keep[:3]],
            float(problem.rate_cap), float(problem.mem_cap),
            float(problem.effective_weight()), float(problem.mean_rate),
            float(problem.mean_mem),
            cur.ctypes.data_as(_native.i32p) if cur is not None else None,
            cost.ctypes.data_as(dp) if cost is not None else None,
            float(problem.change_budget))

    def check(self, rc: int, what: str):
        if rc == 2:
            raise PartitionError(f"{what}: invalid problem for the device search")
        if rc != 0:
            raise RuntimeError(f"{what} failed (status {rc})")


def brute_force(problem: PartitionProblem, device: int = 0) -> SolveResult:
    """Exhaustive optimum over l^m assignments (partitioner.py:422-435)."""
    m, l = problem.n_models, problem.subclusters
    if l ** m > 4_000_000:
        raise PartitionError(f"instance too large to enumerate: {l}^{m}")
    d = _Device(problem, device)
    x = np.zeros(m, np.int32)
    obj, feas = C.c_double(0.0), C.c_int32(0)
    d.check(d.lib.sym_part_brute_force(C.byref(d.p), device, x.ctypes.data_as(C.POINTER(C.c_int32)),
                                       C.byref(obj), C.byref(feas)), "brute_force")
    best = tuple(int(v) for v in x)
    return SolveResult(best, evaluate(problem, best), 0, 0)


def evaluate_many(problem: PartitionProblem, rows, device: int = 0):
    """Objective and feasibility of every row of an int [count, m] matrix on
    the device, plus the index of the first minimum of (infeasible,
    objective)."""
    d = _Device(problem, device)
    xs = np.ascontiguousarray(rows, np.int32)
    if xs.ndim != 2 or xs.shape[1] != problem.n_models or len(xs) == 0:
        raise PartitionError("rows must be a non-empty [count, m] matrix")
    obj = np.empty(len(xs), np.float64)
    feas = np.empty(len(xs), np.int32)
    best = C.c_int64(-1)
    d.check(d.lib.sym_part_evaluate(C.byref(d.p), device, xs.ctypes.data, len(xs),
                                    obj.ctypes.data, feas.ctypes.data, C.byref(best)),
            "evaluate_many")
    return obj, feas.astype(bool), int(best.value)


def random_solver(problem: PartitionProblem, time_budget_s: float, seed: int,
                  device: int = 0, max_draws: int | None = None) -> SolveResult:
    """Uniform random assignments from the reference's stream
    (substream(seed, 1), 256 x m rows per draw, partitioner.py:392-419); the
    feasible one with the least objective wins, first drawn on ties.  Rows
    are scored on the device RANDOM_BATCHES_PER_LAUNCH draws at a time; the
    deadline is checked between launches.  ``max_draws`` bounds the rows
    (deterministic runs)."""
    if time_budget_s <= 0:
        raise PartitionError("time budget must be > 0")
    deadline = time.monotonic() + time_budget_s
    rng = substream(seed, 1)
    m, l = problem.n_models, problem.subclusters
    best_x, best_key, tried = None, None, 0
    while True:
        batches = RANDOM_BATCHES_PER_LAUNCH
        if max_draws is not None:
            batches = max(1, min(batches, (max_draws - tried + 255) // 256))
        rows = np.concatenate([rng.integers(0, l, size=(256, m)) for _ in range(batches)])
        if max_draws is not None:
            rows = rows[:max_draws - tried]
        obj, feas, k = evaluate_many(problem, rows, device)
        key = (0.0 if feas[k] else 1.0, float(obj[k]))
        if best_key is None or key < best_key:
            best_key, best_x = key, tuple(int(v) for v in rows[k])
        tried += len(rows)
        if time.monotonic() >= deadline or (max_draws is not None and tried >= max_draws):
            return SolveResult(best_x, evaluate(problem, best_x), tried, 0)


def solve(problem: PartitionProblem, time_budget_s: float, seed: int, device: int = 0,
          restarts_per_launch: int = RESTARTS_PER_LAUNCH,
          max_launches: int | None = None) -> SolveResult:
    """Best assignment found by randomized greedy construction plus
    first-improvement local search (single moves, then pairwise swaps) with
    restarts (partitioner.py:344-389).  Each launch runs
    ``restarts_per_launch`` restarts in parallel, one warp each (the lanes
    score 32 candidate moves at once); a restart stops at its local optimum
    or at the deadline, and launches repeat until the budget expires (at
    least one).  The lexicographic
    (violation, objective) score picks the result, so the least-infeasible
    assignment comes back when nothing feasible was found."""
    if time_budget_s <= 0:
        raise PartitionError("time budget must be > 0")
    deadline = time.monotonic() + time_budget_s
    d = _Device(problem, device)
    m = problem.n_models
    order = np.array(sorted(range(m), key=lambda i: (-problem.rates[i],
                                                       -problem.static_mem[i], i)), np.int32)
    R = int(restarts_per_launch)
    xs = np.empty((R, m), np.int32)
    viol, obj = np.empty(R, np.float64), np.empty(R, np.float64)
    steps = np.empty(R, np.int64)
    best_key, best_x = None, None
    r0 = improvements = launches = 0
    while True:
        left = max(deadline - time.monotonic(), 1e-3)
        d.check(d.lib.sym_part_solve(C.byref(d.p), device, order.ctypes.data,
                                     C.c_uint64(seed & (2**64 - 1)), r0, R, left,
                                     xs.ctypes.data, viol.ctypes.data, obj.ctypes.data,
                                     steps.ctypes.data), "solve")
        k = int(np.lexsort((np.arange(R), obj, viol))[0])
        key = (float(viol[k]), float(obj[k]))
        if best_key is None or key < best_key:
            best_key, best_x = key, tuple(int(v) for v in xs[k])
        improvements += int(steps.sum())
        r0 += R
        launches += 1
        if time.monotonic() >= deadline or (max_launches and launches >= max_launches):
            break
    return SolveResult(best_x, evaluate(problem, best_x), r0, improvements)


# -- instances and file formats -------------------------------------------------

def random_instance(n_models: int, subclusters: int, seed: int, mean_rate: float = 100.0,
                    rate_cap_slack: float = 1.5, mem_cap_slack: float = 1.5) -> PartitionProblem:
    """Synthetic instance, exponential rates (partitioner.py:440-457)."""
    rng = substream(seed, 2)
    rates = rng.exponential(mean_rate, size=n_models)
    static = rng.uniform(50.0, 2000.0, size=n_models)
    dynamic = rng.uniform(0.0, 500.0, size=n_models)
    rate_cap = rate_cap_slack * float(rates.sum()) / subclusters
    mem_cap = mem_cap_slack * (float(static.sum()) / subclusters + float(dynamic.max()))
    return PartitionProblem(
        names=tuple(f"m{i}" for i in range(n_models)),
        rates=tuple(round(float(r), 6) for r in rates),
        static_mem=tuple(round(float(s), 6) for s in static),
        dynamic_mem=tuple(round(float(d), 6) for d in dynamic),
        subclusters=subclusters, rate_cap=rate_cap, mem_cap=mem_cap)


PROBLEM_HEADER = ["model", "rate_rps", "static_mem_mb", "dynamic_mem_mb"]


def parse_problem(text: str, source: str = "<problem>") -> PartitionProblem:
    """Problem file (partitioner.py:460-505): '# key=value' lines set l,
    R_max, S_max, w and C_max; the remaining non-blank lines are the CSV
    model,rate_rps,static_mem_mb,dynamic_mem_mb."""
    lines = text.splitlines()
    config = dict(kv.split("=", 1) for kv in
                  (ln[1:].strip() for ln in lines if ln.startswith("#")) if "=" in kv)
    config = {k.strip(): v.strip() for k, v in config.items()}
    rows = list(csv.reader([ln for ln in lines if not ln.startswith("#") and ln.strip()]))
    if not rows or rows[0] != PROBLEM_HEADER:
        raise PartitionError(f"{source}: expected header {','.join(PROBLEM_HEADER)}")
    cols: tuple[list, list, list, list] = ([], [], [], [])
    for lineno, row in enumerate(rows[1:], start=2):
        if len(row) != 4:
            raise PartitionError(f"{source}:{lineno}: expected 4 fields")
        try:
            vals = (row[0], float(row[1]), float(row[2]), float(row[3]))
        except ValueError as exc:
            raise PartitionError(f"{source}:{lineno}: {exc}") from None
        for col, v in zip(cols, vals):
            col.append(v)
    if "l" not in config:
        raise PartitionError(f"{source}: missing '# l=' config line")

    def opt(key):
        return float(config[key]) if config.get(key, "") != "" else INF

    return PartitionProblem(
        names=tuple(cols[0]), rates=tuple(cols[1]), static_mem=tuple(cols[2]),
        dynamic_mem=tuple(cols[3]), subclusters=int(config["l"]), rate_cap=opt("R_max"),
        mem_cap=opt("S_max"), weight=float(config["w"]) if config.get("w") else None,
        change_budget=opt("C_max"))


def load_problem(path: str) -> PartitionProblem:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_problem(fh.read(), source=path)


def assignment_csv(problem: PartitionProblem, assignment) -> str:
    lines = ["model,subcluster"]
    lines.extend(f"{name},{j}" for name, j in zip(problem.names, assignment))
    return "\n".join(lines) + "\n"
