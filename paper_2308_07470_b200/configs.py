"""The benchmark configurations C1-C5 of BASELINE.json / SURVEY.md §8d.

All use the deferred policy, zero network delay, max_batch 256, seed 42 and
10 % warm-up/cool-down, with the A100 model zoo (Table 4) cycled
where a config needs more models than the zoo has.  ``variant`` selects the
parity variants (eager, timeout 30 % of SLO, d_ctrl=30us/d_data=3us).
"""
from __future__ import annotations

import math
from dataclasses import replace

from .network import NetworkModel
from .profile import LatencyProfile, ModelSpec, load_model_zoo
from .scenario import Scenario
from .scheduler import PolicyConfig
from .units import ms_to_ns
from .workload import WorkloadSpec

SEED = 42
NOMINAL_DURATION_S = 60.0


def _zoo_models(n: int, slo_override=None) -> tuple[ModelSpec, ...]:
    zoo = load_model_zoo("a100")
    out = []
    for i in range(n):
        z = zoo[i % len(zoo)]
        slo = z.slo_ms if slo_override is None else slo_override(i)
        out.append(ModelSpec(i, f"{z.name}_{i}", LatencyProfile.linear(z.alpha_ms, z.beta_ms),
                             ms_to_ns(slo)))
    return tuple(out)


def policy_variant(variant: str) -> tuple[PolicyConfig, NetworkModel]:
    if variant == "deferred":
        p = PolicyConfig("deferred")
    elif variant == "eager":
        p = PolicyConfig("eager")
    elif variant == "timeout30":
        p = PolicyConfig("timeout", timeout_slo_frac=0.3)
    elif variant == "delay":
        p = PolicyConfig("deferred", d_ctrl_ns=30_000, d_data_ns=3_000)
    else:
        raise ValueError(f"unknown variant {variant!r}")
    return p, NetworkModel.constant(p.d_ctrl_ns, p.d_data_ns)


def _scenario(name, models, gpus, workload, duration_s, variant, shards=None):
    policy, net = policy_variant(variant)
    return Scenario(name=name, models=models, gpu_count=gpus, policy=policy,
                    workload=workload, duration_s=duration_s, warmup_s=0.1 * duration_s,
                    cooldown_s=0.1 * duration_s, seed=SEED, network=net, shards=shards)


def c1(duration_s: float = NOMINAL_DURATION_S, variant: str = "deferred") -> Scenario:
    """1 ResNet-50 (alpha 1.053, beta 5.072 ms), SLO 50 ms, 8 GPUs, Poisson 2k r/s."""
    m = (ModelSpec(0, "ResNet50", LatencyProfile.linear(1.053, 5.072), ms_to_ns(50.0)),)
    return _scenario("C1", m, 8, WorkloadSpec("poisson", 2000.0), duration_s, variant)


def c2(duration_s: float = NOMINAL_DURATION_S, variant: str = "deferred") -> Scenario:
    """A100 zoo rows 1-10, SLO_i = round(20 + 80 i/9) ms, 64 GPUs, Poisson 40k r/s."""
    m = _zoo_models(10, slo_override=lambda i: float(round(20 + 80 * i / 9)))
    return _scenario("C2", m, 64, WorkloadSpec("poisson", 40_000.0), duration_s, variant)


def c3(duration_s: float = NOMINAL_DURATION_S, variant: str = "deferred") -> Scenario:
    """100 zoo models, zoo SLOs, 1024 GPUs, Gamma CV=4 (k=1/16) at 300k r/s."""
    return _scenario("C3", _zoo_models(100), 1024,
                     WorkloadSpec("gamma", 300_000.0, gamma_shape=1.0 / 16.0),
                     duration_s, variant)


C4_SHARDS = 8


def c4(duration_s: float = NOMINAL_DURATION_S, variant: str = "deferred") -> Scenario:
    """1000 zoo models x 8192 GPUs, Poisson 1.2M r/s aggregate, P=8
    sub-clusters of 125 contiguous models and 1024 GPUs each."""
    per = 1000 // C4_SHARDS
    shards = (tuple(i // per for i in range(1000)), (1024,) * C4_SHARDS)
    return _scenario("C4", _zoo_models(1000), 8192, WorkloadSpec("poisson", 1_200_000.0),
                     duration_s, variant, shards=shards)


def c5_segments(duration_s: float = NOMINAL_DURATION_S, n: int = 24,
                peak: float = 600_000.0):
    """24 equal segments spanning the run (2.5 s each at the nominal 60 s),
    rate_j = peak * (0.55 - 0.45 cos(2 pi j / 24)).  The segments must span
    the duration: the reference's piecewise generator does not clip a
    segment at duration_s (workload.py:131-137)."""
    seg_s = duration_s / n
    return tuple((j * seg_s, peak * (0.55 - 0.45 * math.cos(2 * math.pi * j / n)))
                 for j in range(n))


def c5(duration_s: float = NOMINAL_DURATION_S, variant: str = "deferred") -> Scenario:
    """500 zoo models, 4096 GPUs, diurnal piecewise 24 x 2.5 s segments
    (60k -> 600k -> 60k r/s); the autoscaling series is computed per epoch
    from compute_stats + autoscale_advice (see autoscale.py)."""
    return _scenario("C5", _zoo_models(500), 4096,
                     WorkloadSpec("piecewise", segments=c5_segments(duration_s)), duration_s, variant)


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def shard_scenarios(sc: Scenario):
    """Split a sharded scenario into per-sub-cluster (models, gpus, model-id
    list) triples; the oracle runs each sub-cluster's filtered trace."""
    if sc.shards is None:
        return [(sc.models, sc.gpu_count, list(range(len(sc.models))))]
    som, gps = sc.shards
    out = []
    for s, g in enumerate(gps):
        ids = [i for i, x in enumerate(som) if x == s]
        ms = tuple(replace(sc.models[i], model_id=k) for k, i in enumerate(ids))
        out.append((ms, g, ids))
    return out
