"""Deterministic random scheduler cases (pure numpy/random, no package
imports) shared by the golden generator and the parity tests.  They cover
what the reference's own tests exercise piecemeal: same-tick bursts
(Gamma CV=4 and coarse ticks), table profiles, max_batch caps, network
delays, every policy and gather mode, and deep overload (drops, GPU-timer
evictions)."""
from __future__ import annotations

import random

import numpy as np


def _linear(rng, mb):
    a = int(round(rng.uniform(0, 2) * 1e6))
    b = int(round(rng.uniform(0.5, 10) * 1e6))
    return [a * k + b for k in range(1, mb + 1)]


def _table(rng, mb):
    pts = sorted(set([1] + rng.sample(range(1, mb + 1), min(mb, rng.randint(1, 4)))))
    v, vals = 1.0, []
    for _ in pts:
        v += rng.uniform(0, 3.0)
        vals.append(int(round(v * 1e6)))
    lat = []
    for (b0, v0), (b1, v1) in zip(zip(pts, vals), zip(pts[1:], vals[1:])):
        lat.extend(v0 + (v1 - v0) * (k - b0) // (b1 - b0) for k in range(b0, b1))
    lat.append(vals[-1])
    lat.extend([lat[-1]] * (mb - len(lat)))
    return lat


def make_case(seed: int) -> dict:
    rng = random.Random(seed)
    M = rng.choice([1, 2, 3, 5, 10, 30])
    G = rng.choice([1, 2, 3, 4, 8, 16, 64])
    mbmax = rng.choice([4, 8, 16, 64, 256])
    models = []
    for _ in range(M):
        mb = rng.randint(1, mbmax)
        table = rng.random() < 0.3
        lat = _table(rng, mb) if table else _linear(rng, mb)
        slo = lat[0] + int(round(rng.uniform(0.001, 40) * 1e6))
        models.append({"kind": "table" if table else "linear", "max_batch": mb,
                       "lat": lat, "slo": slo})
    kind = rng.choice(["deferred", "deferred", "eager", "timeout"])
    gather = "drop_head" if rng.random() < 0.2 else "prefix"
    policy = {"kind": kind,
              "timeout_ns": int(round(rng.uniform(0, 10) * 1e6)) if rng.random() < 0.5 else 0,
              "timeout_slo_frac": rng.choice([None, 0.1, 0.3, 0.9]),
              "d_ctrl_ns": rng.choice([0, 0, 30000, 500000]),
              "d_data_ns": rng.choice([0, 0, 3000, 100000]),
              "gather": gather,
              "target_batch": rng.randint(1, 32) if gather == "drop_head" else 0}
    n = rng.choice([50, 300, 2000, 8000])
    rate = rng.choice([0.3, 1, 3, 10]) * G * 1000
    shape = rng.choice([1.0, 1 / 16.0])
    gaps = np.array([rng.gammavariate(shape, 1.0) for _ in range(n)]) / rate
    if rng.random() < 0.5:
        gaps = np.round(gaps * 1e3) / 1e3  # coarse clock: many same-tick arrivals
    ticks = np.cumsum(np.rint(gaps * 1e9).astype(np.int64))
    midx = np.array([rng.randrange(M) if rng.random() < 0.7 else 0 for _ in range(n)],
                    np.int64)
    return {"models": models, "gpus": G, "policy": policy, "ticks": ticks, "midx": midx}
