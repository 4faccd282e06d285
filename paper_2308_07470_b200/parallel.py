"""Multi-GPU execution of independent sub-clusters.

A sub-cluster (disjoint models plus their own GPU sub-pool) is an
independent Engine -- the paper's "no communications between dispatcher
threads", the reference's scalebench shards
(scalebench.py:98-99).  Sub-cluster s runs on rank ``s % world``; there is
no collective on the data path.  The only exchange is one end-of-run
reduction of per-sub-cluster integer summaries (per-model outcome counts,
per-GPU busy time) so every rank can evaluate goodput, idle fraction and
the autoscaling advice of the whole cluster (metrics.py:71-132, 309-322).
Summaries are disjoint slices of one global int64 vector, so the all-reduce
(SUM) over NCCL (or gloo on CPU) is the all-gather.
"""
from __future__ import annotations

import math

import numpy as np

from .metrics import autoscale_advice
from .units import NS_PER_S


def assign(n_shards: int, world: int) -> list[list[int]]:
    """Sub-clusters owned by each rank (round robin, fixed by the scenario,
    so results are identical at any world size)."""
    return [[s for s in range(n_shards) if s % world == r] for r in range(world)]


class SummaryLayout:
    """Global int64 vector: [arrivals|completed|late|dropped] x M, busy x G."""

    def __init__(self, n_models: int, n_gpus: int):
        self.M, self.G = n_models, n_gpus

    @property
    def size(self) -> int:
        return 4 * self.M + self.G

    def empty(self) -> np.ndarray:
        return np.zeros(self.size, np.int64)

    def put(self, vec: np.ndarray, model_ids, gpu_ids, counts: dict) -> None:
        model_ids = np.asarray(model_ids)
        for k, name in enumerate(("arrivals", "completed", "late", "dropped")):
            vec[k * self.M + model_ids] = counts[name]
        vec[4 * self.M + np.asarray(gpu_ids)] = counts["gpu_busy_ns"]

    def split(self, vec: np.ndarray) -> dict:
        M = self.M
        return {"arrivals": vec[:M], "completed": vec[M:2 * M], "late": vec[2 * M:3 * M],
                "dropped": vec[3 * M:4 * M], "gpu_busy_ns": vec[4 * M:]}


def window_counts_host(req_model, req_arrival, req_outcome, batches_gpu, batches_start,
                       batches_finish, n_models, n_gpus, lo, hi) -> dict:
    """The same integer reductions from host arrays (used for CPU ranks and
    to cross-check sym_window_counts)."""
    inw = (req_arrival >= lo) & (req_arrival < hi)
    m = np.asarray(req_model)[inw]
    o = np.asarray(req_outcome)[inw]
    out = {"arrivals": np.bincount(m, minlength=n_models).astype(np.int64)}
    for code, name in ((0, "completed"), (1, "late"), (2, "dropped")):
        out[name] = np.bincount(m[o == code], minlength=n_models).astype(np.int64)
    busy = np.zeros(n_gpus, np.int64)
    clipped = np.maximum(0, np.minimum(batches_finish, hi) - np.maximum(batches_start, lo))
    np.add.at(busy, np.asarray(batches_gpu), clipped)
    out["gpu_busy_ns"] = busy
    return out


def reduce_summaries(vec: np.ndarray, group=None) -> np.ndarray:
    """The single collective: SUM of the disjoint per-rank slices."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return vec
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.from_numpy(vec).to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def cluster_stats(vec: np.ndarray, layout: SummaryLayout, lo: int, hi: int) -> dict:
    """Goodput, bad rate, idle fractions and the autoscaling delta of the
    whole cluster from the reduced summary, with the reference's formulas
    (metrics.py:79-94, 309-322) applied to identical integers."""
    d = layout.split(vec)
    wl = hi - lo
    arrivals = int(d["arrivals"].sum())
    completed = int(d["completed"].sum())
    bad = int(d["dropped"].sum()) + int(d["late"].sum())
    idle = [float(x) for x in 1.0 - d["gpu_busy_ns"] / wl]
    mean_idle = sum(idle) / len(idle) if idle else 1.0
    bad_rate = bad / arrivals if arrivals else 0.0
    # autoscale_advice rejects r == 1 (metrics.py:314); clamp at all-dropped
    r = min(bad_rate, math.nextafter(1.0, 0.0))
    return {"arrivals": arrivals, "completed": completed,
            "goodput_rps": completed / (wl / NS_PER_S), "bad_rate": bad_rate,
            "mean_idle_fraction": mean_idle,
            "autoscale_delta": autoscale_advice(r, mean_idle, layout.G)}
