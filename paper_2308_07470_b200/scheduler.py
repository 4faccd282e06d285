"""Scheduling-policy configuration and plane-protocol types.

Mirrors the public types of batchsym/scheduler.py.  The two planes
(ModelPlane / RankPlane, scheduler.py:138-469) have no Python counterpart
here: they run as the device-resident live-event chain of
csrc/engine_core.cuh, behind the Engine of simulator.py.
"""
from __future__ import annotations

from dataclasses import dataclass

OUTSTANDING = -1  # free_at marker while a grant is in flight (scheduler.py:41)

GATHER_PREFIX = "prefix"
GATHER_DROP_HEAD = "drop_head"

DROP_DEADLINE = "deadline"
DROP_POLICY = "policy"

POLICY_KINDS = ("deferred", "eager", "timeout")


class ProtocolError(RuntimeError):
    """Violation of the plane messaging contract: unknown model/GPU ids or a
    duplicate request id (scheduler.py:50-51)."""


@dataclass(frozen=True)
class PolicyConfig:
    """Dispatch policy and planning bounds (scheduler.py:54-87).

    ``timeout_ns`` is the timeout-policy offset k from the head's arrival
    (k = 0 is eager); ``timeout_slo_frac`` resolves k per model as a
    fraction of its SLO.
    """
    kind: str
    timeout_ns: int = 0
    timeout_slo_frac: float | None = None
    d_ctrl_ns: int = 0
    d_data_ns: int = 0
    gather: str = GATHER_PREFIX
    target_batch: int = 0

    def __post_init__(self) -> None:
        if self.kind not in POLICY_KINDS:
            raise ValueError(f"unknown policy kind {self.kind!r}")
        if self.timeout_ns < 0:
            raise ValueError("timeout must be >= 0")
        if self.timeout_slo_frac is not None and self.timeout_slo_frac < 0:
            raise ValueError("timeout_slo_frac must be >= 0")
        if self.d_ctrl_ns < 0 or self.d_data_ns < 0:
            raise ValueError("negative network delay bound")
        if self.gather not in (GATHER_PREFIX, GATHER_DROP_HEAD):
            raise ValueError(f"unknown gather policy {self.gather!r}")
        if self.gather == GATHER_DROP_HEAD and self.target_batch < 1:
            raise ValueError("drop_head gathering needs target_batch >= 1")

    def resolve_timeout_ns(self, slo_ns: int) -> int:
        if self.timeout_slo_frac is None:
            return self.timeout_ns
        return int(round(self.timeout_slo_frac * slo_ns))


class Request:
    """One inference request (scheduler.py:90-100)."""
    __slots__ = ("rid", "model_id", "arrival", "deadline")

    def __init__(self, rid: int, model_id: int, arrival: int, deadline: int):
        self.rid = rid
        self.model_id = model_id
        self.arrival = arrival
        self.deadline = deadline

    def __repr__(self) -> str:
        return f"Request({self.rid}, m{self.model_id}, a={self.arrival})"


class ExecutionOrder:
    """One dispatched batch (scheduler.py:123-135), rebuilt from the
    engine's batch records."""
    __slots__ = ("gpu_id", "model_id", "size", "start", "finish",
                 "request_ids", "emitted_at")

    def __init__(self, gpu_id, model_id, size, start, finish, request_ids, emitted_at):
        self.gpu_id = gpu_id
        self.model_id = model_id
        self.size = size
        self.start = start
        self.finish = finish
        self.request_ids = request_ids
        self.emitted_at = emitted_at
