"""Engine / RunResult: the drop-in for batchsym/simulator.py on B200.

``Engine(models, gpu_count, policy, network, seed, record_trace,
check_invariants)`` and ``run`` / ``run_stream`` keep the reference
signatures (simulator.py:99-102, 195-226) and return a ``RunResult`` with
the reference's fields and dtypes (simulator.py:65-87).  The discrete-event
loop itself runs on the GPU (csrc/engine.cu); this module only marshals
int64 arrays through the C ABI of include/symphony_b200.h.  There is no CPU
fallback: without the CUDA library or a device the first run raises.

Extension: ``shards=(shard_of_model, gpus_per_shard)`` runs independent
sub-clusters (the paper's multicore partitioning; the
reference's scalebench shards, scalebench.py:98-99) in one call.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from collections.abc import Sequence
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np

from . import _native
from .network import NetworkModel, jitter_tables
from .profile import ModelSpec
from .scheduler import PolicyConfig, ProtocolError
from .units import s_to_ns
from .workload import WorkloadSpec, generate_arrivals

EV_COMPLETION, EV_GPU_TIMER, EV_MODEL_TIMER, EV_DROP_TIMER, EV_ARRIVAL = range(5)
OUTCOME_COMPLETED, OUTCOME_LATE, OUTCOME_DROPPED = 0, 1, 2
OUTCOME_NAMES = ("completed", "late", "dropped")
TRACE_DISPATCH, TRACE_DROP, TRACE_SHRINK = "dispatch", "drop", "shrink"


class InvariantViolation(AssertionError):
    pass


class _GpuLogs(Sequence):
    """gpu_logs[g] = [(start, finish, model, size), ...] in emission order,
    materialised from the batch records on first access (a 7M-batch run
    does not pay for Python tuples unless someone reads them)."""

    def __init__(self, batches: np.ndarray, n_gpus: int):
        self._b = batches
        self._n = n_gpus
        self._logs = None

    def _build(self):
        if self._logs is None:
            logs = [[] for _ in range(self._n)]
            b = self._b
            order = np.argsort(b["gpu"], kind="stable")
            for k in order:
                logs[int(b["gpu"][k])].append((int(b["start"][k]), int(b["finish"][k]),
                                               int(b["model"][k]), int(b["size"][k])))
            self._logs = logs
        return self._logs

    def __getitem__(self, i):
        return self._build()[i]

    def __len__(self):
        return self._n

    def __eq__(self, other):
        return list(self._build()) == list(other)


@dataclass
class RunResult:
    model_names: list[str]
    gpu_count: int
    duration_ns: int
    req_model: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    req_arrival: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    req_deadline: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    req_dispatch: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    req_start: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    req_finish: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    req_batch: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    req_outcome: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    gpu_logs: Sequence = field(default_factory=list)
    trace: list[tuple] = field(default_factory=list)
    drops: int = 0
    completions: int = 0
    late: int = 0
    #: batch records (numpy structured array, _native.BATCH_DTYPE), the
    #: compact form gpu_logs is derived from
    batches: np.ndarray | None = None
    #: (weakref to the Engine, its run id): while the engine's last run is
    #: this one, compute_stats can reduce on the device (sym_window_stats)
    _source: tuple | None = field(default=None, repr=False, compare=False)

    def device_engine(self):
        """The Engine still holding this run on the device, else None."""
        if self._source is None:
            return None
        eng = self._source[0]()
        if eng is None or eng._handle is None or eng._run_id != self._source[1]:
            return None
        return eng

    @property
    def n_requests(self) -> int:
        return len(self.req_model)


_ECHO_CHUNK = 1 << 20


def _echo_chunk(lo, hi, ticks, midx, slo, arrival, model, deadline):
    np.copyto(arrival[lo:hi], ticks[lo:hi])
    np.copyto(model[lo:hi], midx[lo:hi])
    # clip: an unknown model id is reported by the device (ProtocolError)
    np.add(ticks[lo:hi], np.take(slo, midx[lo:hi], mode="clip"), out=deadline[lo:hi])


def _echo_inputs(ticks, midx, slo, arrival, model, deadline):
    """req_arrival / req_model are copies of the inputs and req_deadline =
    arrival + slo[model] (simulator.py:217-219): formed on host threads while
    the device runs (numpy releases the GIL), so none of them crosses PCIe."""
    from concurrent.futures import ThreadPoolExecutor
    n = len(ticks)
    spans = [(lo, min(n, lo + _ECHO_CHUNK)) for lo in range(0, n, _ECHO_CHUNK)]
    if len(spans) <= 1:
        for lo, hi in spans:
            _echo_chunk(lo, hi, ticks, midx, slo, arrival, model, deadline)
        return
    with ThreadPoolExecutor(min(8, len(spans), os.cpu_count() or 1)) as ex:
        list(ex.map(lambda sp: _echo_chunk(sp[0], sp[1], ticks, midx, slo, arrival, model,
                                           deadline), spans))


def _split_shards(models, gpu_count, shards):
    M = len(models)
    if shards is None:
        return np.zeros(M, np.int32), np.array([gpu_count], np.int32)
    shard_of_model, gpus_per_shard = shards
    som = np.asarray(shard_of_model, np.int32)
    gps = np.asarray(gpus_per_shard, np.int32)
    if som.shape != (M,) or len(gps) < 1 or som.min() < 0 or som.max() >= len(gps):
        raise ValueError("bad shard layout")
    if int(gps.sum()) != gpu_count or gps.min() < 1:
        raise ValueError("gpus_per_shard must be >= 1 each and sum to gpu_count")
    if len(np.unique(som)) != len(gps):
        raise ValueError("every shard needs at least one model")
    return som, gps


class Engine:
    """B200 engine with the reference Engine's constructor and run API."""

    def __init__(self, models: list[ModelSpec], gpu_count: int,
                 policy: PolicyConfig, network: NetworkModel | None = None,
                 seed: int = 0, record_trace: bool = False,
                 check_invariants: bool = False, *, shards=None, device: int = 0,
                 devices=None, use_fresh: bool = True, use_fast: bool = True):
        if gpu_count < 1:
            raise ValueError("need at least one GPU")
        self.models = list(models)
        self.policy = policy
        self.network = network or NetworkModel.zero()
        # jittered delays: per-dispatch draws from the engine's numpy Philox
        # substream, reproduced on the device (simulator.py:116-122)
        self._jitter = jitter_tables(self.network, seed)
        self.seed = seed
        self.record_trace = record_trace
        self.check_invariants = check_invariants
        self.gpu_count = gpu_count
        self.device = device
        # several devices in one call: sub-cluster s on devices[s % len]
        self.devices = None if devices is None or len(devices) < 2 else \
            np.ascontiguousarray(devices, np.int32)
        self.use_fresh = use_fresh
        self.use_fast = use_fast
        self.shard_of_model, self.gpus_per_shard = _split_shards(self.models, gpu_count, shards)
        self.n_shards = len(self.gpus_per_shard)
        stride = max(m.profile.max_batch for m in self.models)
        self._lat = np.stack([m.profile.table_array(stride) for m in self.models])
        self._max_batch = np.array([m.profile.max_batch for m in self.models], np.int32)
        self._slo = np.array([m.slo_ns for m in self.models], np.int64)
        self._timeout = np.array([policy.resolve_timeout_ns(m.slo_ns) for m in self.models],
                                 np.int64)
        self._handle = None
        self._run_id = 0
        self._last_ok = False   # the last run succeeded and is still on the device
        self._keep = None       # caller tensors the device views of that run read
        self._lib = None
        # reference-style counters (RankPlane.ops/evictions/registrations,
        # Engine.handler_ops_max), filled after each run
        self.rank = SimpleNamespace(ops=0, evictions=0, registrations=0)
        self.handler_ops_max = 0
        self.stats = {}

    # -- native handle --------------------------------------------------------

    def _ensure(self):
        if self._handle is not None:
            return
        lib = _native.load()
        cfg = _native.SymConfig()
        cfg.n_models = len(self.models)
        cfg.n_gpus = self.gpu_count
        cfg.kind = _native.KIND[self.policy.kind]
        cfg.gather = _native.GATHER[self.policy.gather]
        cfg.target_batch = self.policy.target_batch
        cfg.lat_stride = self._lat.shape[1]
        cfg.d_ctrl_ns = self.policy.d_ctrl_ns
        cfg.d_data_ns = self.policy.d_data_ns
        cfg.lat_ns = self._lat.ctypes.data_as(_native.i64p)
        cfg.max_batch = self._max_batch.ctypes.data_as(_native.i32p)
        cfg.slo_ns = self._slo.ctypes.data_as(_native.i64p)
        cfg.timeout_ns = self._timeout.ctypes.data_as(_native.i64p)
        cfg.n_shards = self.n_shards
        cfg.device = self.device
        cfg.shard_of_model = self.shard_of_model.ctypes.data_as(_native.i32p)
        cfg.gpus_per_shard = self.gpus_per_shard.ctypes.data_as(_native.i32p)
        if self.devices is not None:
            cfg.devices = self.devices.ctypes.data_as(_native.i32p)
            cfg.n_devices = len(self.devices)
        j = self._jitter
        if j is not None:
            self._jit_keep = [np.ascontiguousarray(a) for a in (j.ctrl_vals, j.ctrl_cdf,
                                                                j.data_vals, j.data_cdf)]
            cv, cc, dv, dc = self._jit_keep
            cfg.net_ctrl_n, cfg.net_data_n = len(cv), len(dv)
            cfg.net_ctrl_vals = cv.ctypes.data_as(_native.i64p)
            cfg.net_data_vals = dv.ctypes.data_as(_native.i64p)
            cfg.net_ctrl_cdf = cc.ctypes.data_as(C.POINTER(C.c_double))
            cfg.net_data_cdf = dc.ctypes.data_as(C.POINTER(C.c_double))
            cfg.net_ctrl_const, cfg.net_data_const = int(j.ctrl_const), int(j.data_const)
            cfg.net_key[0], cfg.net_key[1] = int(j.key[0]), int(j.key[1])
        status = C.c_int32(0)
        h = lib.sym_create(C.byref(cfg), C.byref(status))
        if not h:
            if status.value == _native.SYM_EINVAL:
                raise ValueError("invalid engine configuration")
            raise RuntimeError(f"sym_create failed (status {status.value}); "
                               "is a CUDA device visible?")
        self._lib = lib
        self._handle = h

    def close(self):
        if self._handle is not None:
            self._lib.sym_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, rc: int, res: _native.SymResult):
        msg = self._lib.sym_last_error(self._handle).decode()
        if rc == _native.SYM_EPROTO:
            raise ProtocolError(f"request for unknown model (arrival {res.err_index})")
        if rc == _native.SYM_EINVAL:
            raise ValueError(msg)
        if rc == _native.SYM_EINVARIANT:
            raise InvariantViolation(msg)
        raise RuntimeError(f"B200 engine failed ({rc}): {msg}")

    def _flags(self) -> int:
        f = 0
        if self.record_trace:
            f |= _native.FLAG_TRACE
        if not self.use_fresh:
            f |= _native.FLAG_NO_FRESH
        if not self.use_fast:
            f |= _native.FLAG_NO_FAST
        if self.check_invariants:
            # per-event _verify (simulator.py:276-305) inside the device chain
            f |= _native.FLAG_CHECK_INVARIANTS
            if getattr(self, "_inject_fault", False):  # test hook
                f |= _native.FLAG_INJECT_FAULT
        return f

    def _absorb_counters(self, res: _native.SymResult):
        self.rank.ops = res.ops
        self.rank.evictions = res.evictions
        self.rank.registrations = res.registrations
        self.handler_ops_max = res.handler_ops_max
        self.stats = {k: getattr(res, k) for k in (
            "chain_events", "absorbed_arrivals", "fresh_adoptions", "launches", "fast_shards", "fast_fail_mask",
            "ms_ingest", "ms_fresh", "ms_fast", "ms_chain", "ms_expand", "ms_total")}

    # -- reference API --------------------------------------------------------

    def run(self, workload: WorkloadSpec, duration_s: float, seed: int) -> RunResult:
        names = [m.name for m in self.models]
        ticks, midx = generate_arrivals(workload, names, duration_s, seed)
        return self.run_stream(ticks, midx, duration_s)

    def run_stream(self, arr_ticks, arr_midx, duration_s: float) -> RunResult:
        """simulator.py:201-226 on the B200.  Validation (model ids in range,
        time-ordered arrivals) happens on the device; results are written by
        the device straight into page-locked arrays."""
        ticks = np.ascontiguousarray(arr_ticks, dtype=np.int64)
        midx = np.ascontiguousarray(arr_midx, dtype=np.int64)
        n = len(ticks)
        if len(midx) != n:
            raise ValueError("arr_ticks and arr_midx differ in length")
        self._ensure()
        names = ("dispatch", "start", "finish", "batch", "outcome", "arrival", "deadline",
                 "model")
        outs = {k: _native.pinned_empty(n) for k in names}
        res = _native.SymResult()
        res.n = n
        # req_arrival / req_model / req_deadline follow from the inputs: host
        # threads form them while the device runs and its copy engine returns
        # the five computed arrays (simulator.py:217-219, 228-242)
        echo = ("arrival", "model", "deadline")
        for k in names:
            if k not in echo:
                setattr(res, "req_" + k, outs[k].ctypes.data_as(_native.i64p))
        copier = threading.Thread(target=_echo_inputs,
                                  args=(ticks, midx, self._slo, outs["arrival"], outs["model"],
                                        outs["deadline"]))
        copier.start()
        if self.record_trace:
            drop_t = np.empty(n, np.int64)
            drop_ks = np.empty(n, np.int64)
            drop_ka = np.empty(n, np.int32)
            res.drop_t = drop_t.ctypes.data_as(_native.i64p)
            res.drop_key_sub = drop_ks.ctypes.data_as(_native.i64p)
            res.drop_key_a = drop_ka.ctypes.data_as(_native.i32p)
        self._run_id += 1
        self._last_ok, self._keep = False, None
        self._stepping = False
        rc = self._lib.sym_run(self._handle, ticks.ctypes.data, midx.ctypes.data, n,
                               self._flags() | _native.FLAG_MODEL_I64, C.byref(res))
        copier.join()
        if rc != _native.SYM_OK:
            if rc == _native.SYM_EPROTO and 0 <= res.err_index < n:
                raise ProtocolError(f"request for unknown model {int(midx[res.err_index])}")
            self._raise(rc, res)
        self._absorb_counters(res)
        self._last_ok = True
        batches = _native.pinned_empty(res.n_batches, _native.BATCH_DTYPE)
        got = self._lib.sym_last_batches(self._handle, batches.ctypes.data, len(batches))
        if got < 0:
            self._raise(-got, res)
        if got != res.n_batches:
            raise RuntimeError(f"sym_last_batches returned {got}")
        outc = outs["outcome"]
        result = RunResult(
            model_names=[m.name for m in self.models], gpu_count=self.gpu_count,
            duration_ns=s_to_ns(duration_s), req_model=outs["model"],
            req_arrival=outs["arrival"], req_deadline=outs["deadline"],
            req_dispatch=outs["dispatch"], req_start=outs["start"], req_finish=outs["finish"],
            req_batch=outs["batch"], req_outcome=outc,
            gpu_logs=_GpuLogs(batches, self.gpu_count), drops=int(res.drops),
            # n_completed counts every completion event, LATE ones included
            # (simulator.py:251-252)
            completions=n - int(res.drops),
            late=int(np.count_nonzero(outc == OUTCOME_LATE)) if self._jitter is not None else 0,
            batches=batches, _source=(weakref.ref(self), self._run_id))
        if self.record_trace:
            result.trace = self._build_trace(ticks, midx, batches, drop_t, drop_ks, drop_ka)
        if self.check_invariants:
            self._verify(result)
        return result

    # -- step API (scalebench.py:67-84: _record_arrival / on_new_request /
    # _dispatch_event, batched) ----------------------------------------------

    #: until_tick that drains a stepped run
    DRAIN = (1 << 63) - 1

    def reset_steps(self):
        """Start a stepped run (a whole run_stream / run_device ends one)."""
        self._ensure()
        self._last_ok, self._keep = False, None
        rc = self._lib.sym_step_reset(self._handle)
        if rc != _native.SYM_OK:
            self._raise(rc, _native.SymResult())
        self._stepping = True
        self._step_until = None

    def step(self, arr_ticks, arr_midx, until_tick: int) -> dict:
        """Feed the next arrivals and process every event with tick <=
        until_tick; later arrivals must have tick >= until_tick.  State stays
        on the device between calls (sym_step).  Starts a stepped run if
        none is in progress.  Returns the cumulative counters: arrivals,
        batches, dispatched requests, drops."""
        if not getattr(self, "_stepping", False):
            self.reset_steps()
        ticks = np.ascontiguousarray(arr_ticks, dtype=np.int64)
        midx = np.ascontiguousarray(arr_midx, dtype=np.int64)
        if len(midx) != len(ticks):
            raise ValueError("arr_ticks and arr_midx differ in length")
        res = _native.SymResult()
        flags = _native.FLAG_MODEL_I64
        if self.check_invariants:
            flags |= _native.FLAG_CHECK_INVARIANTS
        rc = self._lib.sym_step(self._handle, ticks.ctypes.data, midx.ctypes.data, len(ticks),
                                int(until_tick), flags, C.byref(res))
        if rc != _native.SYM_OK:
            if rc == _native.SYM_EPROTO and 0 <= res.err_index < len(midx):
                raise ProtocolError(f"request for unknown model {int(midx[res.err_index])}")
            self._raise(rc, res)
        self._step_until = int(until_tick)
        self._absorb_counters(res)
        return {"arrivals": res.n, "batches": res.n_batches, "dispatched": res.completions,
                "drops": res.drops, "chain_events": res.chain_events,
                "ms_total": res.ms_total}

    def step_result(self, duration_s: float, drain: bool = True) -> RunResult:
        """RunResult of every arrival stepped so far; with ``drain`` the run is
        first completed (until_tick = +inf), which makes it equal to
        run_stream over the concatenated arrivals."""
        if not getattr(self, "_stepping", False):
            raise RuntimeError("no stepped run in progress")
        if drain and self._step_until != self.DRAIN:
            self.step(np.empty(0, np.int64), np.empty(0, np.int64), self.DRAIN)
        probe = _native.SymResult()
        rc = self._lib.sym_step_result(self._handle, C.byref(probe))  # counts only
        if rc != _native.SYM_OK:
            self._raise(rc, probe)
        n, nb = probe.n, probe.n_batches
        names = ("dispatch", "start", "finish", "batch", "outcome", "arrival", "deadline",
                 "model")
        outs = {k: np.empty(n, np.int64) for k in names}
        batches = np.empty(nb, _native.BATCH_DTYPE)
        res = _native.SymResult()
        for k in names:
            setattr(res, "req_" + k, outs[k].ctypes.data_as(_native.i64p))
        res.batches = batches.ctypes.data
        res.batch_cap = nb
        rc = self._lib.sym_step_result(self._handle, C.byref(res))
        if rc != _native.SYM_OK:
            self._raise(rc, res)
        self._absorb_counters(res)
        # a whole run lists the batches sub-cluster by sub-cluster, each in
        # emission order; a stepped run appends them step by step
        if self.n_shards > 1 and nb:
            batches = batches[np.argsort(self.shard_of_model[batches["model"]], kind="stable")]
        outc = outs["outcome"]
        return RunResult(
            model_names=[m.name for m in self.models], gpu_count=self.gpu_count,
            duration_ns=s_to_ns(duration_s), req_model=outs["model"],
            req_arrival=outs["arrival"], req_deadline=outs["deadline"],
            req_dispatch=outs["dispatch"], req_start=outs["start"], req_finish=outs["finish"],
            req_batch=outs["batch"], req_outcome=outc,
            gpu_logs=_GpuLogs(batches, self.gpu_count), drops=int(res.drops),
            completions=int(res.completions), late=0, batches=batches)

    # -- device-resident entry point -------------------------------------------

    def _require_last_run(self):
        if self._handle is None or not self._last_ok:
            raise RuntimeError("no successful run on the device to reduce")

    def window_counts(self, lo_ns: int, hi_ns: int) -> dict:
        """Integer window reductions of the last run on the device (the
        counting part of compute_stats, metrics.py:79-94): per model
        arrivals/completed/late/dropped among arrivals in [lo, hi), per GPU
        busy ns clipped to the window."""
        self._require_last_run()
        M, G = len(self.models), self.gpu_count
        out = {k: np.zeros(M, np.int64) for k in ("arrivals", "completed", "late", "dropped")}
        busy = np.zeros(G, np.int64)
        rc = self._lib.sym_window_counts(
            self._handle, int(lo_ns), int(hi_ns),
            *(out[k].ctypes.data_as(_native.i64p) for k in ("arrivals", "completed", "late",
                                                               "dropped")),
            busy.ctypes.data_as(_native.i64p))
        if rc != _native.SYM_OK:
            self._raise(rc, _native.SymResult())
        out["gpu_busy_ns"] = busy
        return out

    def window_stats(self, lo_ns: int, hi_ns: int) -> dict:
        """window_counts plus the rest of compute_stats' per-model inputs,
        reduced on the device from the last run (sym_window_stats): p99
        latency by nearest rank (drops as +inf; -1 = inf, 0 = no arrivals),
        largest queueing delay of a served request, and the batch-size
        histogram of batches starting in the window ([M][max_batch + 1])."""
        self._require_last_run()
        M, G = len(self.models), self.gpu_count
        stride = int(self._max_batch.max()) + 1 if M else 1
        keys = ("arrivals", "completed", "late", "dropped")
        out = {k: np.zeros(M, np.int64) for k in keys + ("p99_ns", "max_qd_ns")}
        busy = np.zeros(G, np.int64)
        hist = np.zeros((M, stride), np.int64)
        rc = self._lib.sym_window_stats(
            self._handle, int(lo_ns), int(hi_ns),
            *(out[k].ctypes.data_as(_native.i64p) for k in keys),
            busy.ctypes.data_as(_native.i64p), out["p99_ns"].ctypes.data_as(_native.i64p),
            out["max_qd_ns"].ctypes.data_as(_native.i64p), hist.ctypes.data_as(_native.i64p),
            stride)
        if rc != _native.SYM_OK:
            self._raise(rc, _native.SymResult())
        out["gpu_busy_ns"] = busy
        out["batch_hist"] = hist
        return out

    def kernel_times(self, reset: bool = True) -> dict:
        """{kernel: (launches, total_ms)} from runs made with kernel_times=True."""
        import json
        if self._handle is None:
            return {}
        raw = self._lib.sym_kernel_times(self._handle, int(reset)).decode()
        return {k: (int(v[0]), float(v[1])) for k, v in json.loads(raw).items()}

    def run_device(self, ticks, model, outputs: dict | None = None, expand: bool = True,
                   batches=None, kernel_times: bool = False):
        """Run on arrival tensors already resident on the engine's device
        (torch int64 ticks, int32 model ids).  Per-request outputs are
        written into ``outputs`` (dict of int64 CUDA tensors: dispatch,
        start, finish, batch, outcome), allocated if None.  Returns
        (outputs, counters).  Nothing crosses PCIe but the counters."""
        import torch

        n = int(ticks.numel())
        if ticks.dtype != torch.int64 or model.dtype != torch.int32:
            raise TypeError("ticks must be int64 and model int32 tensors")
        if not (ticks.is_cuda and model.is_cuda):
            raise ValueError("run_device needs CUDA tensors")
        self._ensure()
        dev = ticks.device
        if outputs is None and expand:
            outputs = {k: torch.empty(max(n, 1), dtype=torch.int64, device=dev)
                       for k in ("dispatch", "start", "finish", "batch", "outcome")}
        res = _native.SymResult()
        res.n = n
        if expand:
            res.req_dispatch, res.req_start, res.req_finish, res.req_batch, res.req_outcome = (
                C.cast(outputs[k].data_ptr(), _native.i64p)
                for k in ("dispatch", "start", "finish", "batch", "outcome"))
        if batches is not None:
            res.batches = batches.data_ptr()
            res.batch_cap = batches.numel() // C.sizeof(_native.SymBatch)
        flags = self._flags() & ~_native.FLAG_TRACE
        if not expand:
            flags |= _native.FLAG_NO_EXPAND
        if kernel_times:
            flags |= _native.FLAG_KERNEL_TIMES
        torch.cuda.current_stream(dev).synchronize()
        self._run_id += 1
        self._last_ok, self._keep = False, None
        self._stepping = False
        rc = self._lib.sym_run_device(self._handle, ticks.data_ptr(), model.data_ptr(), n,
                                      flags, C.byref(res))
        if rc != _native.SYM_OK:
            self._raise(rc, res)
        self._absorb_counters(res)
        # the engine's view of this run (window_counts / window_stats) reads
        # these tensors: keep them alive until the next run
        self._keep = (ticks, model, outputs, batches)
        self._last_ok = True
        counters = dict(self.stats, n_batches=res.n_batches, drops=res.drops,
                        registrations=res.registrations, evictions=res.evictions)
        return outputs, counters

    # -- trace / invariants ---------------------------------------------------

    def _build_trace(self, ticks, midx, batches, drop_t, drop_ks, drop_ka):
        """Rebuild the reference's trace list (simulator.py:170-187) in
        processing order from the per-event positions the engine recorded."""
        n = len(ticks)
        shard = self.shard_of_model[midx] if n else np.empty(0, np.int32)
        # rid = 1 + index within the sub-cluster's stream (simulator.py:217)
        rid = np.empty(n, np.int64)
        rank = np.empty(n, np.int64)  # position within the model's queue
        members = {}
        for s in range(self.n_shards):
            idx = np.nonzero(shard == s)[0]
            rid[idx] = np.arange(1, len(idx) + 1)
        for m in range(len(self.models)):
            idx = np.nonzero(midx == m)[0]
            members[m] = idx
            rank[idx] = np.arange(len(idx))
        rows = []  # (shard, t, a, sub, rank, kind_order, entry)
        for b in batches:
            m = int(b["model"])
            first = int(b["first_index"])
            r0 = int(rank[first])
            size = int(b["size"])
            s = int(self.shard_of_model[m])
            gid = int(b["gpu"])
            key = (s, int(b["key_t"]), int(b["key_a"]), int(b["key_sub"]), r0)
            if int(b["shrunk_from"]) > 0:
                rows.append(key + (0, (int(b["emitted"]), TRACE_SHRINK, m, gid, size, -1, -1, ())))
            rids = tuple(int(x) for x in rid[members[m][r0:r0 + size]])
            rows.append(key + (1, (int(b["emitted"]), TRACE_DISPATCH, m, gid, size,
                                   int(b["start"]), int(b["finish"]), rids)))
        for i in np.nonzero(drop_t >= 0)[0]:
            m = int(midx[i])
            rows.append((int(self.shard_of_model[m]), int(drop_t[i]), int(drop_ka[i]),
                         int(drop_ks[i]), int(rank[i]), 1,
                         (int(drop_t[i]), TRACE_DROP, m, -1, 0, -1, -1, (int(rid[i]),))))
        rows.sort(key=lambda r: r[:6])
        return [r[6] for r in rows]

    def _verify(self, res: RunResult):
        """End-of-run invariants on the returned arrays.  The per-event
        _verify of simulator.py:276-305 runs inside the device chain
        (SYM_FLAG_CHECK_INVARIANTS, engine_core.cuh verify_state) after
        every event of a check_invariants run."""
        o = res.req_outcome
        if np.any((o < 0) | (o > 2)):
            raise InvariantViolation("unresolved request outcome")
        served = o != OUTCOME_DROPPED
        if int(np.count_nonzero(served)) + res.drops != res.n_requests:
            raise InvariantViolation("conservation broken")
        if np.any(res.req_finish[served] > res.req_deadline[served]) and res.late == 0:
            raise InvariantViolation("served request misses its deadline")
        b = res.batches
        if b is not None and len(b):
            order = np.lexsort((np.arange(len(b)), b["gpu"]))
            g, st, fi = b["gpu"][order], b["start"][order], b["finish"][order]
            same = g[1:] == g[:-1]
            if np.any(st[1:][same] < fi[:-1][same]):
                raise InvariantViolation("overlapping batches on one GPU")
