"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the C parity oracle.

`symoracle.c` restates the reference's sequential scheduler/event loop
(batchsym scheduler.py + simulator.py:191-272) in plain C.  This module loads
it and runs it on plain arrays.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may import it; the product package never does.

Pinned against the Python reference by tests/golden/ (see
tests/golden/make_golden.py and tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsymoracle.so")

KIND = {"deferred": 0, "eager": 1, "timeout": 2}
GATHER = {"prefix": 0, "drop_head": 1}
ERRORS = {1: "protocol", 2: "invalid argument", 3: "invariant", 5: "out of memory"}

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class _Config(C.Structure):
    _fields_ = [
        ("n_models", C.c_int32), ("n_gpus", C.c_int32), ("kind", C.c_int32),
        ("gather", C.c_int32), ("target_batch", C.c_int32),
        ("record_trace", C.c_int32), ("check_invariants", C.c_int32),
        ("_pad", C.c_int32), ("d_ctrl_ns", C.c_int64), ("d_data_ns", C.c_int64),
        ("lat_ns", _i64p), ("lat_stride", C.c_int32), ("_pad2", C.c_int32),
        ("max_batch", _i32p), ("slo_ns", _i64p), ("timeout_ns", _i64p),
        ("net_ctrl_n", C.c_int32), ("net_data_n", C.c_int32),
        ("net_ctrl_vals", _i64p), ("net_data_vals", _i64p),
        ("net_ctrl_cdf", C.POINTER(C.c_double)), ("net_data_cdf", C.POINTER(C.c_double)),
        ("net_ctrl_const", C.c_int64), ("net_data_const", C.c_int64),
        ("net_key", C.c_uint64 * 2),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("req_dispatch", _i64p), ("req_start", _i64p), ("req_finish", _i64p),
        ("req_batch", _i64p), ("req_outcome", _i64p),
        ("n_orders", C.c_int64),
        ("ord_gpu", _i32p), ("ord_model", _i32p), ("ord_size", _i32p),
        ("ord_start", _i64p), ("ord_finish", _i64p), ("ord_emitted", _i64p),
        ("n_trace", C.c_int64),
        ("tr_t", _i64p), ("tr_start", _i64p), ("tr_finish", _i64p),
        ("tr_kind", _i32p), ("tr_model", _i32p), ("tr_gpu", _i32p),
        ("tr_size", _i32p), ("tr_rid_off", _i64p), ("tr_rids", _i64p),
        ("drops", C.c_int64), ("completions", C.c_int64), ("late", C.c_int64),
        ("ops", C.c_int64), ("evictions", C.c_int64),
        ("registrations", C.c_int64), ("handler_ops_max", C.c_int64),
        ("events_popped", C.c_int64), ("events_pushed", C.c_int64),
        ("err_index", C.c_int64),
    ]


_lib = None


def build() -> str:
    """Compile the oracle with its committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.symo_run.argtypes = [C.POINTER(_Config), _i64p, _i64p, C.c_int64,
                                  C.POINTER(_Result)]
        _lib.symo_run.restype = C.c_int32
        _lib.symo_free_result.argtypes = [C.POINTER(_Result)]
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, where: int):
        self.code = code
        self.where = where
        super().__init__(f"oracle failed: {ERRORS.get(code, code)} (arrival {where})")


def _arr(p, n, dtype):
    if n == 0:
        return np.empty(0, dtype)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dtype, copy=True)


def run(lat_ns, max_batch, slo_ns, timeout_ns, n_gpus, arr_ticks, arr_midx,
        kind="deferred", gather="prefix", target_batch=0, d_ctrl_ns=0,
        d_data_ns=0, record_trace=False, check_invariants=False, net=None) -> dict:
    """Run the restated reference loop on one engine (one sub-cluster).

    lat_ns: int64 [M, stride] with lat_ns[m, b-1] = l_m(b).
    Returns per-request arrays, per-order arrays in emission order, the trace
    and the counters.
    """
    lat = np.ascontiguousarray(lat_ns, dtype=np.int64)
    M = lat.shape[0]
    mb = np.ascontiguousarray(max_batch, dtype=np.int32)
    slo = np.ascontiguousarray(slo_ns, dtype=np.int64)
    tmo = np.ascontiguousarray(timeout_ns, dtype=np.int64)
    ticks = np.ascontiguousarray(arr_ticks, dtype=np.int64)
    midx = np.ascontiguousarray(arr_midx, dtype=np.int64)
    n = len(ticks)
    cfg = _Config(M, int(n_gpus), KIND[kind], GATHER[gather], int(target_batch),
                  int(bool(record_trace)), int(bool(check_invariants)), 0,
                  int(d_ctrl_ns), int(d_data_ns),
                  lat.ctypes.data_as(_i64p), lat.shape[1], 0,
                  mb.ctypes.data_as(_i32p), slo.ctypes.data_as(_i64p),
                  tmo.ctypes.data_as(_i64p))
    keep = []
    if net is not None:  # JitterTables (paper_2308_07470_b200.network)
        cv = np.ascontiguousarray(net.ctrl_vals, np.int64)
        cc = np.ascontiguousarray(net.ctrl_cdf, np.float64)
        dv = np.ascontiguousarray(net.data_vals, np.int64)
        dc = np.ascontiguousarray(net.data_cdf, np.float64)
        keep += [cv, cc, dv, dc]
        cfg.net_ctrl_n, cfg.net_data_n = len(cv), len(dv)
        cfg.net_ctrl_vals = cv.ctypes.data_as(_i64p)
        cfg.net_data_vals = dv.ctypes.data_as(_i64p)
        cfg.net_ctrl_cdf = cc.ctypes.data_as(C.POINTER(C.c_double))
        cfg.net_data_cdf = dc.ctypes.data_as(C.POINTER(C.c_double))
        cfg.net_ctrl_const, cfg.net_data_const = int(net.ctrl_const), int(net.data_const)
        cfg.net_key[0], cfg.net_key[1] = int(net.key[0]), int(net.key[1])
    outs = {k: np.empty(n, np.int64) for k in
            ("dispatch", "start", "finish", "batch", "outcome")}
    res = _Result()
    res.n = n
    res.req_dispatch = outs["dispatch"].ctypes.data_as(_i64p)
    res.req_start = outs["start"].ctypes.data_as(_i64p)
    res.req_finish = outs["finish"].ctypes.data_as(_i64p)
    res.req_batch = outs["batch"].ctypes.data_as(_i64p)
    res.req_outcome = outs["outcome"].ctypes.data_as(_i64p)
    L = lib()
    rc = L.symo_run(C.byref(cfg), ticks.ctypes.data_as(_i64p),
                    midx.ctypes.data_as(_i64p), n, C.byref(res))
    try:
        if rc != 0:
            raise OracleError(rc, res.err_index)
        no, nt = res.n_orders, res.n_trace
        out = {
            "req_dispatch": outs["dispatch"], "req_start": outs["start"],
            "req_finish": outs["finish"], "req_batch": outs["batch"],
            "req_outcome": outs["outcome"],
            "ord_gpu": _arr(res.ord_gpu, no, np.int64),
            "ord_model": _arr(res.ord_model, no, np.int64),
            "ord_size": _arr(res.ord_size, no, np.int64),
            "ord_start": _arr(res.ord_start, no, np.int64),
            "ord_finish": _arr(res.ord_finish, no, np.int64),
            "ord_emitted": _arr(res.ord_emitted, no, np.int64),
            "drops": res.drops, "completions": res.completions,
            "late": res.late, "ops": res.ops, "evictions": res.evictions,
            "registrations": res.registrations,
            "handler_ops_max": res.handler_ops_max,
            "events_popped": res.events_popped,
            "events_pushed": res.events_pushed,
        }
        if record_trace:
            off = _arr(res.tr_rid_off, nt + 1, np.int64) if nt else np.zeros(1, np.int64)
            rids = _arr(res.tr_rids, int(off[-1]), np.int64)
            out["trace"] = {
                "t": _arr(res.tr_t, nt, np.int64),
                "kind": _arr(res.tr_kind, nt, np.int64),
                "model": _arr(res.tr_model, nt, np.int64),
                "gpu": _arr(res.tr_gpu, nt, np.int64),
                "size": _arr(res.tr_size, nt, np.int64),
                "start": _arr(res.tr_start, nt, np.int64),
                "finish": _arr(res.tr_finish, nt, np.int64),
                "rid_off": off, "rids": rids,
            }
        return out
    finally:
        L.symo_free_result(C.byref(res))


def run_shards(shards: list[dict], threads: int | None = None) -> list[dict]:
    """Run independent sub-cluster engines concurrently (ctypes releases the
    GIL), mirroring scalebench.bench_workers' process-per-shard layout."""
    threads = threads or min(len(shards), len(os.sched_getaffinity(0)))
    if threads <= 1 or len(shards) <= 1:
        return [run(**sh) for sh in shards]
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(lambda sh: run(**sh), shards))
