"""ctypes binding of the CUDA engine library (include/symphony_b200.h).

The library is built in-tree by __graft_entry__.build() (nvcc, sm_100a) as
paper_2308_07470_b200/libsymphony_b200.so.  There is no CPU fallback: if
the library or a CUDA device is missing, loading raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libsymphony_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)

SYM_OK, SYM_EPROTO, SYM_EINVAL, SYM_EINVARIANT, SYM_ECUDA, SYM_ENOMEM, SYM_EGUARD = range(7)
FLAG_TRACE, FLAG_NO_FRESH, FLAG_NO_EXPAND, FLAG_NO_FAST, FLAG_KERNEL_TIMES = 1, 2, 4, 8, 16
FLAG_MODEL_I64 = 32
FLAG_CHECK_INVARIANTS, FLAG_INJECT_FAULT = 64, 128
KIND = {"deferred": 0, "eager": 1, "timeout": 2}
GATHER = {"prefix": 0, "drop_head": 1}

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class SymConfig(C.Structure):
    _fields_ = [
        ("n_models", C.c_int32), ("n_gpus", C.c_int32), ("kind", C.c_int32),
        ("gather", C.c_int32), ("target_batch", C.c_int32), ("lat_stride", C.c_int32),
        ("d_ctrl_ns", C.c_int64), ("d_data_ns", C.c_int64),
        ("lat_ns", i64p), ("max_batch", i32p), ("slo_ns", i64p), ("timeout_ns", i64p),
        ("n_shards", C.c_int32), ("device", C.c_int32),
        ("shard_of_model", i32p), ("gpus_per_shard", i32p),
        ("net_ctrl_n", C.c_int32), ("net_data_n", C.c_int32),
        ("net_ctrl_vals", i64p), ("net_data_vals", i64p),
        ("net_ctrl_cdf", C.POINTER(C.c_double)), ("net_data_cdf", C.POINTER(C.c_double)),
        ("net_ctrl_const", C.c_int64), ("net_data_const", C.c_int64),
        ("net_key", C.c_uint64 * 2),
        ("devices", i32p), ("n_devices", C.c_int32), ("_pad_dev", C.c_int32),
    ]


class SymBatch(C.Structure):
    _fields_ = [
        ("emitted", C.c_int64), ("start", C.c_int64), ("finish", C.c_int64),
        ("key_t", C.c_int64), ("key_sub", C.c_int64), ("key_a", C.c_int32),
        ("model", C.c_int32), ("gpu", C.c_int32), ("size", C.c_int32),
        ("first_index", C.c_int32), ("shrunk_from", C.c_int32),
    ]


BATCH_DTYPE = [("emitted", "<i8"), ("start", "<i8"), ("finish", "<i8"),
               ("key_t", "<i8"), ("key_sub", "<i8"), ("key_a", "<i4"),
               ("model", "<i4"), ("gpu", "<i4"), ("size", "<i4"),
               ("first_index", "<i4"), ("shrunk_from", "<i4")]


class SymResult(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("req_dispatch", i64p), ("req_start", i64p), ("req_finish", i64p),
        ("req_batch", i64p), ("req_outcome", i64p),
        ("req_arrival", i64p), ("req_deadline", i64p), ("req_model", i64p),
        ("drop_t", i64p), ("drop_key_sub", i64p), ("drop_key_a", i32p),
        ("batches", C.c_void_p), ("batch_cap", C.c_int64), ("n_batches", C.c_int64),
        ("drops", C.c_int64), ("completions", C.c_int64), ("late", C.c_int64),
        ("ops", C.c_int64), ("evictions", C.c_int64), ("registrations", C.c_int64),
        ("handler_ops_max", C.c_int64),
        ("chain_events", C.c_int64), ("absorbed_arrivals", C.c_int64),
        ("fresh_adoptions", C.c_int64), ("launches", C.c_int64),
        ("fast_shards", C.c_int64), ("fast_fail_mask", C.c_int64),
        ("ms_ingest", C.c_float), ("ms_fresh", C.c_float), ("ms_fast", C.c_float),
        ("ms_chain", C.c_float),
        ("ms_expand", C.c_float), ("ms_total", C.c_float),
        ("err_index", C.c_int64),
    ]


EXPORTS = ("sym_create", "sym_destroy", "sym_run", "sym_run_device",
           "sym_window_counts", "sym_last_error", "sym_version", "sym_kernel_times",
           "sym_last_batches", "sym_window_stats", "sym_text_format", "sym_text_fetch",
           "sym_text_free", "sym_part_brute_force", "sym_part_evaluate", "sym_part_solve",
           "sym_step_reset", "sym_step", "sym_step_result")

TEXT_REQUESTS, TEXT_LATENCY = 0, 1


class SymPartProblem(C.Structure):
    _fields_ = [("m", C.c_int32), ("l", C.c_int32),
                ("rates", C.POINTER(C.c_double)), ("static_mem", C.POINTER(C.c_double)),
                ("dynamic_mem", C.POINTER(C.c_double)),
                ("rate_cap", C.c_double), ("mem_cap", C.c_double), ("weight", C.c_double),
                ("mean_rate", C.c_double), ("mean_mem", C.c_double),
                ("current", C.POINTER(C.c_int32)), ("change_cost", C.POINTER(C.c_double)),
                ("change_budget", C.c_double)]


class SymTextColumns(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(k, i64p) for k in (
        "req_model", "req_arrival", "req_dispatch", "req_start", "req_finish", "req_batch",
        "req_outcome")] + [("n_names", C.c_int32), ("_pad", C.c_int32),
                           ("names", C.c_char_p), ("name_off", i64p)]

_lib = None


class NativeUnavailable(RuntimeError):
    pass


def load(path: str | None = None):
    """Load (once) and type the engine library; raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("SYMPHONY_B200_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    lib.sym_create.argtypes = [C.POINTER(SymConfig), i32p]
    lib.sym_create.restype = C.c_void_p
    lib.sym_destroy.argtypes = [C.c_void_p]
    lib.sym_destroy.restype = None
    for fn in (lib.sym_run, lib.sym_run_device):
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_uint32,
                       C.POINTER(SymResult)]
        fn.restype = C.c_int32
    lib.sym_step_reset.argtypes = [C.c_void_p]
    lib.sym_step_reset.restype = C.c_int32
    lib.sym_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                             C.c_uint32, C.POINTER(SymResult)]
    lib.sym_step.restype = C.c_int32
    lib.sym_step_result.argtypes = [C.c_void_p, C.POINTER(SymResult)]
    lib.sym_step_result.restype = C.c_int32
    lib.sym_window_counts.argtypes = [C.c_void_p, C.c_int64, C.c_int64] + [i64p] * 5
    lib.sym_window_counts.restype = C.c_int32
    lib.sym_window_stats.argtypes = ([C.c_void_p, C.c_int64, C.c_int64] + [i64p] * 8 +
                                     [C.c_int32])
    lib.sym_window_stats.restype = C.c_int32
    lib.sym_last_error.argtypes = [C.c_void_p]
    lib.sym_last_error.restype = C.c_char_p
    lib.sym_version.restype = C.c_int32
    lib.sym_last_batches.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    lib.sym_last_batches.restype = C.c_int64
    lib.sym_kernel_times.argtypes = [C.c_void_p, C.c_int32]
    lib.sym_kernel_times.restype = C.c_char_p
    lib.sym_text_format.argtypes = [C.c_int32, C.POINTER(SymTextColumns), C.c_int32, i64p, i32p]
    lib.sym_text_format.restype = C.c_void_p
    lib.sym_text_fetch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    lib.sym_text_fetch.restype = C.c_int32
    lib.sym_text_free.argtypes = [C.c_void_p]
    lib.sym_text_free.restype = None
    pp = C.POINTER(SymPartProblem)
    lib.sym_part_brute_force.argtypes = [pp, C.c_int32, i32p, C.POINTER(C.c_double), i32p]
    lib.sym_part_evaluate.argtypes = [pp, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                      C.c_void_p, C.POINTER(C.c_int64)]
    lib.sym_part_solve.argtypes = [pp, C.c_int32, C.c_void_p, C.c_uint64, C.c_int64,
                                   C.c_int32, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]
    for fn in (lib.sym_part_brute_force, lib.sym_part_evaluate, lib.sym_part_solve):
        fn.restype = C.c_int32
    _lib = lib
    return lib


def pinned_empty(n: int, dtype=np.int64):
    """A host array in page-locked memory from torch's caching host allocator
    (recycled across calls once the array is freed), so device->host copies
    run at full PCIe speed; plain numpy memory if torch is unavailable."""
    dtype = np.dtype(dtype)
    try:
        import torch
        t = torch.empty(max(int(n), 1) * dtype.itemsize, dtype=torch.uint8, pin_memory=True)
        return t.numpy().view(dtype)[:n]
    except Exception:  # noqa: BLE001 -- no torch / no driver: pageable memory
        return np.empty(n, dtype)
