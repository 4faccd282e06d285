"""DEV TOOL: build tools/hostcheck (the chain + lean fast-path helpers
compiled for the host) and run every golden case through it, reporting the
lean-pointer mismatch counter (counters[9]) and parity with the oracle."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]

from oracle import oracle  # noqa: E402
import cases  # noqa: E402
from conftest import oracle_args  # noqa: E402

LIB = os.path.join(HERE, "libhostcheck.so")
subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", LIB,
                os.path.join(HERE, "hostcheck.cpp")], check=True)
lib = C.CDLL(LIB)
i64p = C.POINTER(C.c_int64)
lib.hc_run.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                       C.c_void_p, C.c_void_p, C.c_void_p]
lib.hc_run.restype = C.c_int32


def cfg_of(models, gpus, policy):
    a = oracle_args(models, gpus, policy)
    lat = np.ascontiguousarray(a["lat_ns"], np.int64)
    mb = np.ascontiguousarray(a["max_batch"], np.int32)
    slo = np.ascontiguousarray(a["slo_ns"], np.int64)
    tmo = np.ascontiguousarray(a["timeout_ns"], np.int64)
    cfg = oracle._Config(len(models), gpus, oracle.KIND[a["kind"]], oracle.GATHER[a["gather"]],
                         int(a["target_batch"]), 0, 0, 0, int(a["d_ctrl_ns"]), int(a["d_data_ns"]),
                         lat.ctypes.data_as(i64p), lat.shape[1], 0,
                         mb.ctypes.data_as(C.POINTER(C.c_int32)), slo.ctypes.data_as(i64p),
                         tmo.ctypes.data_as(i64p))
    return cfg, (lat, mb, slo, tmo)


total_bad = 0
for case in list(cases.bundled()) + list(cases.stress()) + list(cases.config_cases()):
    key, models, gpus, policy, ticks, midx = case[:6]
    cfg, keep = cfg_of(models, gpus, policy)
    n = len(ticks)
    t = np.ascontiguousarray(ticks, np.int64)
    m = np.ascontiguousarray(midx, np.int64)
    req = np.zeros(5 * n, np.int64)
    ords = np.zeros(7 * (n + 1), np.int64)
    nord = C.c_int64(0)
    cnt = np.zeros(10, np.int64)
    rc = lib.hc_run(1, C.addressof(cfg), t.ctypes.data, m.ctypes.data, n, req.ctypes.data,
                    ords.ctypes.data, C.addressof(nord), cnt.ctypes.data)
    bad = int(cnt[9])
    ref = oracle.run(arr_ticks=ticks, arr_midx=midx, **oracle_args(models, gpus, policy))
    diff = [k for j, k in enumerate(("req_dispatch", "req_start", "req_finish", "req_batch",
                                      "req_outcome")) if not np.array_equal(req[j * n:(j + 1) * n],
                                                                            ref[k])]
    total_bad += bad + len(diff)
    if rc or bad or diff:
        print(key, "rc", rc, "mismatch", bad, "certified", int(cnt[8]), "parity", diff or "ok",
              flush=True)
print("cases done; total mismatch", total_bad)
