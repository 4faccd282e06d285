"""Phase timestamps of concurrent engines (dev tool)."""
import ctypes as C
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, ".")
from paper_2308_07470_b200 import _native, scenario as SCN  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

sc = SCN.load_scenario("table2_resnet50").with_rate(11678.8)
ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], sc.duration_s, sc.seed)
T0 = [0.0]


def stamp():
    return round(time.perf_counter() - T0[0], 3)


def one(i):
    log = [("start", stamp())]
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, use_fast=False)
    eng._ensure()
    log.append(("created", stamp()))
    n = len(ticks)
    outs = {k: _native.pinned_empty(n) for k in range(8)}
    log.append(("pinned", stamp()))
    res = _native.SymResult()
    res.n = n
    for k, nm in enumerate(("dispatch", "start", "finish", "batch", "outcome", "arrival",
                            "deadline", "model")):
        setattr(res, "req_" + nm, outs[k].ctypes.data_as(_native.i64p))
    rc = eng._lib.sym_run(eng._handle, ticks.ctypes.data, midx.ctypes.data, n,
                          eng._flags() | _native.FLAG_MODEL_I64, C.byref(res))
    log.append(("sym_run", stamp(), rc, round(res.ms_total, 1)))
    eng.close()
    log.append(("closed", stamp()))
    return i, log


one(0)
for k in (2, 4):
    T0[0] = time.perf_counter()
    with ThreadPoolExecutor(k) as ex:
        for i, log in ex.map(one, range(k)):
            print(k, i, log, flush=True)
