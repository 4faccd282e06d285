"""Cycle attribution of the sequential chain (dev tool).  Builds a separate
library with -DSYM_CHAIN_PROF (clock64 around each chain_step phase) under
/tmp or gpurun_out, runs overloaded cases through it, prints cycles/event."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

LIB = os.path.join(ROOT, "gpurun_out", "libsym_chainprof.so")
if not os.path.exists(LIB) or "--build" in sys.argv:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = [os.path.join(g.CSRC, f) for f in ("engine.cu", "multi.cu", "textfmt.cu",
                                                 "partition.cu")]
    subprocess.run([g._nvcc(), *g.NVCC_FLAGS, "-DSYM_CHAIN_PROF", "-o", LIB, *srcs], check=True)
if "--build" in sys.argv:
    sys.exit(0)
os.environ["SYMPHONY_B200_LIB"] = LIB
from paper_2308_07470_b200 import _native, scenario as SCN  # noqa: E402
from paper_2308_07470_b200.scheduler import PolicyConfig  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

lib = _native.load()
lib.sym_chain_prof.argtypes = [C.c_void_p]
buf = (C.c_ulonglong * 16)()


def report(label):
    lib.sym_chain_prof(buf)
    v = list(buf)
    n = sum(v[4:8]) or 1
    names = ["MT", "DT", "ARR", "GPU"]
    parts = ", ".join(f"{names[i]} {v[4 + i]} x {v[i] / max(v[4 + i], 1):.0f}" for i in range(4))
    tot = sum(v[0:4]) + v[8] + v[9] + v[10]
    print(f"{label}: events {n}, cycles/event {tot / n:.0f} | handler {sum(v[0:4]) / n:.0f} "
          f"dispatch {v[8] / n:.0f} refresh {v[9] / n:.0f} pq {v[10] / n:.0f} "
          f"(refreshed/event {v[11] / n:.2f}) | {parts}", flush=True)
    print(f"    update_candidate {v[13] / n:.2f} calls/event x {v[12] / max(v[13], 1):.0f} cycles; "
          f"scan_model {v[14] / n:.0f} cycles/event; set_gpu_timer {v[15] / n:.0f} cycles/event",
          flush=True)


sc = SCN.load_scenario("table2_resnet50").with_rate(11678.8)
eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
lib.sym_chain_prof(buf)
eng.run(sc.workload, sc.duration_s, sc.seed)
report("table2 overload")
c1 = configs.CONFIGS["C1"](60.0)
t, m = generate_arrivals(c1.workload, [x.name for x in c1.models], 60.0, 42)
eng = Engine(list(c1.models), c1.gpu_count, PolicyConfig("eager"))
eng.run_stream(t, m, 60.0)
report("C1 eager")

for name in ("C3", "C4"):
    sc = configs.CONFIGS[name](1.0, "eager")
    t, m = generate_arrivals(sc.workload, [x.name for x in sc.models], 1.0, 42)
    models, gpus = list(sc.models), sc.gpu_count
    if name == "C4":
        ms, g, ids = configs.shard_scenarios(sc)[0]
        keep = (m >= ids[0]) & (m <= ids[-1])
        t, m, models, gpus = t[keep], m[keep] - ids[0], list(ms), g
    eng = Engine(models, gpus, sc.policy)
    eng.run_stream(t, m, 1.0)
    report(f"{name} eager 1 s ({len(t)} requests, {eng.stats['ms_chain']:.0f} ms chain)")
