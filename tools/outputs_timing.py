"""Time the result-file writers on a large engine result (C4 sub-cluster):
GPU rendering (csrc/textfmt.cu) vs the host formatter, plus the
reference-style per-element loop on a 1M-request slice for scale."""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2308_07470_b200 import outputs as O  # noqa: E402
from paper_2308_07470_b200.simulator import Engine, OUTCOME_NAMES  # noqa: E402


def ref_style_requests(result, limit):
    lines = [O.REQUESTS_HEADER]
    names = result.model_names
    for i in range(limit):
        o = result.req_outcome[i]
        outcome = OUTCOME_NAMES[o] if o >= 0 else ""
        if o == 2:
            lines.append(f"{i + 1},{names[result.req_model[i]]},{result.req_arrival[i]},,,,,{outcome}")
        else:
            lines.append(f"{i + 1},{names[result.req_model[i]]},{result.req_arrival[i]},"
                         f"{result.req_dispatch[i]},{result.req_start[i]},{result.req_finish[i]},"
                         f"{result.req_batch[i]},{outcome}")
    return "\n".join(lines) + "\n"


def main():
    from bench import build_workload
    sc, models, gpus, ticks, midx = build_workload(60.0, 0)
    res = Engine(models, gpus, sc.policy).run_stream(ticks, midx, 60.0)
    n = res.n_requests
    out = {"requests": n}
    O.requests_csv(res, 0)  # warm (context, kernels)
    for dev, key in ((0, "gpu"), (None, "host")):
        t = time.perf_counter()
        txt = O.requests_csv(res, dev)
        out[f"requests_csv_{key}_s"] = round(time.perf_counter() - t, 4)
        out[f"requests_csv_{key}_bytes"] = len(txt)
        t = time.perf_counter()
        O.latency_csv(res, dev)
        out[f"latency_csv_{key}_s"] = round(time.perf_counter() - t, 4)
    lim = min(1_000_000, n)
    t = time.perf_counter()
    ref_style_requests(res, lim)
    el = time.perf_counter() - t
    out["requests_csv_refloop_s_extrapolated"] = round(el * n / lim, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
