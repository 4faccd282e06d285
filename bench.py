"""Benchmark: requests scheduled per second (device-timed) on BASELINE's C4.

Workload (BASELINE.json configs[3]): 1000 A100-zoo models x
8192 simulated GPUs, Poisson 1.2M req/s aggregate over a 60 s trace, seed 42,
partitioned into P=8 sub-clusters of 125 contiguous models and 1024 GPUs.
The configuration is fixed and the GPU count varies (strong scaling): rank r
of N runs sub-clusters {s : s mod N == r} in ONE engine call, so N=1 is the
whole of C4 (72M requests) on one B200 and N=8 is one sub-cluster per B200.

A step is one pass of the hot path over the rank's whole trace, inputs
resident in HBM: ingest (stable partition) -> window/chain pointers (K2) ->
batch chains -> batch order -> matchmaking (K3) -> per-request RunResult
arrays.  The parallel validated path resolves every C4 sub-cluster; the exact
sequential chain would take over any sub-cluster that failed validation.
``value`` is the whole-job throughput (all requests / max-over-ranks device
time); ``e2e`` is the same metric through the public API (Engine.run_stream:
pinned host arrays in, RunResult out, H2D/D2H inside the timed region).
Every rank checks its device results bit for bit against the CPU oracle
(oracle/, a C restatement of batchsym's loop) before printing.

--impl reference times that CPU restatement of the reference algorithm on
the host cores over the same C4 sub-clusters (one thread per sub-cluster,
the reference scalebench's process-per-shard layout).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "requests scheduled/sec (device-timed) at 1/2/4/8 B200; goodput bit-exact vs CPU ref"
UNIT = "requests/s"
N_SUBCLUSTERS = 8
FRESH_REC_BYTES = 128  # sizeof(FreshRec)
BATCH_REC_BYTES = 64   # sizeof(BatchRec) / sizeof(sym_batch)
EV_BATCH_BYTES = 56    # sizeof(EvBatch)

# SURVEY.md §8(d) algorithmic bytes of the three kernels north_star names
# (n requests, nb batches, G simulated GPUs of the launch):
#   K1 ingest       24 B per request (read tick+model 12, write 12 permuted)
#   K2 window       12 B per arrival scanned (the per-model state and the
#                   log2(max_batch) l(b) probes are negligible at this size)
#   K3 matchmaking  8 B per GPU free_at + 24 B per ready candidate + 12 B
#                   written per grant
# K1's 24 B/request cover the whole stable partition; with several
# sub-clusters in one engine it runs as two k_part passes (by sub-cluster,
# then by model), so each pass is credited its share (24 B / passes).
SURVEY_KERNELS = {
    "K1": ("k_part", lambda n, nb, g, passes=1: 24 * n / passes),
    "K2": ("k_nxt_tma", lambda n, nb, g, passes=1: 12 * n),
    "K3": ("k_match_coop", lambda n, nb, g, passes=1: 36 * nb + 8 * g),
}


def design_bytes(kernel: str, n: int, nb: int, shards: int) -> float | None:
    """Minimal DRAM bytes one launch of a kernel outside §8(d)'s three must
    move (DESIGN.md §5 derives each line)."""
    table = {
        "k_part_count": n * 4,
        "k_fresh": n * (8 + 4 + 4 + FRESH_REC_BYTES + 4),
        "k_nxt_general": 0,
        "k_chain_recs": n * (8 + 4 + 4) + nb * (4 + EV_BATCH_BYTES + 8 + 4),
        "k_walk_expand": nb * (64 + 4),   # 4 KB pointer window per 64 batches + the start
        "k_cp_scan": 0,
        "k_tie_fix": 0,
        "k_match_iter": 0,
        "k_token_keys": nb * (4 + 8 + EV_BATCH_BYTES + 8 + 4),
        "k_jump4": n * (4 + 4),
        "k_bkt_scatter": nb * (12 + 12),
        "k_fast_emit": nb * (EV_BATCH_BYTES + 12 + 4 + 8 + BATCH_REC_BYTES),
        "k_bid": nb * BATCH_REC_BYTES + n * (4 + 4),        # records, s_i, bid by request
        "k_out": n * (8 + 4 + 4 + 5 * 8) + nb * BATCH_REC_BYTES,  # tick, model, bid; 5 results
        "k_copy_batches": nb * (BATCH_REC_BYTES + 4 + 64),
    }
    return table.get(kernel)


def kernel_bytes(kernel: str, n: int, nb: int, g: int, shards: int, passes: float = 1):
    """(bytes per launch, source) -- §8(d) for K1/K2/K3, else DESIGN."""
    for tag, (name, fn) in SURVEY_KERNELS.items():
        if name == kernel:
            return fn(n, nb, g, passes), f"SURVEY §8(d) {tag}" + (
                f" / {passes:g} passes" if passes != 1 else "")
    b = design_bytes(kernel, n, nb, shards)
    return b, ("DESIGN.md §5" if b is not None else None)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def my_subclusters(rank: int, world: int) -> list[int]:
    from paper_2308_07470_b200.parallel import assign
    return assign(N_SUBCLUSTERS, world)[rank]


def build_workload(duration_s: float, subclusters: list[int]):
    """The C4 trace restricted to the given sub-clusters, their models
    renumbered contiguously in sub-cluster order.  Returns the scenario,
    the engine arguments and each sub-cluster's (models, gpus, stream
    indices) for the oracle."""
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(duration_s)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], duration_s,
                                    configs.SEED)
    parts = configs.shard_scenarios(sc)
    new_id = np.full(len(sc.models), -1, np.int64)
    models, som, gps, k = [], [], [], 0
    from dataclasses import replace
    for j, s in enumerate(subclusters):
        ms, g, ids = parts[s]
        for i in ids:
            new_id[i] = k
            models.append(replace(sc.models[i], model_id=k))
            som.append(j)
            k += 1
        gps.append(g)
    m2 = new_id[midx]
    keep = m2 >= 0
    t_sel = np.ascontiguousarray(ticks[keep])
    m_sel = np.ascontiguousarray(m2[keep])
    som_a = np.asarray(som, np.int32)
    per = []
    base = 0
    for j, s in enumerate(subclusters):
        ms, g, ids = parts[s]
        idx = np.nonzero(som_a[m_sel] == j)[0]
        per.append((list(ms), g, idx, base))
        base += len(ids)
    return sc, models, int(sum(gps)), (som, gps), t_sel, m_sel, per


def oracle_shard_run(ms, gpus, policy, ticks, midx):
    from oracle import oracle
    stride = max(m.profile.max_batch for m in ms)
    return oracle.run(np.stack([m.profile.table_array(stride) for m in ms]),
                      [m.profile.max_batch for m in ms], [m.slo_ns for m in ms],
                      [policy.resolve_timeout_ns(m.slo_ns) for m in ms], gpus, ticks, midx,
                      kind=policy.kind, gather=policy.gather,
                      target_batch=policy.target_batch, d_ctrl_ns=policy.d_ctrl_ns,
                      d_data_ns=policy.d_data_ns)


def oracle_all(sc, per, ticks, midx, threads):
    """The oracle over every sub-cluster of the rank, one thread each (the
    C library releases the GIL); returns (results, wall seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    def one(p):
        ms, g, idx, base = p
        return oracle_shard_run(ms, g, sc.policy, ticks[idx], midx[idx] - base)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max(1, threads)) as ex:
        res = list(ex.map(one, per))
    return res, time.perf_counter() - t0


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the
    timed region (B200_PROFILING.md clocks line)."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.window = None  # (t0, t1) wall-clock bounds of the timed region
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(1.0)  # nvidia-smi start-up: sampling runs before timing starts

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        import datetime
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            if self.window and not (self.window[0] - 0.25 <= ts <= self.window[1] + 0.25):
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def workload_name(duration_s: float) -> str:
    return (f"C4: 1000 A100-zoo models x 8192 GPUs, Poisson 1.2M req/s, {duration_s:g} s "
            f"trace, seed 42, 8 sub-clusters of 125 models x 1024 GPUs")


def base_config(args, world):
    return {"workload": workload_name(args.duration), "policy": "deferred", "max_batch": 256,
            "subclusters_per_gpu": N_SUBCLUSTERS / world,
            "l2": "256 MB buffer written before every step (> 126 MB L2)",
            "parallelism": f"sub-cluster s on GPU s mod {world}"}


REF_BUDGET_S = 150.0
PYREF_DIR = os.path.join(ROOT, "baseline", "_ref")
PYREF_SECONDS = 2.0


def python_reference_sample():
    """The unmodified Python reference (batchsym, pip-installed into
    baseline/_ref from the reference package) timed on one host
    core: its Engine.run_stream over the first PYREF_SECONDS of C4
    sub-cluster 0, its result checked against the oracle's.  None when the
    install is absent."""
    if not os.path.isdir(os.path.join(PYREF_DIR, "batchsym")):
        return None
    sys.path.insert(0, PYREF_DIR)
    try:
        import batchsym.profile as RP
        import batchsym.scheduler as RS
        from batchsym.simulator import Engine as REngine
    finally:
        sys.path.remove(PYREF_DIR)
    sc, _, _, _, ticks, midx, per = build_workload(PYREF_SECONDS, [0])
    ms, g, idx, base = per[0]
    t, m = ticks[idx], midx[idx] - base
    rmodels = [RP.ModelSpec(x.model_id, x.name,
                            RP.LatencyProfile(x.profile.kind, x.profile.max_batch,
                                              x.profile.alpha_ns, x.profile.beta_ns,
                                              x.profile.lat_ns), x.slo_ns) for x in ms]
    eng = REngine(rmodels, g, RS.PolicyConfig(sc.policy.kind))
    t0 = time.perf_counter()
    res = eng.run_stream(t, m, PYREF_SECONDS)
    el = time.perf_counter() - t0
    ref = oracle_shard_run(ms, g, sc.policy, t, m)
    same = all(np.array_equal(np.asarray(getattr(res, "req_" + k)), ref["req_" + k])
               for k in ("dispatch", "start", "finish", "batch", "outcome"))
    return {"value": len(t) / el, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"batchsym Engine.run_stream (baseline/_ref), C4 sub-cluster 0, first "
                      f"{PYREF_SECONDS:g} s of the trace ({len(t)} requests)",
            "equals_oracle": bool(same)}


def run_reference(args, world):
    """CPU arm: the oracle port over all 8 C4 sub-clusters, one host thread
    per sub-cluster (scalebench.bench_workers' process-per-shard layout)."""
    cores = min(N_SUBCLUSTERS, len(os.sched_getaffinity(0)))
    all_sc = list(range(N_SUBCLUSTERS))
    # bounded sample: the same trace, shortened if K + W steps of the full
    # trace would not fit REF_BUDGET_S (calibrated on one second first)
    sc, _, _, _, t1, m1, per1 = build_workload(1.0, all_sc)
    _, cal = oracle_all(sc, per1, t1, m1, cores)
    dur = round(min(args.duration, max(1.0, REF_BUDGET_S / (cal * (args.steps + args.warmup)))), 2)
    sc, _, _, _, ticks, midx, per = build_workload(dur, all_sc)
    n_total = len(ticks)
    for _ in range(args.warmup):
        oracle_all(sc, per, ticks, midx, cores)
    el = 0.0
    for _ in range(args.steps):
        el += oracle_all(sc, per, ticks, midx, cores)[1]
    value = n_total * args.steps / el
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "impl": "reference", "config": base_config(args, world),
        "requests_per_step": n_total,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"all 8 C4 sub-clusters, first {dur:g} s of the "
                                   f"{args.duration:g} s trace ({n_total} requests) per step; "
                                   "oracle/symoracle.c (C restatement of batchsym's event "
                                   "loop), one host thread per sub-cluster"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        py = python_reference_sample()
    except Exception as exc:  # the reported arm stays the C port
        py = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    if py is not None:
        line["python_reference"] = py
    print(json.dumps(line), flush=True)


def check_parity(res_by_shard, per, outs):
    """Device outputs of the timed runs vs the oracle, element for element."""
    for (ms, g, idx, base), ref in zip(per, res_by_shard):
        for k in ("dispatch", "start", "finish", "batch", "outcome"):
            got = outs[k][idx]
            if not np.array_equal(got, ref["req_" + k]):
                bad = int(np.nonzero(got != ref["req_" + k])[0][0])
                raise SystemExit(f"parity failure vs the oracle on req_{k} "
                                 f"(sub-cluster model base {base}, request {bad})")


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2308_07470_b200.simulator import Engine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    mine = my_subclusters(rank, world)
    sc, models, gpus, shards, ticks, midx, per = build_workload(args.duration, mine)
    n = len(ticks)
    eng = Engine(models, gpus, sc.policy, shards=shards, device=local_rank)
    t_dev = torch.from_numpy(ticks).to(dev)
    m_dev = torch.from_numpy(midx.astype(np.int32)).to(dev)
    outs = {k: torch.empty(n, dtype=torch.int64, device=dev)
            for k in ("dispatch", "start", "finish", "batch", "outcome")}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    for _ in range(args.warmup):
        flush.fill_(1)
        eng.run_device(t_dev, m_dev, outs)
    clk = ClockSampler(local_rank)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dev_ms, batches, launches = 0.0, 0, 0
    phase_keys = ("ms_ingest", "ms_fresh", "ms_fast", "ms_chain", "ms_expand")
    phase_sum = dict.fromkeys(phase_keys, 0.0)
    t0 = time.perf_counter()
    w0 = time.time()
    for _ in range(args.steps):
        flush.fill_(1)
        _, cnt = eng.run_device(t_dev, m_dev, outs)
        dev_ms += cnt["ms_total"]
        batches += cnt["n_batches"]
        launches += cnt["launches"]
        for k in phase_keys:
            phase_sum[k] += cnt[k]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    clk.window = (w0, time.time())
    if world > 1:
        dist.barrier()
    clk.stop()
    stats = dict(cnt)
    stats.update({k: v / args.steps for k, v in phase_sum.items()})  # phases: mean over the K steps
    host_outs = {k: v.cpu().numpy() for k, v in outs.items()}

    # per-kernel device time: the same K steps again with every launch
    # bracketed by CUDA events on the engine's stream
    eng.kernel_times(reset=True)
    for _ in range(args.steps):
        flush.fill_(1)
        eng.run_device(t_dev, m_dev, outs, kernel_times=True)
    ktimes = eng.kernel_times(reset=True)

    # end to end through the public API: host arrays in, RunResult out
    # (steady state: two untimed calls warm the pinned-memory pool; each
    # result is released before the next call, as a streaming caller would)
    def e2e(t_host, m_host, reps):
        for _ in range(2):
            eng.run_stream(t_host, m_host, args.duration)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = eng.run_stream(t_host, m_host, args.duration)
            times.append(time.perf_counter() - t0)
            del r
        return sum(times) / len(times)
    reps = max(3, min(args.steps, 10))
    pin_t = torch.from_numpy(ticks).pin_memory().numpy()
    pin_m = torch.from_numpy(midx).pin_memory().numpy()
    e2e_pinned = e2e(pin_t, pin_m, reps)
    e2e_pageable = e2e(ticks, midx, reps)
    res = eng.run_stream(pin_t, pin_m, args.duration)
    nb_rank = len(res.batches)
    h2d = n * (8 + 8)  # ticks + int64 model ids
    # five computed RunResult arrays + the batch records cross PCIe;
    # req_arrival / req_model / req_deadline are formed on the host
    d2h = n * 5 * 8 + nb_rank * BATCH_REC_BYTES
    for k in ("batch", "outcome", "start"):
        if not np.array_equal(host_outs[k], getattr(res, "req_" + k)):
            raise SystemExit(f"device-resident and API outputs differ on req_{k}")

    # bit-exact against the CPU oracle, every sub-cluster of this rank
    threads = min(len(per), len(os.sched_getaffinity(0)))
    ref, ref_s = oracle_all(sc, per, ticks, midx, threads)
    check_parity(ref, per, host_outs)

    # end of run: the one collective -- per-sub-cluster integer summaries
    # reduced over NCCL into the cluster's goodput / idle / autoscale view
    from paper_2308_07470_b200.parallel import SummaryLayout, cluster_stats, reduce_summaries
    layout = SummaryLayout(1000, 8192)
    lo, hi = int(0.1 * args.duration * 1e9), int(0.9 * args.duration * 1e9)
    w = eng.window_counts(lo, hi)
    vec = layout.empty()
    for j, s in enumerate(mine):
        ms, g, idx, base = per[j]
        k = len(ms)
        layout.put(vec, np.arange(125 * s, 125 * s + k),
                   np.arange(1024 * s, 1024 * s + g),
                   {name: w[name][base:base + k] for name in ("arrivals", "completed", "late",
                                                              "dropped")} |
                   {"gpu_busy_ns": w["gpu_busy_ns"][1024 * j:1024 * j + g]})
    t_red = time.perf_counter()
    vec = reduce_summaries(vec)
    red_ms = 1e3 * (time.perf_counter() - t_red)
    cstats = cluster_stats(vec, layout, lo, hi)

    t = torch.tensor([dev_ms, e2e_pinned, e2e_pageable, wall], dtype=torch.float64, device=dev)
    tot = torch.tensor([n, batches, launches, h2d, d2h], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    dev_ms, e2e_pinned, e2e_pageable, wall = t.tolist()
    n_all, batches_all, launches_all, h2d_all, d2h_all = (int(x) for x in tot.tolist())
    if rank != 0:
        return
    value = n_all * args.steps / (dev_ms / 1e3)
    peak, peak_kind = measured_peak_hbm()
    nb_step = batches // args.steps  # this rank's batches per step
    kern = {}
    k_total = sum(v[1] for v in ktimes.values())
    for name, (cnt_l, k_ms) in ktimes.items():
        per_launch_ms = k_ms / cnt_l
        ab, src = kernel_bytes(name, n, nb_step, gpus, len(mine), cnt_l / args.steps)
        gbs = (ab / (per_launch_ms / 1e3) / 1e9) if ab else None
        kern[name] = {"launches_per_step": cnt_l / args.steps, "ms_per_launch": per_launch_ms,
                      "share": k_ms / k_total, "bytes_per_launch": ab, "bytes_source": src,
                      "gbs": gbs, "frac": gbs / peak if gbs else None}
    dom = max(kern, key=lambda k: kern[k]["share"])
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            summ = json.load(fh)
        if summ.get("workload") == workload_name(args.duration) and summ.get("n_gpus") == world:
            traffic = summ.get("kernels", {}).get(dom, {}).get("dram_bytes_per_launch")
    k123 = {}
    for tag, (name, _) in SURVEY_KERNELS.items():
        if name in kern:
            k123[tag] = {"kernel": name, "achieved_gbs": kern[name]["gbs"],
                         "frac": kern[name]["frac"], "ms_per_launch": kern[name]["ms_per_launch"],
                         "bytes_per_launch": kern[name]["bytes_per_launch"]}
    if "K3" in k123 and "k_tie_fix" in kern:  # the matching phase: the match + the tie groups
        ms3 = sum(kern[k]["ms_per_launch"] * kern[k]["launches_per_step"]
                  for k in ("k_match_coop", "k_tie_fix", "k_match_iter") if k in kern)
        b3 = k123["K3"]["bytes_per_launch"]
        k123["K3"]["phase"] = {"kernels": "k_match_coop + k_tie_fix + k_match_iter", "ms": ms3,
                               "achieved_gbs": b3 / (ms3 / 1e3) / 1e9,
                               "frac": b3 / (ms3 / 1e3) / 1e9 / peak}
    if "K1" in k123:  # the whole ingest phase (counts, scans, passes, readback) vs 24 B/request
        ph = stats["ms_ingest"]
        k123["K1"]["phase"] = {"ms": ph, "achieved_gbs": 24 * n / (ph / 1e3) / 1e9,
                               "frac": 24 * n / (ph / 1e3) / 1e9 / peak}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": base_config(args, world),
        "requests_per_step": n_all,
        "e2e": {"value": n_all / e2e_pinned, "unit": UNIT, "h2d_bytes_per_step": h2d_all,
                "d2h_bytes_per_step": d2h_all, "inputs": "pinned host arrays",
                "ms_per_step": 1e3 * e2e_pinned},
        "e2e_pageable": {"value": n_all / e2e_pageable, "unit": UNIT,
                         "inputs": "pageable numpy arrays", "ms_per_step": 1e3 * e2e_pageable},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": kern[dom]["frac"],
                     "traffic": traffic, "algorithmic_bytes_per_launch":
                         kern[dom]["bytes_per_launch"], "bytes_source": kern[dom]["bytes_source"],
                     "scope": "rank 0's launch"},
        "roofline_k123": k123,
        "kernels": {k: kern[k] for k in sorted(kern, key=lambda k: -kern[k]["share"])[:10]},
        "gpu_launches": launches_all,
        "phases_ms": {k: stats[k] for k in ("ms_ingest", "ms_fresh", "ms_fast", "ms_chain",
                                            "ms_expand")},
        "path": {"fast_shards": stats["fast_shards"], "batches_per_step": batches_all // args.steps,
                 "chain_events": stats["chain_events"]},
        "parity": f"bit-exact vs oracle/symoracle.c on every sub-cluster of every rank "
                  f"({n_all} requests, 5 per-request arrays)",
        "clocks": clk.summary(),
        "wall_ms_per_step": 1e3 * wall / args.steps,
        "cluster": dict(cstats, summary_allreduce_ms=red_ms,
                        scope="all 8 sub-clusters, window [10%, 90%) of the trace"),
    }
    if world > 1:
        line["nccl_world"] = dist.get_world_size()
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = {"value": n / ref_s, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"all {len(per)} sub-clusters, full {args.duration:g} s "
                                          f"trace ({n} requests), oracle/symoracle.c, one host "
                                          "thread per sub-cluster (the parity run above)"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--duration", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank, world, local_rank = dist_env()
    if args.gpus not in (1, 2, 4, 8):
        raise SystemExit("C4 has 8 sub-clusters: --gpus must be 1, 2, 4 or 8")
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus={args.gpus}: launch N>1 with "
                         "torch.distributed.run --nproc-per-node N")
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        print(f"[rank {rank}] NCCL communicator size {dist.get_world_size()}", file=sys.stderr)
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
