"""Benchmark: requests scheduled per second (device-timed) on the C4 workload.

Workload (BASELINE.json configs[3]): 1000 A100-zoo models x
8192 simulated GPUs, Poisson 1.2M req/s aggregate over a 60 s trace, seed 42,
partitioned into P=8 sub-clusters of 125 contiguous models and 1024 GPUs
("models sharded across 8xB200").  Rank r of N runs sub-cluster r, so the
per-GPU work is fixed (weak scaling) and N=8 is exactly C4 on 8 B200s.

A step is one pass of the hot path over the rank's whole sub-cluster trace
(~9.0M requests): ingest -> fresh-start pre-scan -> batch chains ->
per-request RunResult arrays, inputs resident in HBM (the parallel
validated fast path resolves the sub-cluster; the sequential live-event
chain takes over for any sub-cluster that fails validation).  `value` is the
whole-job throughput; `e2e` is the same metric through the public API
(Engine.run_stream: host arrays in, RunResult out, H2D/D2H inside).

--impl reference times the reference algorithm's CPU restatement
(oracle/, a C port of batchsym's event loop) on the host cores over the
same sub-clusters.
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
FRESH_REC_BYTES = 128  # sizeof(FreshRec)
BATCH_REC_BYTES = 64   # sizeof(BatchRec) / sizeof(sym_batch)
EV_BATCH_BYTES = 56    # sizeof(EvBatch)


def algorithmic_bytes(kernel: str, n: int, nb: int, shards: int = 1) -> float | None:
    """Minimal DRAM bytes one launch of `kernel` must move for n requests and
    nb batches over `shards` sub-clusters (DESIGN.md §5 derives each line)."""
    table = {
        # stable partition: read tick+model, write s_tick, s_i, the inverse
        # map, the model slot and the batch-id reset; with several shards
        # also the shard-stream index s_g and the shard-ordered ticks sh_tick
        # (one shard: those alias s_i and the input ticks)
        "k_scatter": n * (8 + 4 + 8 + 4 + 4 + 4 + 4 + (4 + 8 if shards > 1 else 0)),
        "k_hist": n * 4,
        "k_aself": n * (4 + 8 + 8 + 4),
        # fresh-start pre-scan: read each sorted arrival once (tick, A', g),
        # write one FreshRec and one chain pointer per position
        "k_fresh": n * (8 + 4 + 4 + FRESH_REC_BYTES + 4),
        # lean chain pointer: each sorted tick read once (neighbours share
        # the line), one 4-byte pointer written per position
        "k_nxt": n * (8 + 4),
        "k_nxt_pp": n * (8 + 4 + 4),
        "k_nxt_general": n * 4,
        # batch records from the chain positions' fresh scans: the members'
        # ticks/ids once, one EvBatch written per batch
        "k_chain_recs": n * (8 + 4 + 4) + nb * (4 + EV_BATCH_BYTES + 8 + 4),
        "k_walk": 0,
        # match + pointer jumping (~log2(nb/G) rounds) + tie repair, one launch
        "k_match_coop": nb * (8 + 4 + 4 + 4) + nb * 12 * 12,
        "k_token_keys": nb * (4 + 8 + EV_BATCH_BYTES + 8 + 4),
        # J_4k = (J_k)^4: read own pointer, one write; the three gathers
        # re-read the same 4n-byte array, which L2 holds, so they are not
        # counted as DRAM bytes
        "k_jump4": n * (4 + 4),
        # stable merge-path round over the batch runs: read and write key+value
        "k_merge_round": nb * (12 + 12),
        "k_walk_expand": nb * (FRESH_REC_BYTES + 4 + EV_BATCH_BYTES),
        "k_rscatter": nb * (12 + 12),
        "k_rhist": nb * 8,
        "k_scan_up": None, "k_scan_mid": None, "k_scan_down": None,
        "k_fast_emit": nb * (EV_BATCH_BYTES + 12 + 4 + 8 + BATCH_REC_BYTES),
        # per-request RunResult arrays from batch records
        "k_fill32": n * 4,
        "k_bid": nb * BATCH_REC_BYTES + n * 4,
        # one thread per request: inverse map, batch id, tick, model read,
        # five int64 written coalesced; batch records read once
        "k_out": n * (4 + 4 + 8 + 4 + 5 * 8) + nb * BATCH_REC_BYTES,
        "k_copy_batches": nb * (BATCH_REC_BYTES + 4 + 64),
    }
    return table.get(kernel)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def build_workload(duration_s: float, shard: int):
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(duration_s)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], duration_s,
                                    configs.SEED)
    ms, gpus, ids = configs.shard_scenarios(sc)[shard]
    sel = (midx >= ids[0]) & (midx <= ids[-1])
    return sc, list(ms), gpus, np.ascontiguousarray(ticks[sel]), \
        np.ascontiguousarray(midx[sel] - ids[0])


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

    def start(self):
        self.__enter__()
        time.sleep(1.0)  # nvidia-smi start-up; sampling is running before timing

    def stop(self):
        self.__exit__(None, None, None)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
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
        for ln in getattr(self, "lines", []):
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
        return 6650.0, "fallback"


def oracle_shard_run(ms, gpus, policy, ticks, midx):
    from oracle import oracle
    stride = max(m.profile.max_batch for m in ms)
    return oracle.run(np.stack([m.profile.table_array(stride) for m in ms]),
                      [m.profile.max_batch for m in ms], [m.slo_ns for m in ms],
                      [policy.resolve_timeout_ns(m.slo_ns) for m in ms], gpus, ticks, midx,
                      kind=policy.kind, gather=policy.gather,
                      target_batch=policy.target_batch, d_ctrl_ns=policy.d_ctrl_ns,
                      d_data_ns=policy.d_data_ns)


REF_BUDGET_S = 120.0


def run_reference(args, world):
    """CPU arm: the oracle port over every rank's sub-cluster, one thread
    per sub-cluster (scalebench.bench_workers' process-per-shard layout)."""
    from concurrent.futures import ThreadPoolExecutor
    # Bounded sample: a shorter prefix of the same trace when many steps are
    # asked for, so the whole arm stays near REF_BUDGET_S.  The port's speed
    # on this host is calibrated on one second of the trace first.
    cores = min(world, len(os.sched_getaffinity(0)))
    waves = -(-world // cores)
    cal = build_workload(1.0, 0)
    t0 = time.perf_counter()
    oracle_shard_run(cal[1], cal[2], cal[0].policy, cal[3], cal[4])
    per_trace_s = (time.perf_counter() - t0) * waves  # step seconds per trace second
    dur = round(min(args.duration, max(1.0, REF_BUDGET_S / (per_trace_s * (args.steps + args.warmup)))), 2)
    work = [build_workload(dur, s) for s in range(world)]
    n_total = sum(len(w[3]) for w in work)

    def one_step():
        with ThreadPoolExecutor(cores) as ex:
            list(ex.map(lambda w: oracle_shard_run(w[1], w[2], w[0].policy, w[3], w[4]), work))

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    el = time.perf_counter() - t0
    value = n_total * args.steps / el
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"C4 sub-clusters 0..{world - 1} (125 models x 1024 GPUs each, "
                               f"Poisson 150k req/s each, {dur:g} s of the seed-42 trace)",
                   "requests_per_step": n_total, "policy": "deferred"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"first {dur:g} s of the {args.duration:g} s trace of {world} "
                                   "sub-cluster(s) per step, oracle/symoracle.c (C restatement "
                                   "of batchsym's loop), one thread per sub-cluster"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2308_07470_b200.simulator import Engine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    sc, ms, gpus, ticks, midx = build_workload(args.duration, rank)
    n = len(ticks)
    eng = Engine(ms, gpus, sc.policy, device=local_rank)
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
    if True:
        t0 = time.perf_counter()
        w0 = time.time()
        for _ in range(args.steps):
            flush.fill_(1)
            _, cnt = eng.run_device(t_dev, m_dev, outs)
            dev_ms += cnt["ms_total"]
            batches += cnt["n_batches"]
            launches += cnt["launches"] + 1  # + the L2 flush
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        clk.window = (w0, time.time())
    clk.stop()
    if world > 1:
        dist.barrier()
    stats = dict(cnt)
    # per-kernel device time: the same K steps again with every launch
    # bracketed by CUDA events on the engine's stream
    eng.kernel_times(reset=True)
    for _ in range(args.steps):
        flush.fill_(1)
        eng.run_device(t_dev, m_dev, outs, kernel_times=True)
    ktimes = eng.kernel_times(reset=True)

    # end to end through the public API: pinned host arrays in, RunResult out
    # (steady state: two untimed calls warm the pinned-memory pool, and each
    # result is released before the next call, as a streaming caller would)
    pin_t = torch.from_numpy(ticks).pin_memory().numpy()
    pin_m = torch.from_numpy(midx).pin_memory().numpy()
    for _ in range(2):
        eng.run_stream(pin_t, pin_m, args.duration)
    e2e_s = []
    res = None
    for _ in range(max(3, min(args.steps, 10))):
        res = None
        t0 = time.perf_counter()
        res = eng.run_stream(pin_t, pin_m, args.duration)
        e2e_s.append(time.perf_counter() - t0)
    e2e_time = sum(e2e_s) / len(e2e_s)
    h2d = n * (8 + 8)                      # ticks + int64 model ids
    # six computed RunResult arrays + batch records cross PCIe; req_arrival and
    # req_model (copies of the inputs) are filled by a host thread meanwhile
    d2h = n * 6 * 8 + len(res.batches) * BATCH_REC_BYTES

    # parity spot check of the timed outputs against the API result
    for k, ref in (("batch", res.req_batch), ("outcome", res.req_outcome)):
        if not np.array_equal(outs[k].cpu().numpy(), ref):
            raise SystemExit(f"device-resident and API outputs differ on {k}")

    # end of run: the one collective -- per-sub-cluster integer summaries
    # reduced over NCCL into the cluster's goodput / idle / autoscale view
    from paper_2308_07470_b200.parallel import SummaryLayout, cluster_stats, reduce_summaries
    layout = SummaryLayout(len(sc.models), sc.gpu_count)
    lo, hi = int(0.1 * args.duration * 1e9), int(0.9 * args.duration * 1e9)
    ids = np.arange(125 * rank, 125 * (rank + 1))
    vec = layout.empty()
    layout.put(vec, ids, np.arange(1024 * rank, 1024 * (rank + 1)), eng.window_counts(lo, hi))
    t_red = time.perf_counter()
    vec = reduce_summaries(vec)
    red_ms = 1e3 * (time.perf_counter() - t_red)
    world_layout = SummaryLayout(125 * world, 1024 * world)
    cstats = cluster_stats(np.concatenate([vec[k * layout.M:k * layout.M + 125 * world]
                                           for k in range(4)] + [vec[4 * layout.M:4 * layout.M
                                                                      + 1024 * world]]),
                           world_layout, lo, hi)
    t = torch.tensor([dev_ms, e2e_time, wall], dtype=torch.float64, device=dev)
    tot = torch.tensor([n, batches], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    dev_ms, e2e_time, wall = t.tolist()
    n_all = int(tot[0].item())
    if rank != 0:
        return
    value = n_all * args.steps / (dev_ms / 1e3)
    peak, peak_kind = measured_peak_hbm()
    nb_step = batches // args.steps
    kern = {}
    k_total = sum(v[1] for v in ktimes.values())
    for name, (cnt_l, k_ms) in ktimes.items():
        per_launch_ms = k_ms / cnt_l
        ab = algorithmic_bytes(name, n, nb_step)
        kern[name] = {"launches_per_step": cnt_l / args.steps, "ms_per_launch": per_launch_ms,
                      "share": k_ms / k_total,
                      "gbs": (ab / (per_launch_ms / 1e3) / 1e9) if ab else None}
    dom = max(kern, key=lambda k: kern[k]["ms_per_launch"] * kern[k]["launches_per_step"])
    ab = algorithmic_bytes(dom, n, nb_step)
    achieved = kern[dom]["gbs"]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get("kernels", {}).get(dom, {}).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"C4: 1000 A100-zoo models x 8192 GPUs, Poisson 1.2M req/s, "
                               f"{args.duration:g} s trace, seed 42, 8 sub-clusters of 125 "
                               f"models x 1024 GPUs; rank r runs sub-cluster r",
                   "requests_per_step": n_all, "policy": "deferred", "max_batch": 256,
                   "l2": "256 MB flush written before every step",
                   "parallelism": f"sub-cluster-per-gpu x{world}"},
        "e2e": {"value": n_all / e2e_time, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": d2h * world},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "algorithmic_bytes_per_launch": ab},
        "kernels": {k: kern[k] for k in sorted(kern, key=lambda k: -kern[k]["share"])[:8]},
        "gpu_launches": launches,
        "phases_ms": {k: stats[k] for k in ("ms_ingest", "ms_fresh", "ms_fast", "ms_chain",
                                            "ms_expand")},
        "path": {"fast_shards": stats["fast_shards"], "batches": stats["n_batches"],
                 "chain_events": stats["chain_events"]},
        "clocks": clk.summary(),
        "wall_ms_per_step": 1e3 * wall / args.steps,
        "cluster": dict(cstats, summary_allreduce_ms=red_ms,
                        scope=f"sub-clusters 0..{world - 1}, window [10%, 90%) of the trace"),
    }
    if world == 1 and not args.no_cpu_baseline:
        t0 = time.perf_counter()
        oracle_shard_run(ms, gpus, sc.policy, ticks, midx)
        el = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n / el, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"sub-cluster 0, full {args.duration:g} s trace "
                                          f"({n} requests), oracle/symoracle.c single thread"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--duration", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank, world, local_rank = dist_env()
    if world != args.gpus and world != 1:
        print(f"warning: WORLD_SIZE={world} but --gpus={args.gpus}", file=sys.stderr)
    world = max(world, 1)
    if args.gpus > 8:
        raise SystemExit("C4 has 8 sub-clusters: at most 8 GPUs")
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, max(world, args.gpus))
        return
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
