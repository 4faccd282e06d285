"""Summarise ncu --set full reports into profiles/ncu_summary.json (dev tool):
python tools/ncu_summary.py out.json [--workload W --n-gpus N] report1.ncu-rep [...]
bench.py reads dram_bytes_per_launch of its dominant kernel from the summary
when workload / n_gpus match its own line."""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
        "sm__inst_executed.avg.per_cycle_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")
        name = name.replace("void ", "").split("<")[0].strip()  # k_part<1>, <2> -> k_part
        launch = out.setdefault(name, {"_launches": []})["_launches"]
        d = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                try:
                    d[w] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
        t = d.get("gpu__time_duration.sum", 0)
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        launch.append({"duration_us": round(t * 1e6, 1), "dram_bytes_per_launch": int(b),
                     "dram_gbs_cold": round(b / t / 1e9, 1) if t else None,
                     "dram_pct_peak": d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                     "sm_pct_peak": d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                     "ipc": d.get("sm__inst_executed.avg.per_cycle_elapsed"),
                     "l1_hit_pct": d.get("l1tex__t_sector_hit_rate.pct"),
                     "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"),
                     "ld_sectors_per_request": (d["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"] /
                                                d["l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"])
                     if d.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum") else None,
                     "stall_long_scoreboard": d.get("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
                     "stall_lg_throttle": d.get("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"),
                     "registers": d.get("launch__registers_per_thread"),
                     "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size")})
    # one entry per kernel: the mean over its captured launches (k_part runs
    # twice per step with several sub-clusters), every launch kept
    res = {}
    for name, v in out.items():
        ls = v["_launches"]
        first = dict(ls[0])
        first["duration_us"] = round(sum(x["duration_us"] for x in ls) / len(ls), 1)
        first["dram_bytes_per_launch"] = int(sum(x["dram_bytes_per_launch"] for x in ls) / len(ls))
        first["launches_captured"] = len(ls)
        if len(ls) > 1:
            first["per_launch"] = ls
        res[name] = first
    return res


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--workload", default=None)
    ap.add_argument("--n-gpus", type=int, default=1)
    a = ap.parse_args()
    res = {}
    for p in a.reports:
        res.update(summarize(p))
    for k, v in res.items():
        print(k, json.dumps(v))
    doc = {"workload": a.workload, "n_gpus": a.n_gpus, "reports": a.reports, "kernels": res}
    json.dump(doc, open(a.out, "w"), indent=1)
