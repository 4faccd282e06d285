"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_* --csv` launch list
per kernel (dev tool): python tools/ncu_launches.py launches.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; per = collections.defaultdict(dict); order = []
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")[:40])
        v = float(d["Metric Value"].replace(",", "")); u = d.get("Metric Unit", "")
        scale = {"ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        per[key][d["Metric Name"]] = v * scale
        if key not in order: order.append(key)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for k in order:
    a = agg[k[1]]; a[0] += 1; t = per[k].get("gpu__time_duration.sum", 0); a[1] += t; a[3] = max(a[3], t)
    a[2] += per[k].get("dram__bytes_read.sum", 0) + per[k].get("dram__bytes_write.sum", 0)
tot = sum(v[1] for v in agg.values())
print(f"total kernel time {tot/1e3:.3f} ms over {len(order)} launches")
for k, (c, us, b, mx) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k:40s} n={c:3d} ms={us/1e3:9.3f} max={mx/1e3:8.3f} share={100*us/tot:5.1f}%  dram={b/1e6:9.1f} MB  GB/s={b/us/1e3 if us else 0:8.1f}")
