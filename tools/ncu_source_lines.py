"""Map ncu SASS-level stall samples to CUDA source lines via nvdisasm line info
(dev tool): python tools/ncu_source_lines.py <kernel> <sass.csv> [top]"""
import csv, re, sys, collections
sass = open("/tmp/dev/cubin/all.sass").read().splitlines()
fn = sys.argv[1]
# collect line info for the function section
mangled = f"{len(fn)}{fn}E"  # exact Itanium-mangled function name component
start = next(i for i, l in enumerate(sass) if l.startswith("//---") and ".text." in l and mangled in l)
end = next((i for i in range(start + 1, len(sass)) if sass[i].startswith("//---")), len(sass))
cur = None; off2line = {}
for l in sass[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        inl = re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))
        cur = (m.group(1).split("/")[-1] + ":" + m.group(2), tuple(f.split("/")[-1] + ":" + n for f, n in inl[:2]))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sys.argv[2])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
ia = hdr.index("Address"); isamp = hdr.index("Warp Stall Sampling (All Samples)"); iex = hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
agg = collections.Counter(); ex = collections.Counter(); agg_ctx = collections.Counter()
seen = set()
for r in data:
    a = int(r[ia], 16)
    if a in seen: continue
    seen.add(a)
    ln = off2line.get(a - base, ("?", ()))
    s = float(r[isamp] or 0)
    agg[ln[0]] += s; ex[ln[0]] += float(r[iex] or 0)
    agg_ctx[(ln[0],) + ln[1][:1]] += s
tot = sum(agg.values())
print("total samples", tot)
for k, v in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{100*v/tot:5.1f}%  exec={ex[k]:10.0f}  {k}")
print("--- with first inline context")
for k, v in agg_ctx.most_common(25):
    print(f"{100*v/tot:5.1f}%  {k}")
