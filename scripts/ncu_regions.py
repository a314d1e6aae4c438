"""Group ncu cuda,sass per-line samples into des.cu regions (dev tool)."""
import csv, re, sys
from collections import defaultdict
src = open(sys.argv[2]).read().splitlines()
regions = []
for i, l in enumerate(src, 1):
    m = re.search(r"auto (\w+) = \[&\]", l) or re.search(r"// ---- (on_\w+)", l) or re.search(r"^__global__ .*?(\w+_kernel)", l) or re.search(r"^__device__ .*? (\w+)\(", l)
    if m:
        regions.append((i, m.group(1)))
regions.sort()
def region(line):
    name = "prologue"
    for s, n in regions:
        if s <= line: name = n
    return name
rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(lambda: [0, 0]); cur = ""; hdr = None
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[2] != "-": continue
    try: ln = int(r[0])
    except ValueError: continue
    key = region(ln) if cur == "des.cu" else cur
    agg[key][0] += int(r[4] or 0); agg[key][1] += int(r[7] or 0)
ts = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:22s} samples {100*v[0]/ts:5.1f}%  inst {100*v[1]/ti:5.1f}%")
