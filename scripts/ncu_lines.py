"""Summarise an ncu 'cuda,sass' source CSV per CUDA source line: instructions
executed and warp-stall samples (dev tool)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(lambda: [0, 0, 0, ""])
hdr = None
cur_file = ""
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    key = (cur_file, line)
    a = agg[key]
    a[0] += int(r[4] or 0)   # stall samples (all)
    a[1] += int(r[7] or 0)   # instructions executed (warp-level)
    a[3] = r[1][:90]
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
by = sys.argv[2] if len(sys.argv) > 2 else "samples"
idx = 0 if by == "samples" else 1
print(f"total samples {tot_s}  total warp-inst {tot_i}")
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][idx])[: int(sys.argv[3]) if len(sys.argv) > 3 else 45]:
    print(f"{f}:{ln:5d} samp {100*v[0]/tot_s:5.1f}%  inst {100*v[1]/tot_i:5.1f}%  {v[3]}")
