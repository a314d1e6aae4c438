"""Per source line of des.cu in [lo, hi]: samples and the top stall reasons
from an ncu 'cuda,sass' source CSV (dev tool).  Usage: FILE.csv SRC.cu LO HI"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
src = open(sys.argv[2]).read().splitlines()
lo, hi = int(sys.argv[3]), int(sys.argv[4])
hdr = None; cur = ""; tot = 0; out = []
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[2] != "-": continue
    try: ln = int(r[0]); s = int(r[4] or 0)
    except ValueError: continue
    tot += s
    if cur != "des.cu" or not (lo <= ln <= hi): continue
    st = {hdr[i].replace("stall_", ""): int(r[i] or 0) for i in range(len(hdr))
          if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i] not in ("", "0")}
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    out.append((ln, s, int(r[7] or 0), top))
ssum = sum(o[1] for o in out)
print(f"lines {lo}-{hi}: {100*ssum/tot:.1f}% of all samples")
for ln, s, inst, top in out:
    if s * 400 < ssum: continue
    print(f"{ln:5d} {100*s/tot:5.2f}% inst {inst:>11d}  " + " ".join(f"{k}={100*v/max(s,1):.0f}%" for k, v in top)
          + "  | " + src[ln - 1].strip()[:70])
