"""Static SASS size per des.cu region for one kernel (nvdisasm -g output). Dev tool."""
import re, sys
from collections import Counter
sass, src, fn = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(src).read().splitlines()
regions = []
for i, l in enumerate(lines, 1):
    m = re.search(r"auto (\w+) = \[&\]", l) or re.search(r"// ---- (on_\w+|decode hand-off|prefill passes)", l) or re.search(r"^__global__ .*?(\w+_kernel)", l) or re.search(r"^__device__ .*? (\w+)\(", l) or re.search(r"// (event loop)", l)
    if m: regions.append((i, m.group(1)))
def region(ln):
    name = "prologue"
    for s, n in regions:
        if s <= ln: name = n
    return name
cnt = Counter(); infn = False; cur = "?"
for l in open(sass):
    if l.startswith("\t.text.") or ".section" in l and ".text." in l:
        infn = fn in l
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        f, ln = m.group(1), int(m.group(2))
        cur = region(ln) if f.endswith("des.cu") else f.split("/")[-1]
        continue
    if infn and re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l):
        cnt[cur] += 1
tot = sum(cnt.values())
print("total", tot)
for k, v in cnt.most_common(30):
    print(f"{k:28s} {v:6d} {100*v/tot:5.1f}%")
