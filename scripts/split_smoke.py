"""Quick split-mode parity on a few golden cases (dev tool)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2512_16134_b200 as P
from tests.common import CASES, load_case
names = sys.argv[1:] or ["decode_dp32", "short_3k", "cfg2_20s"]
for n in names:
    t0 = time.time()
    g = P.run_experiment(CASES[n], per_request=True)
    want = load_case(n)
    bad = [c for c in ("dispatch", "prefill_start", "first_token", "completion") if not np.array_equal(g["requests"][c], want[c])]
    print(n, "OK" if not bad else f"BAD {bad}", "err", g["agg"]["error"], f"{time.time()-t0:.2f}s", flush=True)
