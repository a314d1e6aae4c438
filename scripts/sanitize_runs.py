"""compute-sanitizer driver (dev tool; logs committed under profiles/).

Runs three golden decode cases through the two-warp replicas (SBS_SPLIT=2:
des_cluster_kernel, SBS_SPLIT=1: des_split_kernel), in parity mode, checks the
per-request timestamps against the committed reference fixtures, then one
small batch through each allocation kernel (pbaa register + shared-memory
paths, iqr register + shared-memory paths, sched) and device trace generation.
Usage (under compute-sanitizer): python scripts/sanitize_runs.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2512_16134_b200 as P  # noqa: E402
from tests.common import CASES, GOLD  # noqa: E402

names = ["cfg2_20s", "faults_decode_capped_tps3", "decode_dp32_random"]
pts = [P.experiment_from_config(CASES[n]) for n in names]
trs = [P.generate_workload(p) for p in pts]
sim = P.Simulator(pts, trs, per_request=True)
sim.launch()
res = sim.results()
for i, n in enumerate(names):
    fx = np.load(GOLD / f"sim_{n}.npz")
    rq = sim.requests(i)
    for col in ("dispatch", "prefill_start", "first_token", "completion"):
        assert np.array_equal(rq[col], fx[col]), (n, col)
print("des ok", [r["completed"] for r in res], [r["error"] for r in res])
rng = np.random.default_rng(1)
wins = []
for t in range(64):
    k = int(rng.integers(0, 80 if t % 2 else 20))
    D = int(rng.integers(1, 40 if t % 2 else 9))
    rows = [[int(i), int(rng.integers(1, 3000)), int(rng.integers(0, 3))] for i in range(k)]
    wins.append({"pending": rows[: k // 3], "new": rows[k // 3:],
                 "caps": rng.integers(-100, 3000, D).tolist(), "n_limit": 2})
P.allocate_batch(wins)
calls = [(rng.integers(0, 3, U), rng.integers(0, 5000, U)) for U in (1, 7, 32, 320, 700)]
P.select_decode_unit(calls)
P.schedule_decode_batch([([[1, 900, 500], [2, 700, 300]], [0, 1, 0], [100, 900, 50])])
g = P.generate_workload_device([P.experiment_from_config(CASES["decode_dp32"])]) \
    if hasattr(P, "generate_workload_device") else None
print("alloc ok", g is not None)
