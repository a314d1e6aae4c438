"""Small multi-case run for compute-sanitizer (dev tool)."""
import sys
sys.path.insert(0, '.')
import paper_2512_16134_b200 as P
from tests.common import CASES
names = ["short_3k", "decode_dp32", "faults_prefill", "faults_decode_capped_tps3", "oracle_n8",
         "cfg3_seed11_150s_random", "overload_dp1"]
pts = [P.experiment_from_config(CASES[n]) for n in names]
trs = [P.generate_workload(p) for p in pts]
sim = P.Simulator(pts, trs, per_request=True, logs=True)
sim.launch()
res = sim.results()
print([r["completed"] for r in res], [r["error"] for r in res])
w = P.allocate_batch([{"pending": [[0, 500, 0]], "new": [[1, 900, 0], [2, 7, 0]], "caps": [1000, 3],
                       "n_limit": 8}])
pos, fb, th = P.select_decode_unit([([0, 1, 0, 2], [10, 10, 10, 100])])
print("ok", w[0]["mapping"].tolist(), pos.tolist())
