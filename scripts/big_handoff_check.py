import copy, sys, subprocess, os, json
sys.path.insert(0, '.')
import numpy as np
import paper_2512_16134_b200 as P
from tests.common import CASES
from oracle import ref
# one EndForward finishes > 1024 decode-bound requests: tiny prompts, huge chunk
c = copy.deepcopy(CASES["decode_dp32"])
c["cluster"].update({"c_chunk": 100000, "dp_degree": 1, "n_instances_prefill": 1, "t_default_s": 0.5})
c["workload"].update({"rate_qps": 3000.0, "duration_s": 3.0, "initial_burst": 2000,
                      "prompt": {"dist": "constant", "value": 1}, "output": {"dist": "uniform", "min": 2, "max": 20}})
g = P.run_experiment(c, per_request=True)
r = ref.run(c, per_request=True)
ok = np.array_equal(g["requests"]["completion"], r["requests"][:, 7])
print("OK" if ok else "DIFF", g["agg"]["error"], g["n"])
