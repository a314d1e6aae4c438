"""Dev fuzz: multi-instance decode pools with topology/dead faults, batch caps
and tps > 1, GPU (default two-warp replicas) vs the compiled reference."""
import copy, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2512_16134_b200 as P
from oracle import ref
from tests.common import CASES
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
for t in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    c = copy.deepcopy(CASES[["decode_dp32", "cfg2_20s"][t % 2]])
    Pn = int(rng.integers(1, 4)); Dn = int(rng.choice([2, 3, 5]))
    c["cluster"]["n_instances_prefill"] = Pn
    c["cluster"]["n_instances_decode"] = Dn
    c["cluster"]["dp_degree_decode"] = int(rng.choice([4, 16, 40]))
    c["cluster"]["decode_max_batch_per_dp"] = int(rng.choice([0, 3, 20]))
    c["cluster"]["decode_tokens_per_step"] = int(rng.choice([1, 2, 5]))
    c["workload"]["duration_s"] = float(rng.uniform(5, 25))
    c["scheduler"]["decode_policy"] = str(rng.choice(["iqr", "iqr", "random", "round_robin"]))
    c["sim"]["seed"] = int(rng.integers(0, 10**6))
    dur = c["workload"]["duration_s"]
    f = {"topology": [], "dead": []}
    for k in range(int(rng.integers(0, 4))):
        inst = int(rng.integers(0, Pn + Dn))
        f["topology"].append({"instance": inst, "time_s": float(rng.uniform(0, dur)), "healthy": bool(rng.random() < 0.5)})
    if rng.random() < 0.5:
        f["dead"].append({"instance": int(rng.integers(Pn, Pn + Dn)), "time_s": float(rng.uniform(0, dur))})
    c["faults"] = f
    g = P.run_experiment(c, per_request=True)
    r = ref.run(c, per_request=True)
    rq = r["requests"]
    ok = all(np.array_equal(g["requests"][k], rq[:, i]) for k, i in
             (("dispatch", 4), ("prefill_start", 5), ("first_token", 6), ("completion", 7)))
    ok = ok and np.array_equal(g["requests"]["status"], rq[:, 3].astype(np.int8))
    ok = ok and int(g["agg"]["decode_steps"]) == int(r["agg"]["decode_steps"])
    print(t, "OK" if ok else "DIFF", Pn, Dn, c["scheduler"]["decode_policy"], flush=True)
    bad += not ok
print("bad", bad)
