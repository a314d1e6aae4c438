"""Dev tool: split modes vs serial on random configs, one subprocess per case
(so a hang is attributed).  Usage: split_fuzz.py MODE N [SEED]"""
import copy, json, os, subprocess, sys
sys.path.insert(0, '.')
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import paper_2512_16134_b200 as P
    c = json.loads(sys.argv[2])
    g = P.run_experiment(c, per_request=True)
    print(json.dumps({"err": int(g["agg"]["error"]), "digest": int(sum(int(x) for x in g["requests"]["completion"][:50000:7])),
                      "tpot": float(g["agg"].get("tpot_mean_s", 0) or 0), "done": int(g["agg"]["completed"])}))
    sys.exit(0)
from tests.common import CASES
mode, n = sys.argv[1], int(sys.argv[2])
rng = np.random.default_rng(int(sys.argv[3]) if len(sys.argv) > 3 else 77)
for t in range(n):
    c = copy.deepcopy(CASES[["decode_dp32", "cfg2_20s"][t % 2]])
    c["workload"]["duration_s"] = float(rng.uniform(3, 20))
    c["workload"]["rate_qps"] = float(c["workload"].get("rate_qps", 10) * rng.uniform(0.5, 2.5))
    c["cluster"]["dp_degree"] = int(rng.choice([1, 4, 17, 64]))
    c["cluster"]["l_net_s"] = float(rng.choice([0.0, 0.001, 0.02]))
    c["scheduler"]["decode_policy"] = str(rng.choice(["iqr", "random", "round_robin"]))
    c["sim"]["seed"] = int(rng.integers(0, 10**6))
    outs = []
    for m in ("0", mode):
        try:
            r = subprocess.run([sys.executable, __file__, "--one", json.dumps(c)], capture_output=True, text=True,
                               timeout=60, env=dict(os.environ, SBS_SPLIT=m))
            outs.append(r.stdout.strip().splitlines()[-1] if r.returncode == 0 else "RC%d %s" % (r.returncode, r.stderr[-300:]))
        except subprocess.TimeoutExpired:
            outs.append("HANG")
    print(t, "OK" if outs[0] == outs[1] else "DIFF", c["cluster"]["dp_degree"], c["scheduler"]["decode_policy"],
          outs if outs[0] != outs[1] else "", flush=True)
