"""Dev fuzz: random configurations over every feature (policies, decode
policies, faults, caps, tps, cache-aware PBAA, shared prefixes, multi-instance
pools), GPU default path vs the compiled reference, per request.
Usage: fuzz_all.py N SEED"""
import copy, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2512_16134_b200 as P
from oracle import ref
from tests.common import CASES

N = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for t in range(N):
    base = ["short_3k", "decode_dp32", "cfg2_20s", "oracle_n8", "cache_short", "cache_pd"][t % 6]
    c = copy.deepcopy(CASES[base])
    cl, wl = c["cluster"], c["workload"]
    Pn, Dn = int(rng.integers(1, 6)), int(rng.integers(1, 4))
    cl.update({"n_instances_prefill": Pn, "n_instances_decode": Dn,
               "dp_degree": int(rng.choice([1, 2, 3, 8, 17, 40])),
               "dp_degree_decode": int(rng.choice([1, 4, 32, 100])),
               "l_net_s": float(rng.choice([0.0, 0.001, 0.01])),
               "n_limit": int(rng.choice([0, 1, 3, 64])),
               "decode_max_batch_per_dp": int(rng.choice([0, 0, 2, 30])),
               "decode_tokens_per_step": int(rng.choice([1, 1, 3]))})
    wl["duration_s"] = float(rng.uniform(2, 12))
    wl["rate_qps"] = float(wl.get("rate_qps", 10) * rng.uniform(0.3, 2.0))
    if rng.random() < 0.3:
        wl["initial_burst"] = int(rng.integers(1, 200))
    c["scheduler"]["policy"] = str(rng.choice(["sbs", "sbs", "immediate", "round_robin", "least_outstanding"]))
    c["scheduler"]["decode_policy"] = str(rng.choice(["iqr", "iqr", "random", "round_robin"]))
    c["sim"]["seed"] = int(rng.integers(0, 10**6))
    dur = wl["duration_s"]
    f = {}
    if rng.random() < 0.4:
        f["topology"] = [{"instance": int(rng.integers(0, Pn + Dn)), "time_s": float(rng.uniform(0, dur)),
                          "healthy": bool(rng.random() < 0.5)} for _ in range(int(rng.integers(1, 4)))]
    if rng.random() < 0.3:
        f["dead"] = [{"instance": int(rng.integers(0, Pn + Dn)), "time_s": float(rng.uniform(0, dur))}]
    if rng.random() < 0.3:
        f["drop_end_forward"] = [{"instance": int(rng.integers(-1, Pn)), "from_s": float(rng.uniform(0, dur / 2)),
                                  "until_s": float(rng.uniform(dur / 2, dur))}]
    if f:
        c["faults"] = f
    try:
        g = P.run_experiment(c, per_request=True)
    except P.ConfigError as e:
        print(t, "config", e); continue
    r = ref.run(c, per_request=True)
    rq = r["requests"]
    ok = all(np.array_equal(np.asarray(g["requests"][k], np.int64), rq[:, i]) for k, i in
             (("status", 3), ("dispatch", 4), ("prefill_start", 5), ("first_token", 6), ("completion", 7)))
    for k in ("completed", "throttled", "passes", "decode_steps", "output_tokens", "deferrals",
              "mask_events", "fallback_events", "watchdog_fires", "dropped_end_forwards"):
        ok = ok and int(g["agg"][k]) == int(r["agg"][k])
    print(t, "OK" if ok else "DIFF", base, c["scheduler"], Pn, Dn, flush=True)
    bad += not ok
print("bad", bad, "of", N)
