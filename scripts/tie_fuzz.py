"""Dev tool: configs with round engine coefficients make EndForward / decode-step
ties at equal ns common; report which ones need the two-warp replica's one-warp
rerun (kErrSplitTie) and check them against the compiled reference."""
import copy, json, os, subprocess, sys
sys.path.insert(0, '.')
import numpy as np

def cfg(t, rng):
    from tests.common import CASES
    c = copy.deepcopy(CASES["decode_dp32"])
    c["workload"]["duration_s"] = 20.0
    c["workload"]["rate_qps"] = float(rng.choice([5, 20, 50]))
    c["cluster"]["l_net_s"] = 0.0
    c["cluster"]["engine"] = {"prefill_base_s": 0.01, "prefill_per_token_s": 0.0, "decode_base_s": 0.01,
                              "decode_per_request_s": 0.0, "decode_per_kv_token_s": 0.0}
    c["cluster"]["dp_degree"] = int(rng.choice([1, 2, 4]))
    c["cluster"]["dp_degree_decode"] = int(rng.choice([1, 4, 32]))
    c["workload"]["output"] = {"dist": "uniform", "min": 2, "max": int(rng.choice([3, 10, 50]))}
    c["workload"]["prompt"] = {"dist": "uniform", "min": 10, "max": 100}
    c["sim"]["seed"] = int(rng.integers(0, 10**6))
    return c

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import paper_2512_16134_b200 as P
    from oracle import ref
    c = json.loads(sys.argv[2])
    g = P.run_experiment(c, per_request=True)
    r = ref.run(c, per_request=True)
    ok = all(np.array_equal(g["requests"][k], r["requests"][:, i])
             for k, i in (("dispatch", 4), ("prefill_start", 5), ("first_token", 6), ("completion", 7)))
    print("OK" if ok else "DIFF")
    sys.exit(0)
rng = np.random.default_rng(5)
ties = []
for t in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    c = cfg(t, rng)
    p = subprocess.run([sys.executable, __file__, "--one", json.dumps(c)], capture_output=True, text=True,
                       env=dict(os.environ, SBS_DEBUG="1"), timeout=120)
    tie = "split ties" in p.stderr
    print(t, p.stdout.strip(), "TIE-RERUN" if tie else "", flush=True)
    if tie: ties.append(c)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(ties, open("gpurun_out/tie_configs.json", "w"), indent=1)
