"""Regenerate tests/golden/ from the compiled reference (oracle/_ref).

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
Everything here is produced by the UNMODIFIED reference sources through
oracle/ref_harness.cpp; the GPU box only reads the committed outputs.

  configs/*.json            the reference's committed scenarios (proj/configs)
  cases.json                the parity cases (name -> config)
  sim_<case>.npz            per-request dispatch/prefill_start/first_token/
                            completion/status + aggregates + digest + counts
  csv_sha256.json           sha256 of the reference's four report CSVs per case
  windows_short_3k.npz      every allocate_batch window of short_3k (inputs and
                            outputs), flat int64 records (ref_harness.cpp)
  windows_cache_aware.npz   random cache-aware windows with their Len_hit matrices
  decodes_decode_dp32.npz   every select_decode_unit call of decode_dp32
  smoke_decode_dp32_30s.npz the __graft_entry__.smoke() fixture
"""
from __future__ import annotations

import copy
import hashlib
import json
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

REF_CONFIGS = Path("/root/reference/proj/configs")


def load(name):
    return json.load(open(HERE / "configs" / f"{name}.json"))


def with_(cfg, **kw):
    c = copy.deepcopy(cfg)
    for path, v in kw.items():
        keys = path.split("__")
        d = c
        for k in keys[:-1]:
            d = d.setdefault(k, {})
        d[keys[-1]] = v
    return c


def cfg2(duration=20.0, seed=11):
    return {
        "cluster": {"n_instances_prefill": 4, "n_instances_decode": 1, "dp_degree": 8,
                    "dp_degree_decode": 320, "c_chunk": 3000, "t_default_s": 0.35, "w_size": 64,
                    "l_net_s": 0.002, "n_limit": 64,
                    "engine": {"prefill_base_s": 0.05, "prefill_per_token_s": 1e-4,
                               "decode_base_s": 0.004, "decode_per_request_s": 2e-4,
                               "decode_per_kv_token_s": 1e-6}},
        "workload": {"process": "poisson", "rate_qps": 200, "duration_s": duration,
                     "prompt": {"dist": "lognormal", "mu": 6.2, "sigma": 1.2, "min": 1, "max": 3000},
                     "output": {"dist": "lognormal", "mu": 5.0, "sigma": 0.8, "min": 1, "max": 2000}},
        "scheduler": {"policy": "sbs", "decode_policy": "iqr"},
        "sim": {"seed": seed, "warmup_fraction": 0.1},
    }


def cases():
    s3k, n8, live, d32 = load("short_3k"), load("oracle_n8"), load("liveness"), load("decode_dp32")
    cfg3 = with_(d32, workload__rate_qps=10.4, workload__duration_s=150.0,
                 workload__initial_burst=256,
                 workload__output={"dist": "lognormal", "mu": 6.5, "sigma": 1.0, "min": 1, "max": 8000},
                 sim__warmup_fraction=0.2)
    faults = with_(s3k, workload__duration_s=12.0,
                   faults={"dead": [{"instance": 2, "time_s": 4.0}],
                           "topology": [{"instance": 5, "time_s": 3.0, "healthy": False},
                                        {"instance": 5, "time_s": 7.5, "healthy": True},
                                        {"instance": 1, "time_s": 6.0, "healthy": False}],
                           "drop_end_forward": [{"instance": 3, "from_s": 2.0, "until_s": 5.0}]})
    dec_faults = with_(d32, workload__duration_s=60.0, cluster__n_instances_decode=2,
                       cluster__dp_degree_decode=16, cluster__decode_max_batch_per_dp=20,
                       cluster__decode_tokens_per_step=3,
                       faults={"dead": [{"instance": 3, "time_s": 40.0}],
                               "topology": [{"instance": 2, "time_s": 20.0, "healthy": False},
                                            {"instance": 2, "time_s": 30.0, "healthy": True}]})
    cache = {"enabled": True, "probe_lens": [64, 256, 512, 1024], "budget_tokens": 3000}
    cache_short = with_(s3k, workload__duration_s=8.0, workload__shared_prefix_fraction=0.6,
                        workload__prefix_pool=6, workload__prefix_len=1024, cluster__cache=cache,
                        scheduler__prefill_mode="cache_aware")
    cache_pd = with_(cfg2(12.0, seed=3), workload__shared_prefix_fraction=0.5,
                     workload__prefix_pool=12, workload__prefix_len=600,
                     cluster__cache={"enabled": True, "probe_lens": [32, 128, 512, 600],
                                     "budget_tokens": 1500},
                     scheduler__prefill_mode="cache_aware")
    return {
        "short_3k": s3k,
        "short_3k_immediate": with_(s3k, scheduler__policy="immediate"),
        "short_3k_least_outstanding": with_(s3k, scheduler__policy="least_outstanding"),
        "cfg1_sbs": with_(s3k, workload__duration_s=23.25),
        "cfg1_immediate": with_(s3k, workload__duration_s=23.25, scheduler__policy="immediate"),
        "oracle_n8": n8,
        "oracle_n8_immediate": with_(n8, scheduler__policy="immediate"),
        "liveness": live,
        "decode_dp32": d32,
        "decode_dp32_random": with_(d32, scheduler__decode_policy="random"),
        "decode_dp32_round_robin": with_(d32, scheduler__decode_policy="round_robin"),
        "cfg2_20s": cfg2(20.0),
        "cfg3_seed11_150s": cfg3,
        "cfg3_seed11_150s_random": with_(cfg3, scheduler__decode_policy="random"),
        "faults_prefill": faults,
        "faults_decode_capped_tps3": dec_faults,
        "overload_dp1": with_(s3k, cluster__dp_degree=1, workload__duration_s=6.0,
                              cluster__n_limit=3),
        "nlimit0": with_(s3k, cluster__dp_degree=2, workload__duration_s=4.0, cluster__n_limit=0),
        # round engine coefficients: EndForward / decode-step ties at equal ns
        # deep enough that a two-warp replica reruns on one warp (kErrSplitTie)
        "split_tie_round_coeffs": {"cluster": {"n_instances_prefill": 2, "n_instances_decode": 1, "dp_degree": 2, "dp_degree_decode": 32, "c_chunk": 4000, "t_default_s": 0.06, "w_size": 64, "l_net_s": 0.0, "n_limit": 64, "decode_max_batch_per_dp": 0, "engine": {"prefill_base_s": 0.01, "prefill_per_token_s": 0.0, "decode_base_s": 0.01, "decode_per_request_s": 0.0, "decode_per_kv_token_s": 0.0}}, "workload": {"process": "poisson", "rate_qps": 50.0, "duration_s": 20.0, "prompt": {"dist": "uniform", "min": 10, "max": 100}, "output": {"dist": "uniform", "min": 2, "max": 3}}, "scheduler": {"policy": "sbs", "decode_policy": "iqr"}, "sim": {"seed": 361518, "warmup_fraction": 0.7}},
        # cache-aware PBAA + per-DP PrefixCache
        "cache_short": cache_short,
        "cache_short_basic": with_(cache_short, scheduler__prefill_mode="basic"),
        "cache_short_tiny_budget": with_(cache_short, cluster__cache__budget_tokens=300,
                                         cluster__cache__probe_lens=[32, 128, 256, 128]),
        "cache_pd": cache_pd,
        "cache_pd_dp33": with_(cache_pd, cluster__dp_degree=33, cluster__n_instances_prefill=2,
                               workload__prefix_pool=40, sim__seed=5),
    }


def dump_sim(name, cfg, path):
    r = ref.run(cfg, per_request=True)
    rq = r["requests"]
    np.savez_compressed(
        path, arrival=rq[:, 0], prompt=rq[:, 1], output=rq[:, 2], status=rq[:, 3].astype(np.int8),
        dispatch=rq[:, 4], prefill_start=rq[:, 5], first_token=rq[:, 6], completion=rq[:, 7],
        agg_json=json.dumps(r["agg"]), digest=np.uint64(r["digest"]),
        alloc_calls=r["alloc_calls"], decode_selects=r["decode_selects"])
    print(f"{name}: n={r['n']} completed={int(r['agg']['completed'])} digest={r['digest']:016x}")


def pbaa_cache_windows(path, n=400, seed=99):
    """Random cache-aware allocate_batch windows with given Len_hit matrices.

    Flat records: [n_pending, n_new, D, n_limit, (id,len,wait)*, caps*D,
    hits*(n*D), n_map, (id,dp)*, n_def, (id,wait)*, n_thr, id*, caps_out*D, flow]."""
    rng = np.random.default_rng(seed)
    rec = []
    for w in range(n):
        D = int(rng.choice([1, 2, 3, 8, 17, 33, 64]))
        npend, nnew = int(rng.integers(0, 24)), int(rng.integers(0, 40))
        k = npend + nnew
        ids = rng.permutation(10 * k + 10)[:k]
        lens = rng.integers(1, 3000, k)
        if k and rng.random() < 0.3:
            lens[rng.integers(0, k, k // 2)] = lens[0]  # prompt ties
        waits = rng.integers(0, 5, k) * (np.arange(k) < npend)
        caps = rng.integers(-500, 4000, D)
        hits = np.where(rng.random((k, D)) < 0.4, rng.integers(0, 3000, (k, D)), 0)
        hits = np.minimum(hits, lens[:, None])
        nlim = int(rng.integers(0, 6))
        rows = np.stack([ids, lens, waits], 1) if k else np.zeros((0, 3), np.int64)
        r = ref.allocate_batch(rows[:npend], rows[npend:], caps.copy(), nlim, hits=hits)
        rec += [npend, nnew, D, nlim] + rows.ravel().tolist() + caps.tolist() + hits.ravel().tolist()
        rec += [len(r["mapping"])] + r["mapping"].ravel().tolist()
        rec += [len(r["deferred"])] + r["deferred"].ravel().tolist()
        rec += [len(r["throttled"])] + r["throttled"].tolist() + r["caps"].tolist() + [int(r["flow"])]
    np.savez_compressed(path, records=np.array(rec, np.int64))
    print("cache-aware windows:", n)


def main():
    (HERE / "configs").mkdir(exist_ok=True)
    if REF_CONFIGS.exists():
        for f in sorted(REF_CONFIGS.glob("*.json")):
            shutil.copy(f, HERE / "configs" / f.name)
    cs = cases()
    json.dump(cs, open(HERE / "cases.json", "w"), indent=1)
    sha = {}
    for name, cfg in cs.items():
        dump_sim(name, cfg, HERE / f"sim_{name}.npz")
        csv = ref.run(cfg, csv=True)["csv"]
        sha[name] = {k: hashlib.sha256(v.encode()).hexdigest() for k, v in csv.items()}
    json.dump(sha, open(HERE / "csv_sha256.json", "w"), indent=1, sort_keys=True)
    smoke = with_(load("decode_dp32"), workload__duration_s=30.0,
                  workload__output={"dist": "uniform", "min": 20, "max": 60},
                  sim__warmup_fraction=0.2)
    dump_sim("smoke", smoke, HERE / "smoke_decode_dp32_30s.npz")
    with np.load(HERE / "smoke_decode_dp32_30s.npz") as z:
        d = dict(z)
    d["cfg_json"] = json.dumps(smoke)
    np.savez_compressed(HERE / "smoke_decode_dp32_30s.npz", **d)
    r = ref.run(load("short_3k"), windows=True)
    np.savez_compressed(HERE / "windows_short_3k.npz", records=r["windows"])
    print("windows:", r["alloc_calls"])
    pbaa_cache_windows(HERE / "windows_cache_aware.npz")
    r = ref.run(load("decode_dp32"), decodes=True)
    np.savez_compressed(HERE / "decodes_decode_dp32.npz", records=r["decodes"])
    print("decodes:", r["decode_selects"])


if __name__ == "__main__":
    main()
