"""CPU: pin the plain-C restatement of the whole simulator (oracle/sbs_oracle_des.c)
against the golden fixtures recorded from the reference (all 18 cases) and,
where available, the compiled reference on random configs."""
import copy

import numpy as np
import pytest

import paper_2512_16134_b200 as P
from oracle import orc, ref
from tests.common import CASES, load_case

AGG = ["generated", "completed", "throttled", "in_flight", "window_requests", "ttft_mean_s",
       "ttft_p50_s", "ttft_p95_s", "scheduler_wait_mean_s", "device_wait_mean_s",
       "total_wait_mean_s", "passes", "chunk_util_mean", "decode_steps", "output_tokens",
       "output_tokens_per_s", "kv_mean_time_avg", "kv_sigma_time_avg", "completed_per_s",
       "watchdog_fires", "dropped_end_forwards", "rejected_samples", "deferrals",
       "flow_control_events", "mask_events", "fallback_events"]


def _check(name, got, want_req, want_agg):
    r = got["requests"]
    for j, col in enumerate(("status", "dispatch", "prefill_start", "first_token", "completion")):
        w = want_req[col]
        d = np.nonzero(r[:, j] != w)[0]
        assert len(d) == 0, f"{name}: {col} differs at request {d[0]}: {r[d[0], j]} vs {w[d[0]]}"
    for k in AGG:  # same FP64 operation order as the reference: exact equality
        assert got["agg"][k] == want_agg[k], f"{name}: {k} {got['agg'][k]!r} vs {want_agg[k]!r}"


def _prefixes(cfg, g):
    """Shared-prefix columns of a golden trace.  The reference harness exports
    (arrival, prompt, output) only; the prefixes come from the host generator,
    whose workload_digest (which folds in every request's first prefix token
    and prefix size, workload.cpp:153-159) must equal the reference's."""
    if cfg.get("workload", {}).get("shared_prefix_fraction", 0) <= 0:
        return None, None
    tr = P.generate_workload(cfg)
    assert tr.digest == int(g["digest"])
    assert np.array_equal(tr.prompt_len, g["prompt"])
    return tr.prefix_pool_id, tr.prefix_size


@pytest.mark.parametrize("name", sorted(CASES))
def test_des_restatement_matches_reference_fixtures(name):
    g = load_case(name)
    pp, ps = _prefixes(CASES[name], g)
    out = orc.run(CASES[name], g["arrival"], g["prompt"], g["output"], prefix_pool=pp,
                  prefix_size=ps)
    assert out["agg"]["error"] == 0
    _check(name, out, g, g["agg"])
    assert out["agg"]["alloc_calls"] == int(g["alloc_calls"])


@pytest.mark.skipif(not ref.available(), reason="compiled reference unavailable")
def test_des_restatement_random_vs_reference():
    rng = np.random.default_rng(31)
    for t in range(25):
        c = copy.deepcopy(CASES[["short_3k", "decode_dp32", "cfg2_20s", "oracle_n8"][t % 4]])
        c["workload"]["duration_s"] = float(rng.uniform(2, 10))
        c["cluster"]["dp_degree"] = int(rng.choice([1, 2, 5, 8, 16]))
        c["cluster"]["n_instances_prefill"] = int(rng.integers(1, 7))
        c["cluster"]["n_limit"] = int(rng.choice([0, 2, 64]))
        c["scheduler"]["policy"] = str(rng.choice(["sbs", "immediate", "least_outstanding"]))
        c["scheduler"]["decode_policy"] = str(rng.choice(["iqr", "random", "round_robin"]))
        c["sim"]["seed"] = int(rng.integers(0, 10**6))
        a, p, o, _ = ref.generate_workload(c)
        r = ref.run(c, per_request=True)
        rq = r["requests"]
        want = {"status": rq[:, 3], "dispatch": rq[:, 4], "prefill_start": rq[:, 5],
                "first_token": rq[:, 6], "completion": rq[:, 7]}
        _check(f"random#{t}", orc.run(c, a, p, o), want, r["agg"])


@pytest.mark.skipif(not ref.available(), reason="compiled reference unavailable")
def test_des_restatement_cache_aware_random_vs_reference():
    """Cache-aware PBAA + per-DP PrefixCache on random settings."""
    rng = np.random.default_rng(77)
    for t in range(16):
        c = copy.deepcopy(CASES[["cache_short", "cache_pd"][t % 2]])
        c["workload"]["duration_s"] = float(rng.uniform(2, 8))
        c["workload"]["shared_prefix_fraction"] = float(rng.choice([0.2, 0.7, 1.0]))
        c["workload"]["prefix_pool"] = int(rng.integers(1, 30))
        c["workload"]["prefix_len"] = int(rng.choice([16, 300, 2000]))
        c["cluster"]["dp_degree"] = int(rng.choice([1, 3, 8, 20]))
        c["cluster"]["cache"] = {"enabled": True,
                                 "probe_lens": [int(x) for x in rng.integers(1, 1500, int(rng.integers(1, 6)))],
                                 "budget_tokens": int(rng.choice([1, 200, 2000, 100000]))}
        c["sim"]["seed"] = int(rng.integers(0, 10**6))
        a, p, o, dg = ref.generate_workload(c)
        tr = P.generate_workload(c)
        assert tr.digest == dg
        r = ref.run(c, per_request=True)
        rq = r["requests"]
        want = {"status": rq[:, 3], "dispatch": rq[:, 4], "prefill_start": rq[:, 5],
                "first_token": rq[:, 6], "completion": rq[:, 7]}
        _check(f"cache#{t}", orc.run(c, a, p, o, prefix_pool=tr.prefix_pool_id,
                                     prefix_size=tr.prefix_size), want, r["agg"])
