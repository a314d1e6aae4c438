"""GPU: the persistent DES kernel reproduces the reference simulator.

Bit-exact: every per-request timestamp (dispatch, prefill_start, first_token,
completion), every status, allocation-window counts, integer aggregates.
FP64 aggregates within AGG_RTOL (1e-9 relative; north star: 1e-6).
Full-size cases compare against the compiled reference when it is present and
otherwise check size-independent properties (determinism, conservation,
timestamp monotonicity)."""
import copy

import numpy as np
import pytest

import paper_2512_16134_b200 as P
from oracle import ref
from tests.common import CASES, agg_close, load_case

pytestmark = pytest.mark.gpu
HAVE_REF = ref.available()
COLS = ("dispatch", "prefill_start", "first_token", "completion")
INT_AGGS = ("generated", "completed", "throttled", "in_flight", "window_requests", "passes",
            "decode_steps", "output_tokens", "watchdog_fires", "dropped_end_forwards",
            "rejected_samples", "deferrals", "flow_control_events", "mask_events",
            "fallback_events")


def check_against(name, got_req, got_agg, want):
    for c in COLS:
        d = np.nonzero(got_req[c] != want[c])[0]
        assert len(d) == 0, f"{name}: {c} differs at request {d[0]}: {got_req[c][d[0]]} vs {want[c][d[0]]}"
    assert np.array_equal(got_req["status"], want["status"]), f"{name}: status"
    for k in P.REFERENCE_AGG_KEYS:
        if k in INT_AGGS:
            assert int(got_agg[k]) == int(want["agg"][k]), f"{name}: {k}"
        else:
            assert agg_close(got_agg[k], want["agg"][k]), f"{name}: {k} {got_agg[k]!r} vs {want['agg'][k]!r}"
    assert int(got_agg["alloc_calls"]) == int(want["alloc_calls"]), f"{name}: alloc_calls"


@pytest.mark.parametrize("name", sorted(CASES))
def test_case_bit_exact(name):
    out = P.run_experiment(CASES[name], per_request=True)
    assert out["digest"] == int(load_case(name)["digest"])
    check_against(name, out["requests"], out["agg"], load_case(name))


def test_all_cases_in_one_launch():
    """Mixed shapes/policies in one persistent launch (one warp per replica)."""
    names = sorted(CASES)
    pts = [P.experiment_from_config(CASES[n]) for n in names]
    trs = [P.generate_workload(p) for p in pts]
    sim = P.Simulator(pts, trs, per_request=True)
    try:
        for rep in range(2):  # relaunch: state fully reset between runs
            sim.launch()
            aggs = sim.results()
            for i, n in enumerate(names):
                check_against(n, sim.requests(i), aggs[i], load_case(n))
    finally:
        sim.close()


def test_shared_trace_points():
    """Points sharing one uploaded trace (sweep over l_net / dp on one seed)."""
    base = CASES["cfg1_sbs"]
    cfgs = []
    for ln in (0.0, 0.005, 0.05):
        for dp in (4, 8, 16):
            c = copy.deepcopy(base)
            c["cluster"]["l_net_s"] = ln
            c["cluster"]["dp_degree"] = dp
            cfgs.append(c)
    pts = [P.experiment_from_config(c) for c in cfgs]
    tr = P.generate_workload(pts[0])
    sim = P.Simulator(pts, [tr], trace_of_point=[0] * len(pts), per_request=True)
    try:
        sim.launch()
        aggs = sim.results()
        for i, c in enumerate(cfgs):
            if HAVE_REF:
                r = ref.run(c, per_request=True)
                g = sim.requests(i)
                assert np.array_equal(g["first_token"], r["requests"][:, 6])
                assert np.array_equal(g["dispatch"], r["requests"][:, 4])
                assert aggs[i]["alloc_calls"] == r["alloc_calls"]
            else:
                assert aggs[i]["error"] == 0 and aggs[i]["generated"] == tr.n
    finally:
        sim.close()


def test_random_configs_vs_reference():
    """vs the compiled reference when present, else the pinned C restatement
    (oracle/sbs_oracle_des.c, built from source with gcc on the box)."""
    from oracle import orc
    rng = np.random.default_rng(2024)
    for t in range(40):
        c = copy.deepcopy(CASES[["short_3k", "decode_dp32", "cfg2_20s", "oracle_n8"][t % 4]])
        c["workload"]["duration_s"] = float(rng.uniform(2, 15))
        c["workload"]["rate_qps"] = float(c["workload"].get("rate_qps", 10) * rng.uniform(0.3, 1.8))
        c["cluster"]["dp_degree"] = int(rng.choice([1, 2, 3, 8, 17, 33]))
        c["cluster"]["n_instances_prefill"] = int(rng.integers(1, 9))
        c["cluster"]["l_net_s"] = float(rng.choice([0.0, 0.001, 0.02]))
        c["cluster"]["n_limit"] = int(rng.choice([0, 1, 4, 64]))
        c["scheduler"]["policy"] = str(rng.choice(["sbs", "sbs", "immediate", "least_outstanding"]))
        c["scheduler"]["decode_policy"] = str(rng.choice(["iqr", "random", "round_robin"]))
        c["sim"]["seed"] = int(rng.integers(0, 10**6))
        g = P.run_experiment(c, per_request=True)
        if HAVE_REF:
            r = ref.run(c, per_request=True)
            rq = r["requests"]
            want = {"dispatch": rq[:, 4], "prefill_start": rq[:, 5], "first_token": rq[:, 6],
                    "completion": rq[:, 7], "status": rq[:, 3].astype(np.int8), "agg": r["agg"],
                    "alloc_calls": r["alloc_calls"]}
        else:
            tr = g["trace"]
            r = orc.run(c, tr.arrival_ns, tr.prompt_len, tr.output_len)
            rq = r["requests"]
            want = {"status": rq[:, 0].astype(np.int8), "dispatch": rq[:, 1],
                    "prefill_start": rq[:, 2], "first_token": rq[:, 3], "completion": rq[:, 4],
                    "agg": r["agg"], "alloc_calls": r["agg"]["alloc_calls"]}
        check_against(f"random#{t}", g["requests"], g["agg"], want)


def _cfg2(duration, seed=11):
    c = copy.deepcopy(CASES["cfg2_20s"])
    c["workload"]["duration_s"] = duration
    c["sim"]["seed"] = seed
    return c


@pytest.mark.slow
def test_config2_full_size():
    """100k requests, DP 320 decode."""
    c = _cfg2(500.0)
    g = P.run_experiment(c, per_request=True)
    rq = g["requests"]
    done = rq["status"] == 4
    # size-independent properties
    assert g["agg"]["generated"] == g["n"] and g["agg"]["error"] == 0
    assert g["agg"]["completed"] + g["agg"]["throttled"] + g["agg"]["in_flight"] == g["n"]
    tr = g["trace"]
    assert np.all(tr.arrival_ns[done] <= rq["dispatch"][done])
    assert np.all(rq["dispatch"][done] <= rq["prefill_start"][done])
    assert np.all(rq["prefill_start"][done] <= rq["first_token"][done])
    assert np.all(rq["first_token"][done] <= rq["completion"][done])
    g2 = P.run_experiment(c, per_request=True)
    assert all(np.array_equal(g2["requests"][k], rq[k]) for k in COLS)
    if HAVE_REF:
        r = ref.run(c, per_request=True)
        want = {"dispatch": r["requests"][:, 4], "prefill_start": r["requests"][:, 5],
                "first_token": r["requests"][:, 6], "completion": r["requests"][:, 7],
                "status": r["requests"][:, 3].astype(np.int8), "agg": r["agg"],
                "alloc_calls": r["alloc_calls"]}
        check_against("cfg2_full", rq, g["agg"], want)


@pytest.mark.slow
@pytest.mark.skipif(not HAVE_REF, reason="compiled reference unavailable on this box")
def test_config5_replica_full_size():
    """SURVEY §8d config 5 replica: ~1M requests (reference ~40 s on one core)."""
    c = _cfg2(5000.0, seed=12)
    g = P.run_experiment(c)
    r = ref.run(c)
    for k in P.REFERENCE_AGG_KEYS:
        assert agg_close(g["agg"][k], r["agg"][k]), k
    assert g["agg"]["alloc_calls"] == r["alloc_calls"]
    assert g["agg"]["decode_selects"] == r["decode_selects"]


def test_cache_aware_random_vs_reference():
    """Cache-aware PBAA + per-DP prefix caches on random settings:
    pool sizes, prefix lengths, probe sets (with repeats), budgets that evict
    constantly or never, DP degrees on both kernel variants."""
    from oracle import orc
    rng = np.random.default_rng(4242)
    for t in range(24):
        c = copy.deepcopy(CASES[["cache_short", "cache_pd"][t % 2]])
        c["workload"]["duration_s"] = float(rng.uniform(2, 10))
        c["workload"]["shared_prefix_fraction"] = float(rng.choice([0.1, 0.6, 1.0]))
        c["workload"]["prefix_pool"] = int(rng.integers(1, 50))
        c["workload"]["prefix_len"] = int(rng.choice([8, 300, 1200, 4000]))
        c["cluster"]["dp_degree"] = int(rng.choice([1, 3, 8, 20, 40]))
        c["cluster"]["n_instances_prefill"] = int(rng.integers(1, 6))
        probes = [int(x) for x in rng.integers(1, 1500, int(rng.integers(1, 9)))]
        c["cluster"]["cache"] = {"enabled": True, "probe_lens": probes + probes[:1],
                                 "budget_tokens": int(rng.choice([1, 150, 2500, 10**7]))}
        c["sim"]["seed"] = int(rng.integers(0, 10**6))
        g = P.run_experiment(c, per_request=True)
        if HAVE_REF:
            r = ref.run(c, per_request=True)
            rq = r["requests"]
            want = {"dispatch": rq[:, 4], "prefill_start": rq[:, 5], "first_token": rq[:, 6],
                    "completion": rq[:, 7], "status": rq[:, 3].astype(np.int8), "agg": r["agg"],
                    "alloc_calls": r["alloc_calls"]}
        else:
            tr = g["trace"]
            r = orc.run(c, tr.arrival_ns, tr.prompt_len, tr.output_len,
                        prefix_pool=tr.prefix_pool_id, prefix_size=tr.prefix_size)
            rq = r["requests"]
            want = {"status": rq[:, 0].astype(np.int8), "dispatch": rq[:, 1],
                    "prefill_start": rq[:, 2], "first_token": rq[:, 3], "completion": rq[:, 4],
                    "agg": r["agg"], "alloc_calls": r["agg"]["alloc_calls"]}
        check_against(f"cache#{t}", g["requests"], g["agg"], want)


def test_trace_reupload_pinned_gather_and_pageable():
    """sbs_sim_upload_traces: pinned host traces go up in one gather launch,
    pageable ones by copies; both give the same simulation."""
    names = ["decode_dp32", "short_3k", "cfg2_20s", "cache_short"]
    pts = [P.experiment_from_config(CASES[n]) for n in names]
    pinned = [P.generate_workload(p, pinned=True) for p in pts]
    pageable = [P.generate_workload(p) for p in pts]
    sim = P.Simulator(pts, pageable, per_request=True)
    try:
        outs = []
        for trs in (pinned, pageable, pinned):
            sim.upload_traces(trs)
            sim.launch()
            aggs = sim.results()
            outs.append([sim.requests(i)["completion"].copy() for i in range(len(names))])
            for i, n in enumerate(names):
                assert aggs[i]["error"] == 0
                assert np.array_equal(outs[-1][i], load_case(n)["completion"]), n
    finally:
        sim.close()


def test_trace_slots_alternate():
    """Two trace slots: launches alternate slots (uploads into the idle one)
    and every launch reproduces the reference; relaunch reuses the last slot."""
    names = ["decode_dp32", "cfg2_20s", "cache_short"]
    pts = [P.experiment_from_config(CASES[n]) for n in names]
    trs = [P.generate_workload(p, pinned=True) for p in pts]
    sim = P.Simulator(pts, trs, per_request=True)
    try:
        sim.enable_trace_slots(2)
        sim.upload_traces(slot=1)
        for k in range(4):
            sim.launch(slot=k & 1)
            aggs = sim.results()
            for i, n in enumerate(names):
                assert aggs[i]["error"] == 0
                assert np.array_equal(sim.requests(i)["completion"], load_case(n)["completion"]), (k, n)
    finally:
        sim.close()
