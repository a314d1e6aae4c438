"""GPU: trace generation on the device (sbs_generate_workload_device, csrc/gen.cu)
against the host generator (the reference's generate_workload restated over
the same glibc) — per request and by workload_digest (workload.cpp:144-162),
pinned to the reference's own digests in tests/golden."""
import copy
import json
import random

import numpy as np
import pytest

import paper_2512_16134_b200 as P
from paper_2512_16134_b200 import api
from tests.common import CASES, GOLD, load_case

pytestmark = pytest.mark.gpu


def same(dev, host, name):
    h = dev.to_host()
    assert dev.n == host.n, f"{name}: n {dev.n} vs {host.n}"
    for col in ("arrival_ns", "prompt_len", "output_len"):
        a, b = getattr(h, col), getattr(host, col)
        d = np.nonzero(a != b)[0]
        assert len(d) == 0, f"{name}: {col} differs at {d[0]}: {a[d[0]]} vs {b[d[0]]}"
    if host.prefix_pool_id is not None:
        assert np.array_equal(h.prefix_pool_id, host.prefix_pool_id), f"{name}: pool"
        assert np.array_equal(h.prefix_size, host.prefix_size), f"{name}: psize"
    assert dev.digest == host.digest, f"{name}: digest"


def test_golden_cases_digest_and_arrays():
    """Every golden case: the device trace's digest is the reference's."""
    names = sorted(CASES)
    devs = api.generate_workload_device([CASES[n] for n in names])
    for name, dev in zip(names, devs):
        want = load_case(name)
        assert dev.digest == int(want["digest"]), name
        h = dev.to_host()
        assert np.array_equal(h.arrival_ns, want["arrival"]), name
        assert np.array_equal(h.prompt_len, want["prompt"]), name
        assert np.array_equal(h.output_len, want["output"]), name


def _length(rng):
    d = rng.choice(["constant", "uniform", "lognormal"])
    if d == "constant":
        return {"dist": "constant", "value": rng.randint(0, 3000)}
    if d == "uniform":
        lo = rng.randint(-5, 500)
        return {"dist": "uniform", "min": lo, "max": lo + rng.randint(-3, 4000)}
    lo = rng.randint(-2, 200)
    return {"dist": "lognormal", "mu": rng.uniform(-1.0, 9.0), "sigma": rng.uniform(0.0, 2.5),
            "min": lo, "max": lo + rng.randint(0, 20000)}


def random_cfg(rng):
    c = copy.deepcopy(CASES["short_3k"])
    w = c["workload"]
    w["process"] = rng.choice(["poisson", "uniform", "uniform_jitter"])
    w["rate_qps"] = rng.choice([0.5, 3.0, 47.3, 200.0, 1234.5])
    w["duration_s"] = rng.choice([0.001, 0.7, 3.0, 10.0, 21.1])
    w["initial_burst"] = rng.choice([0, 0, 1, 37, 256])
    w["prompt"] = _length(rng)
    w["output"] = _length(rng)
    if rng.random() < 0.4:
        w["shared_prefix_fraction"] = rng.choice([0.1, 0.5, 1.0])
        w["prefix_pool"] = rng.randint(1, 40)
        w["prefix_len"] = rng.randint(1, 3000)
    c["sim"]["seed"] = rng.randrange(0, 2**63)
    return c


def test_random_specs_vs_host():
    """300 random workload specs: every arrival process, length distribution
    (incl. degenerate clamps), shared prefixes, initial bursts, seeds."""
    rng = random.Random(20261019)
    cfgs = [random_cfg(rng) for _ in range(300)]
    devs = api.generate_workload_device(cfgs)
    for i, (c, dev) in enumerate(zip(cfgs, devs)):
        same(dev, P.generate_workload(c), f"cfg {i} {json.dumps(c['workload'])}")


def test_full_size_config5_traces():
    """Config 5 traces at full size (5000 s, ~1M requests): 16 seeds."""
    base = copy.deepcopy(CASES["cfg2_20s"])
    base["workload"]["duration_s"] = 5000.0
    cfgs = []
    for s in range(11, 27):
        c = copy.deepcopy(base)
        c["sim"]["seed"] = s
        cfgs.append(c)
    devs = api.generate_workload_device(cfgs)
    for c, dev in zip(cfgs, devs):
        assert dev.n > 990000
        same(dev, P.generate_workload(c), f"cfg5 seed {c['sim']['seed']}")


def test_capacity_overflow_is_reported():
    c = copy.deepcopy(CASES["short_3k"])
    with pytest.raises(P.SbsError):
        api.generate_workload_device([c], caps=[10])


# ---------------------------------------------------------------- simulator on device traces
def _run_host(cfgs):
    pts = [P.experiment_from_config(c) for c in cfgs]
    sim = P.Simulator(pts, [P.generate_workload(p) for p in pts], per_request=True)
    try:
        sim.launch()
        return sim.results(), [sim.requests(i) for i in range(len(cfgs))]
    finally:
        sim.close()


def _same_results(a, b, ra, rb, name):
    for k in P.REFERENCE_AGG_KEYS + ["alloc_calls", "decode_selects", "tpot_count", "tpot_mean_s"]:
        assert a[k] == b[k], f"{name}: {k} {a[k]} vs {b[k]}"
    for col in ("dispatch", "prefill_start", "first_token", "completion", "status"):
        assert np.array_equal(ra[col], rb[col]), f"{name}: {col}"


def test_generated_simulator_matches_golden():
    """Simulator whose traces never leave the device: every golden case per
    request against the reference's columns."""
    names = sorted(CASES)
    pts = [P.experiment_from_config(CASES[n]) for n in names]
    sim = P.Simulator(pts, None, per_request=True)
    try:
        sim.generate(digest=True)
        sim.launch()
        aggs = sim.results()
        for i, name in enumerate(names):
            want = load_case(name)
            assert sim.trace_stats(i)["digest"] == int(want["digest"]), name
            r = sim.requests(i)
            for col in ("dispatch", "prefill_start", "first_token", "completion"):
                assert np.array_equal(r[col], want[col]), f"{name}: {col}"
            assert aggs[i]["generated"] == len(want["arrival"])
    finally:
        sim.close()


def test_generated_slots_new_seeds_match_fresh_host_runs():
    """Regenerate into the second slot with new seeds (the bench's step loop)
    and compare with host-generated simulators of those seeds."""
    base = ["cfg2_20s", "decode_dp32", "short_3k", "cache_pd", "faults_decode_capped_tps3"]
    cfgs = [copy.deepcopy(CASES[n]) for n in base]
    pts = [P.experiment_from_config(c) for c in cfgs]
    sim = P.Simulator(pts, None, per_request=True)
    try:
        sim.enable_trace_slots(2)
        for step, slot in ((1, 1), (2, 0), (3, 1)):
            seeds = [1000 * step + i for i in range(len(cfgs))]
            sim.generate(seeds, slot=slot)
            sim.launch(slot=slot)
            aggs = sim.results()
            got = [sim.requests(i) for i in range(len(cfgs))]
            for c, s_ in zip(cfgs, seeds):
                c["sim"]["seed"] = s_
            want_aggs, want_req = _run_host(cfgs)
            for i in range(len(cfgs)):
                _same_results(aggs[i], want_aggs[i], got[i], want_req[i], f"{base[i]} step {step}")
    finally:
        sim.close()


def test_reupload_checks_shape_bounds():
    """a re-uploaded trace whose outputs exceed the
    create-time completion ring is refused; one that fits gives the same
    results as a fresh simulator."""
    c = copy.deepcopy(CASES["decode_dp32"])
    pt = P.experiment_from_config(c)
    tr = P.generate_workload(pt)
    sim = P.Simulator([pt], [tr], per_request=True)
    try:
        longer = copy.deepcopy(tr)
        longer.output_len = tr.output_len.copy()
        longer.output_len[0] = int(tr.output_len.max()) * 4 + 64
        with pytest.raises(P.ConfigError):
            sim.upload_traces([longer])
        shorter = copy.deepcopy(tr)
        shorter.output_len = np.maximum(tr.output_len // 2, 1).astype(np.int32)
        sim.upload_traces([shorter])
        sim.launch()
        a = sim.results()
        ra = sim.requests(0)
    finally:
        sim.close()
    sim2 = P.Simulator([pt], [shorter], per_request=True)
    try:
        sim2.launch()
        _same_results(a[0], sim2.results()[0], ra, sim2.requests(0), "reupload")
    finally:
        sim2.close()
