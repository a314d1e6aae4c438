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
