"""CPU: pin the plain-C oracle (oracle/sbs_oracle.c) before trusting it.

Sources of truth, in order: the reference's own known-answer values
(acceptance.cpp:275-295; SPEC.md worked examples), the committed golden
vectors recorded from the reference simulator (tests/golden), and — where the
compiled reference (oracle/_ref) is available — the reference itself on the
exhaustive PBAA grid (acceptance.cpp:415-446) and random cases.
"""
import itertools
import random

import numpy as np
import pytest

from oracle import orc, ref
from tests.common import GOLD, records_decodes, records_windows, records_windows_ca

HAVE_REF = ref.available()


# ---- known-answer values (acceptance.cpp:275-295) ----
def test_iqr_hand_values():
    assert orc.outlier_threshold([10, 20, 30, 40], 1.5) == pytest.approx(55.0, abs=1e-9)
    assert orc.outlier_threshold([10, 10, 10, 100], 1.5) == pytest.approx(66.25, abs=1e-9)
    assert orc.outlier_threshold([7, 7, 7, 7], 1.5) == pytest.approx(7.0, abs=1e-9)
    assert orc.percentile([10, 20, 30, 40], 25) == pytest.approx(17.5, abs=1e-9)
    assert orc.percentile([10, 20, 30, 40], 75) == pytest.approx(32.5, abs=1e-9)
    assert orc.percentile([5], 90) == pytest.approx(5.0, abs=1e-9)


def test_spec_pbaa_examples():
    # q_pending=[r1(L=500)], q_new=[r2(L=900)], one DP c_avail=1000
    r = orc.allocate_batch([[1, 500, 0]], [[2, 900, 0]], [1000], 8)
    assert r["mapping"].tolist() == [[1, 0], [2, 0]] and r["caps"].tolist() == [-400]
    # guard on the pre-assignment headroom: nothing placed on c_avail <= 0
    r = orc.allocate_batch([], [[1, 10, 0], [2, 20, 0]], [0, -5], 1)
    assert len(r["mapping"]) == 0 and r["deferred"].tolist() == [[1, 1], [2, 1]]
    # aging beyond n_limit throttles and raises flow control
    r = orc.allocate_batch([[1, 10, 2]], [], [0], 2)
    assert r["throttled"].tolist() == [1] and r["flow"]
    # longest first, ties by id; argmax capacity, lowest index on ties
    r = orc.allocate_batch([], [[5, 3, 0], [4, 3, 0], [6, 7, 0]], [7, 7], 8)
    assert r["mapping"].tolist() == [[6, 0], [4, 1], [5, 1]]


def test_lex_order_and_fallback():
    # lex-min (B, K), first position on ties; fallback when the mask empties
    pos, fb, th = orc.select_decode_unit([1, 0, 0, 0], [5, 9, 9, 7])
    assert pos == 3 and not fb
    pos, fb, th = orc.select_decode_unit([2, 1], [50, 40])
    assert pos == 1


# ---- golden vectors recorded from the reference simulator ----
def test_recorded_windows_short_3k():
    wins = records_windows(np.load(GOLD / "windows_short_3k.npz")["records"])
    assert len(wins) == 934
    for w in wins:
        r = orc.allocate_batch(w["pending"], w["new"], w["caps"], w["n_limit"])
        assert r["mapping"].tolist() == w["mapping"]
        assert r["deferred"].tolist() == w["deferred"]
        assert r["throttled"].tolist() == w["throttled"]
        assert r["caps"].tolist() == w["caps_out"]
        assert r["flow"] == w["flow"]


def test_recorded_windows_cache_aware():
    """Cache-aware allocate_batch (capacity_after with Len_hit) vs windows the
    reference computed with its own PrefixCache (make_golden.pbaa_cache_windows)."""
    wins = records_windows_ca(np.load(GOLD / "windows_cache_aware.npz")["records"])
    assert len(wins) == 400
    for w in wins:
        r = orc.allocate_batch(w["pending"], w["new"], w["caps"], w["n_limit"], hits=w["hits"])
        assert r["mapping"].tolist() == w["mapping"]
        assert r["deferred"].tolist() == w["deferred"]
        assert r["throttled"].tolist() == w["throttled"]
        assert r["caps"].tolist() == w["caps_out"]
        assert r["flow"] == w["flow"]


def test_spec_cache_aware_example():
    # L=1000, DP0 c_avail=1000/hit=0, DP1 c_avail=800/hit=900 -> DP1
    r = orc.allocate_batch([], [[1, 1000, 0]], [1000, 800], 8, hits=[[0, 900]])
    assert r["mapping"].tolist() == [[1, 1]] and r["caps"].tolist() == [1000, 700]


def test_recorded_decodes_decode_dp32():
    calls = records_decodes(np.load(GOLD / "decodes_decode_dp32.npz")["records"])
    assert len(calls) == 1280
    for c in calls:
        pos, fb, _ = orc.select_decode_unit(c["batch"], c["kv"], 1.5)
        assert pos == c["selected"] and fb == c["fallback"]


# ---- against the compiled reference ----
def pbaa_grid():
    """Exhaustive grid of acceptance.cpp:415-446 (restated enumeration)."""
    chunk = 7
    for dp in (1, 2, 3):
        for k in range(1, 7):
            for lens in itertools.product((1, 2, 3, 4, 5, chunk), repeat=k):
                for split in (0, k // 2, k):
                    for nl in (0, 2):
                        yield dp, lens, split, nl


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference unavailable")
def test_pbaa_grid_vs_reference_sampled():
    # full grid (1,007,748 cases) runs on the GPU side in test_gpu_alloc; here a
    # deterministic 1-in-37 sample keeps the CPU suite fast
    n = 0
    for i, (dp, lens, split, nl) in enumerate(pbaa_grid()):
        if i % 37:
            continue
        rows = [[j, L, 0] for j, L in enumerate(lens)]
        a = orc.allocate_batch(rows[:split], rows[split:], [7] * dp, nl)
        b = ref.allocate_batch(rows[:split], rows[split:], [7] * dp, nl)
        for key in ("mapping", "deferred", "throttled", "caps"):
            assert np.array_equal(a[key], b[key]), (dp, lens, split, nl, key)
        assert a["flow"] == b["flow"]
        n += 1
    assert n > 20000


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference unavailable")
def test_pbaa_random_vs_reference():
    rng = random.Random(1234)
    for _ in range(3000):
        D = rng.randint(1, 40)
        k = rng.randint(0, 60)
        ids = rng.sample(range(10 * k + 10), k)
        rows = [[i, rng.choice([1, rng.randint(1, 4000)]), rng.randint(0, 5)] for i in ids]
        split = rng.randint(0, k)
        caps = [rng.randint(-3000, 3000) for _ in range(D)]
        nl = rng.randint(0, 6)
        a = orc.allocate_batch(rows[:split], rows[split:], caps, nl)
        b = ref.allocate_batch(rows[:split], rows[split:], caps, nl)
        for key in ("mapping", "deferred", "throttled", "caps"):
            assert np.array_equal(a[key], b[key])
        assert a["flow"] == b["flow"]


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference unavailable")
def test_iqr_random_vs_reference():
    rng = np.random.default_rng(7)
    for _ in range(3000):
        U = int(rng.integers(1, 400))
        B = rng.integers(0, 4, U)
        K = rng.integers(0, 50, U) if rng.random() < 0.5 else rng.integers(0, 10**6, U)
        if rng.random() < 0.2:
            K[rng.integers(0, U)] = 10**9  # an outlier
        k = float(rng.choice([0.0, 0.5, 1.5, 3.0]))
        a = orc.select_decode_unit(B, K, k)
        b = ref.select_decode_unit(B, K, k)
        assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference unavailable")
def test_percentile_vs_reference():
    rng = np.random.default_rng(3)
    for _ in range(500):
        v = rng.random(int(rng.integers(1, 300))) * 10
        for p in (0, 25, 50, 75, 95, 100, 33.3):
            assert orc.percentile(v, p) == ref.percentile(v, p)


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference unavailable")
def test_golden_fixtures_match_reference():
    """The committed fixtures are what the reference produces now."""
    import json
    from tests.common import CASES, load_case
    for name in ("short_3k", "decode_dp32", "faults_prefill"):
        r = ref.run(CASES[name], per_request=True)
        g = load_case(name)
        assert np.array_equal(r["requests"][:, 6], g["first_token"])
        assert r["digest"] == int(g["digest"])
        assert json.dumps(r["agg"]) == json.dumps(g["agg"])
