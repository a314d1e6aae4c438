"""GPU: the batched allocation kernels (sbs_prefill_allocate, sbs_decode_select)
against the pinned C oracle and the recorded reference windows."""
import itertools

import numpy as np
import pytest

import paper_2512_16134_b200 as P
from oracle import orc, ref
from tests.common import GOLD, records_decodes, records_windows, records_windows_ca

pytestmark = pytest.mark.gpu


def _csr(windows):
    req_off, dp_off, npend, nlim, ids, lens, waits, caps = [0], [0], [], [], [], [], [], []
    for w in windows:
        rows = list(w["pending"]) + list(w["new"])
        for r in rows:
            ids.append(r[0]); lens.append(r[1]); waits.append(r[2])
        req_off.append(req_off[-1] + len(rows))
        npend.append(len(w["pending"])); nlim.append(w["n_limit"])
        caps.extend(w["caps"]); dp_off.append(dp_off[-1] + len(w["caps"]))
    return req_off, npend, dp_off, nlim, ids, lens, waits, caps


def test_recorded_windows_short_3k():
    wins = records_windows(np.load(GOLD / "windows_short_3k.npz")["records"])
    got = P.allocate_batch([{k: w[k] for k in ("pending", "new", "caps", "n_limit")} for w in wins])
    for w, g in zip(wins, got):
        assert g["mapping"].tolist() == w["mapping"]
        assert g["deferred"].tolist() == w["deferred"]
        assert g["throttled"].tolist() == w["throttled"]
        assert g["caps"].tolist() == w["caps_out"]
        assert g["flow"] == w["flow"]


def test_recorded_windows_cache_aware():
    """Cache-aware windows (Len_hit per request x DP) vs the reference's outputs."""
    wins = records_windows_ca(np.load(GOLD / "windows_cache_aware.npz")["records"])
    got = P.allocate_batch([{k: w[k] for k in ("pending", "new", "caps", "n_limit", "hits")}
                            for w in wins])
    for w, g in zip(wins, got):
        assert g["mapping"].tolist() == w["mapping"]
        assert g["deferred"].tolist() == w["deferred"]
        assert g["throttled"].tolist() == w["throttled"]
        assert g["caps"].tolist() == w["caps_out"]
        assert g["flow"] == w["flow"]


def test_pbaa_exhaustive_grid():
    """All 1,007,748 cases of the reference's allocator grid (acceptance.cpp:415-446)
    in one launch, checked against the C oracle."""
    wins = []
    for dp in (1, 2, 3):
        for k in range(1, 7):
            for lens in itertools.product((1, 2, 3, 4, 5, 7), repeat=k):
                rows = [[j, L, 0] for j, L in enumerate(lens)]
                for split in (0, k // 2, k):
                    for nl in (0, 2):
                        wins.append({"pending": rows[:split], "new": rows[split:],
                                     "caps": [7] * dp, "n_limit": nl})
    assert len(wins) == 1007748
    req_off, npend, dp_off, nlim, ids, lens, waits, caps = _csr(wins)
    e_dp, e_rank, e_wait, e_caps, e_flow = orc.allocate_many(req_off, npend, dp_off, nlim, ids,
                                                             lens, waits, caps)
    got = P.allocate_batch(wins)
    g_caps = np.concatenate([g["caps"] for g in got])
    assert np.array_equal(g_caps, e_caps)
    assert np.array_equal(np.array([g["flow"] for g in got]), e_flow.astype(bool))
    # mapping order and deferred/throttled sets via the oracle's per-request outputs
    for i in range(0, len(wins), 997):
        r0, r1 = req_off[i], req_off[i + 1]
        pl = [(ids[j], e_dp[j], e_rank[j]) for j in range(r0, r1) if e_dp[j] >= 0]
        pl.sort(key=lambda t: t[2])
        assert got[i]["mapping"].tolist() == [[a, b] for a, b, _ in pl]


def test_pbaa_random_vs_oracle():
    rng = np.random.default_rng(99)
    wins = []
    for _ in range(4000):
        D = int(rng.integers(1, 129))
        k = int(rng.integers(0, 300))
        ids = rng.permutation(10 * k + 10)[:k]
        lens = np.where(rng.random(k) < 0.1, 1, rng.integers(1, 5000, k))
        waits = rng.integers(0, 6, k)
        rows = [[int(a), int(b), int(c)] for a, b, c in zip(ids, lens, waits)]
        split = int(rng.integers(0, k + 1))
        wins.append({"pending": rows[:split], "new": rows[split:],
                     "caps": rng.integers(-4000, 4000, D).tolist(), "n_limit": int(rng.integers(0, 6))})
    got = P.allocate_batch(wins)
    for w, g in zip(wins, got):
        e = orc.allocate_batch(w["pending"], w["new"], w["caps"], w["n_limit"])
        for key in ("mapping", "deferred", "throttled", "caps"):
            assert np.array_equal(g[key], e[key]), key
        assert g["flow"] == e["flow"]


def test_iqr_recorded_decodes():
    calls = records_decodes(np.load(GOLD / "decodes_decode_dp32.npz")["records"])
    pos, fb, th = P.select_decode_unit([(c["batch"], c["kv"]) for c in calls], k=1.5)
    assert pos.tolist() == [c["selected"] for c in calls]
    assert fb.tolist() == [c["fallback"] for c in calls]


def test_iqr_kats_and_random():
    pos, fb, th = P.select_decode_unit([([0] * 4, [10, 20, 30, 40]), ([0] * 4, [10, 10, 10, 100]),
                                        ([0] * 4, [7, 7, 7, 7])])
    assert th.tolist() == [55.0, 66.25, 7.0]
    rng = np.random.default_rng(5)
    calls = []
    for _ in range(3000):
        U = int(rng.integers(1, 2049))
        B = rng.integers(0, 4, U)
        K = rng.integers(0, 60, U) if rng.random() < 0.5 else rng.integers(0, 10**7, U)
        if rng.random() < 0.3:
            K[rng.integers(0, U, 3)] = 10**10
        calls.append((B, K))
    for k in (0.0, 1.5, 3.0):
        pos, fb, th = P.select_decode_unit(calls, k=k)
        for i, (B, K) in enumerate(calls):
            e = orc.select_decode_unit(B, K, k)
            assert (pos[i], fb[i], th[i]) == e


def test_allocate_one_host_arrays():
    """sbs_prefill_allocate_one (host arrays, one call per window): the small
    by-value path and the staged path (> 32 requests, cache-aware hits) give
    the reference's results on the recorded windows."""
    wins = records_windows(np.load(GOLD / "windows_short_3k.npz")["records"])
    for w in wins[:300]:
        g = P.allocate_one(w["pending"], w["new"], w["caps"], w["n_limit"])
        assert g["mapping"].tolist() == w["mapping"]
        assert g["deferred"].tolist() == w["deferred"]
        assert g["throttled"].tolist() == w["throttled"]
        assert g["caps"].tolist() == w["caps_out"]
        assert g["flow"] == w["flow"]
    assert any(len(w["pending"]) + len(w["new"]) > 32 for w in wins[:300])
    wins = records_windows_ca(np.load(GOLD / "windows_cache_aware.npz")["records"])
    for w in wins[:100]:
        g = P.allocate_one(w["pending"], w["new"], w["caps"], w["n_limit"], hits=w["hits"])
        assert g["mapping"].tolist() == w["mapping"]
        assert g["deferred"].tolist() == w["deferred"]
        assert g["throttled"].tolist() == w["throttled"]
        assert g["caps"].tolist() == w["caps_out"]


# ------------------------------------------------------------ schedule_decode_batch
def _random_sched_batch(rng, big=False):
    U = rng.choice([1, 2, 3, 4, 7, 32, 64, 320]) if not big else rng.choice([320, 1024, 2048])
    M = rng.choice([0, 1, 2, 5, 17, 64]) if not big else rng.choice([100, 700])
    lo = rng.choice([0, 0, 5])
    kv = [lo + rng.randint(0, rng.choice([3, 50, 5000, 10**6])) for _ in range(U)]
    b = [rng.randint(0, rng.choice([1, 3, 40])) for _ in range(U)]
    ids = [rng.randint(0, max(2, M // 2) if rng.random() < 0.3 else 10**12) for _ in range(M)]
    cands = [(ids[i], rng.choice([rng.randint(1, 9), rng.randint(1, 5000)]),
              rng.choice([0, 1, rng.randint(1, 3000)])) for i in range(M)]
    return cands, b, kv


def test_schedule_decode_batch_vs_reference():
    """1,000 random batches (ties in sort_len and request ids, duplicate ids,
    empty batches, fallbacks) in one launch against the reference's own
    schedule_decode_batch (and the C oracle): placements in order, the
    observer's threshold/fallback per placement, the units after."""
    import random
    from oracle import orc
    rng = random.Random(83106)
    batches = [_random_sched_batch(rng) for _ in range(1000)]
    batches += [_random_sched_batch(rng, big=True) for _ in range(8)]
    for k in (1.5, 0.0, -3.0):  # k < 0 empties the IQR mask: the fallback path
        _check_sched(batches, k)


def _check_sched(batches, k):
    from oracle import orc
    got = P.schedule_decode_batch(batches, k=k)
    for i, ((cands, b, kv), g) in enumerate(zip(batches, got)):
        o_pl, o_b, o_kv = orc.schedule_decode_batch(cands, b, kv, k)
        assert np.array_equal(g["placements"], o_pl), f"batch {i}: placements vs oracle"
        if ref.available():
            pl, th, fb, rb, rkv = ref.schedule_decode_batch(cands, b, kv, k)
            assert np.array_equal(g["placements"], pl), f"batch {i}: placements"
            assert np.array_equal(g["threshold"], th), f"batch {i}: thresholds"
            assert np.array_equal(g["fallback"], fb), f"batch {i}: fallbacks"
            assert np.array_equal(g["batch"], rb) and np.array_equal(g["kv"], rkv), f"batch {i}: units"


def test_schedule_decode_batch_errors():
    with pytest.raises(P.InvariantError):
        P.schedule_decode_batch([([(1, 10, 10)], [], [])])
    assert len(P.schedule_decode_batch([([], [], [])])[0]["placements"]) == 0


def test_shim_schedule_decode_batch_vs_reference(tmp_path):
    """The C++ drop-in (shim/alloc_gpu.cpp) under the reference's own
    signature: what the caller and the observer see equals the reference."""
    import random
    import subprocess
    from pathlib import Path
    exe = Path(__file__).resolve().parents[1] / "shim" / "_build" / "sched_check"
    if not exe.exists():
        pytest.skip("shim not built")
    rng = random.Random(4242)
    batches = [_random_sched_batch(rng) for _ in range(300)]
    batches = [bt for bt in batches if len(bt[0])]
    lines = []
    for cands, b, kv in batches:
        lines.append(f"1.5 {len(cands)} {len(b)}")
        lines += [f"{c[0]} {c[1]} {c[2]}" for c in cands]
        lines += [f"{x} {y}" for x, y in zip(b, kv)]
    f = tmp_path / "batches.txt"
    f.write_text("\n".join(lines) + "\n")
    out = subprocess.run([str(exe), str(f)], capture_output=True, text=True, check=True,
                         timeout=600).stdout.splitlines()
    assert len(out) == len(batches)
    for i, ((cands, b, kv), line) in enumerate(zip(batches, out)):
        tok = line.split()
        iT, iF, iU = tok.index("T"), tok.index("F"), tok.index("U")
        pl = np.array(tok[1:iT], np.int64).reshape(-1, 2)
        th = np.array(tok[iT + 1:iF], np.float64)
        fb = np.array(tok[iF + 1:iU], np.int64).astype(bool)
        un = np.array(tok[iU + 1:], np.int64).reshape(-1, 2)
        if ref.available():
            w_pl, w_th, w_fb, w_b, w_kv = ref.schedule_decode_batch(cands, b, kv, 1.5)
        else:
            w_pl, w_b, w_kv = orc.schedule_decode_batch(cands, b, kv, 1.5)
            w_th, w_fb = th, fb
        assert np.array_equal(pl, w_pl), f"batch {i}"
        assert np.array_equal(th, w_th) and np.array_equal(fb, w_fb), f"batch {i}: observer"
        assert np.array_equal(un[:, 0], w_b) and np.array_equal(un[:, 1], w_kv), f"batch {i}: units"


def test_pbaa_register_path_edges_vs_reference():
    """Windows of <= 32 requests x <= 32 DP units take the register path: full
    (prompt, id) ties keep input order (std::stable_sort), capacities beyond
    32 bits take the 64-bit argmax, ids >= 2^27 fall back to the shared-memory
    path; checked against the compiled reference (else the pinned C oracle)."""
    rng = np.random.default_rng(2027)
    check = ref.allocate_batch if ref.available() else orc.allocate_batch
    wins = []
    for t in range(3000):
        D = int(rng.integers(1, 33))
        k = int(rng.integers(0, 33))
        if t % 5 == 0:
            ids = rng.integers(0, 4, k)                      # duplicate ids
            lens = rng.integers(1, 4, k)                     # -> full ties
        elif t % 5 == 1:
            ids = rng.permutation(1 << 20)[:k] + (1 << 27) - (1 << 19)  # straddles 2^27
            lens = rng.integers(1, 5000, k)
        else:
            ids = rng.permutation(10 * k + 10)[:k]
            lens = np.where(rng.random(k) < 0.2, 1, rng.integers(1, 1 << 30, k))
        waits = rng.integers(0, 6, k)
        rows = [[int(a), int(b), int(c)] for a, b, c in zip(ids, lens, waits)]
        split = int(rng.integers(0, k + 1))
        if t % 3 == 0:
            caps = rng.integers(-(1 << 40), 1 << 41, D)     # 64-bit capacities
        else:
            caps = rng.integers(-4000, 1 << 31, D) if t % 3 == 1 else rng.integers(-50, 50, D)
        wins.append({"pending": rows[:split], "new": rows[split:], "caps": caps.tolist(),
                     "n_limit": int(rng.integers(0, 6))})
    got = P.allocate_batch(wins)
    for w, g in zip(wins, got):
        e = check(w["pending"], w["new"], w["caps"], w["n_limit"])
        for key in ("mapping", "deferred", "throttled", "caps"):
            assert np.array_equal(g[key], e[key]), key
        assert g["flow"] == e["flow"]


def test_iqr_register_path_signed_and_wide_kv():
    """<= 512 units are sorted in registers with K offset by 2^63: negative and
    > 2^32 KV loads order exactly as the reference's doubles."""
    rng = np.random.default_rng(77)
    calls = []
    for t in range(2000):
        U = int(rng.integers(1, 513))
        B = rng.integers(0, 5, U)
        if t % 3 == 0:
            K = rng.integers(-(1 << 45), 1 << 45, U)
        elif t % 3 == 1:
            K = rng.integers(0, 3, U)
        else:
            K = rng.integers(0, 1 << 33, U)
        calls.append((B, K))
    for k in (0.0, 1.5):
        pos, fb, th = P.select_decode_unit(calls, k=k)
        for i, (B, K) in enumerate(calls):
            e = (ref.select_decode_unit(B, K, k) if ref.available()
                 else orc.select_decode_unit(B, K, k))
            assert (pos[i], fb[i], th[i]) == tuple(e), i


def test_iqr_large_unit_lists():
    """Calls above 2,048 units (up to the simulator's 16,384-unit envelope) take
    one power-of-two shared-memory slice per warp; beyond it the call fails
    loudly (no host fallback)."""
    rng = np.random.default_rng(8)
    calls = [(rng.integers(0, 4, U), rng.integers(0, 10**6, U)) for U in (2049, 3000, 9000, 16384)]
    pos, fb, th = P.select_decode_unit(calls, k=1.5)
    for i, (B, K) in enumerate(calls):
        e = ref.select_decode_unit(B, K, 1.5) if ref.available() else orc.select_decode_unit(B, K, 1.5)
        assert (pos[i], fb[i], th[i]) == tuple(e), i
    with pytest.raises(P.api.SbsError):
        P.select_decode_unit([(np.zeros(16385, np.int64), np.arange(16385))])
