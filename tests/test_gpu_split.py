"""GPU: two-warp replicas (a prefill warp and a decode warp per replica, see
DESIGN.md "Two-warp replicas") give exactly the serial one-warp result:
every per-request timestamp and every aggregate, including the non-reference
extensions (TPOT sum, TTFT percentiles, histograms) whose FP64 sums depend on
the lane that accumulated each request.  Mode 1: both warps in one CTA;
mode 2: the two CTAs of a cluster (SBS_SPLIT)."""
import copy
import json

import numpy as np
import pytest

import paper_2512_16134_b200 as P
from tests.common import CASES, load_case

pytestmark = pytest.mark.gpu
COLS = ("dispatch", "prefill_start", "first_token", "completion", "status")


def _run(cfg, split, monkeypatch):
    monkeypatch.setenv("SBS_SPLIT", str(split))
    return P.run_experiment(cfg, per_request=True)


def _same(a, b, name):
    for c in COLS:
        assert np.array_equal(a["requests"][c], b["requests"][c]), f"{name}: {c}"
    for k, v in a["agg"].items():
        w = b["agg"][k]
        if isinstance(v, np.ndarray):
            assert np.array_equal(v, w), f"{name}: {k}"
        elif isinstance(v, float) and np.isnan(v):
            assert np.isnan(w), f"{name}: {k}"
        else:
            assert v == w, f"{name}: {k} {v!r} vs {w!r}"


@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("name", ["decode_dp32", "cfg2_20s", "short_3k", "oracle_n8", "cache_pd", "cache_pd_dp33"])
def test_split_equals_serial(name, mode, monkeypatch):
    _same(_run(CASES[name], mode, monkeypatch), _run(CASES[name], 0, monkeypatch), name)


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_split_equals_serial_random(mode, monkeypatch):
    rng = np.random.default_rng(77)
    for t in range(16):
        c = copy.deepcopy(CASES[["decode_dp32", "cfg2_20s"][t % 2]])
        c["workload"]["duration_s"] = float(rng.uniform(3, 20))
        c["workload"]["rate_qps"] = float(c["workload"].get("rate_qps", 10) * rng.uniform(0.5, 2.5))
        c["cluster"]["dp_degree"] = int(rng.choice([1, 4, 17, 64]))
        c["cluster"]["l_net_s"] = float(rng.choice([0.0, 0.001, 0.02]))
        c["scheduler"]["decode_policy"] = str(rng.choice(["iqr", "random", "round_robin"]))
        c["sim"]["seed"] = int(rng.integers(0, 10**6))
        _same(_run(c, mode, monkeypatch), _run(c, 0, monkeypatch), f"random#{t}")


def test_split_tie_rerun_is_exact():
    """A case whose equal-ns EndForward/step ties exceed the two-warp ordering
    rules: the replica reports kErrSplitTie and the host reruns it on one warp
    (SBS_DEBUG reports the rerun); the result is still the reference's."""
    import json
    import os
    import subprocess
    import sys
    from tests.common import load_case
    code = ("import json,sys; sys.path.insert(0,'.'); import paper_2512_16134_b200 as P; "
            "from tests.common import CASES; g=P.run_experiment(CASES['split_tie_round_coeffs'], "
            "per_request=True); print(json.dumps({k: g['requests'][k].tolist() for k in "
            "('dispatch','prefill_start','first_token','completion')}))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for mode in ("1", "2"):
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root,
                           env=dict(os.environ, SBS_DEBUG="1", SBS_SPLIT=mode), timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        assert "split ties" in p.stderr, "the case no longer exercises the one-warp rerun"
        got = json.loads(p.stdout.strip().splitlines()[-1])
        want = load_case("split_tie_round_coeffs")
        for k in got:
            assert np.array_equal(np.array(got[k], np.int64), want[k]), (mode, k)


def test_multi_instance_decode_with_faults_vs_reference():
    """Two-warp replicas with several decode instances, decode/prefill topology
    changes, dead decode instances, batch caps and tps > 1 (the decode warp's
    own topology handling) against the reference (or the C restatement)."""
    from oracle import orc, ref
    have_ref = ref.available()
    rng = np.random.default_rng(3)
    for t in range(12):
        c = copy.deepcopy(CASES[["decode_dp32", "cfg2_20s"][t % 2]])
        Pn, Dn = int(rng.integers(1, 4)), int(rng.choice([2, 3, 5]))
        c["cluster"].update({"n_instances_prefill": Pn, "n_instances_decode": Dn,
                             "dp_degree_decode": int(rng.choice([4, 16, 40])),
                             "decode_max_batch_per_dp": int(rng.choice([0, 3, 20])),
                             "decode_tokens_per_step": int(rng.choice([1, 2, 5]))})
        dur = float(rng.uniform(5, 20))
        c["workload"]["duration_s"] = dur
        c["scheduler"]["decode_policy"] = str(rng.choice(["iqr", "iqr", "random", "round_robin"]))
        c["sim"]["seed"] = int(rng.integers(0, 10**6))
        c["faults"] = {"topology": [{"instance": int(rng.integers(0, Pn + Dn)),
                                     "time_s": float(rng.uniform(0, dur)),
                                     "healthy": bool(rng.random() < 0.5)} for _ in range(3)],
                       "dead": [{"instance": int(rng.integers(Pn, Pn + Dn)),
                                 "time_s": float(rng.uniform(0, dur))}]}
        g = P.run_experiment(c, per_request=True)
        if have_ref:
            rq = ref.run(c, per_request=True)["requests"]
            want = {"status": rq[:, 3], "dispatch": rq[:, 4], "prefill_start": rq[:, 5],
                    "first_token": rq[:, 6], "completion": rq[:, 7]}
        else:
            tr = g["trace"]
            rq = orc.run(c, tr.arrival_ns, tr.prompt_len, tr.output_len)["requests"]
            want = {"status": rq[:, 0], "dispatch": rq[:, 1], "prefill_start": rq[:, 2],
                    "first_token": rq[:, 3], "completion": rq[:, 4]}
        for k in COLS:
            assert np.array_equal(np.asarray(g["requests"][k], np.int64),
                                  np.asarray(want[k], np.int64)), (t, k)


def test_oversized_handoff_falls_back_to_one_warp():
    """An EndForward that finishes more decode-bound requests than the hand-off
    key ring holds (here > 1,024: one-token prompts, a 100k-token chunk) makes
    the replica rerun on one warp instead of blocking; the result equals the
    one-warp run and, per request, the compiled reference.  Run in a
    subprocess with a timeout so a regression cannot hang the suite."""
    import copy
    import json
    import os
    import subprocess
    import sys
    from oracle import ref
    from tests.common import CASES
    c = copy.deepcopy(CASES["decode_dp32"])
    c["cluster"].update({"c_chunk": 100000, "dp_degree": 1, "n_instances_prefill": 1, "t_default_s": 0.5})
    c["workload"].update({"rate_qps": 3000.0, "duration_s": 3.0, "initial_burst": 2000,
                          "prompt": {"dist": "constant", "value": 1},
                          "output": {"dist": "uniform", "min": 2, "max": 20}})
    code = ("import json,sys; sys.path.insert(0,'.'); import paper_2512_16134_b200 as P; "
            "c=json.loads(sys.argv[1]); g=P.run_experiment(c, per_request=True); "
            "print(json.dumps(g['requests']['completion'].tolist()))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode in ("2", "3", "0"):
        p = subprocess.run([sys.executable, "-c", code, json.dumps(c)], capture_output=True, text=True,
                           cwd=root, env=dict(os.environ, SBS_SPLIT=mode), timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1] == outs[2]
    if ref.available():
        want = ref.run(copy.deepcopy(c), per_request=True)["requests"][:, 7].tolist()
        assert outs[0] == want


def test_pair3_not_coresident_falls_back_to_clusters():
    """If the two pair-mode-3 kernels are not co-resident (forced here), both
    give up after the bounded check-in and the host reruns the launch as 2-CTA
    clusters: the results are still the reference's."""
    import os
    import subprocess
    import sys
    code = ("import json,sys; sys.path.insert(0,'.'); import paper_2512_16134_b200 as P; "
            "from tests.common import CASES; g=P.run_experiment(CASES['decode_dp32'], per_request=True); "
            "print(json.dumps(g['requests']['completion'].tolist()))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root, timeout=300,
                       env=dict(os.environ, SBS_SPLIT="3", SBS_PAIR3_NOT_CORESIDENT="1", SBS_DEBUG="1"))
    assert p.returncode == 0, p.stderr[-2000:]
    assert "not co-resident" in p.stderr
    got = np.array(json.loads(p.stdout.strip().splitlines()[-1]))
    want = load_case("decode_dp32")
    assert np.array_equal(got, want["completion"])
