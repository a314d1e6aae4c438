"""GPU: the integer envelope of the device path is an explicit error, never a
silent wrap: a decode unit whose KV load reaches 2^32 stops the
replica with SBS_ERR_ENVELOPE (6), and the reference-compatible configs just
below the envelope still match the compiled reference."""
import copy
import json

import pytest

import paper_2512_16134_b200 as P
from oracle import ref
from tests.common import GOLD

pytestmark = pytest.mark.gpu


def _big_kv_cfg(prompt, rate=40.0):
    c = json.load(open(GOLD / "configs" / "decode_dp32.json"))
    c["cluster"].update({"n_instances_prefill": 1, "dp_degree": 1, "dp_degree_decode": 1,
                         "c_chunk": (1 << 31) - 1})
    c["cluster"]["engine"].update({"prefill_per_token_s": 0.0, "decode_per_kv_token_s": 0.0})
    c["workload"].update({"rate_qps": rate, "duration_s": 2.0,
                          "prompt": {"dist": "constant", "value": prompt},
                          "output": {"dist": "constant", "value": 3000}})
    c["sim"]["warmup_fraction"] = 0.0
    return c


def test_decode_kv_envelope_is_an_error():
    # every request lands on the single decode unit with 2^29 prompt tokens:
    # the 8th resident takes K to 2^32
    cfg = _big_kv_cfg((1 << 29))
    with pytest.raises(P.api.SbsError, match="rc=6"):
        P.run_experiment(cfg)


def test_large_kv_below_envelope_matches_reference():
    # 2^25-token prompts: K stays below 2^32 for the whole run; per request
    # identical to the reference
    cfg = _big_kv_cfg(1 << 25, rate=20.0)
    out = P.run_experiment(cfg, per_request=True)
    if not ref.available():
        pytest.skip("compiled reference absent")
    want = ref.run(copy.deepcopy(cfg), per_request=True)
    got = out["requests"]
    for i, col in enumerate(("dispatch", "prefill_start", "first_token", "completion")):
        assert (got[col] == want["requests"][:, 4 + i]).all(), col
