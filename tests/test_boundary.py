"""CPU: the C-ABI library loads, exports every declared symbol, mirrors the
reference's config/error behaviour, and generates bit-identical traces.
No GPU compute calls here."""
import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2512_16134_b200 as P
from tests.common import CASES, GOLD, load_case
from tests.conftest import HAS_GPU

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "sbs_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sbs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = P.lib()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/sbs_b200.h but not exported"
    assert set(P.api.EXPORTED_SYMBOLS) == set(names)
    assert b"sm_100a" in lib.sbs_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(P.library_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_sizes_match_header():
    # layout guard between include/sbs_b200.h and the ctypes mirror
    assert ctypes.sizeof(P.api.Cluster) == 128
    assert ctypes.sizeof(P.api.LengthSpec) == 48
    assert ctypes.sizeof(P.api.Experiment) == ctypes.sizeof(P.api.Cluster) + \
        ctypes.sizeof(P.api.Workload) + 4 * 4 + 8 + 8 + 3 * 8 + 8


@pytest.mark.parametrize("name", sorted(CASES))
def test_trace_generation_bit_identical(name):
    g = load_case(name)
    tr = P.generate_workload(CASES[name])
    assert tr.digest == int(g["digest"])
    assert np.array_equal(tr.arrival_ns, g["arrival"])
    assert np.array_equal(tr.prompt_len, g["prompt"])
    assert np.array_equal(tr.output_len, g["output"])


def test_digests_of_reference_scenarios():
    # workload_digest values of proj/configs
    want = {"short_3k": 0x3c57d0633a6534f1, "oracle_n8": 0x19ba658d80ff840c,
            "liveness": 0x3c3a202aa3f7d20f, "decode_dp32": 0xe231ea128ca9feae}
    for name, d in want.items():
        cfg = json.load(open(GOLD / "configs" / f"{name}.json"))
        assert P.generate_workload(cfg).digest == d


def test_config_rejects_unknown_keys_like_reference():
    with pytest.raises(P.ConfigError, match='unknown key "cluster.bogus"'):
        P.experiment_from_config({"cluster": {"bogus": 1}})
    with pytest.raises(P.ConfigError, match="must be an integer"):
        P.experiment_from_config({"cluster": {"c_chunk": 1.5}})
    with pytest.raises(P.ConfigError, match="scheduler.policy"):
        P.experiment_from_config({"scheduler": {"policy": "fifo"}})


def _sim_create_rc(cfg):
    pt = P.experiment_from_config(cfg)
    exp = (P.api.Experiment * 1)(pt.exp)
    tr = P.api.Trace()
    h = ctypes.c_void_p()
    return P.lib().sbs_sim_create(exp, 1, ctypes.byref(tr), 1, None, 0, 0, ctypes.byref(h)), \
        P.lib().sbs_last_error().decode()


def test_validate_errors_are_config_errors():
    # validate() messages (core.cpp:79-114) as SBS_ERR_CONFIG, before any GPU work
    rc, msg = _sim_create_rc({"cluster": {"c_chunk": 0}})
    assert rc == 1 and msg == "c_chunk must be >= 1"
    rc, msg = _sim_create_rc({"cluster": {"t_default_s": 0}})
    assert rc == 1 and msg == "t_default_s must be > 0"
    rc, msg = _sim_create_rc({"workload": {"rate_qps": 0}})
    assert rc == 1 and msg == "workload rate_qps must be > 0"
    rc, msg = _sim_create_rc({"faults": {"dead": [{"instance": 9, "time_s": 1}]}})
    assert rc == 1 and msg == "faults.dead: instance out of range"


def test_gpu_envelope_is_explicit():
    rc, msg = _sim_create_rc({"scheduler": {"prefill_mode": "cache_aware"}})
    assert rc == 1 and "out of scope" in msg


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(P.SbsError, match="no CUDA device"):
        P.run_experiment(CASES["liveness"])
