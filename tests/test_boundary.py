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
    assert ctypes.sizeof(P.api.Cluster) == 144
    assert ctypes.sizeof(P.api.LengthSpec) == 48
    assert ctypes.sizeof(P.api.Trace) == 56
    assert ctypes.sizeof(P.api.WindowBatch) == 8 + 14 * 8 + 8
    assert ctypes.sizeof(P.api.Experiment) == ctypes.sizeof(P.api.Cluster) + \
        ctypes.sizeof(P.api.Workload) + 4 * 4 + 8 + 8 + 3 * 8 + 8


def test_struct_layouts_match_c_compiler(tmp_path):
    """sizeof/offsetof of every ABI struct as gcc sees include/sbs_b200.h."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc absent")
    A = P.api
    structs = {"sbs_cluster": A.Cluster, "sbs_length_spec": A.LengthSpec, "sbs_workload": A.Workload,
               "sbs_experiment": A.Experiment, "sbs_trace": A.Trace, "sbs_aggregates": A.Aggregates,
               "sbs_histograms": A.Histograms, "sbs_window_batch": A.WindowBatch,
               "sbs_decode_batch": A.DecodeBatch}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sbs_b200.h"', "int main(void){"]
    for cn, py in structs.items():
        lines.append(f'printf("{cn} %zu\\n", sizeof({cn}));')
        for f, _ in py._fields_:
            if not f.startswith("_"):
                lines.append(f'printf("{cn}.{f} %zu\\n", offsetof({cn}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True,
                                                           text=True).stdout.splitlines())
    for cn, py in structs.items():
        assert int(got[cn]) == ctypes.sizeof(py), cn
        for f, _ in py._fields_:
            if not f.startswith("_"):
                assert int(got[f"{cn}.{f}"]) == getattr(py, f).offset, f"{cn}.{f}"


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
    rc, msg = _sim_create_rc({"cluster": {"dp_degree": 129}})
    assert rc == 1 and msg == "GPU path supports dp_degree <= 128"
    rc, msg = _sim_create_rc({"cluster": {"cache": {"enabled": True,
                                                    "probe_lens": list(range(1, 40)),
                                                    "budget_tokens": 10}},
                              "scheduler": {"prefill_mode": "cache_aware"}})
    assert rc == 1 and msg == "GPU path supports at most 32 distinct probe lengths"


def test_cache_settings_validated_like_reference():
    # core.cpp:106-113
    rc, msg = _sim_create_rc({"cluster": {"cache": {"enabled": True, "budget_tokens": 10}}})
    assert rc == 1 and msg == "cache.probe_lens must be non-empty when the cache is enabled"
    rc, msg = _sim_create_rc({"cluster": {"cache": {"enabled": True, "probe_lens": [0],
                                                    "budget_tokens": 10}}})
    assert rc == 1 and msg == "cache.probe_lens entries must be >= 1"
    rc, msg = _sim_create_rc({"cluster": {"cache": {"enabled": True, "probe_lens": [8]}}})
    assert rc == 1 and msg == "cache.budget_tokens must be >= 1 when the cache is enabled"
    rc, msg = _sim_create_rc({"workload": {"shared_prefix_fraction": 0.5}})
    assert rc == 1 and "prefix_pool and prefix_len must be positive" in msg


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(P.SbsError, match="no CUDA device"):
        P.run_experiment(CASES["liveness"])
