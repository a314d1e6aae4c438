"""The C++ drop-in (shim/): the reference's own acceptance suite linked against
the B200 path.  The build needs the reference sources (this container); the
binary travels to the GPU box like the other built artefacts."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SHIM = ROOT / "shim"
BIN = SHIM / "_build" / "acceptance_gpu"
REF = Path("/root/reference/proj")


@pytest.mark.skipif(not REF.exists(), reason="reference sources not present on this machine")
def test_shim_builds_against_reference_headers():
    r = subprocess.run(["make", "-s", "-j8", "-C", str(SHIM), "all"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert BIN.exists()
    # the shim replaces exactly the three reference translation units
    nm = subprocess.run(["nm", "-C", "--defined-only", str(SHIM / "_build" / "libsbsim_gpu.a")],
                        capture_output=True, text=True).stdout
    for sym in ("sbsim::allocate_batch", "sbsim::select_decode_unit", "sbsim::run_experiment",
                "sbsim::find_peak_qps", "sbsim::greedy_dispatch", "sbsim::schedule_decode_batch"):
        assert sym in nm, sym


@pytest.mark.gpu
@pytest.mark.skipif(not BIN.exists(), reason="shim/_build/acceptance_gpu not built")
def test_reference_acceptance_suite_on_gpu_path():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    out = r.stdout
    assert "9/9 acceptance checks passed" in out, out[-3000:]
    assert r.returncode == 0
