"""CPU: glibc_libm.cuh (the device trace generator's log/cos/exp) against the
host's glibc, bit for bit, on the generator's own input domains and on wide
ranges (tests/native/libm_check.cpp).  The device compiles the same header
with __fma_rn/__dmul_rn/...; here it compiles with std::fma and
-ffp-contract=off, so the operation sequence checked is the one the GPU runs.

The 10^8-draw run is recorded in profiles/ (scripts/libm_check.sh); the test
suite runs 3 x 10^6 per domain."""
import json
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "native" / "libm_check.cpp"


def build(tmp_path):
    exe = tmp_path / "libm_check"
    subprocess.run(["g++", "-O2", "-mfma", "-ffp-contract=off", "-std=c++17", str(SRC), "-o",
                    str(exe)], check=True)
    return exe


@pytest.mark.skipif(shutil.which("g++") is None, reason="no host compiler")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_libm_restatement_matches_host_glibc(tmp_path, seed):
    exe = build(tmp_path)
    out = subprocess.run([str(exe), "1000000", str(seed)], check=True, capture_output=True,
                         text=True).stdout
    res = json.loads(out)
    for dom, (n, bad, first) in res.items():
        assert n >= 1000000
        assert bad == 0, f"{dom}: {bad} mismatches of {n}, first at x={first!r}"


def test_tables_header_pins_libm_build():
    """The generated tables name the libm build they were read from."""
    h = (ROOT / "paper_2512_16134_b200" / "csrc" / "glibc_libm_tables.h").read_text()
    assert "glibc 2.39" in h and "kLibmCodeSha256" in h
    assert h.count("0x") > 900
