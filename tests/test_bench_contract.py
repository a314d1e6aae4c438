"""CPU: bench.py's reference arm (the compiled reference on the host cores)
prints the contract's JSON line; the workload slices are what DESIGN.md says."""
import json
import subprocess
import sys
from collections import Counter
from pathlib import Path

import numpy as np
import pytest

from oracle import ref

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_workload_slices():
    d, c5 = bench.workload_points("cfg5", 0, 1)
    assert len(c5) == 512 and c5[0]["workload"]["duration_s"] == 5000.0
    seeds = {c["sim"]["seed"] for r in range(8) for c in bench.workload_points("cfg5", r, 8)[1]}
    assert len(seeds) == 8 * 512  # the 4096-replica sweep, no seed twice
    for r in range(8):  # cfg4: every rank gets every dp_degree
        _, c4 = bench.workload_points("cfg4", r, 8)
        assert Counter(c["cluster"]["dp_degree"] for c in c4) == {d: 16 for d in (1, 2, 4, 8, 16, 32, 64, 128)}


@pytest.mark.skipif(not ref.available(), reason="compiled reference unavailable")
def test_reference_arm_json_line():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1",
                        "--replicas", "4", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.skipif(not ref.available(), reason="compiled reference unavailable")
def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks
    (torch.distributed.run, 127.0.0.1); exactly one line, n_gpus 2."""
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                        "--workload", "cfg1", "--replicas", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"


def test_cpu_arm_is_same_config():
    """The CPU arm runs full-size replicas of the GPU arm's workload."""
    for w in ("cfg5", "cfg2", "cfg3", "cfg1"):
        assert bench.cpu_sample_spec(w)["duration"] is None


@pytest.mark.skipif(not ref.available(), reason="compiled reference unavailable")
def test_alloc_reference_arm_and_inputs():
    """`--workload alloc --impl reference`: the reference's allocate_batch /
    select_decode_unit over the calls a cfg2 replica makes (recorded from the
    reference), timed on the host cores; the parsed windows replay to the
    recorded outputs through the C oracle."""
    from oracle import orc
    wrec, drec = bench.alloc_inputs()
    wins, calls = bench.parse_windows(wrec), bench.parse_decodes(drec)
    assert len(wins) > 500 and len(calls) > 10000 and all(len(c[0]) == 320 for c in calls)
    for np_, nlim, rows, caps, mapping, caps_out, flow in wins[:200]:
        e = orc.allocate_batch(rows[:np_], rows[np_:], caps, nlim)
        assert np.array_equal(e["mapping"], mapping) and np.array_equal(e["caps"], caps_out)
        assert e["flow"] == bool(flow)
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "alloc",
                        "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "allocations_per_s" and line["value"] > 0
    assert line["decode_selects_per_s"] > 0 and line["unit"] == "windows/s"


def test_compact_extra_lines():
    line = {"metric": "m", "value": 10.0, "unit": "u", "ms_per_step": 1.0, "config": {},
            "cpu_baseline": {"value": 2.0}, "e2e": {"value": 5.0}, "clocks": None}
    c = bench.compact(line)
    assert c["ratio_vs_cpu"] == 5.0 and c["e2e_ratio_vs_cpu"] == 2.5 and "clocks" not in c
