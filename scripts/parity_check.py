"""Quick GPU-vs-reference parity sweep (development tool; the real gate is tests/)."""
import copy
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2512_16134_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402

CFG = ROOT / "tests" / "golden" / "configs"


def variants():
    base = {n: json.load(open(CFG / f"{n}.json")) for n in ["short_3k", "oracle_n8", "liveness", "decode_dp32"]}
    out = []
    for n, c in base.items():
        out.append((n, c))
        for pol in ["immediate", "least_outstanding"]:
            c2 = copy.deepcopy(c); c2["scheduler"]["policy"] = pol
            out.append((f"{n}/{pol}", c2))
    for dp in ["random", "round_robin"]:
        c2 = copy.deepcopy(base["decode_dp32"]); c2["scheduler"]["decode_policy"] = dp
        out.append((f"decode_dp32/{dp}", c2))
    return out


def compare(name, cfg):
    t0 = time.time()
    g = P.run_experiment(cfg, per_request=True)
    t1 = time.time()
    r = ref.run(cfg, per_request=True)
    t2 = time.time()
    rq = r["requests"]
    gq = g["requests"]
    bad = []
    for col, j in [("dispatch", 4), ("prefill_start", 5), ("first_token", 6), ("completion", 7)]:
        d = np.nonzero(gq[col] != rq[:, j])[0]
        if len(d):
            bad.append(f"{col}: {len(d)} diffs, first id {d[0]} gpu={gq[col][d[0]]} ref={rq[d[0], j]}")
    d = np.nonzero(gq["status"] != rq[:, 3])[0]
    if len(d):
        bad.append(f"status: {len(d)} diffs, first id {d[0]} gpu={gq['status'][d[0]]} ref={rq[d[0],3]}")
    ga, ra = g["agg"], r["agg"]
    for k in P.REFERENCE_AGG_KEYS:
        a, b = float(ga[k]), float(ra[k])
        if not (a == b or abs(a - b) <= 1e-9 * max(abs(a), abs(b))):
            bad.append(f"agg {k}: gpu={a!r} ref={b!r}")
    if ga["alloc_calls"] != r["alloc_calls"]:
        bad.append(f"alloc_calls gpu={ga['alloc_calls']} ref={r['alloc_calls']}")
    if cfg["scheduler"].get("decode_policy", "iqr") == "iqr" and ga["decode_selects"] != r["decode_selects"]:
        bad.append(f"decode_selects gpu={ga['decode_selects']} ref={r['decode_selects']}")
    print(f"[{'OK ' if not bad else 'BAD'}] {name}: n={g['n']} gpu {t1-t0:.2f}s ref {t2-t1:.2f}s err={ga['error']}")
    for b in bad[:12]:
        print("     ", b)
    return not bad


if __name__ == "__main__":
    ok = all([compare(n, c) for n, c in variants()])
    print("ALL OK" if ok else "MISMATCHES")
    sys.exit(0 if ok else 1)
