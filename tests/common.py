"""Shared helpers for the parity tests (test infrastructure)."""
import json
from pathlib import Path

import numpy as np

GOLD = Path(__file__).resolve().parent / "golden"
CASES = json.load(open(GOLD / "cases.json"))

# FP64 aggregates: the device sums exact int64 ns / integer-exact FP64 partials;
# the reference sums doubles in request-id order.  North-star tolerance 1e-6
# relative; we hold them to 1e-9.
AGG_RTOL = 1e-9


def load_case(name):
    z = np.load(GOLD / f"sim_{name}.npz")
    d = {k: z[k] for k in z.files}
    d["agg"] = json.loads(str(d.pop("agg_json")))
    return d


def records_windows(rec):
    """Parse ref_harness.cpp's flat allocate_batch records."""
    out, i = [], 0
    rec = [int(x) for x in rec]
    while i < len(rec):
        np_, nn, D, nlim = rec[i:i + 4]; i += 4
        pend = [rec[i + 3 * k:i + 3 * k + 3] for k in range(np_)]; i += 3 * np_
        new = [rec[i + 3 * k:i + 3 * k + 3] for k in range(nn)]; i += 3 * nn
        caps = rec[i:i + D]; i += D
        nm = rec[i]; i += 1
        mapping = [rec[i + 2 * k:i + 2 * k + 2] for k in range(nm)]; i += 2 * nm
        nd = rec[i]; i += 1
        deferred = [rec[i + 2 * k:i + 2 * k + 2] for k in range(nd)]; i += 2 * nd
        nt = rec[i]; i += 1
        thr = rec[i:i + nt]; i += nt
        caps_out = rec[i:i + D]; i += D
        flow = bool(rec[i]); i += 1
        out.append({"pending": pend, "new": new, "caps": caps, "n_limit": nlim,
                    "mapping": mapping, "deferred": deferred, "throttled": thr,
                    "caps_out": caps_out, "flow": flow})
    return out


def records_windows_ca(rec):
    """Parse make_golden.pbaa_cache_windows records (windows with Len_hit)."""
    out, i = [], 0
    rec = [int(x) for x in rec]
    while i < len(rec):
        np_, nn, D, nlim = rec[i:i + 4]; i += 4
        rows = [rec[i + 3 * k:i + 3 * k + 3] for k in range(np_ + nn)]; i += 3 * (np_ + nn)
        caps = rec[i:i + D]; i += D
        hits = [rec[i + D * k:i + D * k + D] for k in range(np_ + nn)]; i += D * (np_ + nn)
        nm = rec[i]; i += 1
        mapping = [rec[i + 2 * k:i + 2 * k + 2] for k in range(nm)]; i += 2 * nm
        nd = rec[i]; i += 1
        deferred = [rec[i + 2 * k:i + 2 * k + 2] for k in range(nd)]; i += 2 * nd
        nt = rec[i]; i += 1
        thr = rec[i:i + nt]; i += nt
        caps_out = rec[i:i + D]; i += D
        flow = bool(rec[i]); i += 1
        out.append({"pending": rows[:np_], "new": rows[np_:], "caps": caps, "n_limit": nlim,
                    "hits": hits, "mapping": mapping, "deferred": deferred, "throttled": thr,
                    "caps_out": caps_out, "flow": flow})
    return out


def records_decodes(rec):
    out, i = [], 0
    rec = [int(x) for x in rec]
    while i < len(rec):
        U = rec[i]; i += 1
        b = rec[i:i + 2 * U:2]; k = rec[i + 1:i + 2 * U:2]; i += 2 * U
        sel, fb = rec[i], bool(rec[i + 1]); i += 2
        out.append({"batch": b, "kv": k, "selected": sel, "fallback": fb})
    return out


def agg_close(a, b, rtol=AGG_RTOL):
    a, b = float(a), float(b)
    return a == b or abs(a - b) <= rtol * max(abs(a), abs(b))
