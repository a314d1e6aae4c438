"""Report files from a GPU run, byte-identical to the reference's writers
(MetricsCollector::requests_csv / passes_csv / kvband_csv / control_csv,
metrics.cpp:194-273) — built from the per-request arrays and the run records
the DES kernel keeps under SBS_FLAG_LOGS."""
from __future__ import annotations

import numpy as np

LOG_DISPATCH, LOG_CONTROL, LOG_PASS, LOG_STEP, LOG_KV, LOG_KVLOADS = 1, 2, 3, 4, 5, 6
STATUS_COMPLETED = 4


def parse_log(words):
    """int64 words -> dict of record lists."""
    w = [int(x) for x in words]
    out = {"dispatch": [], "control": [], "pass": [], "step": [], "kv": [], "kv_loads": []}
    i = 0
    while i < len(w):
        kind, n = w[i] & 0xFF, w[i] >> 8
        pl = w[i + 1:i + 1 + n]
        i += 1 + n
        if kind == LOG_DISPATCH:
            out["dispatch"].append((pl[0], pl[1]))
        elif kind == LOG_CONTROL:
            out["control"].append(tuple(pl[:4]))
        elif kind == LOG_PASS:
            out["pass"].append((pl[0], pl[1], pl[2:]))
        elif kind == LOG_STEP:
            out["step"].append((pl[0], pl[1]))
        elif kind == LOG_KV:
            mean = np.int64(pl[1]).view(np.float64).item()
            sigma = np.int64(pl[2]).view(np.float64).item()
            out["kv"].append((pl[0], mean, sigma, pl[3], pl[4]))
        elif kind == LOG_KVLOADS:
            out["kv_loads"].append((pl[0], pl[1:]))
        else:
            raise ValueError(f"bad log record kind {kind} at word {i}")
    return out


def requests_csv(arrival, req) -> str:
    """metrics.cpp:194-220: completed requests in id order."""
    lines = ["id,arrival_ns,dispatch_ns,prefill_start_ns,first_token_ns,completion_ns,"
             "scheduler_wait_ns,device_wait_ns,ttft_ns\n"]
    st = req["status"]
    ids = np.nonzero(st == STATUS_COMPLETED)[0]
    a, d, p, f, c = (arrival[ids], req["dispatch"][ids], req["prefill_start"][ids],
                     req["first_token"][ids], req["completion"][ids])
    for row in zip(ids.tolist(), a.tolist(), d.tolist(), p.tolist(), f.tolist(), c.tolist(),
                   (d - a).tolist(), (p - d).tolist(), (f - a).tolist()):
        lines.append(",".join(map(str, row)) + "\n")
    return "".join(lines)


def chunk_utilization(assigned, c_chunk):
    """metrics.cpp:193-202 with the same FP64 operation order."""
    s = 0.0
    for a in assigned:
        s += float(min(a, c_chunk)) / float(c_chunk)
    return s / float(len(assigned))


def passes_csv(log, c_chunk) -> str:
    out = ["time_ns,instance,dp,assigned_tokens,utilization\n"]
    for t, inst, assigned in log["pass"]:
        u = "%.6f" % chunk_utilization(assigned, c_chunk)
        for d, a in enumerate(assigned):
            out.append(f"{t},{inst},{d},{a},{u}\n")
    return "".join(out)


def kvband_csv(log) -> str:
    out = ["time_ns,mean,lo,hi,min,max\n"]
    for t, mean, sigma, mn, mx in log["kv"]:
        out.append(f"{t},{'%.3f' % mean},{'%.3f' % (mean - sigma)},{'%.3f' % (mean + sigma)},"
                   f"{mn},{mx}\n")
    return "".join(out)


def control_csv(log) -> str:
    out = ["time_ns,i_opt_ns,t_fwd_bar_ns,n_active\n"]
    for t, i_opt, tbar, na in log["control"]:
        out.append(f"{t},{i_opt},{tbar},{na}\n")
    return "".join(out)


def all_csvs(run) -> dict:
    """From run_experiment(cfg, logs=True): the four report files."""
    log = parse_log(run["log"])
    return {"requests": requests_csv(run["trace"].arrival_ns, run["requests"]),
            "passes": passes_csv(log, run["c_chunk"]),
            "kvband": kvband_csv(log),
            "control": control_csv(log)}
