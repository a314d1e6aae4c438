"""TEST INFRASTRUCTURE ONLY — ctypes view of the compiled reference (oracle/_ref).

Loads ``oracle/_ref/libsbsim_ref.so`` (the unmodified reference sources plus
``oracle/ref_harness.cpp``, built by ``oracle/Makefile``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this module;
the product (``paper_2512_16134_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libsbsim_ref.so"
REF_SRC = Path(os.environ.get("SBS_REFERENCE", "/root/reference")) / "proj"

# aggregates_json order (reference simulation.cpp:545-576)
AGG_FIELDS = [
    "generated", "completed", "throttled", "in_flight", "window_requests",
    "ttft_mean_s", "ttft_p50_s", "ttft_p95_s", "scheduler_wait_mean_s",
    "device_wait_mean_s", "total_wait_mean_s", "passes", "chunk_util_mean",
    "decode_steps", "output_tokens", "output_tokens_per_s", "kv_mean_time_avg",
    "kv_sigma_time_avg", "completed_per_s", "watchdog_fires",
    "dropped_end_forwards", "rejected_samples", "deferrals",
    "flow_control_events", "mask_events", "fallback_events",
    "warmup_cutoff_s", "duration_s",
]

_lib = None
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


def available() -> bool:
    return LIB_PATH.exists() or REF_SRC.exists()


def build() -> None:
    """Compile oracle/_ref from the reference sources (needs /root/reference)."""
    if not REF_SRC.exists():
        if LIB_PATH.exists():
            return
        raise RuntimeError("reference sources absent and oracle/_ref not prebuilt")
    subprocess.run(["make", "-s", "-j8", "ref", f"REF={REF_SRC}"], cwd=HERE, check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.ref_last_error.restype = C.c_char_p
        L.ref_run_json.argtypes = [C.c_char_p, _f64p, _i64p, _i64p, C.c_int64,
                                   _i64p, _i64p, _i64p, _i64p, C.c_char_p, _i64p]
        L.ref_generate_workload.argtypes = [C.c_char_p, _i64p, C.c_int64, _i64p]
        L.ref_allocate_batch.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, _i64p,
                                         C.c_int64, C.c_int, _i64p, _i64p, _i64p, _i64p]
        L.ref_allocate_batch_ca.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, _i64p,
                                            C.c_int64, C.c_int, _i64p, _i64p, _i64p, _i64p,
                                            _i64p]
        L.ref_select_decode_unit.argtypes = [_i64p, _i64p, C.c_int64, C.c_double,
                                             C.POINTER(C.c_int), _f64p]
        L.ref_percentile.argtypes = [_f64p, C.c_int64, C.c_double]
        L.ref_percentile.restype = C.c_double
        L.ref_schedule_decode_batch.argtypes = [_i64p, C.c_int64, _i64p, _i64p, C.c_int64,
                                                C.c_double, _i64p, C.POINTER(C.c_double),
                                                C.POINTER(C.c_int)]
        L.ref_find_peak_qps.argtypes = [C.c_char_p, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.POINTER(C.c_double), C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.ref_outlier_threshold.argtypes = [_i64p, C.c_int64, C.c_double]
        L.ref_outlier_threshold.restype = C.c_double
        L.ref_run_batch.argtypes = [C.POINTER(C.c_char_p), C.c_int64, C.c_int, _f64p,
                                    _i64p, _f64p]
        L.ref_bench_allocate.argtypes = [_i64p, C.c_int64, C.c_int, C.c_int, _f64p, _i64p, _i64p]
        L.ref_bench_select.argtypes = [_i64p, C.c_int64, C.c_double, C.c_int, C.c_int, _f64p,
                                       _i64p, _i64p]
        _lib = L
    return _lib


def _p(a, t=_i64p):
    return a.ctypes.data_as(t) if a is not None else None


def _check(rc):
    if rc not in (0,):
        raise RuntimeError(f"reference rc={rc}: {lib().ref_last_error().decode()}")


def run(cfg: dict, per_request=False, windows=False, decodes=False, csv=False,
        win_cap=1 << 24, dec_cap=1 << 26):
    """Run one experiment through the reference; returns a dict."""
    L = lib()
    text = json.dumps(cfg).encode()
    agg = np.zeros(len(AGG_FIELDS), np.float64)
    meta = np.zeros(5, np.int64)
    n_est = 0
    if per_request:
        m = np.zeros(2, np.int64)
        _check(L.ref_generate_workload(text, None, 0, _p(m)))
        n_est = int(m[0])
    pr = np.zeros((max(n_est, 1), 8), np.int64) if per_request else None
    win = np.zeros(win_cap, np.int64) if windows else None
    wl = np.array([win_cap], np.int64)
    dec = np.zeros(dec_cap, np.int64) if decodes else None
    dl = np.array([dec_cap], np.int64)
    csv_cap = 1 << 28
    cbuf = C.create_string_buffer(csv_cap) if csv else None
    cl = np.array([csv_cap], np.int64)
    rc = L.ref_run_json(text, _p(agg, _f64p), _p(meta), _p(pr), n_est,
                        _p(win), _p(wl) if windows else None,
                        _p(dec), _p(dl) if decodes else None,
                        cbuf, _p(cl) if csv else None)
    _check(rc)
    out = {"agg": dict(zip(AGG_FIELDS, agg.tolist())),
           "digest": int(meta[0]) & 0xFFFFFFFFFFFFFFFF,
           "alloc_calls": int(meta[1]), "decode_selects": int(meta[2]),
           "n": int(meta[3]), "horizon": int(meta[4])}
    if per_request:
        out["requests"] = pr[: out["n"]]
    if windows:
        out["windows"] = win[: int(wl[0])].copy()
    if decodes:
        out["decodes"] = dec[: int(dl[0])].copy()
    if csv:
        parts = cbuf.value.decode().split("\x1e")
        out["csv"] = dict(zip(["requests", "passes", "kvband", "control"], parts))
    return out


def generate_workload(cfg: dict):
    """(arrival_ns, prompt_len, output_len) arrays + digest from the reference."""
    L = lib()
    text = json.dumps(cfg).encode()
    m = np.zeros(2, np.int64)
    _check(L.ref_generate_workload(text, None, 0, _p(m)))
    n = int(m[0])
    buf = np.zeros((max(n, 1), 3), np.int64)
    _check(L.ref_generate_workload(text, _p(buf), n, _p(m)))
    return buf[:n, 0].copy(), buf[:n, 1].copy(), buf[:n, 2].copy(), int(m[1]) & (2**64 - 1)


def allocate_batch(pending, fresh, caps, n_limit, hits=None):
    """pending/fresh: int64 arrays (k,3) of (id, prompt_len, wait_cycles);
    hits (optional, (k_pending + k_new, D)): cache-aware mode with these Len_hit."""
    L = lib()
    pending = np.ascontiguousarray(pending, np.int64).reshape(-1, 3)
    fresh = np.ascontiguousarray(fresh, np.int64).reshape(-1, 3)
    caps = np.array(caps, np.int64)
    n = len(pending) + len(fresh)
    om = np.zeros((max(n, 1), 2), np.int64)
    od = np.zeros((max(n, 1), 2), np.int64)
    ot = np.zeros(max(n, 1), np.int64)
    cnt = np.zeros(3, np.int64)
    if hits is None:
        flow = L.ref_allocate_batch(_p(pending), len(pending), _p(fresh), len(fresh), _p(caps),
                                    len(caps), int(n_limit), _p(om), _p(od), _p(ot), _p(cnt))
    else:
        h = np.ascontiguousarray(hits, np.int64).reshape(n, len(caps))
        flow = L.ref_allocate_batch_ca(_p(pending), len(pending), _p(fresh), len(fresh),
                                       _p(caps), len(caps), int(n_limit), _p(h), _p(om), _p(od),
                                       _p(ot), _p(cnt))
    return {"mapping": om[: cnt[0]].copy(), "deferred": od[: cnt[1]].copy(),
            "throttled": ot[: cnt[2]].copy(), "caps": caps, "flow": bool(flow)}


def schedule_decode_batch(cands, batch, kv, k=1.5):
    """The reference's schedule_decode_batch: returns (placements (id, pos) in
    placement order, thresholds, fallbacks, batch after, kv after)."""
    c = np.ascontiguousarray(cands, np.int64).reshape(-1, 3)
    b = np.array(batch, np.int64)
    kv = np.array(kv, np.int64)
    m = max(len(c), 1)
    out = np.zeros((m, 2), np.int64)
    th = np.zeros(m, np.float64)
    fb = np.zeros(m, np.int32)
    rc = lib().ref_schedule_decode_batch(_p(c), len(c), _p(b), _p(kv), len(b), float(k), _p(out),
                                         th.ctypes.data_as(C.POINTER(C.c_double)),
                                         fb.ctypes.data_as(C.POINTER(C.c_int)))
    if rc:
        raise RuntimeError(lib().ref_last_error().decode())
    n = len(c)
    return out[:n], th[:n], fb[:n].astype(bool), b, kv


def find_peak_qps(cfg, slo, rmin, rmax, res):
    """The reference's find_peak_qps: (probes [(rate, ttft, window, feasible)], peak, attainable)."""
    buf = np.zeros((4096, 4), np.float64)
    peak = C.c_double(0)
    att = C.c_int(0)
    n = lib().ref_find_peak_qps(json.dumps(cfg).encode(), slo, rmin, rmax, res,
                                buf.ctypes.data_as(C.POINTER(C.c_double)), 4096, C.byref(peak),
                                C.byref(att))
    if n < 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return buf[:n].copy(), peak.value, bool(att.value)


def select_decode_unit(batch, kv, k=1.5):
    L = lib()
    b = np.ascontiguousarray(batch, np.int64)
    kv = np.ascontiguousarray(kv, np.int64)
    fb = C.c_int(0)
    th = C.c_double(0)
    pos = L.ref_select_decode_unit(_p(b), _p(kv), len(b), float(k), C.byref(fb), C.byref(th))
    return pos, bool(fb.value), th.value


def percentile(values, p):
    v = np.ascontiguousarray(values, np.float64)
    return lib().ref_percentile(_p(v, _f64p), len(v), float(p))


def outlier_threshold(kv, k):
    v = np.ascontiguousarray(kv, np.int64)
    return lib().ref_outlier_threshold(_p(v), len(v), float(k))


def run_batch(cfgs, threads):
    """CPU baseline: run_experiment over cfgs on `threads` std::threads."""
    L = lib()
    texts = [json.dumps(c).encode() for c in cfgs]
    arr = (C.c_char_p * len(texts))(*texts)
    agg = np.zeros((len(cfgs), len(AGG_FIELDS)), np.float64)
    meta = np.zeros((len(cfgs), 3), np.int64)
    wall = C.c_double(0)
    _check(L.ref_run_batch(arr, len(cfgs), int(threads), _p(agg, _f64p), _p(meta),
                           C.byref(wall)))
    return wall.value, agg, meta


def bench_allocate(window_records, threads, reps):
    """CPU baseline: the reference's allocate_batch over recorded windows
    (Recorder records), `reps` passes on `threads` threads.  Returns
    (wall_s, calls, checksum)."""
    rec = np.ascontiguousarray(window_records, np.int64)
    wall, n, cs = np.zeros(1), np.zeros(1, np.int64), np.zeros(1, np.int64)
    _check(lib().ref_bench_allocate(_p(rec), len(rec), int(threads), int(reps), _p(wall, _f64p),
                                    _p(n), _p(cs)))
    return float(wall[0]), int(n[0]) * max(1, int(reps)), int(cs[0])


def bench_select(decode_records, k, threads, reps):
    """CPU baseline: the reference's select_decode_unit over recorded calls."""
    rec = np.ascontiguousarray(decode_records, np.int64)
    wall, n, cs = np.zeros(1), np.zeros(1, np.int64), np.zeros(1, np.int64)
    _check(lib().ref_bench_select(_p(rec), len(rec), float(k), int(threads), int(reps),
                                  _p(wall, _f64p), _p(n), _p(cs)))
    return float(wall[0]), int(n[0]) * max(1, int(reps)), int(cs[0])
