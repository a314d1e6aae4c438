"""TEST INFRASTRUCTURE ONLY — ctypes view of the plain-C restatement (oracle/_ref/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU leg may use this."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "liboracle.so"
_lib = None
_i64p = C.POINTER(C.c_int64)


def lib():
    global _lib
    if _lib is None:
        srcs = [HERE / "sbs_oracle.c", HERE / "sbs_oracle.h"]
        if not LIB_PATH.exists() or any(s.stat().st_mtime > LIB_PATH.stat().st_mtime for s in srcs):
            subprocess.run(["make", "-s", "oracle"], cwd=HERE, check=True)
        L = C.CDLL(str(LIB_PATH))
        L.orc_allocate_batch.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, _i64p, C.c_int64,
                                         C.c_int, _i64p, _i64p, _i64p, _i64p]
        L.orc_percentile.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_double]
        L.orc_percentile.restype = C.c_double
        L.orc_outlier_threshold.argtypes = [_i64p, C.c_int64, C.c_double]
        L.orc_outlier_threshold.restype = C.c_double
        L.orc_select_decode_unit.argtypes = [_i64p, _i64p, C.c_int64, C.c_double,
                                             C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.orc_schedule_decode_batch.argtypes = [_i64p, C.c_int64, _i64p, _i64p, C.c_int64,
                                                C.c_double, _i64p]
        L.orc_allocate_many.argtypes = [C.c_int64] + [C.c_void_p] * 12
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_i64p)


def allocate_batch(pending, fresh, caps, n_limit):
    L = lib()
    pending = np.ascontiguousarray(pending, np.int64).reshape(-1, 3)
    fresh = np.ascontiguousarray(fresh, np.int64).reshape(-1, 3)
    caps = np.array(caps, np.int64)
    n = max(len(pending) + len(fresh), 1)
    om, od, ot = np.zeros((n, 2), np.int64), np.zeros((n, 2), np.int64), np.zeros(n, np.int64)
    cnt = np.zeros(3, np.int64)
    flow = L.orc_allocate_batch(_p(pending), len(pending), _p(fresh), len(fresh), _p(caps),
                                len(caps), int(n_limit), _p(om), _p(od), _p(ot), _p(cnt))
    return {"mapping": om[: cnt[0]].copy(), "deferred": od[: cnt[1]].copy(),
            "throttled": ot[: cnt[2]].copy(), "caps": caps, "flow": bool(flow)}


def percentile(values, p):
    v = np.ascontiguousarray(values, np.float64)
    return lib().orc_percentile(v.ctypes.data_as(C.POINTER(C.c_double)), len(v), float(p))


def outlier_threshold(kv, k):
    v = np.ascontiguousarray(kv, np.int64)
    return lib().orc_outlier_threshold(_p(v), len(v), float(k))


def select_decode_unit(batch, kv, k=1.5):
    b = np.ascontiguousarray(batch, np.int64)
    kv = np.ascontiguousarray(kv, np.int64)
    fb, th = C.c_int(0), C.c_double(0)
    pos = lib().orc_select_decode_unit(_p(b), _p(kv), len(b), float(k), C.byref(fb), C.byref(th))
    return pos, bool(fb.value), th.value


def schedule_decode_batch(cands, batch, kv, k=1.5):
    c = np.ascontiguousarray(cands, np.int64).reshape(-1, 3)
    b = np.array(batch, np.int64)
    kv = np.array(kv, np.int64)
    out = np.zeros((max(len(c), 1), 2), np.int64)
    lib().orc_schedule_decode_batch(_p(c), len(c), _p(b), _p(kv), len(b), float(k), _p(out))
    return out[: len(c)], b, kv


def allocate_many(req_off, n_pending, dp_off, n_limit, req_id, prompt_len, wait_in, caps):
    """CSR batch (same layout as sbs_prefill_allocate); returns out_dp, out_rank,
    wait_out, caps_after, flow."""
    a = lambda x, t: np.ascontiguousarray(x, t)
    req_off, dp_off = a(req_off, np.int64), a(dp_off, np.int64)
    n_pending, n_limit, wait_in = a(n_pending, np.int32), a(n_limit, np.int32), a(wait_in, np.int32)
    req_id, prompt_len, caps = a(req_id, np.int64), a(prompt_len, np.int64), np.array(caps, np.int64)
    n = len(req_id)
    od, orank, ow = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
    flow = np.zeros(max(len(n_pending), 1), np.uint8)
    lib().orc_allocate_many(len(n_pending), *[x.ctypes.data for x in
                            (req_off, n_pending, dp_off, n_limit, req_id, prompt_len, wait_in,
                             caps, od, orank, ow, flow)])
    return od[:n], orank[:n], ow[:n], caps, flow[:len(n_pending)]
