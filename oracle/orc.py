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
        srcs = [HERE / "sbs_oracle.c", HERE / "sbs_oracle_des.c", HERE / "sbs_oracle.h"]
        if not LIB_PATH.exists() or any(s.stat().st_mtime > LIB_PATH.stat().st_mtime for s in srcs):
            subprocess.run(["make", "-s", "oracle"], cwd=HERE, check=True)
        L = C.CDLL(str(LIB_PATH))
        L.orc_allocate_batch.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, _i64p, C.c_int64,
                                         C.c_int, _i64p, _i64p, _i64p, _i64p]
        L.orc_allocate_batch_hits.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, _i64p,
                                              C.c_int64, C.c_int, _i64p, _i64p, _i64p, _i64p,
                                              _i64p]
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


def allocate_batch(pending, fresh, caps, n_limit, hits=None):
    """hits (optional, rows pending-then-new x DP): cache-aware Len_hit."""
    L = lib()
    pending = np.ascontiguousarray(pending, np.int64).reshape(-1, 3)
    fresh = np.ascontiguousarray(fresh, np.int64).reshape(-1, 3)
    caps = np.array(caps, np.int64)
    n = max(len(pending) + len(fresh), 1)
    om, od, ot = np.zeros((n, 2), np.int64), np.zeros((n, 2), np.int64), np.zeros(n, np.int64)
    cnt = np.zeros(3, np.int64)
    h = None
    if hits is not None:
        h = np.ascontiguousarray(hits, np.int64).reshape(len(pending) + len(fresh), len(caps))
    flow = L.orc_allocate_batch_hits(_p(pending), len(pending), _p(fresh), len(fresh), _p(caps),
                                     len(caps), int(n_limit), _p(h) if h is not None else None,
                                     _p(om), _p(od), _p(ot), _p(cnt))
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


# ---------------- full simulator restatement (sbs_oracle_des.c) ----------------
class _Drop(C.Structure):
    _fields_ = [("instance", C.c_int), ("from_s", C.c_double), ("until_s", C.c_double)]


class _Dead(C.Structure):
    _fields_ = [("instance", C.c_int), ("time_s", C.c_double)]


class _Topo(C.Structure):
    _fields_ = [("instance", C.c_int), ("healthy", C.c_int), ("time_s", C.c_double)]


class OrcConfig(C.Structure):
    _fields_ = [("n_instances_prefill", C.c_int), ("n_instances_decode", C.c_int),
                ("dp_degree", C.c_int), ("dp_degree_decode", C.c_int), ("c_chunk", C.c_int64),
                ("w_size", C.c_int64), ("decode_tokens_per_step", C.c_int64),
                ("t_default_s", C.c_double), ("l_net_s", C.c_double), ("iqr_k", C.c_double),
                ("watchdog_multiplier", C.c_double), ("n_limit", C.c_int),
                ("decode_max_batch_per_dp", C.c_int), ("prefill_base_s", C.c_double),
                ("prefill_per_token_s", C.c_double), ("decode_base_s", C.c_double),
                ("decode_per_request_s", C.c_double), ("decode_per_kv_token_s", C.c_double),
                ("policy", C.c_int), ("decode_policy", C.c_int), ("seed", C.c_uint64),
                ("duration_s", C.c_double), ("warmup_fraction", C.c_double),
                ("drops", C.POINTER(_Drop)), ("n_drops", C.c_int), ("deads", C.POINTER(_Dead)),
                ("n_deads", C.c_int), ("topology", C.POINTER(_Topo)), ("n_topology", C.c_int),
                ("prefill_mode", C.c_int), ("cache_enabled", C.c_int),
                ("cache_budget_tokens", C.c_int64), ("cache_probe_lens", C.c_void_p),
                ("n_probe_lens", C.c_int)]


class OrcResult(C.Structure):
    _fields_ = ([(k, C.c_uint64) for k in ("generated", "completed", "throttled", "in_flight",
                                           "window_requests")]
                + [(k, C.c_double) for k in ("ttft_mean_s", "ttft_p50_s", "ttft_p95_s",
                                             "scheduler_wait_mean_s", "device_wait_mean_s",
                                             "total_wait_mean_s")]
                + [("passes", C.c_uint64), ("chunk_util_mean", C.c_double),
                   ("decode_steps", C.c_uint64), ("output_tokens", C.c_uint64)]
                + [(k, C.c_double) for k in ("output_tokens_per_s", "kv_mean_time_avg",
                                             "kv_sigma_time_avg", "completed_per_s")]
                + [(k, C.c_uint64) for k in ("watchdog_fires", "dropped_end_forwards",
                                             "rejected_samples", "deferrals",
                                             "flow_control_events", "mask_events",
                                             "fallback_events")]
                + [("warmup_cutoff_s", C.c_double), ("duration_s", C.c_double),
                   ("alloc_calls", C.c_uint64), ("decode_selects", C.c_uint64),
                   ("error", C.c_int)])


def _config(cfg):
    """Reference JSON schema (defaults: config.h / core.h) -> OrcConfig."""
    c = cfg.get("cluster", {})
    e = c.get("engine", {})
    w = cfg.get("workload", {})
    s = cfg.get("scheduler", {})
    sim = cfg.get("sim", {})
    f = cfg.get("faults", {})
    oc = OrcConfig(
        n_instances_prefill=c.get("n_instances_prefill", 1),
        n_instances_decode=c.get("n_instances_decode", 1), dp_degree=c.get("dp_degree", 1),
        dp_degree_decode=c.get("dp_degree_decode", 0), c_chunk=c.get("c_chunk", 1),
        w_size=c.get("w_size", 64), decode_tokens_per_step=c.get("decode_tokens_per_step", 1),
        t_default_s=c.get("t_default_s", 0.1), l_net_s=c.get("l_net_s", 0.0),
        iqr_k=c.get("iqr_k", 1.5), watchdog_multiplier=c.get("watchdog_multiplier", 5.0),
        n_limit=c.get("n_limit", 8), decode_max_batch_per_dp=c.get("decode_max_batch_per_dp", 0),
        prefill_base_s=e.get("prefill_base_s", 0.0),
        prefill_per_token_s=e.get("prefill_per_token_s", 0.0),
        decode_base_s=e.get("decode_base_s", 0.0),
        decode_per_request_s=e.get("decode_per_request_s", 0.0),
        decode_per_kv_token_s=e.get("decode_per_kv_token_s", 0.0),
        policy={"sbs": 0, "immediate": 1, "round_robin": 1, "least_outstanding": 3}[s.get("policy", "sbs")],
        decode_policy={"iqr": 0, "random": 1, "round_robin": 2}[s.get("decode_policy", "iqr")],
        seed=sim.get("seed", 1), duration_s=w.get("duration_s", 1.0),
        warmup_fraction=sim.get("warmup_fraction", 0.1),
        prefill_mode=1 if s.get("prefill_mode", "basic") == "cache_aware" else 0)
    keep = []
    cc = c.get("cache", {})
    if cc.get("enabled", False):
        oc.cache_enabled = 1
        oc.cache_budget_tokens = cc.get("budget_tokens", 0)
        pl = (C.c_int64 * max(len(cc.get("probe_lens", [])), 1))(*cc.get("probe_lens", []))
        keep.append(pl)
        oc.cache_probe_lens = C.cast(pl, C.c_void_p)
        oc.n_probe_lens = len(cc.get("probe_lens", []))
    d = [_Drop(x.get("instance", -1), x.get("from_s", 0.0), x.get("until_s", float("inf")))
         for x in f.get("drop_end_forward", [])]
    dd = [_Dead(x.get("instance", 0), x.get("time_s", 0.0)) for x in f.get("dead", [])]
    t = [_Topo(x.get("instance", 0), 1 if x.get("healthy") else 0, x.get("time_s", 0.0))
         for x in f.get("topology", [])]
    if d:
        arr = (_Drop * len(d))(*d); keep.append(arr)
        oc.drops, oc.n_drops = C.cast(arr, C.POINTER(_Drop)), len(d)
    if dd:
        arr = (_Dead * len(dd))(*dd); keep.append(arr)
        oc.deads, oc.n_deads = C.cast(arr, C.POINTER(_Dead)), len(dd)
    if t:
        arr = (_Topo * len(t))(*t); keep.append(arr)
        oc.topology, oc.n_topology = C.cast(arr, C.POINTER(_Topo)), len(t)
    return oc, keep


def run(cfg, arrival, prompt, output, per_request=True, prefix_pool=None, prefix_size=None):
    """Run the C restatement on a given trace (e.g. the reference's own);
    prefix_pool/prefix_size: the requests' shared prefixes (None: none)."""
    L = lib()
    if not hasattr(L, "_orc_run_bound"):
        L.orc_run_prefix.argtypes = [C.POINTER(OrcConfig), C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(OrcResult),
                                     C.c_void_p]
        L._orc_run_bound = True
    oc, keep = _config(cfg)
    a = np.ascontiguousarray(arrival, np.int64)
    p = np.ascontiguousarray(prompt, np.int32)
    o = np.ascontiguousarray(output, np.int32)
    res = OrcResult()
    pr = np.zeros((max(len(a), 1), 5), np.int64) if per_request else None
    pp = ps = None
    if prefix_pool is not None:
        pp = np.ascontiguousarray(prefix_pool, np.int32)
        ps = np.ascontiguousarray(prefix_size, np.int32)
    L.orc_run_prefix(C.byref(oc), a.ctypes.data, p.ctypes.data, o.ctypes.data,
                     pp.ctypes.data if pp is not None else None,
                     ps.ctypes.data if ps is not None else None, len(a), C.byref(res),
                     pr.ctypes.data if per_request else None)
    out = {"agg": {k: getattr(res, k) for k, _ in OrcResult._fields_}}
    if per_request:
        out["requests"] = pr[: len(a)]
    return out
