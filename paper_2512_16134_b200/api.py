"""Python view of the sm_100a SBS hot path (ctypes over include/sbs_b200.h).

Mirrors the reference's public interface for this path
(``proj/include/sbsim/*.h``): experiment configs use the reference JSON schema
(config.cpp:405-435, unknown keys rejected), ``run_experiment`` returns the
reference ``Aggregates`` fields (metrics.h:67-102), and ``allocate_batch`` /
``select_decode_unit`` have the reference's argument meaning.  There is no CPU
fallback: every entry point fails loudly when the CUDA library or a GPU is
missing.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SBS_LIB"]) if os.environ.get("SBS_LIB") else PKG / "lib" / "libsbs_b200.so"

OK, ERR_CONFIG, ERR_INVARIANT, ERR_OVERFLOW, ERR_CUDA, ERR_ENVELOPE = 0, 1, 3, 4, 5, 6


class ConfigError(RuntimeError):
    """≙ sbsim::ConfigError (core.h:34-37)."""


class InvariantError(RuntimeError):
    """≙ std::logic_error raised by a reference invariant check."""


class SbsError(RuntimeError):
    pass


# ----------------------------------------------------------------- structs
class Cluster(C.Structure):
    _fields_ = [
        ("n_instances_prefill", C.c_int32), ("n_instances_decode", C.c_int32),
        ("dp_degree", C.c_int32), ("dp_degree_decode", C.c_int32),
        ("c_chunk", C.c_int64), ("t_default_s", C.c_double), ("w_size", C.c_int64),
        ("l_net_s", C.c_double), ("n_limit", C.c_int32),
        ("decode_max_batch_per_dp", C.c_int32), ("iqr_k", C.c_double),
        ("watchdog_multiplier", C.c_double), ("prefill_base_s", C.c_double),
        ("prefill_per_token_s", C.c_double), ("decode_base_s", C.c_double),
        ("decode_per_request_s", C.c_double), ("decode_per_kv_token_s", C.c_double),
        ("decode_tokens_per_step", C.c_int64), ("cache_enabled", C.c_int32),
        ("cache_n_probes", C.c_int32), ("cache_budget_tokens", C.c_int64),
        ("cache_probe_lens", C.c_void_p),
    ]


class LengthSpec(C.Structure):
    _fields_ = [("dist", C.c_int32), ("_pad", C.c_int32), ("value", C.c_int64),
                ("min", C.c_int64), ("max", C.c_int64), ("mu", C.c_double),
                ("sigma", C.c_double)]


class Workload(C.Structure):
    _fields_ = [("process", C.c_int32), ("initial_burst", C.c_int32),
                ("rate_qps", C.c_double), ("duration_s", C.c_double),
                ("prompt", LengthSpec), ("output", LengthSpec),
                ("shared_prefix_fraction", C.c_double), ("prefix_pool", C.c_int32),
                ("_pad", C.c_int32), ("prefix_len", C.c_int64)]


class DropFault(C.Structure):
    _fields_ = [("instance", C.c_int32), ("_pad", C.c_int32), ("from_s", C.c_double),
                ("until_s", C.c_double)]


class DeadFault(C.Structure):
    _fields_ = [("instance", C.c_int32), ("_pad", C.c_int32), ("time_s", C.c_double)]


class TopologyFault(C.Structure):
    _fields_ = [("instance", C.c_int32), ("healthy", C.c_int32), ("time_s", C.c_double)]


class Experiment(C.Structure):
    _fields_ = [("cluster", Cluster), ("workload", Workload), ("policy", C.c_int32),
                ("prefill_mode", C.c_int32), ("decode_policy", C.c_int32),
                ("n_drops", C.c_int32), ("seed", C.c_uint64), ("warmup_fraction", C.c_double),
                ("drops", C.POINTER(DropFault)), ("deads", C.POINTER(DeadFault)),
                ("topology", C.POINTER(TopologyFault)), ("n_deads", C.c_int32),
                ("n_topology", C.c_int32)]


class Trace(C.Structure):
    _fields_ = [("arrival_ns", C.POINTER(C.c_int64)), ("prompt_len", C.POINTER(C.c_int32)),
                ("output_len", C.POINTER(C.c_int32)), ("n", C.c_int64), ("digest", C.c_uint64),
                ("prefix_pool_id", C.POINTER(C.c_int32)), ("prefix_size", C.POINTER(C.c_int32))]


AGG_FIELDS = [
    ("generated", C.c_uint64), ("completed", C.c_uint64), ("throttled", C.c_uint64),
    ("in_flight", C.c_uint64), ("window_requests", C.c_uint64), ("ttft_mean_s", C.c_double),
    ("ttft_p50_s", C.c_double), ("ttft_p95_s", C.c_double),
    ("scheduler_wait_mean_s", C.c_double), ("device_wait_mean_s", C.c_double),
    ("total_wait_mean_s", C.c_double), ("passes", C.c_uint64), ("chunk_util_mean", C.c_double),
    ("decode_steps", C.c_uint64), ("output_tokens", C.c_uint64),
    ("output_tokens_per_s", C.c_double), ("kv_mean_time_avg", C.c_double),
    ("kv_sigma_time_avg", C.c_double), ("completed_per_s", C.c_double),
    ("watchdog_fires", C.c_uint64), ("dropped_end_forwards", C.c_uint64),
    ("rejected_samples", C.c_uint64), ("deferrals", C.c_uint64),
    ("flow_control_events", C.c_uint64), ("mask_events", C.c_uint64),
    ("fallback_events", C.c_uint64), ("warmup_cutoff_s", C.c_double), ("duration_s", C.c_double),
    ("alloc_calls", C.c_uint64), ("decode_selects", C.c_uint64), ("events", C.c_uint64),
    ("tpot_mean_s", C.c_double), ("tpot_count", C.c_uint64), ("ttft_sum_ns", C.c_int64),
    ("sched_sum_ns", C.c_int64), ("device_sum_ns", C.c_int64), ("error", C.c_int32),
    ("_pad", C.c_int32),
]
REFERENCE_AGG_KEYS = [f for f, _ in AGG_FIELDS[:28]]


class Aggregates(C.Structure):
    _fields_ = AGG_FIELDS

    def to_dict(self):
        return {f: getattr(self, f) for f, _ in AGG_FIELDS if not f.startswith("_")}


_NP_OF = {C.c_uint64: "<u8", C.c_int64: "<i8", C.c_double: "<f8", C.c_int32: "<i4"}
# numpy view of an Aggregates array (bulk conversion in results())
_AGG_NAMES = [f for f, _ in AGG_FIELDS if not f.startswith("_")]
_AGG_DTYPE = np.dtype({"names": _AGG_NAMES,
                       "formats": [_NP_OF[t] for f, t in AGG_FIELDS if not f.startswith("_")],
                       "offsets": [getattr(Aggregates, f).offset for f in _AGG_NAMES],
                       "itemsize": C.sizeof(Aggregates)})


HIST_BINS = 64


class Histograms(C.Structure):
    _fields_ = [("ttft", C.c_int64 * HIST_BINS), ("tpot", C.c_int64 * HIST_BINS)]


class WindowBatch(C.Structure):
    _fields_ = [("n_windows", C.c_int32), ("max_requests", C.c_int32), ("req_off", C.c_void_p),
                ("n_pending", C.c_void_p), ("dp_off", C.c_void_p), ("n_limit", C.c_void_p),
                ("req_id", C.c_void_p), ("prompt_len", C.c_void_p), ("wait_in", C.c_void_p),
                ("caps", C.c_void_p), ("out_dp", C.c_void_p), ("out_rank", C.c_void_p),
                ("wait_out", C.c_void_p), ("flow", C.c_void_p), ("hit_off", C.c_void_p),
                ("hit", C.c_void_p), ("max_dp", C.c_int32), ("_pad", C.c_int32)]


class DecodeBatch(C.Structure):
    _fields_ = [("n_calls", C.c_int32), ("max_units", C.c_int32), ("unit_off", C.c_void_p),
                ("batch", C.c_void_p), ("kv", C.c_void_p), ("k", C.c_double),
                ("pos_out", C.c_void_p), ("fallback_out", C.c_void_p),
                ("threshold_out", C.c_void_p)]


class GenStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("digest", C.c_uint64), ("max_prompt", C.c_int32),
                ("max_output", C.c_int32), ("n_pools", C.c_int32), ("max_psize", C.c_int32),
                ("error", C.c_int32), ("_pad", C.c_int32), ("draws", C.c_int64)]


class GenJob(C.Structure):
    _fields_ = [("spec", Workload), ("seed", C.c_uint64), ("cap", C.c_int64),
                ("arrival_ns", C.c_void_p), ("prompt_len", C.c_void_p),
                ("output_len", C.c_void_p), ("prefix_pool_id", C.c_void_p),
                ("prefix_size", C.c_void_p), ("stats", C.c_void_p)]


# ----------------------------------------------------------------- library
_lib = None


def library_path() -> Path:
    return LIB_PATH


def lib():
    """Load the sm_100a library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise SbsError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(str(LIB_PATH))
        L.sbs_last_error.restype = C.c_char_p
        L.sbs_version.restype = C.c_char_p
        L.sbs_generate_workload.argtypes = [C.POINTER(Workload), C.c_uint64, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_int64, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_uint64)]
        L.sbs_generate_workload_device.argtypes = [C.POINTER(GenJob), C.c_int32, C.c_void_p,
                                                   C.c_int32, C.c_void_p]
        L.sbs_workload_capacity.argtypes = [C.POINTER(Workload)]
        L.sbs_workload_capacity.restype = C.c_int64
        L.sbs_sim_create.argtypes = [C.POINTER(Experiment), C.c_int32, C.POINTER(Trace),
                                     C.c_int32, C.c_void_p, C.c_uint32, C.c_int32,
                                     C.POINTER(C.c_void_p)]
        L.sbs_sim_create_generated.argtypes = [C.POINTER(Experiment), C.c_int32, C.c_void_p,
                                               C.c_int32, C.c_uint32, C.c_int32,
                                               C.POINTER(C.c_void_p)]
        L.sbs_sim_generate_slot.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                            C.c_void_p]
        L.sbs_sim_trace_stats.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(GenStats)]
        L.sbs_sim_trace_arrays.argtypes = [C.c_void_p, C.c_int32, C.c_int32] + [C.c_void_p] * 5 + \
            [C.c_int64, C.POINTER(C.c_int64)]
        L.sbs_sim_upload_traces.argtypes = [C.c_void_p, C.POINTER(Trace), C.c_void_p]
        L.sbs_sim_launch.argtypes = [C.c_void_p, C.c_void_p]
        L.sbs_sim_enable_trace_slots.argtypes = [C.c_void_p, C.c_int32]
        L.sbs_sim_upload_traces_slot.argtypes = [C.c_void_p, C.POINTER(Trace), C.c_int32, C.c_void_p]
        L.sbs_sim_launch_slot.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.sbs_sim_results.argtypes = [C.c_void_p, C.POINTER(Aggregates), C.POINTER(Histograms),
                                      C.c_void_p]
        L.sbs_sim_requests.argtypes = [C.c_void_p, C.c_int32] + [C.c_void_p] * 5
        L.sbs_sim_log.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64,
                                  C.POINTER(C.c_int64)]
        L.sbs_sim_launches_per_run.argtypes = [C.c_void_p]
        L.sbs_sim_des_ms.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.sbs_sim_profile_counters.argtypes = [C.c_void_p, C.c_void_p]
        L.sbs_sim_device_bytes.argtypes = [C.c_void_p]
        L.sbs_sim_device_bytes.restype = C.c_int64
        L.sbs_sim_destroy.argtypes = [C.c_void_p]
        L.sbs_sim_destroy.restype = None
        L.sbs_run_experiments.argtypes = [C.POINTER(Experiment), C.c_int32,
                                          C.POINTER(Aggregates), C.c_int32]
        L.sbs_prefill_allocate.argtypes = [C.POINTER(WindowBatch), C.c_void_p]
        L.sbs_decode_select.argtypes = [C.POINTER(DecodeBatch), C.c_void_p]
        L.sbs_decode_schedule_batch.argtypes = [C.c_void_p, C.c_void_p]
        L.sbs_prefill_allocate_one.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                               C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


EXPORTED_SYMBOLS = [
    "sbs_generate_workload", "sbs_sim_create", "sbs_sim_upload_traces", "sbs_sim_launch",
    "sbs_sim_results", "sbs_sim_requests", "sbs_sim_log", "sbs_sim_launches_per_run",
    "sbs_sim_device_bytes",
    "sbs_sim_destroy", "sbs_run_experiments", "sbs_prefill_allocate",
    "sbs_prefill_allocate_async", "sbs_decode_select", "sbs_decode_select_async",
    "sbs_last_error", "sbs_version", "sbs_sim_profile_counters", "sbs_sim_des_ms",
    "sbs_sim_enable_trace_slots", "sbs_sim_upload_traces_slot", "sbs_sim_launch_slot",
    "sbs_prefill_allocate_one", "sbs_generate_workload_device", "sbs_workload_capacity",
    "sbs_sim_create_generated", "sbs_sim_generate_slot", "sbs_sim_trace_stats",
    "sbs_sim_trace_arrays", "sbs_decode_schedule_batch", "sbs_decode_schedule_batch_async",
]


def _check(rc):
    if rc == OK:
        return
    msg = lib().sbs_last_error().decode()
    if rc == ERR_CONFIG:
        raise ConfigError(msg)
    if rc == ERR_INVARIANT:
        raise InvariantError(msg)
    raise SbsError(f"sbs rc={rc}: {msg}")


# ----------------------------------------------------------------- configs
_CLUSTER_KEYS = {"n_instances_prefill", "n_instances_decode", "dp_degree", "dp_degree_decode",
                 "c_chunk", "t_default_s", "w_size", "l_net_s", "n_limit", "iqr_k",
                 "watchdog_multiplier", "engine", "decode_tokens_per_step",
                 "decode_max_batch_per_dp", "cache"}
_ENGINE_KEYS = {"prefill_base_s", "prefill_per_token_s", "decode_base_s",
                "decode_per_request_s", "decode_per_kv_token_s"}
_WORKLOAD_KEYS = {"process", "rate_qps", "duration_s", "prompt", "output",
                  "shared_prefix_fraction", "prefix_pool", "prefix_len", "initial_burst",
                  "reference_peak_qps"}
_LEN_KEYS = {"dist", "value", "min", "max", "mu", "sigma"}
_POLICIES = {"sbs": 0, "immediate": 1, "round_robin": 2, "least_outstanding": 3}
_DECODE = {"iqr": 0, "random": 1, "round_robin": 2}
_PROCESS = {"poisson": 0, "uniform": 1, "uniform_jitter": 2}
_DIST = {"constant": 0, "uniform": 1, "lognormal": 2}


def _keys(obj, path, allowed):
    if not isinstance(obj, dict):
        raise ConfigError(f"{path} must be an object")
    for k in obj:
        if k not in allowed:
            raise ConfigError(f'unknown key "{path}.{k}"')


def _int(obj, key, default, path):
    if key not in obj:
        return default
    v = obj[key]
    if isinstance(v, bool) or not isinstance(v, int):
        raise ConfigError(f"{path}.{key} must be an integer")
    return v


def _num(obj, key, default, path):
    if key not in obj:
        return default
    v = obj[key]
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise ConfigError(f"{path}.{key} must be a number")
    return float(v)


def _length(obj, path):
    _keys(obj, path, _LEN_KEYS)
    s = LengthSpec(dist=0, value=1, min=1, max=1, mu=0.0, sigma=1.0)
    if "dist" in obj:
        if obj["dist"] not in _DIST:
            raise ConfigError(f"{path}.dist must be constant, uniform, or lognormal")
        s.dist = _DIST[obj["dist"]]
    s.value = _int(obj, "value", s.value, path)
    s.min = _int(obj, "min", s.min, path)
    s.max = _int(obj, "max", s.max, path)
    s.mu = _num(obj, "mu", s.mu, path)
    s.sigma = _num(obj, "sigma", s.sigma, path)
    return s


@dataclass
class Point:
    """One replica: the ctypes Experiment plus the fault arrays it points to."""
    exp: Experiment
    probes: object = None
    drops: object = None
    deads: object = None
    topo: object = None


def experiment_from_config(cfg: dict) -> Point:
    """Reference JSON schema (config.cpp:24-435) -> sbs_experiment."""
    _keys(cfg, "$", {"cluster", "workload", "scheduler", "sim", "faults"})
    cl = Cluster(n_instances_prefill=1, n_instances_decode=1, dp_degree=1, dp_degree_decode=0,
                 c_chunk=1, t_default_s=0.1, w_size=64, l_net_s=0.0, n_limit=8,
                 decode_max_batch_per_dp=0, iqr_k=1.5, watchdog_multiplier=5.0,
                 decode_tokens_per_step=1)
    c = cfg.get("cluster", {})
    _keys(c, "cluster", _CLUSTER_KEYS)
    for k in ("n_instances_prefill", "n_instances_decode", "dp_degree", "dp_degree_decode",
              "c_chunk", "w_size", "n_limit", "decode_tokens_per_step",
              "decode_max_batch_per_dp"):
        setattr(cl, k, _int(c, k, getattr(cl, k), "cluster"))
    for k in ("t_default_s", "l_net_s", "iqr_k", "watchdog_multiplier"):
        setattr(cl, k, _num(c, k, getattr(cl, k), "cluster"))
    if "engine" in c:
        _keys(c["engine"], "cluster.engine", _ENGINE_KEYS)
        for k in _ENGINE_KEYS:
            setattr(cl, k, _num(c["engine"], k, 0.0, "cluster.engine"))
    probes = None
    if "cache" in c:
        cc = c["cache"]
        _keys(cc, "cluster.cache", {"enabled", "probe_lens", "budget_tokens"})
        if "enabled" in cc and not isinstance(cc["enabled"], bool):
            raise ConfigError("cluster.cache.enabled must be a boolean")
        cl.cache_enabled = 1 if cc.get("enabled", False) else 0
        cl.cache_budget_tokens = _int(cc, "budget_tokens", 0, "cluster.cache")
        if "probe_lens" in cc:
            if not isinstance(cc["probe_lens"], list):
                raise ConfigError("cluster.cache.probe_lens must be an array")
            for v in cc["probe_lens"]:
                if isinstance(v, bool) or not isinstance(v, int):
                    raise ConfigError("cluster.cache.probe_lens entries must be integers")
            if cc["probe_lens"]:
                probes = (C.c_int64 * len(cc["probe_lens"]))(*cc["probe_lens"])
                cl.cache_probe_lens = C.cast(probes, C.c_void_p)
                cl.cache_n_probes = len(cc["probe_lens"])
    w = cfg.get("workload", {})
    _keys(w, "workload", _WORKLOAD_KEYS)
    wl = Workload(process=0, initial_burst=0, rate_qps=1.0, duration_s=1.0,
                  prompt=LengthSpec(dist=0, value=1, min=1, max=1, mu=0.0, sigma=1.0),
                  output=LengthSpec(dist=0, value=1, min=1, max=1, mu=0.0, sigma=1.0))
    if "process" in w:
        if w["process"] not in _PROCESS:
            raise ConfigError("workload.process must be poisson, uniform, or uniform_jitter")
        wl.process = _PROCESS[w["process"]]
    wl.rate_qps = _num(w, "rate_qps", wl.rate_qps, "workload")
    wl.duration_s = _num(w, "duration_s", wl.duration_s, "workload")
    if "prompt" in w:
        wl.prompt = _length(w["prompt"], "workload.prompt")
    if "output" in w:
        wl.output = _length(w["output"], "workload.output")
    wl.shared_prefix_fraction = _num(w, "shared_prefix_fraction", 0.0, "workload")
    wl.prefix_pool = _int(w, "prefix_pool", 0, "workload")
    wl.prefix_len = _int(w, "prefix_len", 0, "workload")
    wl.initial_burst = _int(w, "initial_burst", 0, "workload")
    x = Experiment(cluster=cl, workload=wl, policy=0, prefill_mode=0, decode_policy=0,
                   seed=1, warmup_fraction=0.1)
    s = cfg.get("scheduler", {})
    _keys(s, "scheduler", {"policy", "prefill_mode", "decode_policy"})
    if "policy" in s:
        if s["policy"] not in _POLICIES:
            raise ConfigError("scheduler.policy must be sbs, immediate, round_robin, or "
                              "least_outstanding")
        x.policy = _POLICIES[s["policy"]]
    if "prefill_mode" in s:
        if s["prefill_mode"] not in ("basic", "cache_aware"):
            raise ConfigError("scheduler.prefill_mode must be basic or cache_aware")
        x.prefill_mode = 0 if s["prefill_mode"] == "basic" else 1
    if "decode_policy" in s:
        if s["decode_policy"] not in _DECODE:
            raise ConfigError("scheduler.decode_policy must be iqr, random, or round_robin")
        x.decode_policy = _DECODE[s["decode_policy"]]
    sim = cfg.get("sim", {})
    _keys(sim, "sim", {"seed", "warmup_fraction", "trace"})
    seed = _int(sim, "seed", 1, "sim")
    if seed < 0:
        raise ConfigError("sim.seed must be non-negative")
    x.seed = seed
    x.warmup_fraction = _num(sim, "warmup_fraction", 0.1, "sim")
    if not (0.0 <= x.warmup_fraction < 1.0):
        raise ConfigError("sim.warmup_fraction must be in [0, 1)")
    pt = Point(exp=x, probes=probes)
    f = cfg.get("faults", {})
    _keys(f, "faults", {"drop_end_forward", "dead", "topology"})
    drops = [DropFault(instance=e.get("instance", -1), from_s=float(e.get("from_s", 0.0)),
                       until_s=float(e.get("until_s", math.inf)))
             for e in f.get("drop_end_forward", [])]
    deads = [DeadFault(instance=e.get("instance", 0), time_s=float(e.get("time_s", 0.0)))
             for e in f.get("dead", [])]
    topo = [TopologyFault(instance=e.get("instance", 0), healthy=1 if e.get("healthy") else 0,
                          time_s=float(e.get("time_s", 0.0))) for e in f.get("topology", [])]
    if drops:
        pt.drops = (DropFault * len(drops))(*drops)
        x.drops, x.n_drops = C.cast(pt.drops, C.POINTER(DropFault)), len(drops)
    if deads:
        pt.deads = (DeadFault * len(deads))(*deads)
        x.deads, x.n_deads = C.cast(pt.deads, C.POINTER(DeadFault)), len(deads)
    if topo:
        pt.topo = (TopologyFault * len(topo))(*topo)
        x.topology, x.n_topology = C.cast(pt.topo, C.POINTER(TopologyFault)), len(topo)
    return pt


# ----------------------------------------------------------------- traces
@dataclass
class HostTrace:
    arrival_ns: np.ndarray
    prompt_len: np.ndarray
    output_len: np.ndarray
    digest: int
    prefix_pool_id: np.ndarray = None  # shared-prefix pool per request (-1: none)
    prefix_size: np.ndarray = None     # prefix tokens per request

    @property
    def n(self):
        return len(self.arrival_ns)

    def as_c(self) -> Trace:
        i32 = C.POINTER(C.c_int32)
        return Trace(self.arrival_ns.ctypes.data_as(C.POINTER(C.c_int64)),
                     self.prompt_len.ctypes.data_as(i32),
                     self.output_len.ctypes.data_as(i32),
                     self.n, self.digest,
                     self.prefix_pool_id.ctypes.data_as(i32) if self.prefix_pool_id is not None
                     else None,
                     self.prefix_size.ctypes.data_as(i32) if self.prefix_size is not None
                     else None)


def generate_workload(point_or_cfg, pinned: bool = False) -> HostTrace:
    """generate_workload (workload.cpp:67-142) for a point's workload and seed."""
    pt = point_or_cfg if isinstance(point_or_cfg, Point) else experiment_from_config(point_or_cfg)
    L = lib()
    n = C.c_int64(0)
    dg = C.c_uint64(0)
    _check(L.sbs_generate_workload(C.byref(pt.exp.workload), pt.exp.seed, None, None, None,
                                   None, None, 0, C.byref(n), C.byref(dg)))
    cnt = max(n.value, 1)
    if pinned:
        import torch
        a = torch.empty(cnt, dtype=torch.int64, pin_memory=True).numpy()
        p = torch.empty(cnt, dtype=torch.int32, pin_memory=True).numpy()
        o = torch.empty(cnt, dtype=torch.int32, pin_memory=True).numpy()
    else:
        a = np.empty(cnt, np.int64)
        p = np.empty(cnt, np.int32)
        o = np.empty(cnt, np.int32)
    pp = ps = None
    if pt.exp.workload.shared_prefix_fraction > 0:
        if pinned:
            import torch
            pp = torch.empty(cnt, dtype=torch.int32, pin_memory=True).numpy()
            ps = torch.empty(cnt, dtype=torch.int32, pin_memory=True).numpy()
        else:
            pp = np.empty(cnt, np.int32)
            ps = np.empty(cnt, np.int32)
    _check(L.sbs_generate_workload(C.byref(pt.exp.workload), pt.exp.seed, a.ctypes.data,
                                   p.ctypes.data, o.ctypes.data,
                                   pp.ctypes.data if pp is not None else None,
                                   ps.ctypes.data if ps is not None else None, cnt,
                                   C.byref(n), C.byref(dg)))
    k = n.value
    if pp is not None:
        pp, ps = pp[:k], ps[:k]
    return HostTrace(a[:k], p[:k], o[:k], dg.value, pp, ps)


@dataclass
class DeviceTrace:
    """A trace generated on the GPU (torch tensors in HBM) and its stats."""
    arrival_ns: object
    prompt_len: object
    output_len: object
    prefix_pool_id: object
    prefix_size: object
    n: int
    digest: int
    stats: dict

    def to_host(self) -> HostTrace:
        k = self.n
        pp = self.prefix_pool_id[:k].cpu().numpy() if self.prefix_pool_id is not None else None
        ps = self.prefix_size[:k].cpu().numpy() if self.prefix_size is not None else None
        return HostTrace(self.arrival_ns[:k].cpu().numpy(), self.prompt_len[:k].cpu().numpy(),
                         self.output_len[:k].cpu().numpy(), self.digest, pp, ps)


def workload_capacity(point_or_cfg) -> int:
    pt = point_or_cfg if isinstance(point_or_cfg, Point) else experiment_from_config(point_or_cfg)
    return int(lib().sbs_workload_capacity(C.byref(pt.exp.workload)))


def generate_workload_device(points, digest: bool = True, device: int = 0, caps=None):
    """generate_workload for each point's (workload, seed) ON THE GPU (one
    warp per trace, sbs_generate_workload_device); bit-identical to the host
    generator.  Returns DeviceTrace objects."""
    import torch
    L = lib()
    pts = [p if isinstance(p, Point) else experiment_from_config(p) for p in points]
    n = len(pts)
    dev = torch.device("cuda", device)
    jobs = (GenJob * n)()
    stats = torch.zeros((n, C.sizeof(GenStats) // 8), dtype=torch.int64, device=dev)
    keep = []
    for i, p in enumerate(pts):
        w = p.exp.workload
        cap = int(caps[i]) if caps is not None else int(L.sbs_workload_capacity(C.byref(w)))
        cap = max(cap, 1)
        a = torch.empty(cap, dtype=torch.int64, device=dev)
        pr = torch.empty(cap, dtype=torch.int32, device=dev)
        o = torch.empty(cap, dtype=torch.int32, device=dev)
        pp = ps = None
        if w.shared_prefix_fraction > 0:
            pp = torch.empty(cap, dtype=torch.int32, device=dev)
            ps = torch.empty(cap, dtype=torch.int32, device=dev)
        keep.append((a, pr, o, pp, ps))
        jobs[i] = GenJob(spec=w, seed=p.exp.seed, cap=cap, arrival_ns=a.data_ptr(),
                         prompt_len=pr.data_ptr(), output_len=o.data_ptr(),
                         prefix_pool_id=pp.data_ptr() if pp is not None else None,
                         prefix_size=ps.data_ptr() if ps is not None else None,
                         stats=stats[i].data_ptr())
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        _check(L.sbs_generate_workload_device(jobs, n, None, 1 if digest else 0,
                                              C.c_void_p(stream)))
        torch.cuda.synchronize()
    raw = stats.cpu().numpy()
    out = []
    for i in range(n):
        g = GenStats.from_buffer_copy(raw[i].tobytes())
        st = {f: getattr(g, f) for f, _ in GenStats._fields_ if not f.startswith("_")}
        if g.error:
            raise (ConfigError if g.error == ERR_CONFIG else SbsError)(
                f"device trace generation failed for point {i}: error {g.error}")
        a, pr, o, pp, ps = keep[i]
        out.append(DeviceTrace(a, pr, o, pp, ps, int(g.n), int(g.digest), st))
    return out


# ----------------------------------------------------------------- simulator
class Simulator:
    """Many replicas, one warp each, resident on one GPU (sbs_sim_*)."""

    def __init__(self, points, traces=None, trace_of_point=None, per_request=False, logs=False,
                 device=0):
        """traces: HostTrace list (uploaded), or None: every trace is
        generated ON THE DEVICE from its points' (workload, seed)
        (sbs_sim_create_generated) and regenerated by generate()."""
        L = lib()
        self.points = list(points)
        self.generated = traces is None
        n = len(self.points)
        self._exp = (Experiment * n)(*[p.exp for p in self.points])
        self._map = None
        if trace_of_point is not None:
            self._map = (C.c_int32 * n)(*trace_of_point)
        mp = C.cast(self._map, C.c_void_p) if self._map is not None else None
        flags = (1 if per_request else 0) | (2 if logs else 0)
        h = C.c_void_p()
        if self.generated:
            self.traces = None
            self.n_traces = (max(trace_of_point) + 1) if trace_of_point is not None else n
            _check(L.sbs_sim_create_generated(self._exp, n, mp, self.n_traces, flags, device,
                                              C.byref(h)))
        else:
            self.traces = list(traces)
            self.n_traces = len(self.traces)
            self._tr = (Trace * len(self.traces))(*[t.as_c() for t in self.traces])
            _check(L.sbs_sim_create(self._exp, n, self._tr, len(self.traces), mp, flags, device,
                                    C.byref(h)))
        self.handle = h
        self.n = n
        self._slot = 0

    def generate(self, seeds=None, slot=0, stream=0, digest=False):
        """Regenerate every trace on the device into `slot` (one seed per
        trace; None = the current seeds).  Enqueued on `stream`."""
        arr = None
        if seeds is not None:
            arr = (C.c_uint64 * self.n_traces)(*[int(x) for x in seeds])
        _check(lib().sbs_sim_generate_slot(self.handle, arr, slot, 1 if digest else 0,
                                           C.c_void_p(stream)))

    def trace_stats(self, trace, slot=0):
        st = GenStats()
        _check(lib().sbs_sim_trace_stats(self.handle, trace, slot, C.byref(st)))
        return {f: getattr(st, f) for f, _ in GenStats._fields_ if not f.startswith("_")}

    def trace(self, trace, slot=0) -> HostTrace:
        """A trace as the device holds it (copied back)."""
        L = lib()
        n = C.c_int64(0)
        _check(L.sbs_sim_trace_arrays(self.handle, trace, slot, None, None, None, None, None, 0,
                                      C.byref(n)))
        k = max(n.value, 1)
        a, p, o = np.empty(k, np.int64), np.empty(k, np.int32), np.empty(k, np.int32)
        pp, ps = np.empty(k, np.int32), np.empty(k, np.int32)
        _check(L.sbs_sim_trace_arrays(self.handle, trace, slot, a.ctypes.data, p.ctypes.data,
                                      o.ctypes.data, pp.ctypes.data, ps.ctypes.data, k,
                                      C.byref(n)))
        k = n.value
        dg = self.trace_stats(trace, slot)["digest"] if self.generated else self.traces[trace].digest
        w = self.points[0].exp.workload
        has_pfx = self.generated and any(pt.exp.workload.shared_prefix_fraction > 0
                                         for pt in self.points)
        return HostTrace(a[:k], p[:k], o[:k], dg, pp[:k] if has_pfx else None,
                         ps[:k] if has_pfx else None)

    def upload_traces(self, traces=None, stream=0, slot=0):
        # The copy reads the host buffers asynchronously on `stream`: the
        # previous upload's traces stay referenced until this call returns,
        # by which point the library has waited for that copy to finish.
        prev = (self.traces, self._tr)
        if traces is not None:
            self.traces = list(traces)
            self._tr = (Trace * len(self.traces))(*[t.as_c() for t in self.traces])
        _check(lib().sbs_sim_upload_traces_slot(self.handle, self._tr, slot, C.c_void_p(stream)))
        self._inflight = (self.traces, self._tr)
        del prev

    def enable_trace_slots(self, n=2):
        """Second trace buffer set: upload step k+1 while step k runs."""
        _check(lib().sbs_sim_enable_trace_slots(self.handle, n))

    def launch(self, stream=0, slot=0):
        _check(lib().sbs_sim_launch_slot(self.handle, slot, C.c_void_p(stream)))
        self._slot = slot

    def results(self, stream=0, histograms=False):
        out = (Aggregates * self.n)()
        hist = Histograms() if histograms else None
        _check(lib().sbs_sim_results(self.handle, out, C.byref(hist) if hist else None,
                                     C.c_void_p(stream)))
        rows = np.frombuffer(out, dtype=_AGG_DTYPE).tolist()
        res = [dict(zip(_AGG_NAMES, r)) for r in rows]
        return (res, hist) if histograms else res

    def requests(self, point: int):
        t = self._map[point] if self._map is not None else point
        if self.generated:
            m = C.c_int64(0)
            _check(lib().sbs_sim_trace_arrays(self.handle, t, self._slot, None, None, None, None,
                                              None, 0, C.byref(m)))
            n = m.value
        else:
            n = self.traces[t].n
        cols = [np.empty(max(n, 1), np.int64) for _ in range(4)]
        st = np.empty(max(n, 1), np.int8)
        _check(lib().sbs_sim_requests(self.handle, point, *[c.ctypes.data for c in cols],
                                      st.ctypes.data))
        return {"dispatch": cols[0][:n], "prefill_start": cols[1][:n],
                "first_token": cols[2][:n], "completion": cols[3][:n], "status": st[:n]}

    def log(self, point: int) -> np.ndarray:
        """Run records of one point (SBS_FLAG_LOGS), int64 words."""
        n = C.c_int64(0)
        _check(lib().sbs_sim_log(self.handle, point, None, 0, C.byref(n)))
        buf = np.empty(max(n.value, 1), np.int64)
        _check(lib().sbs_sim_log(self.handle, point, buf.ctypes.data, len(buf), C.byref(n)))
        return buf[: n.value]

    def profile_counters(self):
        out = (C.c_int64 * 24)()
        lib().sbs_sim_profile_counters(self.handle, out)
        return list(out)

    def des_ms(self):
        """Device ms of the DES kernels of the last launch (CUDA events)."""
        ms = C.c_double(0)
        _check(lib().sbs_sim_des_ms(self.handle, C.byref(ms)))
        return ms.value

    @property
    def launches_per_run(self):
        return lib().sbs_sim_launches_per_run(self.handle)

    @property
    def device_bytes(self):
        return lib().sbs_sim_device_bytes(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            lib().sbs_sim_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_experiment(cfg: dict, per_request=False, logs=False, device=0):
    """≙ sbsim::run_experiment (simulation.h:33) on the GPU: returns a dict with
    the Aggregates fields (and per-request arrays / run records on request)."""
    pt = experiment_from_config(cfg)
    tr = generate_workload(pt)
    sim = Simulator([pt], [tr], per_request=per_request or logs, logs=logs, device=device)
    try:
        sim.launch()
        agg = sim.results()[0]
        out = {"agg": agg, "digest": tr.digest, "n": tr.n, "trace": tr}
        if per_request or logs:
            out["requests"] = sim.requests(0)
        if logs:
            out["log"] = sim.log(0)
            out["c_chunk"] = int(pt.exp.cluster.c_chunk)
        return out
    finally:
        sim.close()


# ----------------------------------------------------------------- allocators
def allocate_one(pending, new, caps, n_limit, hits=None):
    """One allocate_batch call from host arrays (sbs_prefill_allocate_one):
    pending/new rows (id, prompt_len, wait_cycles); returns the same dict as
    allocate_batch's windows."""
    p = np.asarray(pending, np.int64).reshape(-1, 3)
    q = np.asarray(new, np.int64).reshape(-1, 3)
    rows = np.ascontiguousarray(np.concatenate([p, q]) if len(p) + len(q) else np.zeros((0, 3), np.int64))
    caps = np.array(caps, np.int64)
    n, D = len(rows), len(caps)
    h = None if hits is None else np.ascontiguousarray(np.asarray(hits, np.int64).reshape(n, D))
    dp, rk, wo = (np.zeros(max(n, 1), np.int32) for _ in range(3))
    flow = C.c_uint8(0)
    _check(lib().sbs_prefill_allocate_one(rows.ctypes.data, len(p), len(q), caps.ctypes.data, D,
                                          int(n_limit), h.ctypes.data if h is not None else None,
                                          dp.ctypes.data, rk.ctypes.data, wo.ctypes.data,
                                          C.byref(flow)))
    placed = np.nonzero(dp[:n] >= 0)[0]
    placed = placed[np.argsort(rk[placed], kind="stable")]
    ids = rows[:, 0]
    return {"mapping": np.stack([ids[placed], dp[placed]], 1) if len(placed) else np.zeros((0, 2), np.int64),
            "deferred": np.stack([ids[dp[:n] == -1], wo[:n][dp[:n] == -1]], 1)
            if (dp[:n] == -1).any() else np.zeros((0, 2), np.int64),
            "throttled": ids[dp[:n] == -2], "caps": caps, "flow": bool(flow.value)}


def allocate_batch(windows, device="cuda"):
    """Batched allocate_batch (prefill_alloc.cpp:61-88).

    windows: list of dicts {pending: (k,3) int array of (id, prompt_len,
    wait_cycles), new: (k,3), caps: [c_avail per DP], n_limit} and, for the
    cache-aware mode, hits: (k_pending + k_new, D) Len_hit(r, d).
    Returns per window {mapping: [(id, dp)] in placement order, deferred:
    [(id, wait)], throttled: [id], caps: working capacities, flow: bool}.
    """
    import torch
    req_off, dp_off, npend, nlim = [0], [0], [], []
    ids, lens, waits, caps = [], [], [], []
    for w in windows:
        p = np.asarray(w["pending"], np.int64).reshape(-1, 3)
        q = np.asarray(w["new"], np.int64).reshape(-1, 3)
        allr = np.concatenate([p, q]) if len(p) + len(q) else np.zeros((0, 3), np.int64)
        ids.append(allr[:, 0]); lens.append(allr[:, 1]); waits.append(allr[:, 2])
        npend.append(len(p)); nlim.append(int(w["n_limit"]))
        req_off.append(req_off[-1] + len(allr))
        caps.append(np.asarray(w["caps"], np.int64)); dp_off.append(dp_off[-1] + len(w["caps"]))
    dev = torch.device(device)
    T = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)
    t_req_off, t_dp_off = T(req_off, torch.int64), T(dp_off, torch.int64)
    t_np, t_nl = T(npend, torch.int32), T(nlim, torch.int32)
    t_id, t_len = T(cat(ids), torch.int64), T(cat(lens), torch.int64)
    t_wait, t_caps = T(cat(waits), torch.int32), T(cat(caps), torch.int64)
    total = req_off[-1]
    t_dp = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    t_rank = torch.empty_like(t_dp)
    t_wout = torch.empty_like(t_dp)
    t_flow = torch.empty(max(len(windows), 1), dtype=torch.uint8, device=dev)
    t_hoff = t_hit = None
    if any("hits" in w for w in windows):
        hoff, hits = [0], []
        for w, n0, n1, d0, d1 in zip(windows, req_off, req_off[1:], dp_off, dp_off[1:]):
            h = np.asarray(w.get("hits", np.zeros((n1 - n0, d1 - d0))), np.int64)
            h = h.reshape(n1 - n0, d1 - d0)
            hits.append(h.ravel())
            hoff.append(hoff[-1] + h.size)
        t_hoff, t_hit = T(hoff, torch.int64), T(cat(hits), torch.int64)
    b = WindowBatch(n_windows=len(windows), req_off=t_req_off.data_ptr(), n_pending=t_np.data_ptr(),
                    dp_off=t_dp_off.data_ptr(), n_limit=t_nl.data_ptr(), req_id=t_id.data_ptr(),
                    prompt_len=t_len.data_ptr(), wait_in=t_wait.data_ptr(),
                    caps=t_caps.data_ptr(), out_dp=t_dp.data_ptr(), out_rank=t_rank.data_ptr(),
                    wait_out=t_wout.data_ptr(), flow=t_flow.data_ptr(),
                    hit_off=t_hoff.data_ptr() if t_hoff is not None else None,
                    hit=t_hit.data_ptr() if t_hit is not None else None,
                    max_requests=max(np.diff(req_off).max(initial=0), 1),
                    max_dp=max(np.diff(dp_off).max(initial=0), 1))
    stream = torch.cuda.current_stream(dev).cuda_stream
    _check(lib().sbs_prefill_allocate(C.byref(b), C.c_void_p(stream)))
    o_dp, o_rank, o_w = t_dp.cpu().numpy(), t_rank.cpu().numpy(), t_wout.cpu().numpy()
    o_caps, o_flow = t_caps.cpu().numpy(), t_flow.cpu().numpy()
    all_ids = cat(ids)
    out = []
    for i, w in enumerate(windows):
        r0, r1 = req_off[i], req_off[i + 1]
        sl = slice(r0, r1)
        dpv, rk, wv, idv = o_dp[sl], o_rank[sl], o_w[sl], all_ids[sl]
        placed = np.nonzero(dpv >= 0)[0]
        placed = placed[np.argsort(rk[placed], kind="stable")]
        mapping = np.stack([idv[placed], dpv[placed]], 1) if len(placed) else np.zeros((0, 2), np.int64)
        dmask = np.nonzero(dpv == -1)[0]  # input order: pending first, then new
        deferred = np.stack([idv[dmask], wv[dmask]], 1) if len(dmask) else np.zeros((0, 2), np.int64)
        throttled = idv[dpv == -2]
        out.append({"mapping": mapping.astype(np.int64), "deferred": deferred.astype(np.int64),
                    "throttled": throttled.astype(np.int64),
                    "caps": o_caps[dp_off[i]:dp_off[i + 1]].copy(), "flow": bool(o_flow[i])})
    return out


def select_decode_unit(calls, k=1.5, device="cuda"):
    """Batched select_decode_unit (decode_alloc.cpp:38-81).

    calls: list of (batch[], kv[]) arrays.  Returns (pos, fallback, threshold) arrays.
    """
    import torch
    off = [0]
    for b, kv in calls:
        off.append(off[-1] + len(b))
    dev = torch.device(device)
    t_off = torch.as_tensor(off, dtype=torch.int64, device=dev)
    t_b = torch.as_tensor(np.concatenate([np.asarray(b, np.int32) for b, _ in calls]),
                          dtype=torch.int32, device=dev)
    t_k = torch.as_tensor(np.concatenate([np.asarray(kv, np.int64) for _, kv in calls]),
                          dtype=torch.int64, device=dev)
    n = len(calls)
    t_pos = torch.empty(n, dtype=torch.int32, device=dev)
    t_fb = torch.empty(n, dtype=torch.uint8, device=dev)
    t_th = torch.empty(n, dtype=torch.float64, device=dev)
    b = DecodeBatch(n_calls=n, max_units=max(np.diff(off).max(initial=0), 1),
                    unit_off=t_off.data_ptr(), batch=t_b.data_ptr(), kv=t_k.data_ptr(),
                    k=float(k), pos_out=t_pos.data_ptr(), fallback_out=t_fb.data_ptr(),
                    threshold_out=t_th.data_ptr())
    stream = torch.cuda.current_stream(dev).cuda_stream
    _check(lib().sbs_decode_select(C.byref(b), C.c_void_p(stream)))
    return t_pos.cpu().numpy(), t_fb.cpu().numpy().astype(bool), t_th.cpu().numpy()


class DecodeSchedule(C.Structure):
    _fields_ = [("n_batches", C.c_int32), ("max_candidates", C.c_int32),
                ("max_units", C.c_int32), ("_pad", C.c_int32), ("cand_off", C.c_void_p),
                ("request_id", C.c_void_p), ("sort_len", C.c_void_p), ("kv_len", C.c_void_p),
                ("unit_off", C.c_void_p), ("batch", C.c_void_p), ("kv", C.c_void_p),
                ("k", C.c_double), ("order_out", C.c_void_p), ("pos_out", C.c_void_p),
                ("fallback_out", C.c_void_p), ("threshold_out", C.c_void_p)]


def schedule_decode_batch(batches, k=1.5, device="cuda"):
    """Batched schedule_decode_batch (decode_alloc.cpp:83-106), one warp per batch.

    batches: list of (candidates[(request_id, sort_len, kv_len)], batch[], kv[]).
    Returns, per batch, a dict: placements (request_id, unit position) in
    placement order, threshold / fallback per placement, and the units'
    batch / kv after the call (the reference mutates its units in place)."""
    import torch
    dev = torch.device(device)
    co, uo = [0], [0]
    rows, bs, ks = [], [], []
    for cands, b, kv in batches:
        c = np.asarray(cands, np.int64).reshape(-1, 3)
        rows.append(c)
        bs.append(np.asarray(b, np.int32))
        ks.append(np.asarray(kv, np.int64))
        co.append(co[-1] + len(c))
        uo.append(uo[-1] + len(b))
    allc = np.concatenate(rows) if rows else np.zeros((0, 3), np.int64)
    M = max(1, co[-1])
    t = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x), dtype=dt, device=dev)
    t_co, t_uo = t(co, torch.int64), t(uo, torch.int64)
    t_id = t(allc[:, 0] if len(allc) else np.zeros(1, np.int64), torch.int64)
    t_sl = t(allc[:, 1] if len(allc) else np.zeros(1, np.int64), torch.int64)
    t_kl = t(allc[:, 2] if len(allc) else np.zeros(1, np.int64), torch.int64)
    t_b = t(np.concatenate(bs) if uo[-1] else np.zeros(1, np.int32), torch.int32)
    t_k = t(np.concatenate(ks) if uo[-1] else np.zeros(1, np.int64), torch.int64)
    t_ord = torch.empty(M, dtype=torch.int32, device=dev)
    t_pos = torch.empty(M, dtype=torch.int32, device=dev)
    t_fb = torch.empty(M, dtype=torch.uint8, device=dev)
    t_th = torch.empty(M, dtype=torch.float64, device=dev)
    s = DecodeSchedule(n_batches=len(batches),
                       max_candidates=max([len(r) for r in rows] + [1]),
                       max_units=max([len(b) for b in bs] + [1]),
                       cand_off=t_co.data_ptr(), request_id=t_id.data_ptr(),
                       sort_len=t_sl.data_ptr(), kv_len=t_kl.data_ptr(), unit_off=t_uo.data_ptr(),
                       batch=t_b.data_ptr(), kv=t_k.data_ptr(), k=float(k),
                       order_out=t_ord.data_ptr(), pos_out=t_pos.data_ptr(),
                       fallback_out=t_fb.data_ptr(), threshold_out=t_th.data_ptr())
    stream = torch.cuda.current_stream(dev).cuda_stream
    _check(lib().sbs_decode_schedule_batch(C.byref(s), C.c_void_p(stream)))
    ordv, pos = t_ord.cpu().numpy(), t_pos.cpu().numpy()
    fb, th = t_fb.cpu().numpy().astype(bool), t_th.cpu().numpy()
    b_after, k_after = t_b.cpu().numpy(), t_k.cpu().numpy()
    out = []
    for i in range(len(batches)):
        c0, c1, u0, u1 = co[i], co[i + 1], uo[i], uo[i + 1]
        ids = allc[c0:c1, 0][ordv[c0:c1]] if c1 > c0 else np.zeros(0, np.int64)
        out.append({"placements": np.stack([ids, pos[c0:c1].astype(np.int64)], 1)
                    if c1 > c0 else np.zeros((0, 2), np.int64),
                    "threshold": th[c0:c1], "fallback": fb[c0:c1],
                    "batch": b_after[u0:u1], "kv": k_after[u0:u1]})
    return out
