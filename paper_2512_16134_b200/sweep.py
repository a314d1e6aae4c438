"""Replica sweeps across GPUs (one process per GPU, torch.distributed).

Replicas are independent, so the data path has no collective:
rank r simulates the points {i : i mod world == r} (interleaving balances the
cost of a grid whose point cost grows with rate and dp_degree).  After the
kernels, one fixed-size int64 buffer of exact sums and TTFT/TPOT histogram bins
is all-reduced (NCCL over NVLink on GPUs, gloo in the CPU tests) — KB-sized and
order-independent, so results are bit-stable for any GPU count — and the
per-point aggregate records are gathered to every rank.
"""
from __future__ import annotations

import numpy as np

SUM_KEYS = ["generated", "completed", "throttled", "in_flight", "window_requests", "passes",
            "decode_steps", "output_tokens", "alloc_calls", "decode_selects", "events",
            "ttft_sum_ns", "sched_sum_ns", "device_sum_ns", "tpot_count"]
HIST_BINS = 64
BUF_LEN = len(SUM_KEYS) + 2 * HIST_BINS


def shard(items, rank: int, world: int):
    """Interleaved shard of a sweep: positions i with i % world == rank."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return [x for i, x in enumerate(items) if i % world == rank]


def shard_indices(n: int, rank: int, world: int):
    return list(range(rank, n, world))


def summary_vector(aggs, hist=None) -> np.ndarray:
    """Exact int64 summary of this rank's replicas (+ histogram bins)."""
    v = np.zeros(BUF_LEN, np.int64)
    for i, k in enumerate(SUM_KEYS):
        v[i] = sum(int(a[k]) for a in aggs)
    if hist is not None:
        v[len(SUM_KEYS):len(SUM_KEYS) + HIST_BINS] = np.asarray(list(hist.ttft), np.int64)
        v[len(SUM_KEYS) + HIST_BINS:] = np.asarray(list(hist.tpot), np.int64)
    return v


def unpack_summary(v) -> dict:
    v = np.asarray(v, np.int64)
    out = {k: int(v[i]) for i, k in enumerate(SUM_KEYS)}
    out["ttft_hist"] = v[len(SUM_KEYS):len(SUM_KEYS) + HIST_BINS].copy()
    out["tpot_hist"] = v[len(SUM_KEYS) + HIST_BINS:].copy()
    if out["window_requests"]:
        out["ttft_mean_s"] = out["ttft_sum_ns"] / 1e9 / out["window_requests"]
    return out


def all_reduce_summary(vec: np.ndarray, device=None, group=None) -> np.ndarray:
    """Sum the int64 summary across ranks (single collective)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(vec, dtype=torch.int64)
    if device is not None:
        t = t.to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


# per-point record: the fields a sweep consumer needs (e.g. find_peak_qps)
POINT_KEYS = ["generated", "completed", "window_requests", "ttft_mean_s", "ttft_p50_s",
              "ttft_p95_s", "chunk_util_mean", "output_tokens_per_s", "kv_sigma_time_avg",
              "alloc_calls", "error"]


def gather_points(aggs, n_total: int, rank: int, world: int, device=None, group=None):
    """All-gather per-point records into global point order (float64 rows)."""
    import torch
    import torch.distributed as dist
    idx = shard_indices(n_total, rank, world)
    per = (n_total + world - 1) // world
    local = np.full((per, 1 + len(POINT_KEYS)), np.nan)
    for r, (i, a) in enumerate(zip(idx, aggs)):
        local[r, 0] = i
        local[r, 1:] = [float(a[k]) for k in POINT_KEYS]
    t = torch.as_tensor(local, dtype=torch.float64)
    if device is not None:
        t = t.to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, t, group=group)
        allrows = torch.cat(parts).cpu().numpy()
    else:
        allrows = t.cpu().numpy()
    out = [None] * n_total
    for row in allrows:
        if np.isnan(row[0]):
            continue
        out[int(row[0])] = dict(zip(POINT_KEYS, row[1:].tolist()))
    return out


def run_sweep(cfgs, rank: int = 0, world: int = 1, device: int = 0, group=None):
    """Simulate this rank's shard of `cfgs` on GPU `device`; returns
    (per-point aggregates for every point, reduced summary dict)."""
    import paper_2512_16134_b200 as P
    mine = shard(cfgs, rank, world)
    pts = [P.experiment_from_config(c) for c in mine]
    traces, tmap, seen = [], [], {}
    for p in pts:
        key = (bytes(p.exp.workload), int(p.exp.seed))
        if key not in seen:
            seen[key] = len(traces)
            traces.append(P.generate_workload(p))
        tmap.append(seen[key])
    aggs, hist = [], None
    if pts:
        sim = P.Simulator(pts, traces, trace_of_point=tmap, device=device)
        try:
            sim.launch()
            aggs, hist = sim.results(histograms=True)
        finally:
            sim.close()
    vec = all_reduce_summary(summary_vector(aggs, hist), device=f"cuda:{device}", group=group) \
        if world > 1 else summary_vector(aggs, hist)
    points = gather_points(aggs, len(cfgs), rank, world, device=f"cuda:{device}", group=group) \
        if world > 1 else gather_points(aggs, len(cfgs), 0, 1)
    return points, unpack_summary(vec)
