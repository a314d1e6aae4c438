"""CPU: the N>1 host logic (sharding, summary all-reduce, per-point gather)
with world_size 2 over gloo.  The NCCL leg runs in bench.py on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2512_16134_b200 import sweep


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_aggs(indices):
    out = []
    for i in indices:
        a = {k: 0 for k in sweep.SUM_KEYS}
        a.update({"generated": 1000 + i, "completed": 900 + i, "window_requests": 800 + i,
                  "ttft_sum_ns": 10**9 * (i + 1), "alloc_calls": 7 * i, "events": 3 * i})
        a.update({k: float(i) for k in sweep.POINT_KEYS if k not in a})
        a["error"] = 0
        out.append(a)
    return out


def _worker(rank, world, port, n_points, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = sweep.shard_indices(n_points, rank, world)
    aggs = _fake_aggs(idx)
    vec = sweep.all_reduce_summary(sweep.summary_vector(aggs))
    pts = sweep.gather_points(aggs, n_points, rank, world)
    q.put((rank, vec.tolist(), [p["generated"] if p else None for p in pts]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partition():
    items = list(range(37))
    parts = [sweep.shard(items, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == items
    assert all(len(p) in (9, 10) for p in parts)
    assert parts[1][:3] == [1, 5, 9]


@pytest.mark.parametrize("n_points", [5, 8])
def test_gloo_world2_reduce_and_gather(n_points):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_points, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = sweep.summary_vector(_fake_aggs(range(n_points)))
    for rank, vec, gen in res:
        assert np.array_equal(np.asarray(vec), want)  # identical on every rank
        assert gen == [1000 + i for i in range(n_points)]  # global point order
    s = sweep.unpack_summary(want)
    assert s["generated"] == sum(1000 + i for i in range(n_points))
