"""Dev probe: per-replica speed of the cfg5 slice vs replicas per cluster, with
distinct seeds (independent event chains) or one seed for all replicas (warps
walk the same code in near lockstep: shared instruction-cache lines).
Usage: density_probe.py [duration_s]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_16134_b200 as P  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 50.0
for same in (False, True):
    for R in (148, 296, 444, 518):
        cfgs = [bench.cfg2(seed=11 if same else 11 + i, duration=dur) for i in range(R)]
        sim = P.Simulator([P.experiment_from_config(c) for c in cfgs], None)
        sim.launch(); sim.results()
        torch.cuda.synchronize()
        t = time.perf_counter()
        sim.launch(); res = sim.results()
        dt = time.perf_counter() - t
        n = sum(r["generated"] for r in res)
        print(f"{'same' if same else 'distinct'} seeds, {R} replicas: {n / dt / 1e6:.2f} M sim-req/s, "
              f"{n / dt / R / 1e3:.1f} k per replica", flush=True)
        sim.close()
