"""One profiler range around a single DES launch of the cfg5 slice (dev tool).

ncu's default kernel replay serialises kernels, so the default pair mode 3
(two co-resident kernels talking through HBM) cannot be captured per kernel.
Application-range replay profiles the whole range with both kernels running
concurrently:

  ncu --replay-mode app-range --profile-from-start off --clock-control none \
      --metrics sm__inst_executed.sum,... python scripts/range_profile.py
"""
import sys

sys.path.insert(0, ".")
import torch

import bench
import paper_2512_16134_b200 as P

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dur = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
desc, cfgs = bench.workload_points("cfg5", 0, 1, reps, dur)
pts = [P.experiment_from_config(c) for c in cfgs]
trs = [P.generate_workload(p) for p in pts]
sim = P.Simulator(pts, trs)
for _ in range(2):
    sim.launch()
    sim.results()
rt = torch.cuda.cudart()
torch.cuda.synchronize()
rt.cudaProfilerStart()
sim.launch()
torch.cuda.synchronize()
rt.cudaProfilerStop()
res = sim.results()
print(desc, "requests", sum(r["generated"] for r in res))
