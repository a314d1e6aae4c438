"""Per-region clock64 breakdown for a filtered set of bench points (dev tool;
SBS_PROF=1 build via SBS_LIB).  Usage: prof_points.py WORKLOAD KEY=VALUE (cluster key filter)"""
import sys
sys.path.insert(0, '.')
import bench, paper_2512_16134_b200 as P
wl = sys.argv[1]
key, val = sys.argv[2].split("=")
desc, cfgs = bench.workload_points(wl, 0, 1)
cfgs = [c for c in cfgs if str(c["cluster"].get(key)) == val]
pts = [P.experiment_from_config(c) for c in cfgs]
trs = [P.generate_workload(p) for p in pts]
sim = P.Simulator(pts, trs)
sim.launch(); res = sim.results()
sim.launch(); res = sim.results()
print(len(cfgs), "points,", sim.des_ms(), "ms")
c = sim.profile_counters()
n = sum(r["generated"] for r in res)
names = ["select", "arrival", "finish_pass", "finish_step", "drain", "iqr_select", "S_update",
         "rebuild_S", "try_start_pass", "dispatch_chain", "begin_step", "fs.completers",
         "fs.unit_loop", "fs.reduce", "fs.band", "D.drain_after_step", "D.wait_P", "P.wait_recroom",
         "D.wait_comproom", "P.consume", "D.total", "P.total"]
print("requests", n, "events/req %.2f" % (sum(r["events"] for r in res) / n),
      "alloc_calls/req %.3f" % (sum(r["alloc_calls"] for r in res) / n),
      "passes/req %.3f" % (sum(r["passes"] for r in res) / n))
for i, nm in enumerate(names):
    if c[i]: print(f"{nm:16s} {c[i] / n:10.1f} cycles/request")
