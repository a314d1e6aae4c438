"""Per-region clock64 breakdown (needs SBS_PROF=1 build; SBS_LIB=.../libsbs_b200_prof.so)."""
import sys, time
sys.path.insert(0, '.')
import bench, paper_2512_16134_b200 as P
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 512
dur = float(sys.argv[3]) if len(sys.argv) > 3 else 50.0
desc, cfgs = bench.workload_points(wl, 0, 1, reps, dur if wl == "cfg5" else None)
pts = [P.experiment_from_config(c) for c in cfgs]
trs = [P.generate_workload(p) for p in pts]
sim = P.Simulator(pts, trs)
sim.launch(); res = sim.results()
sim.launch(); res = sim.results()
c = sim.profile_counters()
n = sum(r["generated"] for r in res)
names = ["select", "arrival", "finish_pass", "finish_step", "drain", "iqr_select", "S_update",
         "rebuild_S", "try_start_pass", "dispatch_chain", "begin_step", "fs.completers",
         "fs.unit_loop", "fs.reduce", "fs.band", "D.n_drains_with_waiters", "D.wait_P(~cyc)", "P.wait_recroom(cyc)",
         "D.n_sorts", "D.admit_book(incl S_upd)", "D.total", "P.total", "sum_np_per_dispatch", "sum_nn"]
ev = sum(r["events"] for r in res)
steps = sum(r["decode_steps"] for r in res)
print("steps/request %.3f (post-warmup)" % (steps / n))
print(desc, "requests", n, "events", ev, "events/req %.2f" % (ev / n))
for i, nm in enumerate(names):
    print(f"{nm:16s} {c[i] / n:10.1f} cycles/request")
