"""Write profiles/<tag>_ncu_des_summary.txt from gpurun_out/prof_des_<tag>.ncu-rep and the
launch list gpurun_out/launches_<tag>.csv (scripts/profile_run.sh <tag>).  Also prints the
DRAM bytes per request for profiles/traffic.json.  Usage: ncu_summary.py TAG REQUESTS"""
import collections, csv, subprocess, sys
tag, nreq = sys.argv[1], int(sys.argv[2])
rep = f"gpurun_out/prof_des_{tag}.ncu-rep"
run = lambda *a: subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
r = list(csv.reader(run("--page", "raw", "--csv").splitlines())); d = dict(zip(r[0], r[2]))
det = run("--page", "details").splitlines()
keys = ["Memory Throughput", "DRAM Throughput", "Duration", "Executed Ipc Active", "Issue Slots Busy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Executed Instructions ", "Block Size", "Cluster Size ", "Grid Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy",
        "Achieved Active Warps Per SM"]
seen, lines = set(), []
for l in det:
    s = " ".join(l.split())
    if any(s.startswith(k.strip()) for k in keys) and s not in seen:
        seen.add(s); lines.append(s)
rb, wb = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
st = []
for k in r[0]:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio"):
        try: st.append((float(d[k]), k))
        except ValueError: pass
tt = sum(x for x, _ in st)
rows = [x for x in csv.reader(open(f"gpurun_out/launches_{tag}.csv")) if len(x) > 10 and x[0].isdigit()]
t = collections.defaultdict(float)
for x in rows: t[x[4].split("(")[0]] += float(x[-1])
tot = sum(t.values())
with open(f"profiles/{tag}_ncu_des_summary.txt", "w") as f:
    f.write(f"# ncu --set full --clock-control none, {d['Kernel Name']}, cfg5 slice: 512 replicas x 20 s "
            f"({nreq:,} requests), B200\n# command: scripts/profile_run.sh {tag}\n")
    f.write("\n".join(lines) + "\n\n")
    f.write(f"# dram bytes (read+write) per launch: {rb:.1f} MB + {wb:.1f} MB = {rb + wb:.1f} MB = "
            f"{(rb + wb) * 1e6 / nreq:.1f} B/request (algorithmic: 16 B/request)\n")
    f.write("# launch list of the same command (profiles/" + f"{tag}_ncu_launches_cfg5_slice.csv): "
            + ", ".join(f"{k} {100 * v / tot:.2f} %" for k, v in t.items()) + "\n\n")
    f.write("# warp-stall ratios per issued instruction (smsp__average_warps_issue_stalled_*)\n")
    f.write(", ".join("%s %.2f (%.0f%%)" % (k.replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", ""), x, 100 * x / tt)
                      for x, k in sorted(st, reverse=True)[:10]) + "\n")
    f.write(f"# shared-memory bank conflicts: {float(d['l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']) / 1e6:.1f} M"
            f" over {float(d['smsp__sass_inst_executed_op_shared_ld.sum']) / 1e6:.1f} M shared loads\n")
    # the two CTAs of a cluster run different roles: the busiest SMs are the
    # decode SMs (the critical path), the least busy the prefill SMs
    f.write("# issue slots busy per SM (sm__issue_active.{avg,max,min}): "
            f"avg {float(d['sm__issue_active.avg.pct_of_peak_sustained_elapsed']):.1f} %, "
            f"max {float(d['sm__issue_active.max.pct_of_peak_sustained_elapsed']):.1f} % (decode SMs), "
            f"min {float(d['sm__issue_active.min.pct_of_peak_sustained_elapsed']):.1f} % (prefill SMs); "
            f"warp-instructions per request {float(d['smsp__inst_executed.sum']) / nreq:.0f}\n")
print(f"{(rb + wb) * 1e6 / nreq:.2f} B/request")
