M=sm__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__issue_active.max.pct_of_peak_sustained_elapsed,sm__issue_active.min.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.per_cycle_active,smsp__inst_executed.avg.per_cycle_active
timeout 300 python scripts/range_profile.py > gpurun_out/rp_plain.log 2>&1; echo plain rc=$?; tail -1 gpurun_out/rp_plain.log
timeout 900 ncu --replay-mode app-range --clock-control none --metrics $M --csv --log-file gpurun_out/rp_ncu.csv python scripts/range_profile.py > gpurun_out/rp_ncu.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/rp_ncu.log; cat gpurun_out/rp_ncu.csv | tail -15
