#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_runs.py
# with cluster pairs (SBS_SPLIT=2) and one-CTA pairs (SBS_SPLIT=1); logs to gpurun_out/.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for sp in 2 1; do
  for tool in memcheck racecheck synccheck; do
    SBS_SPLIT=$sp timeout 1200 $CS --tool $tool --print-limit 50 python scripts/sanitize_runs.py \
      > gpurun_out/sanitize_${tool}_split${sp}.log 2>&1
    echo "split=$sp $tool rc=$? $(tail -1 gpurun_out/sanitize_${tool}_split${sp}.log)"
  done
done
