#!/bin/bash
# ncu --set full of the DES kernel, two-warp (split) and one-warp replicas, small cfg5 slice.
TAG=${1:-dev}
SMALL="python bench.py --workload cfg5 --replicas 512 --duration 20 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
for sp in ${SPLITS:-1 0}; do
  SBS_SPLIT=$sp $SMALL > gpurun_out/small_plain_${TAG}_s$sp.log 2>&1 && \
  SBS_SPLIT=$sp ncu --set full --clock-control none --import-source on -k regex:'des_.*kernel' -s 1 -c 1 \
     -o gpurun_out/prof_${TAG}_s$sp -f $SMALL > gpurun_out/ncu_${TAG}_s$sp.log 2>&1
  echo "split=$sp rc=$?"
done
