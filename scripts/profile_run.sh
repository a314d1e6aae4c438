#!/bin/bash
# Usage: scripts/profile_run.sh TAG  — plain default bench, then ncu on a small slice.
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
SMALL="python bench.py --workload cfg5 --replicas 512 --duration 20 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
$SMALL > gpurun_out/small_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $SMALL > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
$SMALL > gpurun_out/small_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-des_.*kernel} -s 1 -c 1 -o gpurun_out/prof_des_${TAG} -f $SMALL > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ls -la gpurun_out
