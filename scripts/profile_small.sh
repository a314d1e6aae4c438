#!/bin/bash
# ncu --set full of the DES kernel on a small cfg5 slice (and optional cfg1).
TAG=${1:-dev}
WL=${2:-cfg5}
EXTRA=${3:-"--replicas 512 --duration 20"}
SMALL="python bench.py --workload $WL $EXTRA --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
$SMALL > gpurun_out/small_plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:des_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} -f $SMALL > gpurun_out/ncu_${TAG}.log 2>&1
echo "rc=$?"
