#!/bin/bash
# A/B on one box: SBS_LIB=A vs B for cfg5 slice and cfg3 (dev tool)
for lib in "$@"; do
  for w in "cfg5 --replicas 512 --duration 100" "cfg3"; do
    SBS_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$w'.split()[0], round(d['value']/1e6,2))"
  done
done
