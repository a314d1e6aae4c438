#!/bin/bash
for sp in ${SPLITS:-0 1 2 0 1 2}; do
  for w in "cfg5 --replicas 512 --duration 100" "cfg3" "cfg1"; do
    SBS_SPLIT=$sp timeout 300 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$sp', '$w'.split()[0], round(d['value']/1e6,2), 'launches', d['gpu_launches'])"
  done
done
