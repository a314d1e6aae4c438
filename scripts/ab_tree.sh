#!/bin/bash
# Same-box A/B: the current tree vs a reference copy in ab_base/ (dev tool).
WLS=${WLS:-"cfg1|cfg5 --replicas 512 --duration 100|cfg3"}
IFS='|' read -ra W <<< "$WLS"
for rep in 1 2; do
  for tree in . ab_base; do
    for w in "${W[@]}"; do
      (cd $tree && timeout 300 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tree', '$w'.split()[0], round(d['value']/1e6,2))")
    done
  done
done
