#!/bin/bash
# quick GPU check: parity subset + three bench points
timeout 900 python -m pytest tests -x -q -m gpu -k "not exhaustive and not config5" 2>&1 | tail -3
for w in "cfg5 --replicas 512 --duration 100" "cfg1" "cfg3"; do
  timeout 300 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],1), 'ms')"
done
