#!/bin/bash
# Step throughput vs the number of CUDA streams the views are spread over (short bench runs).
for s in "$@"; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs --no-random-order --streams $s 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams', $s, round(d['value'],1), 'fps e2e', round(d['e2e']['value'],1))"
done
