#!/bin/bash
# A/B of full library builds on the bench step (same box, alternating): bash tools/gpu_ab.sh a b ...
for rep in 1 2; do
  for v in "$@"; do
    TRIPS_LIB=build/var/$v.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-random-order 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'clk', d.get('clocks'), {k: round(v['ms_in_step'],4) for k, v in d['kernels'].items()})"
  done
done
