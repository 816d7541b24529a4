python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for o in random lib-morton; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --order $o > gpurun_out/b_$o.json 2>gpurun_out/b_$o.err; tail -2 gpurun_out/b_$o.err; python -c "
import json; d=json.load(open('gpurun_out/b_$o.json')); print('$o', round(d['value'],1), 'fps', {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'e2e', round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3))"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python tools/prof_views.py --views 3 > gpurun_out/pv.log 2>&1
