python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_q.json 2>gpurun_out/b_q.err; tail -2 gpurun_out/b_q.err
python -c "
import json; d=json.load(open('gpurun_out/b_q.json')); print(round(d['value'],1), 'fps', {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'e2e', round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), 'random', d.get('random_point_order'))"
