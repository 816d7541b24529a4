#!/bin/bash
# Full measurement pass (one gpurun call): tests, smoke, bench (default flags), the ncu launch
# list of the same bench command, and an ncu --set full capture of the two dominant kernels.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-random-order > gpurun_out/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_raster|k_backward|k_count|k_emit" -s 4 -c 4 \
    -o gpurun_out/full python tools/prof_views.py --views 2 --order morton > gpurun_out/full.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
lscpu | grep -E "Model name|^CPU\(s\)"
