#!/bin/bash
# Full measurement pass (one gpurun call): tests, smoke, bench (default flags), the ncu launch
# list of the same bench command, ncu --set full captures of the per-view kernels and of the
# decoder's convolution, and the reference arm.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-random-order --no-configs > gpurun_out/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_raster|k_backward|k_count|k_emit" -s 4 -c 4 \
    -o gpurun_out/full python tools/prof_views.py --views 2 --order morton > gpurun_out/full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dec_conv|k_dec_prep" -s 6 -c 2 \
    -o gpurun_out/ncu_dec_full python tools/dec_time.py --iters 1 > gpurun_out/dec_full.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
lscpu | grep -E "Model name|^CPU\(s\)"
