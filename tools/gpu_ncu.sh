#!/bin/bash
# ncu --set full of the per-view kernels (one launch each, view 2 of C4, Morton layout)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:"${1:-k_raster|k_backward|k_count|k_emit}" -s ${2:-4} -c ${3:-4} \
    -o gpurun_out/full python tools/prof_views.py --views 2 --order morton > gpurun_out/full.log 2>&1
tail -3 gpurun_out/full.log
