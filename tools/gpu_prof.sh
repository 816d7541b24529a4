#!/bin/bash
# One ncu --set full capture of the four per-view kernels (one launch each, view 2 of C4,
# Morton layout) plus the k_raster per-phase clock shares; reports land in gpurun_out/.
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_raster|k_backward|k_count|k_emit" -s 4 -c 4 \
    -o gpurun_out/full python tools/prof_views.py --views 2 --order morton > gpurun_out/full.log 2>&1
tail -2 gpurun_out/full.log
python paper_2401_06003_b200/build.py --out /tmp/pc.so -DTRIPS_PHASE_CLOCK > /dev/null && \
    TRIPS_LIB=/tmp/pc.so python tools/phase_clocks.py > gpurun_out/phase_clocks.txt 2>&1
cat gpurun_out/phase_clocks.txt | tail -12
