#!/bin/bash
# Full measurement pass B: ncu --set full (with source) of k_raster and k_backward_pairs (one C4
# view, Morton order) and of the decoder's layer-0 prep + convolution.
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_raster|k_backward" -s 2 -c 2 \
    -o gpurun_out/full_r02 -f python tools/prof_views.py --views 2 --order morton > gpurun_out/full.log 2>&1
echo "raster/backward rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_dec_conv|k_dec_prep" -s 6 -c 2 \
    -o gpurun_out/dec_full_r02 -f python tools/dec_time.py --iters 1 > gpurun_out/dec_full.log 2>&1
echo "decoder rc=$?"
ls -la gpurun_out/*.ncu-rep
