#!/bin/bash
# ncu --set full of the decoder's layer-0 conv (current build/var/$1.so), reduced on the box to CSV
v=${1:-ds4}
TRIPS_LIB=build/var/$v.so ncu --set full --clock-control none --import-source on -k regex:"k_dec_conv" -s 3 -c 1 \
    -o gpurun_out/ncu_dec_$v -f python tools/dec_time.py --iters 1 > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu_dec_$v.ncu-rep --page raw --csv > gpurun_out/dec_conv_raw.csv
ncu -i gpurun_out/ncu_dec_$v.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/dec_conv_src.csv.gz
ncu -i gpurun_out/ncu_dec_$v.ncu-rep --page details --csv > gpurun_out/dec_conv_details.csv
rm -f gpurun_out/ncu_dec_$v.ncu-rep
