#!/bin/bash
# Full measurement pass B: ncu --set full (with source) of k_raster, k_backward_pairs (one C4 view,
# Morton order), the decoder's layer-0 prep + convolution and the kNN query; each report is
# reduced on the box to its raw-metric CSV and per-line source CSV (gpurun copies back <= 64 MiB).
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
cap() {   # name, kernel regex, skip, count, command...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c $c -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  echo "$name rc=$?"
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_src.csv 2>/dev/null
  gzip -f gpurun_out/${name}_src.csv
}
cap r02f_raster "k_raster" 1 1 python tools/prof_views.py --views 2 --order morton
cap r02f_backward "k_backward" 1 1 python tools/prof_views.py --views 2 --order morton
cap r02f_dec "k_dec_conv|k_dec_prep" 6 2 python tools/dec_time.py --iters 1
cap r02f_knn "k_knn_query" 0 1 python tools/knn_time.py
ls -la gpurun_out/
