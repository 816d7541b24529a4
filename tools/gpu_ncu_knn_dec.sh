#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
cap() {
  local name=$1 k=$2 s=$3 c=$4; shift 4
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c $c -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  echo "$name rc=$?"
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_src.csv 2>/dev/null
  gzip -f gpurun_out/${name}_src.csv
}
cap r02b_knn "k_knn_query" 0 1 python tools/knn_time.py
cap r02b_dec "k_dec_conv|k_dec_prep" 6 2 python tools/dec_time.py --iters 1
