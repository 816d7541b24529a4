#!/bin/bash
# per-kernel DRAM bytes per launch for C2, C3, C4, C5 (ncu, cold-ish: views after 2 warm-up views)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
specs=""
for cfg in C4 C2 C3 C5; do
  skip=10; [ $cfg = C2 ] && skip=8                 # the first two views' launches are warm-up
  ncu -s $skip --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"k_count|k_tscan|k_emit|k_raster|k_backward" --csv --log-file gpurun_out/traffic_$cfg.csv \
      python tools/traffic_views.py --config $cfg --views 4 > gpurun_out/traffic_$cfg.log 2>&1
  specs="$specs $cfg=gpurun_out/traffic_$cfg.csv"
done
python tools/traffic_json.py gpurun_out/dram_traffic_r02.json $specs
