#!/bin/bash
# One exploratory gpurun call: GPU tests, list-length probe, k_raster phase clocks, and the
# per-stage times of prebuilt variants (build/var/<name>.so, FC4-only experiment builds).
# usage: bash tools/gpu_explore.sh [tests] [probe] -- base v1 v2 ...
[ "$1" = nobuild ] && shift || { python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1; }
for a in "$@"; do
  case "$a" in
    tests) timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 ;;
    ptest:*) v=${a#ptest:}; TRIPS_LIB=build/var/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q \
        -k "c1 or tiny or adversarial or dense or empty or deterministic or multi_view or batch_step or full_size or whole or tmin or coarse or camera" 2>&1 | grep -E "passed|failed|FAILED|Error" | head -30 ;;
    probe) python tools/count_probe.py ;;
    knnncu) ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_knn|k_sort|k_bbox" -c 22 --csv \
        --log-file gpurun_out/knn_launches.csv python tools/knn_time.py > /dev/null 2>&1; echo "knnncu rc=$?" ;;
    knnst) TRIPS_LIB=build/var/knnst.so python tools/knn_stats.py ;;
    dectest:*) v=${a#dectest:}; TRIPS_LIB=build/var/$v.so timeout 900 python -m pytest tests/test_gpu_decoder.py -q -x 2>&1 | tail -15 ;;
    knntime:*) v=${a#knntime:}; TRIPS_LIB=build/var/$v.so python tools/knn_time.py ;;
    dectime:*) v=${a#dectime:}; TRIPS_LIB=build/var/$v.so python tools/dec_time.py; TRIPS_LIB=build/var/$v.so python tools/dec_time.py --W 3840 --H 2160 ;;
    knntest:*) v=${a#knntest:}; TRIPS_LIB=build/var/$v.so timeout 900 python -m pytest tests/test_gpu_knn.py -q 2>&1 | tail -3 ;;
    decncu:*) v=${a#decncu:}; TRIPS_LIB=build/var/$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dec" -c 12 --csv \
        --log-file gpurun_out/dec_launches.csv python tools/dec_time.py --iters 1 > /dev/null 2>&1; echo "decncu rc=$?" ;;
    decfull:*) v=${a#decfull:}; TRIPS_LIB=build/var/$v.so ncu --set full --clock-control none --import-source on -k regex:"k_dec_conv" -s 3 -c 1 \
        -o gpurun_out/ncu_dec -f python tools/dec_time.py --iters 1 > /dev/null 2>&1; echo "decfull rc=$?" ;;
    knn) timeout 900 python -m pytest tests/test_gpu_knn.py -q 2>&1 | tail -5; python tools/knn_time.py ;;
    ncu:*) v=${a#ncu:}; k=${NCU_K:-k_raster}; TRIPS_LIB=build/var/$v.so ncu --set full --clock-control none --import-source on \
        -k regex:$k -s 1 -c 1 -o gpurun_out/ncu_$v -f python tools/prof_views.py --views 2 --order morton > /dev/null 2>&1; echo "ncu $v rc=$?" ;;
    pc*) TRIPS_LIB=build/var/$a.so python tools/phase_clocks.py ;;
    *) TRIPS_LIB=build/var/$a.so python tools/stage_times.py --views 8 --order lib-morton --label $a ;;
  esac
done
# ncu:<variant> -> gpurun_out/ncu_<variant>.ncu-rep (k_raster, one launch, --set full with source)
