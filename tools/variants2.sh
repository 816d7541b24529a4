#!/bin/bash
# Time prebuilt library variants (build/var/*.so) on C4: per-stage us per view (Morton order).
# usage (on the GPU box): bash tools/variants2.sh base reg u1 ...
for name in "$@"; do
  TRIPS_LIB=build/var/$name.so python tools/stage_times.py --views 8 --order lib-morton --label $name
done
