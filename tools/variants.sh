#!/bin/bash
# Build experiment variants of libtrips.so (flags per variant) and time stages on C4.
# usage (on the GPU box): bash tools/variants.sh "base:" "nored:-DTRIPS_EXP_NORED" ...
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  if [ -z "$flags" ]; then lib=paper_2401_06003_b200/libtrips.so; else
    lib=/tmp/libtrips_$name.so; python paper_2401_06003_b200/build.py --out $lib $flags >/dev/null || continue; fi
  for o in lib-morton random; do TRIPS_LIB=$lib python tools/stage_times.py --views 8 --order $o --label $name; done
done
