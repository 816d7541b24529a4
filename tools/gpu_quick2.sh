#!/bin/bash
# tests + per-stage times (C4 Morton / random), one gpurun call
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for o in lib-morton random; do python tools/stage_times.py --views 8 --order $o; done
