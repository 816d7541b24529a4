#!/usr/bin/env python
"""kNN query counters on the C4 cloud (experiment build with -DTRIPS_KNN_STATS):
candidates evaluated, box area (quantisation steps^2, x * y), BIGMIN jumps, queries with a box."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import _abi, knn_sizes  # noqa: E402
from synth import scenes  # noqa: E402

sc = scenes.make_config("C4", n_views=1)
pos = torch.from_numpy(np.ascontiguousarray(sc.pos)).cuda()
fn = _abi.lib().trips_debug_knn_stats
fn.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 4)()
fn(buf, 1)
knn_sizes(pos)
torch.cuda.synchronize()
fn(buf, 1)
n = pos.shape[0]
cand, area, jumps, boxes = list(buf)
print(f"n={n} candidates/query {cand / n:.1f}  boxes {boxes / n:.3f}/query  box area {area / max(boxes, 1):.1f} steps^2"
      f"  BIGMIN jumps/box {jumps / max(boxes, 1):.1f}")
