#!/usr/bin/env python
"""Times trips_knn_sizes on the C4 cloud (8M points, generator and Morton order).

  python tools/knn_time.py [--n N]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import knn_sizes, morton_order  # noqa: E402
from synth import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=None)
args = ap.parse_args()
sc = scenes.make_config("C4", n=args.n, n_views=1)
dev = torch.device("cuda:0")
pos = torch.from_numpy(np.ascontiguousarray(sc.pos)).to(dev)
for name, p in (("generator", pos), ("morton", pos[morton_order(pos)].contiguous())):
    knn_sizes(p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        knn_sizes(p)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"knn {name} order: n={p.shape[0]} {ms:.2f} ms ({p.shape[0] / ms / 1e3:.1f} M points/s)")
