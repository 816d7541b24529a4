#!/usr/bin/env python
"""Renders `--views` views of one config (library Morton layout, forward+backward unless the config
is forward only) for an ncu DRAM-traffic capture of the per-view kernels.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      python tools/traffic_views.py --config C4 --views 3
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Rasterizer, morton_order  # noqa: E402
from synth import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--views", type=int, default=3)
args = ap.parse_args()
sc = scenes.make_config(args.config)
dev = torch.device("cuda:0")
cam = sc.cams[0]
d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
perm = morton_order(d[0])
d = [a[perm].contiguous() for a in d]
r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
bwd = not sc.forward_only
G = torch.from_numpy(scenes.grad_pyramid(r.pyramid_floats)).to(dev)
grad = r.new_grad(sc.n)
for v in range(args.views):
    r.project(sc.cams[v % len(sc.cams)], *d)
    r.forward(save=bwd)
    if bwd:
        r.backward(G, grad)
torch.cuda.synchronize()
print(args.config, r.stats())
