#!/usr/bin/env python
"""Runs a few C4 views (forward + backward) for ncu launch lists / captures.

  python tools/prof_views.py [--views 3] [--order random|morton] [--config C4]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Rasterizer  # noqa: E402
from synth import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=3)
ap.add_argument("--order", default="random")
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=None)
args = ap.parse_args()
sc = scenes.make_config(args.config, n=args.n, order=args.order)
dev = torch.device("cuda:0")
cam0 = sc.cams[0]
r = Rasterizer(cam0.width, cam0.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
G = torch.from_numpy(scenes.grad_pyramid(r.pyramid_floats)).to(dev)
grad = r.new_grad(sc.n)
for v in range(args.views):
    cam = sc.cams[v % len(sc.cams)]
    r.project(cam, *d)
    r.forward(save=True)
    r.backward(G, grad)
torch.cuda.synchronize()
print(r.stats())
