#!/usr/bin/env python
"""Per-stage device times (CUDA events inside libtrips) for a few C4 views.

  python tools/stage_times.py [--views 8] [--order lib-morton|random] [--label X]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Rasterizer, morton_order  # noqa: E402
from synth import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=8)
ap.add_argument("--order", default="lib-morton")
ap.add_argument("--config", default="C4")
ap.add_argument("--label", default="")
args = ap.parse_args()
sc = scenes.make_config(args.config, order="random")
dev = torch.device("cuda:0")
cam0 = sc.cams[0]
r = Rasterizer(cam0.width, cam0.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
if args.order == "lib-morton":
    perm = morton_order(d[0])
    d = [a[perm].contiguous() for a in d]
G = torch.from_numpy(scenes.grad_pyramid(r.pyramid_floats)).to(dev)
grad = r.new_grad(sc.n)


def run(nv):
    for v in range(nv):
        cam = sc.cams[v % len(sc.cams)]
        r.project(cam, *d)
        r.forward(save=not sc.forward_only)
        if not sc.forward_only:
            r.backward(G, grad)


run(3)
torch.cuda.synchronize()
r.stage_ms(reset=True)
r.set_profiling(True)
run(args.views)
torch.cuda.synchronize()
st = r.stage_ms(reset=True)
out = {k: round(v[0] / args.views * 1000, 1) for k, v in st.items()}
out["total_us"] = round(sum(out.values()), 1)
print(json.dumps({"label": args.label, "order": args.order, "config": args.config, "us_per_view": out}))
