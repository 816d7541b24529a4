#!/usr/bin/env python
"""Distribution of per-warp maximum list lengths (2 pixel rows x 16 of a tile) for one C4 view:
which sorting-network sizes would the raster kernel's warps need."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Rasterizer, morton_order  # noqa: E402
from synth import scenes  # noqa: E402

sc = scenes.make_config("C4", order="random")
dev = torch.device("cuda:0")
cam = sc.cams[0]
r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
r.project(cam, *d)
r.forward(save=True)
cnt = r.export_counts().cpu().numpy().astype(np.int64)
W, H = cam.width, cam.height
off = 0
allmax = []
for l in range(sc.n_layers):
    h, w = -(-H // (1 << l)), -(-W // (1 << l))
    c = cnt[off:off + h * w].reshape(h, w)
    off += h * w
    hp, wp = -(-h // 16) * 16, -(-w // 16) * 16
    cp = np.zeros((hp, wp), np.int64)
    cp[:h, :w] = c
    g = cp.reshape(hp // 2, 2, wp // 16, 16).transpose(0, 2, 1, 3).reshape(-1, 32)
    mx = g.max(1)
    allmax.append(mx)
    print("layer", l, "pixels", h * w, "mean list", c.mean().round(2),
          "warp-max pct <=4/8/12/16/32:", [round(float((mx <= k).mean()) * 100, 1) for k in (4, 8, 12, 16, 32)])
mx = np.concatenate(allmax)
print("all warps", mx.size, "pct <=4/8/12/16/32:", [round(float((mx <= k).mean()) * 100, 1) for k in (4, 8, 12, 16, 32)])
