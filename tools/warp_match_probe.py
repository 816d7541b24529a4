#!/usr/bin/env python
"""How much would warp-aggregated gradient reductions save?  For one C4 view, per warp of a
tile (2 pixel rows x 16) and per kept-list position m: distinct point ids among the lanes
whose list reaches m, vs the number of such lanes (= reductions issued today)."""
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
perm = morton_order(d[0])
d = [a[perm].contiguous() for a in d]
r.project(cam, *d)
r.forward(save=True)
kept = r.export_kept().cpu().numpy()
W, H = cam.width, cam.height
off = 0
tot_lanes = tot_same_m = tot_pairs = 0
for l in range(sc.n_layers):
    h, w = -(-H // (1 << l)), -(-W // (1 << l))
    K = kept[off:off + h * w].reshape(h, w, 16)
    off += h * w
    hp, wp = -(-h // 16) * 16, -(-w // 16) * 16
    Kp = np.full((hp, wp, 16), -1, np.int64)
    Kp[:h, :w] = K
    # warps: tile rows of 2 x 16 pixels -> (hp/2, wp/16) groups of 32 lanes
    g = Kp.reshape(hp // 2, 2, wp // 16, 16, 16).transpose(0, 2, 4, 1, 3).reshape(-1, 16, 32)  # [warp, m, lane]
    valid = g >= 0
    tot_lanes += int(valid.sum())
    # distinct ids per (warp, m)
    s = np.sort(np.where(valid, g, -1), axis=2)
    distinct = ((s[:, :, 1:] != s[:, :, :-1]) & (s[:, :, 1:] >= 0)).sum(2) + (s[:, :, 0] >= 0)
    tot_same_m += int(distinct.sum())
    # distinct ids per warp over all m (the best any per-warp aggregation can do)
    gw = g.reshape(g.shape[0], -1)
    sw_ = np.sort(gw, axis=1)
    tot_pairs += int((((sw_[:, 1:] != sw_[:, :-1]) & (sw_[:, 1:] >= 0)).sum(1) + (sw_[:, 0] >= 0)).sum())
print({"kept_fragments": tot_lanes, "warp_aggregated_same_m": tot_same_m,
       "warp_aggregated_any_m": tot_pairs, "ratio_same_m": tot_lanes / tot_same_m,
       "ratio_any_m": tot_lanes / tot_pairs})
