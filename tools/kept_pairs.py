#!/usr/bin/env python
"""Kept (point, tile) pairs vs kept fragments per C4 view (sizing the pair-wise backward)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Rasterizer, morton_order  # noqa: E402
from synth import scenes  # noqa: E402

sc = scenes.make_config(sys.argv[1] if len(sys.argv) > 1 else "C4", order="random")
dev = torch.device("cuda:0")
cam0 = sc.cams[0]
r = Rasterizer(cam0.width, cam0.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
perm = morton_order(d[0])
d = [a[perm].contiguous() for a in d]
tile_of = []
for l, (h, w, off) in enumerate(r.dims):
    ys, xs = torch.meshgrid(torch.arange(h, device=dev), torch.arange(w, device=dev), indexing="ij")
    tile_of.append((l * 1000000 + (ys // 16) * 1000 + xs // 16).reshape(-1))
tile_of = torch.cat(tile_of).long()
for v in range(3):
    r.project(sc.cams[v], *d)
    r.forward(save=True)
    st = r.stats()
    kept = r.export_kept().long()
    valid = kept >= 0
    t = tile_of[:, None].expand_as(kept)[valid]
    i = kept[valid]
    pairs = torch.unique(t * (1 << 28) + i).numel()
    print(v, "kept frags", int(valid.sum()), "kept pairs", pairs, "all pairs", st["n_pairs"], "ratio", int(valid.sum()) / pairs)
