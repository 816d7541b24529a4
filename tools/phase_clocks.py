#!/usr/bin/env python
"""k_raster per-phase clock shares (experiment build with -DTRIPS_PHASE_CLOCK).

  python paper_2401_06003_b200/build.py --out /tmp/pc.so -DTRIPS_PHASE_CLOCK
  TRIPS_LIB=/tmp/pc.so python tools/phase_clocks.py [--order lib-morton]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Rasterizer, _abi, morton_order  # noqa: E402
from synth import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", default="lib-morton")
ap.add_argument("--views", type=int, default=4)
args = ap.parse_args()
sc = scenes.make_config("C4", order="random")
dev = torch.device("cuda:0")
cam0 = sc.cams[0]
r = Rasterizer(cam0.width, cam0.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
if args.order == "lib-morton":
    perm = morton_order(d[0])
    d = [a[perm].contiguous() for a in d]
fn = _abi.lib().trips_debug_phase_clocks
fn.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 8)()
for v in range(args.views):
    r.project(sc.cams[v], *d)
    r.forward(save=True)
torch.cuda.synchronize()
fn(buf, 1)
for v in range(args.views):
    r.project(sc.cams[v], *d)
    r.forward(save=True)
torch.cuda.synchronize()
fn(buf, 1)
names = ["A (fragments, ranks)", "scan", "B (scatter)", "C (sort/merge)", "kept keys to smem", "D (blend)",
         "E (store)", "F (kept pairs)"]
vals = np.array(list(buf)[:8], dtype=np.float64)
tot = vals.sum()
print(os.environ.get("TRIPS_LIB", "in-tree"), f"total {tot:.4g} CTA-cycles")
for n, v in zip(names, vals):
    print(f"{n:22s} {100 * v / tot:5.1f}%")
