#!/usr/bin/env python
"""Time a batch of C4 views (project -> forward -> backward) with the views spread over k
CUDA streams (one Rasterizer workspace per stream), k = 1, 2, 3, 4.

  python tools/streams_probe.py [--views 32]
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
ap.add_argument("--views", type=int, default=32)
args = ap.parse_args()
sc = scenes.make_config("C4", order="random")
dev = torch.device("cuda:0")
cam0 = sc.cams[0]
d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
perm = morton_order(d[0])
d = [a[perm].contiguous() for a in d]
rasts = [Rasterizer(cam0.width, cam0.height, sc.n_layers, sc.F, max_points=sc.n, device=dev) for _ in range(4)]
G = torch.from_numpy(scenes.grad_pyramid(rasts[0].pyramid_floats)).to(dev)
grad = rasts[0].new_grad(sc.n)
streams = [torch.cuda.Stream() for _ in range(4)]
main = torch.cuda.current_stream()


def step(k):
    grad.zero_()
    ev = torch.cuda.Event()
    ev.record(main)
    for s in streams[:k]:
        s.wait_event(ev)
    for j in range(args.views):
        i = j % k
        with torch.cuda.stream(streams[i]):
            r = rasts[i]
            r.project(sc.cams[j % len(sc.cams)], *d)
            r.forward(save=True)
            r.backward(G, grad)
    for s in streams[:k]:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


for k in (1, 2, 3, 4, 1, 2):
    for _ in range(2):
        step(k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(3):
        step(k)
    b.record(main)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(json.dumps({"streams": k, "ms_per_batch": ms, "us_per_view": 1e3 * ms / args.views}), flush=True)
