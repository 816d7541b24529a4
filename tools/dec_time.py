#!/usr/bin/env python
"""Times trips_decode (gated-conv decoder) on a 1080p, 4-layer, F = 4 pyramid -> 3 channels.

  python tools/dec_time.py [--W 1920 --H 1080 --n 4 --F 4 --out 3]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Decoder, Rasterizer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--W", type=int, default=1920)
ap.add_argument("--H", type=int, default=1080)
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--F", type=int, default=4)
ap.add_argument("--out", type=int, default=3)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda:0")
r = Rasterizer(a.W, a.H, a.n, a.F, max_points=16, device=dev)
dec = Decoder(r, a.out)
rng = np.random.default_rng(0)
pyr = torch.from_numpy(rng.normal(0, 0.5, r.pyramid_floats).astype(np.float32)).to(dev)
prm = torch.from_numpy(rng.normal(0, 0.1, dec.param_count).astype(np.float32)).to(dev)
out = dec(prm, pyr)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    dec(prm, pyr, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
alg = 0.0
for l in range(a.n):
    h, w = -(-a.H // (1 << l)), -(-a.W // (1 << l))
    C = a.F + 1 if l == a.n - 1 else 32 + a.F + 1
    alg += 2.0 * h * w * (2 * 32 * C * 9 + 32 * C)
alg += 2.0 * a.H * a.W * 32 * a.out
print(f"decoder {a.W}x{a.H} n={a.n} F={a.F} out={a.out}: {ms:.3f} ms/frame, {1e3 / ms:.1f} frames/s, "
      f"{alg / ms / 1e9:.1f} algorithmic TFLOP/s")
