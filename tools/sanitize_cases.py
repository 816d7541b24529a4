#!/usr/bin/env python
"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): C1, the
adversarial scene and a dense-tile scene (several chunks, lists >> 16), each through project ->
forward (saved) -> backward (+ camera gradient) -> SCREEN_GRADS export, plus the T_min and
coarse-layer variants, the kNN / Morton utilities (incl. a clustered, duplicate-heavy cloud: both
kNN query modes) and the gated-conv decoder (TMA + tcgen05; odd sizes, 1 and 3 layers).

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import Decoder, Rasterizer, knn_sizes, morton_order  # noqa: E402
from synth import scenes  # noqa: E402

dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
cases = [("C1", scenes.c1(), {}), ("adversarial", scenes.adversarial_scene(), {}),
         ("dense", scenes.tiny_scene(11, n=30000, F=4, W=40, H=24, n_layers=3), {}),
         ("tmin", scenes.c1(), {"t_min": 0.2}), ("coarse", scenes.tiny_scene(3, n=3000), {"coarse_layers": 2}),
         ("F6", scenes.tiny_scene(5, n=2000, F=6), {})]
for name, sc, kw in cases:
    cam = sc.cams[0]
    r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=max(sc.n, 1), device=dev, **kw)
    pos, sw, al, de = (T(a) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
    r.project(cam, pos, sw, al, de)
    r.forward(save=True)
    G = T(scenes.grad_pyramid(r.pyramid_floats, seed=1))
    gcam = torch.zeros(17, device=dev)
    g = r.backward(G, grad_camera=gcam)
    r.export_counts(); r.export_kept(); r.export_screen_grads()
    torch.cuda.synchronize()
    print(name, r.stats(), float(g.abs().sum()), flush=True)
pos = T(scenes.c1(n=5000).pos)
knn_sizes(pos)
morton_order(pos)
rng = np.random.default_rng(5)
cl = np.concatenate([rng.normal(size=(400, 3)) * 1e-3 + rng.uniform(-5, 5, 3) for _ in range(5)] +
                    [np.repeat([[0.5, 0.5, 0.5]], 300, 0), [[np.nan, 0, 0]]]).astype(np.float32)
knn_sizes(T(cl))
for (W, H, n, F) in ((100, 77, 3, 4), (130, 40, 1, 8)):
    r = Rasterizer(W, H, n, F, max_points=16, device=dev)
    dec = Decoder(r, 3)
    prm = torch.randn(dec.param_count, device=dev) * 0.1
    out = dec(prm, torch.randn(r.pyramid_floats, device=dev))
    print("decoder", W, H, n, F, float(out.abs().sum()), flush=True)
torch.cuda.synchronize()
print("sanitize cases done")
