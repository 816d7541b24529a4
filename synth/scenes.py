"""Synthetic scenes shaped like the paper's workloads (SURVEY.md 8(d) recipe, DESIGN.md
"Input recipe").  numpy PCG64 generators, geometry in float64, cast once to float32.

No method arithmetic lives here (no projection, levels, footprints, blending): the
camera is described only by its intrinsics and a world->view pose.

Configs (BASELINE.json "configs"):
  C1  1k random points, F=4, one 64x64 camera, 4 layers, fwd+bwd
  C2  Tanks&Temples-like, 5M points, 1920x1080, 4 layers, forward only
  C3  Mip-NeRF360-bicycle-like, 6M points, wide sizes, 8 layers, fwd+bwd
  C4  32 views x 8M points (C2-like geometry), 4 layers, fwd+bwd, view-parallel
  C5  large landscape, 25M points, 1920x1080, 8 layers, long lists, fwd+bwd
"""
from dataclasses import dataclass, field
from typing import List

import numpy as np


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    f: float                      # focal length of Eq. (2); = fx when fx == fy (reading Q6)
    R: np.ndarray                 # (3,3) float32 world->view, OpenCV axes (x right, y down, z fwd)
    t: np.ndarray                 # (3,) float32
    width: int
    height: int
    near: float = 0.01


@dataclass
class Scene:
    name: str
    pos: np.ndarray               # (N,3) float32
    sw: np.ndarray                # (N,) float32 world sizes s_w
    alpha: np.ndarray             # (N,) float32 opacities
    desc: np.ndarray              # (N,F) float32 descriptors tau
    cams: List[Camera]
    n_layers: int
    forward_only: bool = False
    meta: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.pos.shape[0]

    @property
    def F(self):
        return self.desc.shape[1]


def look_at(eye, target, width, height, fx, fy=None, up=(0.0, 0.0, 1.0), near=0.01):
    """OpenCV camera at `eye` looking at `target`; world up = +z.  cx = (W-1)/2."""
    fy = fx if fy is None else fy
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    t = -R @ eye
    f = float(np.float32(np.sqrt(np.float64(fx) * np.float64(fy))))
    return Camera(fx=float(np.float32(fx)), fy=float(np.float32(fy)), cx=(width - 1) / 2.0,
                  cy=(height - 1) / 2.0, f=f, R=R.astype(np.float32), t=t.astype(np.float32),
                  width=int(width), height=int(height), near=near)


def _finish(name, pos, sw, rng, F, cams, n_layers, alpha_lo=0.2, forward_only=False, order="random",
            meta=None):
    n = pos.shape[0]
    alpha = rng.uniform(alpha_lo, 1.0, n)
    desc = rng.normal(0.0, 0.5, (n, F))
    if order == "random":
        perm = rng.permutation(n)
    elif order == "morton":
        perm = morton_order(pos)
    else:
        raise ValueError(order)
    m = dict(meta or {}, order=order)
    return Scene(name, pos[perm].astype(np.float32), sw[perm].astype(np.float32),
                 alpha[perm].astype(np.float32), desc[perm].astype(np.float32), cams, n_layers,
                 forward_only, m)


def morton_order(pos):
    """Permutation sorting points by the 3-D Morton code of a 2^21 grid over their
    bounding box: the spatially coherent order MVS / LiDAR point clouds come in."""
    lo = pos.min(0)
    ext = np.maximum(pos.max(0) - lo, 1e-12)
    q = np.clip(((pos - lo) / ext * (2 ** 21 - 1)).astype(np.uint64), 0, 2 ** 21 - 1)

    def spread(v):
        v = v & np.uint64(0x1FFFFF)
        v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
        v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
        v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
        v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
        return v

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable")


def _sizes(rng, n, area, sigma):
    """s_w = 0.82 sqrt(A/N) exp(sigma xi): 0.820/sqrt(rho) is the mean 4-NN distance of a
    planar Poisson process, mirroring the paper's 4-NN size init."""
    return 0.82 * np.sqrt(area / max(n, 1)) * np.exp(sigma * rng.normal(size=n))


def _sphere(rng, n, c, r):
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return c + r * v, 4 * np.pi * r * r


def _box(rng, n, c, half):
    half = np.asarray(half, np.float64)
    areas = np.array([half[1] * half[2], half[0] * half[2], half[0] * half[1]]) * 4
    face = rng.choice(6, size=n, p=np.repeat(areas, 2) / (2 * areas.sum()))
    u = rng.uniform(-1, 1, (n, 3)) * half
    ax = face // 2
    sgn = np.where(face % 2 == 0, -1.0, 1.0)
    u[np.arange(n), ax] = sgn * half[ax]
    return c + u, 2 * areas.sum()


def _disk(rng, n, c, r):
    rad = r * np.sqrt(rng.uniform(size=n))
    th = rng.uniform(0, 2 * np.pi, n)
    p = np.stack([rad * np.cos(th), rad * np.sin(th), np.zeros(n)], 1)
    return c + p, np.pi * r * r


def _torus(rng, n, c, R, r):
    u = rng.uniform(0, 2 * np.pi, n)
    v = rng.uniform(0, 2 * np.pi, n)
    p = np.stack([(R + r * np.cos(v)) * np.cos(u), r * np.sin(v), (R + r * np.cos(v)) * np.sin(u)], 1)
    return c + p, 4 * np.pi ** 2 * R * r


def _cyl(rng, n, c, r, h):
    th = rng.uniform(0, 2 * np.pi, n)
    z = rng.uniform(0, h, n)
    return c + np.stack([r * np.cos(th), r * np.sin(th), z], 1), 2 * np.pi * r * h


def _split(n, fracs):
    k = [int(round(n * f)) for f in fracs]
    k[-1] = n - sum(k[:-1])
    return k


def _tt_geometry(rng, n, sigma):
    """C2/C4: 60% object (unit sphere + 3 boxes at the origin), 40% ground disk r=12."""
    n_obj, n_gnd = _split(n, [0.6, 0.4])
    n_sph, n_b1, n_b2, n_b3 = _split(n_obj, [0.4, 0.2, 0.2, 0.2])
    parts = [
        _sphere(rng, n_sph, np.array([0.0, 0.0, 0.0]), 1.0),
        _box(rng, n_b1, np.array([1.6, 0.3, -0.5]), [0.5, 0.5, 0.5]),
        _box(rng, n_b2, np.array([-1.4, 0.8, -0.6]), [0.4, 0.7, 0.4]),
        _box(rng, n_b3, np.array([0.2, -1.7, -0.3]), [0.6, 0.3, 0.7]),
        _disk(rng, n_gnd, np.array([0.0, 0.0, -1.0]), 12.0),
    ]
    pos, sw = [], []
    for (p, area) in parts:
        pos.append(p)
        sw.append(_sizes(rng, p.shape[0], area, sigma))
    return np.concatenate(pos), np.concatenate(sw)


def _orbit_cam(az, W=1920, H=1080, fx=1150.0, r=4.5, elev_deg=15.0):
    e = np.deg2rad(elev_deg)
    eye = r * np.array([np.cos(e) * np.cos(az), np.cos(e) * np.sin(az), np.sin(e)])
    return look_at(eye, [0.0, 0.0, 0.0], W, H, fx)


def c1(seed=1, n=1000, F=4, W=64, H=64, n_layers=4, order="random"):
    """C1 tiny: covers the eps branch, all 4 layers and the clamp."""
    rng = np.random.default_rng(seed)
    cam = Camera(fx=64.0, fy=64.0, cx=31.5, cy=31.5, f=64.0, R=np.eye(3, dtype=np.float32),
                 t=np.zeros(3, np.float32), width=W, height=H)
    z = rng.uniform(1, 4, n)
    u = rng.uniform(-6, W + 6, n)
    v = rng.uniform(-6, H + 6, n)
    s_star = 2.0 ** rng.uniform(-3, 4.5, n)
    pos = np.stack([(u - cam.cx) * z / cam.fx, (v - cam.cy) * z / cam.fy, z], 1)
    sw = s_star * z / cam.fx
    alpha = rng.uniform(0.05, 0.95, n)
    desc = rng.normal(0, 1, (n, F))
    return Scene("C1", pos.astype(np.float32), sw.astype(np.float32), alpha.astype(np.float32),
                 desc.astype(np.float32), [cam], n_layers, meta=dict(order=order))


def tiny_scene(seed, n=None, F=None, W=None, H=None, n_layers=None):
    """Random tiny scenes for brute-force pins (sizes drawn from the seed)."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 400)) if n is None else n
    F = int(rng.integers(1, 6)) if F is None else F
    W = int(rng.integers(5, 40)) if W is None else W
    H = int(rng.integers(5, 40)) if H is None else H
    n_layers = int(rng.integers(1, 6)) if n_layers is None else n_layers
    fx = float(np.float32(rng.uniform(0.5, 1.5) * max(W, H)))
    cam = Camera(fx=fx, fy=fx, cx=(W - 1) / 2.0, cy=(H - 1) / 2.0, f=fx, R=np.eye(3, dtype=np.float32),
                 t=np.zeros(3, np.float32), width=W, height=H)
    # a random rotation/translation so the full projection is exercised
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    a, b, c, d = q
    Rm = np.array([[a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
                   [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
                   [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]])
    tv = rng.normal(size=3)
    z = rng.uniform(0.5, 5, n)
    u = rng.uniform(-4, W + 4, n)
    v = rng.uniform(-4, H + 4, n)
    pv = np.stack([(u - cam.cx) * z / fx, (v - cam.cy) * z / fx, z], 1)   # view-space targets
    pos = (pv - tv) @ Rm                                                   # world = R^T (p - t)
    cam.R = Rm.astype(np.float32)
    cam.t = tv.astype(np.float32)
    s_star = 2.0 ** rng.uniform(-3, n_layers + 0.5, n)
    sw = s_star * z / fx
    alpha = rng.uniform(0.05, 1.0, n)
    desc = rng.normal(0, 1, (n, F))
    return Scene(f"tiny{seed}", pos.astype(np.float32), sw.astype(np.float32), alpha.astype(np.float32),
                 desc.astype(np.float32), [cam], n_layers)


def adversarial_scene(F=4, W=48, H=40, n_layers=5):
    """Edge cases (SURVEY.md 8(d) C1 note): exact 2^k sizes at exact pixel centres, an
    opaque front point, equal-depth ties, a 40-deep stacked pixel, z <= near, NaN/Inf,
    negative size, off-screen points, points on the image border."""
    rng = np.random.default_rng(77)
    fx = 32.0
    cam = Camera(fx=fx, fy=fx, cx=(W - 1) / 2.0, cy=(H - 1) / 2.0, f=fx, R=np.eye(3, dtype=np.float32),
                 t=np.zeros(3, np.float32), width=W, height=H)
    P, S, A = [], [], []

    def add(u, v, z, s, a=0.7):
        P.append([(u - cam.cx) * z / fx, (v - cam.cy) * z / fx, z])
        S.append(s * z / fx)
        A.append(a)

    # exact powers of two at exact pixel centres (dyadic z so everything is exact)
    for k in range(-2, n_layers + 2):
        add(4.0 + 3 * (k + 2), 4.0, 2.0, 2.0 ** k)
    # an opaque front point over a stack
    add(20.0, 10.0, 1.0, 1.5, a=1.0)
    for j in range(6):
        add(20.0, 10.0, 1.5 + 0.25 * j, 1.5)
    # equal-depth ties at one pixel
    for j in range(8):
        add(30.0, 12.0, 2.0, 1.25)
    # a 40-deep stacked pixel (random depth order)
    zs = rng.permutation(np.linspace(1.0, 3.0, 40))
    for z in zs:
        add(10.25, 20.75, z, 0.75)
    # behind / at the near plane
    add(10, 10, 0.01, 1.0)
    add(10, 10, -1.0, 1.0)
    add(10, 10, 0.005, 1.0)
    # border and off-screen
    add(-1.0, 5.0, 2.0, 1.0)
    add(-0.999, 5.0, 2.0, 1.0)
    add(-1e-10, 7.0, 2.0, 1.0)
    add(W - 1.0, H - 1.0, 2.0, 1.0)
    add(W - 1e-3, 3.0, 2.0, 1.0)
    add(W + 0.5, 3.0, 2.0, 1.0)
    add(5.0, -1.5, 2.0, 1.0)
    # large sizes (coarse layers / clamp) near the border
    add(2.0, 37.0, 2.0, 2.0 ** (n_layers + 3))
    add(45.0, 2.0, 2.0, 2.0 ** (n_layers - 1) - 0.001)
    # zero size and tiny size
    add(12.5, 30.5, 2.0, 0.0)
    add(13.5, 30.5, 2.0, 1e-30)
    pos = np.array(P, np.float64)
    sw = np.array(S, np.float64)
    alpha = np.array(A, np.float64)
    # non-finite and negative-size points
    bad = np.array([[np.nan, 0, 2], [0, np.inf, 2], [0, 0, np.inf], [0.1, 0.1, 2.0]], np.float64)
    pos = np.concatenate([pos, bad])
    sw = np.concatenate([sw, [0.05, 0.05, 0.05, -0.05]])
    alpha = np.concatenate([alpha, [0.5, 0.5, 0.5, 0.5]])
    n = pos.shape[0]
    desc = rng.normal(0, 1, (n, F))
    return Scene("adversarial", pos.astype(np.float32), sw.astype(np.float32), alpha.astype(np.float32),
                 desc.astype(np.float32), [cam], n_layers)


def make_config(name, seed=None, n=None, order="random", n_views=None):
    """C2..C5 at full size unless `n` overrides the point count (tests use smaller n)."""
    if name == "C1":
        return c1(seed or 1, order=order)
    if name == "C2":
        rng = np.random.default_rng(seed or 2)
        n = n or 5_000_000
        pos, sw = _tt_geometry(rng, n, 0.3)
        cams = [_orbit_cam(0.6)]
        return _finish("C2", pos, sw, rng, 4, cams, 4, forward_only=True, order=order)
    if name == "C3":
        rng = np.random.default_rng(seed or 3)
        n = n or 6_000_000
        k_thin, k_gnd, k_bg = _split(n, [0.35, 0.35, 0.30])
        k_tor, k_cyl = _split(k_thin, [0.5, 0.5])
        k_clutter = int(round(0.02 * n))
        k_bg -= k_clutter
        parts = [
            _torus(rng, k_tor // 2, np.array([-0.9, 0.0, 0.0]), 0.7, 0.04),
            _torus(rng, k_tor - k_tor // 2, np.array([0.9, 0.0, 0.0]), 0.7, 0.04),
            _cyl(rng, k_cyl, np.array([0.0, 0.0, -0.7]), 0.05, 1.2),
            _disk(rng, k_gnd, np.array([0.0, 0.0, -0.7]), 15.0),
            _sphere(rng, k_bg, np.array([0.0, 0.0, 0.0]), 40.0),
        ]
        pos, sw = [], []
        for (p, area) in parts:
            pos.append(p)
            sw.append(_sizes(rng, p.shape[0], area, 0.8))
        cam = _orbit_cam(0.3, r=3.5, elev_deg=12.0, fx=1100.0)
        # near clutter: 0.5-1.5 units in front of the camera
        eye = -cam.R.T.astype(np.float64) @ cam.t.astype(np.float64)
        fwd = cam.R[2].astype(np.float64)
        d = rng.uniform(0.5, 1.5, k_clutter)
        lat = rng.normal(0, 0.4, (k_clutter, 3))
        pc = eye + d[:, None] * fwd + lat * d[:, None]
        pos.append(pc)
        sw.append(_sizes(rng, k_clutter, 1.0, 0.8) * 0.05)
        return _finish("C3", np.concatenate(pos), np.concatenate(sw), rng, 4, [cam], 8, order=order)
    if name == "C4":
        rng = np.random.default_rng(seed or 4)
        n = n or 8_000_000
        pos, sw = _tt_geometry(rng, n, 0.3)
        nv = n_views or 32
        cams = [_orbit_cam(2 * np.pi * v / nv) for v in range(nv)]
        return _finish("C4", pos, sw, rng, 4, cams, 4, order=order)
    if name == "C5":
        rng = np.random.default_rng(seed or 5)
        n = n or 25_000_000
        n_gnd, n_tree = _split(n, [0.8, 0.2])
        L = 400.0
        xy = rng.uniform(-L / 2, L / 2, (n_gnd, 2))

        def height(x, y):
            return (8 * np.sin(x / 37.0) * np.cos(y / 53.0) + 4 * np.sin(x / 13.0 + 1.0)
                    + 2 * np.cos(y / 7.0 + x / 11.0))
        gnd = np.stack([xy[:, 0], xy[:, 1], height(xy[:, 0], xy[:, 1])], 1)
        sw_g = _sizes(rng, n_gnd, L * L * 1.15, 0.4)
        n_crowns = 2000
        cc = rng.uniform(-L / 2, L / 2, (n_crowns, 2))
        crad = rng.uniform(2, 5, (n_crowns, 3))
        ch = height(cc[:, 0], cc[:, 1]) + crad[:, 2] + 3.0
        which = rng.integers(0, n_crowns, n_tree)
        v = rng.normal(size=(n_tree, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        v *= rng.uniform(0, 1, (n_tree, 1)) ** (1 / 3)
        tree = np.stack([cc[which, 0], cc[which, 1], ch[which]], 1) + v * crad[which]
        vol_area = (4 * np.pi * crad.prod(1) ** (2 / 3)).sum()
        sw_t = _sizes(rng, n_tree, vol_area, 0.4)
        eye = np.array([-L / 2 + 1.0, 0.0, height(-L / 2 + 1.0, 0.0) + 2.0])
        pitch = np.deg2rad(-5.0)
        target = eye + np.array([np.cos(pitch), 0.0, np.sin(pitch)])
        cam = look_at(eye, target, 1920, 1080, 1150.0)
        return _finish("C5", np.concatenate([gnd, tree]), np.concatenate([sw_g, sw_t]), rng, 4, [cam], 8,
                       order=order)
    raise ValueError(name)


def grad_pyramid(size, seed=100):
    """Upstream gradient dL/d(pyramid) ~ N(0,1), flat float32 of the given length."""
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, 1.0, size).astype(np.float32)
