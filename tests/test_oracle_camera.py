"""Pins of the oracle's camera gradient (the paper optimises camera
intrinsics and poses): fp64 central finite differences over every camera
parameter (R entries, t, fx, fy, cx, cy, f) with the structural guard, and the identity
sum_b dL/dR_ab R_cb-style consistency with the position gradient (dL/dt = sum_i dL/dp_i)."""
import copy

import numpy as np
import pytest

from oracle import oracle
from synth import scenes


def _loss(sc, cam, G):
    r = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, real="double")
    return float(np.dot(r["pyramid"], G.astype(np.float64))), r


def _set(cam, k, v):
    c = copy.deepcopy(cam)
    c.R = np.array(c.R, np.float32).copy()
    c.t = np.array(c.t, np.float32).copy()
    if k < 9:
        c.R.reshape(-1)[k] = np.float32(v)
    elif k < 12:
        c.t[k - 9] = np.float32(v)
    else:
        setattr(c, ("fx", "fy", "cx", "cy", "f")[k - 12], float(np.float32(v)))
    return c


def _get(cam, k):
    if k < 9:
        return float(np.asarray(cam.R, np.float32).reshape(-1)[k])
    if k < 12:
        return float(np.asarray(cam.t, np.float32)[k - 9])
    return float(np.float32(getattr(cam, ("fx", "fy", "cx", "cy", "f")[k - 12])))


@pytest.mark.parametrize("seed", [0, 2, 5])
def test_camera_gradient_finite_differences(seed):
    sc = scenes.tiny_scene(seed, n=150)
    cam = sc.cams[0]
    P = oracle.num_pixels(cam.width, cam.height, sc.n_layers)
    G = scenes.grad_pyramid(P * (sc.F + 1), seed=seed + 7)
    gc = np.zeros(17)
    gcm = np.zeros(17)
    oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, real="double", grad_cam=gc,
                    grad_cam_mag=gcm)
    _, base = _loss(sc, cam, G)
    _, lev0, _ = oracle.project(cam, sc.n_layers, sc.pos, sc.sw, real="double")
    checked = 0
    for k in range(17):
        x0 = _get(cam, k)
        h = max(abs(x0), 1e-2) * 2.0 ** -14
        vals = []
        for sgn in (1, -1):
            c = _set(cam, k, x0 + sgn * h)
            L, r = _loss(sc, c, G)
            _, lev, _ = oracle.project(c, sc.n_layers, sc.pos, sc.sw, real="double")
            if not (np.array_equal(r["counts"], base["counts"]) and np.array_equal(r["kept"], base["kept"])
                    and np.array_equal(lev, lev0)):
                vals = None
                break
            vals.append((L, _get(c, k)))
        if vals is None:
            continue
        (Lp, xp), (Lm, xm) = vals
        fd = (Lp - Lm) / (xp - xm)
        assert abs(fd - gc[k]) <= 1e-4 * gcm[k] + 1e-4 * abs(gc[k]) + 1e-9, (oracle.CAMERA_GRAD_NAMES[k], fd, gc[k])
        checked += 1
    assert checked >= 12


def test_translation_gradient_is_sum_of_view_space_gradients():
    """dL/dt = sum_i dL/dp_i and dL/dx_i = R^T dL/dp_i, so R dL/dt = sum_i dL/dx_i (exact
    algebra of p = R x + t, independent of the rasterizer)."""
    sc = scenes.tiny_scene(4, n=200)
    cam = sc.cams[0]
    P = oracle.num_pixels(cam.width, cam.height, sc.n_layers)
    G = scenes.grad_pyramid(P * (sc.F + 1), seed=3)
    gc = np.zeros(17)
    g, _ = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, real="double", grad_cam=gc)
    R = np.asarray(cam.R, np.float64)
    lhs = R.T @ gc[9:12]
    rhs = g[:, :3].sum(0)
    assert np.allclose(lhs, rhs, rtol=1e-9, atol=1e-9 * np.abs(rhs).max())
