"""Pins of the T_min blend variant (reading Q17): closed forms on a
constant-opacity stack, t_min = 0 is the exact definition, and the backward of a cut list
matches finite differences."""
import numpy as np

from oracle import oracle
from synth import scenes

from test_oracle_pins import point_scene, unit_cam


def test_constant_stack_cut_closed_form():
    cam = unit_cam(16, 16, f=8.0)
    zs = 1.0 + np.arange(10) / 32.0
    desc = np.arange(10, dtype=np.float64) + 1
    pos, sw, a, d = point_scene(cam, [[7.0, 7.0, z] for z in zs], [1.0] * 10, alpha=[0.3] * 10, desc=desc)
    g = float(np.float32(0.3))
    # T after m fragments = 0.7^m; first m with 0.7^m < 0.5 is m = 2 -> two fragments kept
    r = oracle.forward(cam, 3, pos, sw, a, d, t_min=0.5)
    kept = oracle.split_pixels(r["kept"].reshape(-1), 16, 16, 3, 16)[0][7, 7]
    assert list(kept[:3]) == [0, 1, -1]
    lay = oracle.split_pyramid(r["pyramid"], 1, 16, 16, 3)
    assert abs(lay[0][0, 7, 7] - (g * 1 + (1 - g) * g * 2)) < 1e-12
    assert abs(lay[0][1, 7, 7] - (1 - (1 - g) ** 2)) < 1e-12
    # t_min = 0 is the exact definition (no cut)
    r0 = oracle.forward(cam, 3, pos, sw, a, d, t_min=0.0)
    rd = oracle.forward(cam, 3, pos, sw, a, d)
    assert np.array_equal(r0["pyramid"], rd["pyramid"]) and np.array_equal(r0["kept"], rd["kept"])
    assert list(oracle.split_pixels(r0["kept"].reshape(-1), 16, 16, 3, 16)[0][7, 7][:10]) == list(range(10))


def test_cut_list_backward_matches_finite_differences():
    """With the cut held fixed (structural guard includes the kept lists), the backward of
    the T_min variant is the derivative of its forward."""
    sc = scenes.tiny_scene(6, n=150)
    cam = sc.cams[0]
    P = oracle.num_pixels(cam.width, cam.height, sc.n_layers)
    G = scenes.grad_pyramid(P * (sc.F + 1), seed=4)
    tmin = 0.3
    g, gm = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, t_min=tmin)
    base = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, t_min=tmin)
    rng = np.random.default_rng(0)
    checked = 0
    for _ in range(40):
        i = int(rng.integers(sc.n))
        c = int(rng.integers(sc.F))
        x0 = float(sc.desc[i, c])
        h = max(abs(x0), 1e-2) * 2.0 ** -10
        vals = []
        for sgn in (1, -1):
            d = sc.desc.copy()
            d[i, c] = np.float32(x0 + sgn * h)
            r = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, d, t_min=tmin)
            vals.append((float(np.dot(r["pyramid"], G.astype(np.float64))), float(d[i, c])))
            assert np.array_equal(r["kept"], base["kept"])       # tau does not move the cut
        (Lp, xp), (Lm, xm) = vals
        fd = (Lp - Lm) / (xp - xm)
        assert abs(fd - g[i, 5 + c]) <= 1e-6 * gm[i, 5 + c] + 1e-9 + 1e-6 * abs(fd)
        checked += 1
    assert checked == 40


def test_cut_boundary_equal_transmittance_is_not_cut():
    """Reading Q17: the kept list ends with the fragment after which T drops BELOW t_min (strict).
    gamma = 0.5 exactly (pixel centre, s = 1, alpha = 0.5), so T = 0.5, 0.25, 0.125, ... exactly:
    with t_min = 0.25 the second fragment leaves T == t_min (not below) and the third is kept too;
    one ulp above 0.25 the cut falls after the second."""
    cam = unit_cam(16, 16, f=8.0)
    zs = 1.0 + np.arange(6) / 32.0
    pos, sw, a, d = point_scene(cam, [[7.0, 7.0, z] for z in zs], [1.0] * 6, alpha=[0.5] * 6,
                                desc=np.ones(6))
    for t_min, K in ((0.25, 3), (float(np.nextafter(np.float32(0.25), np.float32(1))), 2), (0.5, 2),
                     (float(np.nextafter(np.float32(0.5), np.float32(1))), 1)):
        r = oracle.forward(cam, 3, pos, sw, a, d, t_min=t_min)
        kept = oracle.split_pixels(r["kept"].reshape(-1), 16, 16, 3, 16)[0][7, 7]
        assert list(kept[:K + 1]) == list(range(K)) + [-1], (t_min, kept[:4])
        A = oracle.split_pyramid(r["pyramid"], 1, 16, 16, 3)[0][1, 7, 7]
        assert A == 1.0 - 0.5 ** K                       # exact: sum_m T_m gamma_m of the kept prefix
