"""Pins of coarse-layer inclusion (reading Q22):
hand-computed blends of a coarse point in front of a fine one, a point blended with its own
coarser-layer fragment, full occlusion by an opaque coarse point, the pixel-centric brute force
(O0, written separately), mask restriction, and finite differences of the backward."""
import numpy as np
import pytest

from oracle import brute, oracle
from synth import scenes

from test_oracle_pins import _fd_check, point_scene, unit_cam


def _px(r, cam, n_layers, F, l, x, y):
    lay = oracle.split_pyramid(r["pyramid"], F, cam.width, cam.height, n_layers)[l]
    return lay[:, y, x]


def _kept(r, cam, n_layers, l, x, y, key="kept"):
    return list(oracle.split_pixels(r[key].reshape(-1), cam.width, cam.height, n_layers, 16)[l][y, x])


def test_coarse_point_in_front_of_fine_point():
    cam = unit_cam(16, 16, f=8.0)
    # B: s = 2 (wholly layer 1, iota = 1) at pixel (6, 6) -> x_1 = 3 exactly, beta = 1 at (3, 3)
    # S: s = 1 (layer 0, iota = 1) at pixel (7, 7), behind B
    pos, sw, a, d = point_scene(cam, [[6.0, 6.0, 1.0], [7.0, 7.0, 2.0]], [2.0, 1.0], alpha=[0.6, 0.5],
                                desc=[5.0, 3.0])
    g_b, g_s = float(np.float32(0.6)), 0.5
    plain = oracle.forward(cam, 3, pos, sw, a, d)
    assert np.allclose(_px(plain, cam, 3, 1, 0, 7, 7), [g_s * 3, g_s], atol=1e-12)
    for c in (1, 2):
        r = oracle.forward(cam, 3, pos, sw, a, d, coarse=c)
        assert np.allclose(_px(r, cam, 3, 1, 0, 7, 7), [g_b * 5 + (1 - g_b) * g_s * 3, g_b + (1 - g_b) * g_s],
                           atol=1e-12)
        assert _kept(r, cam, 3, 0, 7, 7)[:3] == [0, 1, -1]
        assert _kept(r, cam, 3, 0, 7, 7, "kept_layer")[:3] == [1, 0, -1]
        assert np.allclose(_px(r, cam, 3, 1, 0, 6, 6), [g_b * 5, g_b], atol=1e-12)
        # (8, 8): B's zero-weight corner (4, 4) of layer 1 and S's zero-weight corner -- both kept
        assert _kept(r, cam, 3, 0, 8, 8)[:3] == [0, 1, -1]
        assert np.all(_px(r, cam, 3, 1, 0, 8, 8) == 0)
        # counts are the pixel's own list, unchanged
        assert np.array_equal(r["counts"], plain["counts"])
        # layer 1 has no coarser fragments here: unchanged
        l1 = oracle.split_pyramid(r["pyramid"], 1, 16, 16, 3)[1]
        assert np.array_equal(l1, oracle.split_pyramid(plain["pyramid"], 1, 16, 16, 3)[1])


def test_point_blends_with_its_own_coarser_fragment():
    cam = unit_cam(16, 16, f=8.0)
    # s = 1.5: layers 0 and 1 with iota = 0.5 each; at pixel (6, 6) beta = 1 in both layers
    pos, sw, a, d = point_scene(cam, [[6.0, 6.0, 1.0]], [1.5], alpha=[0.8], desc=[2.0])
    g = float(np.float32(0.5) * np.float32(0.8))
    r = oracle.forward(cam, 3, pos, sw, a, d, coarse=1)
    assert np.allclose(_px(r, cam, 3, 1, 0, 6, 6), [g * 2 + (1 - g) * g * 2, g + (1 - g) * g], atol=1e-12)
    assert _kept(r, cam, 3, 0, 6, 6)[:3] == [0, 0, -1]                 # (z, i, d): finer layer first
    assert _kept(r, cam, 3, 0, 6, 6, "kept_layer")[:3] == [0, 1, -1]
    plain = oracle.forward(cam, 3, pos, sw, a, d)
    assert np.allclose(_px(plain, cam, 3, 1, 0, 6, 6), [g * 2, g], atol=1e-12)


def test_opaque_coarse_point_occludes_all_descendants():
    cam = unit_cam(32, 32, f=8.0)
    # B: s = 4 (layer 2, iota = 1), alpha = 1, pixel (8, 8) -> x_2 = 2 exactly, beta = 1 at (2, 2)
    pts = [[8.0, 8.0, 1.0]] + [[8.0 + (k % 4), 8.0 + (k // 4) % 4, 1.5 + 0.01 * k] for k in range(20)]
    sizes = [4.0] + [1.0] * 20
    alpha = [1.0] + [0.9] * 20
    desc = [7.0] + list(range(20))
    pos, sw, a, d = point_scene(cam, pts, sizes, alpha=alpha, desc=desc)
    r = oracle.forward(cam, 3, pos, sw, a, d, coarse=2)
    for y in range(8, 12):
        for x in range(8, 12):
            assert np.array_equal(_px(r, cam, 3, 1, 0, x, y), [7.0, 1.0])
            assert _kept(r, cam, 3, 0, x, y)[0] == 0 and _kept(r, cam, 3, 0, x, y, "kept_layer")[0] == 2
    plain = oracle.forward(cam, 3, pos, sw, a, d)
    assert not np.array_equal(_px(plain, cam, 3, 1, 0, 9, 9), [7.0, 1.0])


def test_coarse_zero_and_single_layer_are_the_definition():
    sc = scenes.tiny_scene(3)
    cam = sc.cams[0]
    base = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc)
    r0 = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=0)
    assert np.array_equal(base["pyramid"], r0["pyramid"]) and np.array_equal(base["kept"], r0["kept"])
    b1 = oracle.forward(cam, 1, sc.pos, sc.sw, sc.alpha, sc.desc)
    c1 = oracle.forward(cam, 1, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=3)
    assert np.array_equal(b1["pyramid"], c1["pyramid"]) and np.array_equal(b1["kept"], c1["kept"])
    # coarse >= n_layers - 1 saturates
    ca = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=sc.n_layers - 1)
    cb = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=15)
    assert np.array_equal(ca["pyramid"], cb["pyramid"]) and np.array_equal(ca["kept"], cb["kept"])


def _compare_o0_o1(sc, coarse):
    cam = sc.cams[0]
    r = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=coarse)
    L, Cn, K = brute.render(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=coarse)
    pyr = oracle.split_pyramid(r["pyramid"], sc.F, cam.width, cam.height, sc.n_layers)
    cn = oracle.split_pixels(r["counts"], cam.width, cam.height, sc.n_layers)
    kp = oracle.split_pixels(r["kept"].reshape(-1), cam.width, cam.height, sc.n_layers, 16)
    for l in range(sc.n_layers):
        assert np.array_equal(cn[l], Cn[l]), (sc.name, l)
        assert np.array_equal(kp[l], K[l]), (sc.name, l)
        assert np.abs(pyr[l] - L[l]).max() <= 1e-12, (sc.name, l)
    return r


@pytest.mark.parametrize("coarse", [1, 3])
def test_o1_matches_brute_force_coarse(coarse):
    changed = 0
    for sc in [scenes.c1(), scenes.adversarial_scene()] + [scenes.tiny_scene(s) for s in range(6)]:
        r = _compare_o0_o1(sc, coarse)
        plain = oracle.forward(sc.cams[0], sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc)
        changed += int(not np.array_equal(r["kept"], plain["kept"]))
    assert changed >= 4                                   # the variant does change the lists


def test_mask_restricts_without_changing_marked_pixels():
    sc = scenes.c1()
    cam = sc.cams[0]
    P = oracle.num_pixels(cam.width, cam.height, sc.n_layers)
    rng = np.random.default_rng(5)
    mask = (rng.random(P) < 0.1).astype(np.uint8)
    full = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=3)
    part = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, coarse=3, mask=mask)
    m = mask.astype(bool)
    assert np.array_equal(part["kept"][m], full["kept"][m])
    assert np.array_equal(part["kept_layer"][m], full["kept_layer"][m])
    assert np.array_equal(part["counts"][m], full["counts"][m]) and not part["counts"][~m].any()
    pm = np.repeat(m[None], sc.F + 1, 0)                  # pyramid layout is planar per layer
    pyr_full = oracle.split_pyramid(full["pyramid"], sc.F, cam.width, cam.height, sc.n_layers)
    pyr_part = oracle.split_pyramid(part["pyramid"], sc.F, cam.width, cam.height, sc.n_layers)
    msk = oracle.split_pixels(mask, cam.width, cam.height, sc.n_layers)
    for l in range(sc.n_layers):
        sel = np.broadcast_to(msk[l].astype(bool), pyr_full[l].shape)
        assert np.array_equal(pyr_part[l][sel], pyr_full[l][sel]) and not pyr_part[l][~sel].any()
    del pm
    # backward on the mask == backward of the loss restricted to the marked pixels
    G = scenes.grad_pyramid(P * (sc.F + 1), seed=9)
    Gm = np.concatenate([(g * np.broadcast_to(mk.astype(np.float32), g.shape)).reshape(-1)
                         for g, mk in zip(oracle.split_pyramid(G, sc.F, cam.width, cam.height, sc.n_layers), msk)])
    g1, _ = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, mask=mask, coarse=3)
    g2, _ = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, Gm, coarse=3)
    assert np.abs(g1 - g2).max() <= 1e-12 * max(1.0, np.abs(g2).max())


def test_backward_finite_differences_coarse():
    _fd_check(scenes.c1(), 1, coarse=3)
    for seed in range(3):
        _fd_check(scenes.tiny_scene(seed), seed, n_coords=40, coarse=1 + seed)
