"""O0: pixel-centric brute-force rasterizer for tiny scenes (numpy).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Independent of O1 (trips_oracle.c): instead of emitting fragments per point and
sorting one big array, it visits every pyramid pixel and scans ALL points for the
ones whose 2x2 footprint in that layer contains the pixel (Eq. 3),
then sorts that pixel's list by (z, i), keeps 16 and blends
(Eqs. 5-6).  O(P * N): tiny scenes only.

Layer selection is written from Eq. (4) with frexp (float32 throughout the exact
block, one numpy op per rounding, no contraction -- matching reading Q18).
"""
import numpy as np

CAP = 16
EPS = np.float32(0.25)


def _project(cam, pos, sw):
    f32 = np.float32
    R = np.asarray(cam.R, f32).reshape(3, 3)
    t = np.asarray(cam.t, f32)
    X, Y, Z = pos[:, 0].astype(f32), pos[:, 1].astype(f32), pos[:, 2].astype(f32)
    p = []
    with np.errstate(all="ignore"):
        for r in range(3):
            acc = R[r, 0] * X
            acc = acc + R[r, 1] * Y
            acc = acc + R[r, 2] * Z
            acc = acc + t[r]
            p.append(acc)
        z = p[2]
        xs = (f32(cam.fx) * p[0]) / z + f32(cam.cx)
        ys = (f32(cam.fy) * p[1]) / z + f32(cam.cy)
        s = (f32(cam.f) * sw.astype(f32)) / z
        vis = (z > f32(cam.near)) & np.isfinite(xs) & np.isfinite(ys) & np.isfinite(s) & (s >= 0)
    return xs, ys, z, s, vis


def _layer_weight(s, vis, l, n_layers):
    """iota of layer l per point (0 where layer l is not selected), Eq. (4)."""
    f32 = np.float32
    iota = np.zeros(s.shape, f32)
    sel = np.zeros(s.shape, bool)
    with np.errstate(all="ignore"):
        small = vis & (s < 1)
        if l == 0:
            iota[small] = EPS + (f32(1) - EPS) * s[small]
            sel |= small
        big = vis & (s >= 1)
        mant, ex = np.frexp(s[big])                      # s = mant * 2^ex, mant in [0.5, 1)
        k = ex.astype(np.int64) - 1                     # floor(log2 s)
        m = (mant * f32(2)).astype(f32)                 # s / 2^k in [1, 2), exact
        idx = np.nonzero(big)[0]
        clamp = k >= n_layers - 1
        single = (~clamp) & (m == 1)
        two = (~clamp) & (m != 1)
        hit = clamp & (l == n_layers - 1)
        iota[idx[hit]] = 1
        sel[idx[hit]] = True
        hit = single & (k == l)
        iota[idx[hit]] = 1
        sel[idx[hit]] = True
        lo = two & (k == l)
        iota[idx[lo]] = f32(2) - m[lo]
        sel[idx[lo]] = True
        hi = two & (k + 1 == l)
        iota[idx[hi]] = m[hi] - f32(1)
        sel[idx[hi]] = True
    return sel, iota


def render(cam, n_layers, pos, sw, alpha, desc, coarse=0):
    """Returns (list of (F+1, H_l, W_l) float64 layers, list of (H_l, W_l) counts,
    list of (H_l, W_l, 16) kept indices, -1 padded).

    coarse > 0: coarse-layer inclusion (reading Q22): the list blended at
    (l, u, v) is the union of the fragments of (l + d, u >> d, v >> d), d = 0..min(coarse,
    n_layers - 1 - l), ordered by (z, i, d), 16 kept; counts stay the pixel's own list."""
    if coarse:
        return _render_coarse(cam, n_layers, pos, sw, alpha, desc, coarse)
    pos = np.asarray(pos, np.float32)
    sw = np.asarray(sw, np.float32)
    alpha = np.asarray(alpha, np.float32)
    desc = np.asarray(desc, np.float32)
    n, F = desc.shape
    xs, ys, z, s, vis = _project(cam, pos, sw)
    layers, counts, kepts = [], [], []
    idx_all = np.arange(n)
    for l in range(n_layers):
        Hl = -(-cam.height // (1 << l))
        Wl = -(-cam.width // (1 << l))
        sel, iota = _layer_weight(s, vis, l, n_layers)
        scale = np.float32(2.0 ** -l)
        with np.errstate(all="ignore"):
            xl = xs * scale
            yl = ys * scale
            inb = sel & (xl >= -1) & (xl < Wl) & (yl >= -1) & (yl < Hl)
            x0 = np.floor(np.where(inb, xl, 0)).astype(np.int64)
            y0 = np.floor(np.where(inb, yl, 0)).astype(np.int64)
            fx = (xl - x0.astype(np.float32)).astype(np.float32)
            fy = (yl - y0.astype(np.float32)).astype(np.float32)
        out = np.zeros((F + 1, Hl, Wl))
        cnt = np.zeros((Hl, Wl), np.int64)
        kept = np.full((Hl, Wl, CAP), -1, np.int64)
        for v in range(Hl):
            for u in range(Wl):
                hx = inb & ((x0 == u) | (x0 + 1 == u)) & ((y0 == v) | (y0 + 1 == v))
                ids = idx_all[hx]
                cnt[v, u] = ids.size
                if ids.size == 0:
                    continue
                order = np.lexsort((ids, z[ids]))       # by z, then index
                ids = ids[order][:CAP]
                kept[v, u, :ids.size] = ids
                wx = np.where(x0[ids] + 1 == u, fx[ids], np.float32(1) - fx[ids]).astype(np.float32)
                wy = np.where(y0[ids] + 1 == v, fy[ids], np.float32(1) - fy[ids]).astype(np.float32)
                beta = (wx * wy).astype(np.float32)
                gamma = ((beta * iota[ids]).astype(np.float32) * alpha[ids]).astype(np.float32)
                T, C, A = 1.0, np.zeros(F), 0.0
                for j, i in enumerate(ids):
                    g = float(gamma[j])
                    C += T * g * desc[i].astype(np.float64)
                    A += T * g
                    T *= 1.0 - g
                out[:F, v, u] = C
                out[F, v, u] = A
        layers.append(out)
        counts.append(cnt)
        kepts.append(kept)
    return layers, counts, kepts


def _pixel_fragments(cam, n_layers, xs, ys, s, vis, alpha):
    """Per layer, per pixel: (point ids, gamma float32) of every fragment (Eq. 3), any order."""
    f32 = np.float32
    idx_all = np.arange(xs.shape[0])
    out = []
    for l in range(n_layers):
        Hl = -(-cam.height // (1 << l))
        Wl = -(-cam.width // (1 << l))
        sel, iota = _layer_weight(s, vis, l, n_layers)
        scale = f32(2.0 ** -l)
        with np.errstate(all="ignore"):
            xl = xs * scale
            yl = ys * scale
            inb = sel & (xl >= -1) & (xl < Wl) & (yl >= -1) & (yl < Hl)
            x0 = np.floor(np.where(inb, xl, 0)).astype(np.int64)
            y0 = np.floor(np.where(inb, yl, 0)).astype(np.int64)
            fx = (xl - x0.astype(f32)).astype(f32)
            fy = (yl - y0.astype(f32)).astype(f32)
        grid = {}
        for v in range(Hl):
            for u in range(Wl):
                hx = inb & ((x0 == u) | (x0 + 1 == u)) & ((y0 == v) | (y0 + 1 == v))
                ids = idx_all[hx]
                wx = np.where(x0[ids] + 1 == u, fx[ids], f32(1) - fx[ids]).astype(f32)
                wy = np.where(y0[ids] + 1 == v, fy[ids], f32(1) - fy[ids]).astype(f32)
                beta = (wx * wy).astype(f32)
                gamma = ((beta * iota[ids]).astype(f32) * alpha[ids]).astype(f32)
                grid[(v, u)] = (ids, gamma)
        out.append((Hl, Wl, grid))
    return out


def _render_coarse(cam, n_layers, pos, sw, alpha, desc, coarse):
    pos = np.asarray(pos, np.float32)
    sw = np.asarray(sw, np.float32)
    alpha = np.asarray(alpha, np.float32)
    desc = np.asarray(desc, np.float32)
    n, F = desc.shape
    xs, ys, z, s, vis = _project(cam, pos, sw)
    frags = _pixel_fragments(cam, n_layers, xs, ys, s, vis, alpha)
    layers, counts, kepts = [], [], []
    for l in range(n_layers):
        Hl, Wl, grid = frags[l]
        D = min(coarse, n_layers - 1 - l)
        out = np.zeros((F + 1, Hl, Wl))
        cnt = np.zeros((Hl, Wl), np.int64)
        kept = np.full((Hl, Wl, CAP), -1, np.int64)
        for v in range(Hl):
            for u in range(Wl):
                cnt[v, u] = grid[(v, u)][0].size
                ids, gam, dd = [], [], []
                for d in range(D + 1):
                    a_ids, a_gam = frags[l + d][2][(v >> d, u >> d)]
                    ids.append(a_ids)
                    gam.append(a_gam)
                    dd.append(np.full(a_ids.size, d))
                ids, gam, dd = np.concatenate(ids), np.concatenate(gam), np.concatenate(dd)
                if ids.size == 0:
                    continue
                order = np.lexsort((dd, ids, z[ids]))[:CAP]      # by z, then index, then d
                kept[v, u, :order.size] = ids[order]
                T, C, A = 1.0, np.zeros(F), 0.0
                for j in order:
                    g = float(gam[j])
                    C += T * g * desc[ids[j]].astype(np.float64)
                    A += T * g
                    T *= 1.0 - g
                out[:F, v, u] = C
                out[F, v, u] = A
        layers.append(out)
        counts.append(cnt)
        kepts.append(kept)
    return layers, counts, kepts
