"""ctypes wrapper of the C oracle (oracle/trips_oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Argument marshalling only; all
arithmetic is in trips_oracle.c (point-centric lists, "O1") or oracle/brute.py
(pixel-centric brute force, "O0").
"""
import ctypes as C
import os

import numpy as np

from . import build as _build

_LIBS = {}


class _Camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("f", C.c_float), ("R", C.c_float * 9), ("t", C.c_float * 3),
                ("width", C.c_int32), ("height", C.c_int32), ("near_plane", C.c_float)]


class _Stats(C.Structure):
    _fields_ = [("n_culled", C.c_int64), ("n_visible", C.c_int64), ("n_frag", C.c_int64),
                ("n_kept", C.c_int64), ("n_trunc_pixels", C.c_int64), ("max_list", C.c_int64)]


def _lib(real: str):
    if real not in _LIBS:
        paths = _build.build()
        lib = C.CDLL(paths[real])
        vp = C.c_void_p
        lib.oracle_num_pixels.restype = C.c_int64
        lib.oracle_num_pixels.argtypes = [C.c_int, C.c_int32, C.c_int32]
        lib.oracle_project.restype = C.c_int
        lib.oracle_project.argtypes = [C.POINTER(_Camera), C.c_int, C.c_int64, vp, vp, vp, vp, vp]
        lib.oracle_forward.restype = C.c_int
        lib.oracle_forward.argtypes = [C.POINTER(_Camera), C.c_int, C.c_int, C.c_int64, vp, vp, vp, vp,
                                       vp, vp, vp, vp, vp, C.POINTER(_Stats)]
        lib.oracle_backward.restype = C.c_int
        lib.oracle_backward.argtypes = [C.POINTER(_Camera), C.c_int, C.c_int, C.c_int64, vp, vp, vp, vp,
                                        vp, vp, vp, vp, vp, vp]
        lib.oracle_set_t_min.restype = None
        lib.oracle_set_t_min.argtypes = [C.c_float]
        lib.oracle_set_screen_out.restype = None
        lib.oracle_set_screen_out.argtypes = [vp, vp]
        lib.oracle_set_coarse.restype = None
        lib.oracle_set_coarse.argtypes = [C.c_int, vp]
        lib.oracle_knn4.restype = C.c_int
        lib.oracle_knn4.argtypes = [C.c_int64, vp, C.c_int64, vp, vp, vp]
        _LIBS[real] = lib
    return _LIBS[real]


def knn4(pos, queries=None):
    """4-NN size init (reading Q25): returns (size float32 [q], nbr int32 [q,4])
    for the query indices (all points if None), brute force over all points."""
    pos = _f32(pos, (-1, 3))
    n = pos.shape[0]
    q = None if queries is None else np.ascontiguousarray(queries, dtype=np.int64)
    nq = n if q is None else q.shape[0]
    size = np.zeros(nq, np.float32)
    nbr = np.full((nq, 4), -1, np.int32)
    rc = _lib("float").oracle_knn4(n, _ptr(pos), nq, _ptr(q), _ptr(size), _ptr(nbr))
    assert rc == 0, rc
    return size, nbr


def camera_struct(cam) -> _Camera:
    c = _Camera()
    c.fx, c.fy, c.cx, c.cy, c.f = cam.fx, cam.fy, cam.cx, cam.cy, cam.f
    R = np.asarray(cam.R, dtype=np.float32).reshape(9)
    t = np.asarray(cam.t, dtype=np.float32).reshape(3)
    for k in range(9):
        c.R[k] = float(R[k])
    for k in range(3):
        c.t[k] = float(t[k])
    c.width, c.height, c.near_plane = int(cam.width), int(cam.height), cam.near
    return c


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    if shape is not None:
        a = a.reshape(shape)
    return a


def layer_dims(width: int, height: int, n_layers: int):
    """[(H_l, W_l)] with H_l = ceil(H / 2^l), W_l = ceil(W / 2^l) (reading Q8)."""
    return [(-(-height // (1 << l)), -(-width // (1 << l))) for l in range(n_layers)]


def num_pixels(width, height, n_layers):
    return int(_lib("float").oracle_num_pixels(n_layers, width, height))


def split_pyramid(flat, F, width, height, n_layers):
    """Flat pyramid (layer-major, planar (F+1, H_l, W_l)) -> list of arrays."""
    out, off = [], 0
    for (h, w) in layer_dims(width, height, n_layers):
        sz = (F + 1) * h * w
        out.append(flat[off:off + sz].reshape(F + 1, h, w))
        off += sz
    return out


def split_pixels(flat, width, height, n_layers, per_pixel=1):
    """Per-pixel array in pyramid pixel order -> list of (H_l, W_l[, per_pixel])."""
    out, off = [], 0
    for (h, w) in layer_dims(width, height, n_layers):
        sz = h * w * per_pixel
        a = flat[off:off + sz]
        out.append(a.reshape(h, w) if per_pixel == 1 else a.reshape(h, w, per_pixel))
        off += sz
    return out


def project(cam, n_layers, pos, sw, real="float"):
    """Returns (proj [n,4] (x, y, z, s; NaN if culled), level int8 [n], iota [n,2])."""
    pos = _f32(pos, (-1, 3))
    sw = _f32(sw, (-1,))
    n = pos.shape[0]
    dt = np.float32 if real == "float" else np.float64
    proj = np.zeros((n, 4), dtype=dt)
    level = np.zeros(n, dtype=np.int8)
    iota = np.zeros((n, 2), dtype=dt)
    rc = _lib(real).oracle_project(C.byref(camera_struct(cam)), n_layers, n, _ptr(pos), _ptr(sw),
                                   _ptr(proj), _ptr(level), _ptr(iota))
    assert rc == 0, rc
    return proj, level, iota


def forward(cam, n_layers, pos, sw, alpha, desc, mask=None, real="float", want_kept=True, t_min=0.0, coarse=0):
    """O1 forward.  Returns dict(pyramid float64 flat, mag, counts uint32 [P],
    kept int32 [P,16], kept_layer int8 [P,16] (coarse only), stats dict).  t_min > 0 selects
    the T_min variant (reading Q17), coarse > 0 coarse-layer inclusion (reading Q22)."""
    P = num_pixels(cam.width, cam.height, n_layers)
    kl = np.full((P, 16), -1, dtype=np.int8) if (coarse and want_kept) else None
    _lib(real).oracle_set_t_min(float(np.float32(t_min)))
    _lib(real).oracle_set_coarse(int(coarse), _ptr(kl))
    try:
        r = _forward(cam, n_layers, pos, sw, alpha, desc, mask, real, want_kept)
    finally:
        _lib(real).oracle_set_t_min(0.0)
        _lib(real).oracle_set_coarse(0, None)
    if kl is not None:
        r["kept_layer"] = kl
    return r


def _forward(cam, n_layers, pos, sw, alpha, desc, mask, real, want_kept):
    pos = _f32(pos, (-1, 3))
    n = pos.shape[0]
    sw = _f32(sw, (n,))
    alpha = _f32(alpha, (n,))
    desc = _f32(desc)
    F = desc.shape[1] if desc.ndim == 2 else 1
    desc = desc.reshape(n, F)
    P = num_pixels(cam.width, cam.height, n_layers)
    pyr = np.zeros(P * (F + 1), dtype=np.float64)
    mag = np.zeros(P * (F + 1), dtype=np.float64)
    counts = np.zeros(P, dtype=np.uint32)
    kept = np.full((P, 16), -1, dtype=np.int32) if want_kept else None
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    st = _Stats()
    rc = _lib(real).oracle_forward(C.byref(camera_struct(cam)), n_layers, F, n, _ptr(pos), _ptr(sw),
                                   _ptr(alpha), _ptr(desc), _ptr(pyr), _ptr(mag), _ptr(counts),
                                   _ptr(kept), _ptr(m), C.byref(st))
    assert rc == 0, rc
    stats = {k: int(getattr(st, k)) for k, _ in _Stats._fields_}
    return dict(pyramid=pyr, mag=mag, counts=counts, kept=kept, stats=stats, F=F, P=P)


CAMERA_GRAD_NAMES = ("R00", "R01", "R02", "R10", "R11", "R12", "R20", "R21", "R22", "t0", "t1", "t2",
                     "fx", "fy", "cx", "cy", "f")


def backward(cam, n_layers, pos, sw, alpha, desc, grad_pyramid, mask=None, real="float", grad=None,
             grad_mag=None, grad_cam=None, grad_cam_mag=None, t_min=0.0, coarse=0, screen=None, screen_mag=None):
    """O1 backward.  Returns (grad [n, 5+F] float64, grad_mag [n, 5+F]); rows are
    (d/dx, d/dy, d/dz, d/ds_w, d/dalpha, d/dtau[F]).  If grad / grad_mag are given
    they are accumulated into (multi-view sum, reading Q21).  grad_cam / grad_cam_mag
    (float64 [17], CAMERA_GRAD_NAMES order) receive the camera gradient if given.
    screen / screen_mag (float64 [n, 4+F], overwritten) receive the screen-space gradients
    (d/dx, d/dy, d/ds, d/dalpha, d/dtau) and their magnitudes if given."""
    _lib(real).oracle_set_t_min(float(np.float32(t_min)))
    _lib(real).oracle_set_coarse(int(coarse), None)
    for a in (screen, screen_mag):
        assert a is None or (a.dtype == np.float64 and a.flags.c_contiguous)
    _lib(real).oracle_set_screen_out(_ptr(screen), _ptr(screen_mag))
    try:
        return _backward(cam, n_layers, pos, sw, alpha, desc, grad_pyramid, mask, real, grad, grad_mag, grad_cam,
                         grad_cam_mag)
    finally:
        _lib(real).oracle_set_t_min(0.0)
        _lib(real).oracle_set_coarse(0, None)
        _lib(real).oracle_set_screen_out(None, None)


def _backward(cam, n_layers, pos, sw, alpha, desc, grad_pyramid, mask, real, grad, grad_mag, grad_cam,
              grad_cam_mag):
    pos = _f32(pos, (-1, 3))
    n = pos.shape[0]
    sw = _f32(sw, (n,))
    alpha = _f32(alpha, (n,))
    desc = _f32(desc)
    F = desc.shape[1] if desc.ndim == 2 else 1
    desc = desc.reshape(n, F)
    gp = _f32(grad_pyramid).reshape(-1)
    if grad is None:
        grad = np.zeros((n, 5 + F), dtype=np.float64)
    if grad_mag is None:
        grad_mag = np.zeros((n, 5 + F), dtype=np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    rc = _lib(real).oracle_backward(C.byref(camera_struct(cam)), n_layers, F, n, _ptr(pos), _ptr(sw),
                                    _ptr(alpha), _ptr(desc), _ptr(gp), _ptr(grad), _ptr(grad_mag),
                                    _ptr(m), _ptr(grad_cam), _ptr(grad_cam_mag))
    assert rc == 0, rc
    return grad, grad_mag
