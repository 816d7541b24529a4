"""Thin ctypes binding of include/trips.h (argument marshalling only).

Every step of the rasterizer runs in libtrips.so (hand-written CUDA for sm_100a).  There
is no CPU fallback: if the library is missing or cannot be loaded this module raises.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TRIPS_LIB overrides the library path (kernel experiments build variants elsewhere)
LIB_PATH = os.environ.get("TRIPS_LIB", os.path.join(_HERE, "libtrips.so"))

TRIPS_OK = 0
TRIPS_ERR_ARG = -1
TRIPS_ERR_ALIGN = -2
TRIPS_ERR_CAPACITY = -3
TRIPS_ERR_STATE = -4
TRIPS_ERR_CUDA = -5
TRIPS_FWD_SAVE_FOR_BACKWARD = 1
TRIPS_EXPORT_COUNTS = 1
TRIPS_EXPORT_KEPT = 2
TRIPS_EXPORT_KEPT_LAYER = 3
TRIPS_EXPORT_SCREEN_GRADS = 4
N_STAGES = 5
STAGE_NAMES = ("count", "emit", "tscan", "raster", "backward")


class trips_camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("f", C.c_float), ("R", C.c_float * 9), ("t", C.c_float * 3),
                ("width", C.c_int32), ("height", C.c_int32), ("near_plane", C.c_float)]


class trips_config(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_features", C.c_int32), ("t_min", C.c_float),
                ("coarse_layers", C.c_int32)]


class trips_stats(C.Structure):
    _fields_ = [("n_culled", C.c_int64), ("n_visible", C.c_int64), ("n_pairs", C.c_int64),
                ("n_frag", C.c_int64), ("n_kept", C.c_int64), ("n_trunc_pixels", C.c_int64),
                ("max_list", C.c_int64), ("n_kept_pairs", C.c_int64)]


class TripsError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} ({status})")


_lib = None

# (name, restype, argtypes) for every symbol of include/trips.h
_VP = C.c_void_p
SIGNATURES = [
    ("trips_plan_create", C.c_int, [C.POINTER(trips_config), C.c_int32, C.c_int32, C.c_int64, C.POINTER(_VP)]),
    ("trips_plan_destroy", None, [_VP]),
    ("trips_workspace_bytes", C.c_size_t, [_VP]),
    ("trips_num_pixels", C.c_int64, [_VP]),
    ("trips_pyramid_floats", C.c_int64, [_VP]),
    ("trips_layer_dims", C.c_int, [_VP, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int64)]),
    ("trips_project", C.c_int, [_VP, _VP, C.POINTER(trips_camera), C.c_int64, _VP, _VP, _VP, _VP, _VP, _VP,
                                _VP]),
    ("trips_splat_forward", C.c_int, [_VP, _VP, _VP, C.c_uint32, _VP]),
    ("trips_splat_backward", C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    ("trips_read_stats", C.c_int, [_VP, _VP, C.POINTER(trips_stats), _VP]),
    ("trips_debug_export", C.c_int, [_VP, _VP, C.c_int32, _VP, _VP]),
    ("trips_set_profiling", C.c_int, [_VP, C.c_int32]),
    ("trips_read_stage_ms", C.c_int, [_VP, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32, C.c_int32]),
    ("trips_morton_workspace_bytes", C.c_size_t, [C.c_int64]),
    ("trips_morton_order", C.c_int, [_VP, C.c_int64, _VP, _VP, _VP]),
    ("trips_knn_workspace_bytes", C.c_size_t, [C.c_int64]),
    ("trips_knn_sizes", C.c_int, [_VP, C.c_int64, _VP, _VP, _VP, _VP]),
    ("trips_microbench", C.c_int, [C.c_int32, C.c_int32, _VP, C.c_int64, C.c_int32, C.c_int64, _VP,
                                   C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    ("trips_decoder_param_count", C.c_int64, [_VP, C.c_int32]),
    ("trips_decoder_workspace_bytes", C.c_size_t, [_VP]),
    ("trips_decode", C.c_int, [_VP, _VP, _VP, C.c_int32, _VP, _VP, _VP]),
    ("trips_launch_count", C.c_int64, []),
    ("trips_status_string", C.c_char_p, [C.c_int]),
]


def lib():
    """Loads libtrips.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (the CUDA library is required; there is no fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def status_string(status):
    return lib().trips_status_string(int(status)).decode()


def check(status, where):
    if status != TRIPS_OK:
        raise TripsError(status, where)
    return status


# ---- same names as include/trips.h -------------------------------------------------

def trips_plan_create(num_layers, num_features, width, height, max_points, t_min=0.0, coarse_layers=0):
    cfg = trips_config(num_layers, num_features, t_min, coarse_layers)
    out = _VP()
    check(lib().trips_plan_create(C.byref(cfg), width, height, max_points, C.byref(out)), "trips_plan_create")
    return out.value


def trips_plan_destroy(plan):
    lib().trips_plan_destroy(plan)


def trips_workspace_bytes(plan):
    return int(lib().trips_workspace_bytes(plan))


def trips_num_pixels(plan):
    return int(lib().trips_num_pixels(plan))


def trips_pyramid_floats(plan):
    return int(lib().trips_pyramid_floats(plan))


def trips_layer_dims(plan, l):
    h, w, off = C.c_int32(), C.c_int32(), C.c_int64()
    check(lib().trips_layer_dims(plan, l, C.byref(h), C.byref(w), C.byref(off)), "trips_layer_dims")
    return h.value, w.value, off.value


def camera_struct(cam):
    """Any object with fx, fy, cx, cy, f, R (3x3), t (3), width, height, near."""
    c = trips_camera()
    c.fx, c.fy, c.cx, c.cy, c.f = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), float(cam.f)
    R = np.asarray(cam.R, dtype=np.float32).reshape(9)
    t = np.asarray(cam.t, dtype=np.float32).reshape(3)
    for k in range(9):
        c.R[k] = float(R[k])
    for k in range(3):
        c.t[k] = float(t[k])
    c.width, c.height = int(cam.width), int(cam.height)
    c.near_plane = float(getattr(cam, "near", getattr(cam, "near_plane", 0.01)))
    return c


def trips_project(plan, ws, cam, n, pos, world_size, opacity, desc, level_out=None, proj_out=None, stream=None):
    c = cam if isinstance(cam, trips_camera) else camera_struct(cam)
    return lib().trips_project(plan, ws, C.byref(c), n, pos, world_size, opacity, desc, level_out, proj_out, stream)


def trips_splat_forward(plan, ws, pyramid, flags, stream=None):
    return lib().trips_splat_forward(plan, ws, pyramid, flags, stream)


def trips_splat_backward(plan, ws, grad_pyramid, grad_pos_size, grad_opacity, grad_desc, grad_camera=None,
                         stream=None):
    return lib().trips_splat_backward(plan, ws, grad_pyramid, grad_pos_size, grad_opacity, grad_desc, grad_camera,
                                      stream)


def trips_read_stats(plan, ws, stream=None):
    st = trips_stats()
    check(lib().trips_read_stats(plan, ws, C.byref(st), stream), "trips_read_stats")
    return {k: int(getattr(st, k)) for k, _ in trips_stats._fields_}


def trips_debug_export(plan, ws, what, dst, stream=None):
    return lib().trips_debug_export(plan, ws, what, dst, stream)


def trips_set_profiling(plan, enable):
    check(lib().trips_set_profiling(plan, 1 if enable else 0), "trips_set_profiling")


def trips_read_stage_ms(plan, reset=False):
    ms = (C.c_double * N_STAGES)()
    la = (C.c_int64 * N_STAGES)()
    lib().trips_read_stage_ms(plan, ms, la, N_STAGES, 1 if reset else 0)
    return {STAGE_NAMES[s]: (ms[s], la[s]) for s in range(N_STAGES)}


def trips_morton_workspace_bytes(n):
    return int(lib().trips_morton_workspace_bytes(n))


def trips_morton_order(ws, n, pos, perm_out, stream=None):
    return lib().trips_morton_order(ws, n, pos, perm_out, stream)


def trips_knn_workspace_bytes(n):
    return int(lib().trips_knn_workspace_bytes(n))


def trips_knn_sizes(ws, n, pos, size_out, nbr_out=None, stream=None):
    return lib().trips_knn_sizes(ws, n, pos, size_out, nbr_out, stream)


MB_OPS = {"red_v4_f32": 0, "red_f32": 1, "atomic_add_u32": 2, "store_v4": 3, "load_v4": 4}


def trips_microbench(op, pattern, buf, nbytes, row_bytes, ops, stream=None):
    """Returns (ms, ops_done) of one microbenchmark launch (synchronises the stream)."""
    ms, done = C.c_double(), C.c_int64()
    check(lib().trips_microbench(op, pattern, buf, nbytes, row_bytes, ops, stream, C.byref(ms), C.byref(done)),
          "trips_microbench")
    return ms.value, done.value


def trips_launch_count():
    return int(lib().trips_launch_count())


def trips_decoder_param_count(plan, out_channels):
    n = int(lib().trips_decoder_param_count(plan, out_channels))
    if n < 0:
        raise TripsError(TRIPS_ERR_ARG, "trips_decoder_param_count")
    return n


def trips_decoder_workspace_bytes(plan):
    return int(lib().trips_decoder_workspace_bytes(plan))


def trips_decode(plan, dws, params, out_channels, pyramid, out, stream):
    check(lib().trips_decode(plan, dws, params, out_channels, pyramid, out, stream), "trips_decode")
