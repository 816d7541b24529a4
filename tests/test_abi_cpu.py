"""The C-ABI library loads and exports every symbol include/trips.h declares; host-only
entry points (plan geometry, argument validation) work without a GPU.  No compute calls."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "trips.h")


@pytest.fixture(scope="module")
def A():
    from paper_2401_06003_b200 import build
    build.build()
    from paper_2401_06003_b200 import _abi
    _abi.lib()
    return _abi


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(trips_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(A):
    names = declared_functions()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (trips_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    bound = {s[0] for s in A.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_library_is_sm100a(A):
    out = subprocess.run(["cuobjdump", "--list-elf", A.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plan_geometry(A):
    plan = A.trips_plan_create(4, 4, 1920, 1080, 1000)
    try:
        assert A.trips_num_pixels(plan) == 2_754_000          # P at 1080p, n=4
        assert A.trips_pyramid_floats(plan) == 5 * 2_754_000
        dims = [A.trips_layer_dims(plan, l) for l in range(4)]
        assert [(h, w) for h, w, _ in dims] == [(1080, 1920), (540, 960), (270, 480), (135, 240)]
        assert [o for _, _, o in dims] == [0, 5 * 2073600, 5 * (2073600 + 518400), 5 * (2073600 + 518400 + 129600)]
        assert A.trips_workspace_bytes(plan) % 256 == 0
        with pytest.raises(A.TripsError):
            A.trips_layer_dims(plan, 4)
    finally:
        A.trips_plan_destroy(plan)
    plan = A.trips_plan_create(8, 4, 1920, 1080, 10)
    try:
        assert A.trips_num_pixels(plan) == 2_764_845           # P at 1080p, n=8
        small = A.trips_workspace_bytes(plan)
        # kept lists are dense per tile, 16 slots per pixel: kept-pair key (8 B) + info (4 B) + gamma (4 B)
        assert small >= 2_764_845 * 16 * (8 + 4 + 4)
    finally:
        A.trips_plan_destroy(plan)
    # coarse-layer inclusion: per-pixel kept keys (8 B) + own lists (8 B) + gamma (4 B) per slot
    plan = A.trips_plan_create(8, 4, 1920, 1080, 10, 0.0, 20)
    try:
        assert A.trips_workspace_bytes(plan) >= 2_764_845 * 16 * (8 + 8 + 4)
    finally:
        A.trips_plan_destroy(plan)


@pytest.mark.parametrize("args", [(0, 4, 64, 64, 10), (17, 4, 64, 64, 10), (4, 0, 64, 64, 10),
                                  (4, 33, 64, 64, 10), (4, 4, 0, 64, 10), (4, 4, 64, 64, -1),
                                  (4, 4, 64, 64, 1 << 28), (4, 4, 64, 64, 10, -0.1), (4, 4, 64, 64, 10, 1.0),
                                  (4, 4, 64, 64, 10, 0.0, -1)])
def test_plan_create_rejects(A, args):
    with pytest.raises(A.TripsError) as e:
        A.trips_plan_create(*args)
    assert e.value.status == A.TRIPS_ERR_ARG


def test_host_side_validation(A):
    """Validation happens before any CUDA call, so these run without a GPU."""
    from synth import scenes
    sc = scenes.c1()
    cam = sc.cams[0]
    plan = A.trips_plan_create(4, 4, cam.width, cam.height, 100)
    try:
        ws = 256 * 1024
        assert A.trips_project(plan, ws, cam, 101, 16, 16, 16, 16) == A.TRIPS_ERR_CAPACITY
        assert A.trips_project(plan, ws, cam, -1, 16, 16, 16, 16) == A.TRIPS_ERR_ARG
        assert A.trips_project(plan, ws + 8, cam, 10, 16, 16, 16, 16) == A.TRIPS_ERR_ALIGN
        assert A.trips_project(plan, None, cam, 10, 16, 16, 16, 16) == A.TRIPS_ERR_ARG
        bad = scenes.Camera(fx=0.0, fy=1.0, cx=0, cy=0, f=1.0, R=cam.R, t=cam.t, width=cam.width, height=cam.height)
        assert A.trips_project(plan, ws, bad, 10, 16, 16, 16, 16) == A.TRIPS_ERR_ARG
        wrong = scenes.Camera(fx=1.0, fy=1.0, cx=0, cy=0, f=1.0, R=cam.R, t=cam.t, width=cam.width + 1,
                              height=cam.height)
        assert A.trips_project(plan, ws, wrong, 10, 16, 16, 16, 16) == A.TRIPS_ERR_ARG
        assert A.trips_splat_forward(plan, ws, 256, 1) == A.TRIPS_ERR_STATE
        assert A.trips_splat_backward(plan, ws, 256, 256, 256, 256) == A.TRIPS_ERR_STATE
        assert A.trips_splat_backward(plan, ws, None, 256, 256, 256) == A.TRIPS_ERR_ARG
        assert "STATE" in A.status_string(A.TRIPS_ERR_STATE)
    finally:
        A.trips_plan_destroy(plan)


def test_microbench_validation(A):
    """trips_microbench rejects bad arguments before any CUDA call."""
    import ctypes as C
    ms, done = C.c_double(), C.c_int64()
    L = A.lib()
    assert L.trips_microbench(5, 0, 1 << 20, 1 << 20, 16, 1, None, C.byref(ms), C.byref(done)) == A.TRIPS_ERR_ARG
    assert L.trips_microbench(0, 2, 1 << 20, 1 << 20, 16, 1, None, C.byref(ms), C.byref(done)) == A.TRIPS_ERR_ARG
    assert L.trips_microbench(0, 0, 1 << 20, 1 << 20, 24, 1, None, C.byref(ms), C.byref(done)) == A.TRIPS_ERR_ARG
    assert L.trips_microbench(0, 0, 1 << 20, 512, 16, 1, None, C.byref(ms), C.byref(done)) == A.TRIPS_ERR_ARG
    assert L.trips_microbench(0, 0, (1 << 20) + 4, 1 << 20, 16, 1, None, C.byref(ms), C.byref(done)) == \
        A.TRIPS_ERR_ALIGN


def test_no_cpu_fallback_when_library_missing(A, tmp_path, monkeypatch):
    """The binding raises (it never falls back) when libtrips.so is absent."""
    monkeypatch.setattr(A, "_lib", None)
    monkeypatch.setattr(A, "LIB_PATH", str(tmp_path / "libtrips.so"))
    with pytest.raises(ImportError):
        A.lib()


def test_large_plans_are_accepted(A):
    """More tiles than the shared-memory binning counters hold (8K frames: 172 200 tiles at 4
    layers) select global-counter binning instead of failing; > 2^20 tiles is rejected."""
    plan = A.trips_plan_create(4, 4, 7680, 4320, 10)
    try:
        assert A.trips_pyramid_floats(plan) > 7680 * 4320 * 5
    finally:
        A.trips_plan_destroy(plan)
    with pytest.raises(A.TripsError):
        A.trips_plan_create(1, 4, 32768, 32768, 10)        # 4 194 304 tiles
