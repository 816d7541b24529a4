"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  bit-exact  projected records (x, y, z, s), level codes, per-pixel counts, kept lists
  features   |C_gpu - C_oracle| <= 1e-5 * M_C   (M_C = sum_m T_m gamma_m |tau|, per channel)
  gradients  |g_gpu - g_oracle| <= 1e-3 * M_g   (M_g = the chain with |.| of every factor)
"""
import numpy as np
import pytest
import torch

from oracle import oracle
from synth import scenes

pytestmark = pytest.mark.gpu

FEAT_TOL = 1e-5
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_06003_b200 import _abi
    _abi.lib()
    return torch.device("cuda:0")


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _ovar(var):
    """Rasterizer variant kwargs -> oracle kwargs."""
    return dict(t_min=var.get("t_min", 0.0), coarse=var.get("coarse_layers", 0))


def gpu_run(sc, dev, cam=None, G=None, save=True, export=True, desc_misalign=False, **var):
    """var: Rasterizer variant options (t_min, coarse_layers).  desc_misalign: pass the descriptors
    as a view 4 bytes into a buffer (4-B but not 16-B aligned: the library takes its padded copy)."""
    from paper_2401_06003_b200 import Rasterizer
    cam = cam or sc.cams[0]
    r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=max(sc.n, 1), device=dev, **var)
    pos, sw, al, de = (T(a, dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
    if desc_misalign:
        buf = torch.zeros(de.numel() + 4, dtype=torch.float32, device=dev)
        de = buf[1:1 + de.numel()].view(sc.n, sc.F)
        de.copy_(T(sc.desc, dev))
        assert de.data_ptr() % 16 != 0
    level = torch.empty(sc.n, dtype=torch.int8, device=dev)
    proj = torch.empty(sc.n, 4, dtype=torch.float32, device=dev)
    r.project(cam, pos, sw, al, de, level_out=level, proj_out=proj)
    pyr = r.forward(save=save)
    out = dict(pyr=pyr.cpu().numpy(), level=level.cpu().numpy(), proj=proj.cpu().numpy(), stats=r.stats(), r=r)
    if export:
        out["counts"] = r.export_counts().cpu().numpy().astype(np.uint32)
        if save:
            out["kept"] = r.export_kept().cpu().numpy()
            if var.get("coarse_layers", 0):
                out["kept_layer"] = r.export_kept_layer().cpu().numpy()
    if G is not None:
        g = r.backward(T(G, dev))
        out["grad"] = r.grad_rows(g).cpu().numpy().astype(np.float64)
        out["screen"] = r.export_screen_grads().cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    return out


def check_forward(sc, got, cam=None, mask=None, **var):
    cam = cam or sc.cams[0]
    ref = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, mask=mask, **_ovar(var))
    proj, level, _ = oracle.project(cam, sc.n_layers, sc.pos, sc.sw)
    # bit-exact block
    assert np.array_equal(got["level"], level), "level codes differ"
    assert np.array_equal(got["proj"].view(np.uint32), proj.view(np.uint32)), "projected records differ"
    if mask is None:
        assert np.array_equal(got["counts"], ref["counts"]), "counts differ"
        if "kept" in got:
            assert np.array_equal(got["kept"], ref["kept"]), "kept lists differ"
        if "kept_layer" in got:
            assert np.array_equal(got["kept_layer"], ref["kept_layer"].astype(np.int32)), "kept layers differ"
        st = got["stats"]
        for k in ("n_culled", "n_visible", "n_frag", "n_kept", "n_trunc_pixels", "max_list"):
            assert st[k] == ref["stats"][k], (k, st[k], ref["stats"][k])
        sel = slice(None)
        pix = slice(None)
    else:
        pix = np.nonzero(mask)[0]
        assert np.array_equal(got["counts"][pix], ref["counts"][pix]), "counts differ (sampled)"
        if "kept" in got:
            assert np.array_equal(got["kept"][pix], ref["kept"][pix]), "kept lists differ (sampled)"
        if "kept_layer" in got:
            assert np.array_equal(got["kept_layer"][pix], ref["kept_layer"][pix].astype(np.int32))
        F1 = sc.F + 1
        sel = pixel_float_index(cam, sc.n_layers, F1, pix)
    err = np.abs(got["pyr"].astype(np.float64)[sel] - ref["pyramid"][sel])
    bound = FEAT_TOL * ref["mag"][sel] + 1e-30
    bad = err > bound
    assert not bad.any(), f"{bad.sum()} features out of tolerance, worst {err.max():.3e}"
    return ref


def pixel_float_index(cam, n_layers, F1, pix):
    """Float indices of all channels of the given pyramid pixels."""
    dims = oracle.layer_dims(cam.width, cam.height, n_layers)
    offs = np.cumsum([0] + [h * w for (h, w) in dims])
    out = []
    for l, (h, w) in enumerate(dims):
        sel = pix[(pix >= offs[l]) & (pix < offs[l + 1])] - offs[l]
        for c in range(F1):
            out.append(offs[l] * F1 + c * h * w + sel)
    return np.concatenate(out)


def check_backward(sc, got, G, cam=None, mask=None, **var):
    cam = cam or sc.cams[0]
    scr = np.zeros((sc.n, 4 + sc.F))
    scm = np.zeros((sc.n, 4 + sc.F))
    g, gm = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, mask=mask, screen=scr,
                            screen_mag=scm, **_ovar(var))
    err = np.abs(got["grad"] - g)
    bad = err > GRAD_TOL * gm + 1e-30
    assert not bad.any(), f"{bad.sum()} gradient entries out of tolerance; worst rel " \
                          f"{(err / np.maximum(gm, 1e-30)).max():.3e}"
    if "screen" in got:                                  # SCREEN_GRADS debug export
        serr = np.abs(got["screen"] - scr)
        assert not (serr > GRAD_TOL * scm + 1e-30).any(), "screen-space gradients out of tolerance"
    rel_l2 = np.linalg.norm(got["grad"] - g) / max(np.linalg.norm(g), 1e-30)
    assert rel_l2 < 1e-4, rel_l2


def grads_for(sc, cam, seed=100, mask=None):
    P = oracle.num_pixels(cam.width, cam.height, sc.n_layers)
    G = scenes.grad_pyramid(P * (sc.F + 1), seed=seed)
    if mask is not None:
        keep = np.zeros(G.size, bool)
        keep[pixel_float_index(cam, sc.n_layers, sc.F + 1, np.nonzero(mask)[0])] = True
        G = np.where(keep, G, 0).astype(np.float32)
    return G


# ------------------------------------------------------------------ small scenes

def test_c1_forward_backward(dev):
    sc = scenes.c1()
    G = grads_for(sc, sc.cams[0])
    got = gpu_run(sc, dev, G=G)
    check_forward(sc, got)
    check_backward(sc, got, G)


@pytest.mark.parametrize("seed", range(20))
def test_random_tiny_scenes(dev, seed):
    sc = scenes.tiny_scene(seed)
    G = grads_for(sc, sc.cams[0], seed=seed)
    got = gpu_run(sc, dev, G=G)
    check_forward(sc, got)
    check_backward(sc, got, G)


def test_adversarial_scene(dev):
    sc = scenes.adversarial_scene()
    G = grads_for(sc, sc.cams[0], seed=5)
    got = gpu_run(sc, dev, G=G)
    check_forward(sc, got)
    check_backward(sc, got, G)
    assert got["stats"]["max_list"] >= 40


@pytest.mark.parametrize("F", [1, 3, 5, 6, 8, 13])
def test_feature_counts(dev, F):
    sc = scenes.tiny_scene(3, n=500, F=F, W=50, H=37, n_layers=4)
    G = grads_for(sc, sc.cams[0], seed=F)
    got = gpu_run(sc, dev, G=G)
    check_forward(sc, got)
    check_backward(sc, got, G)


@pytest.mark.parametrize("F", [4, 8])
def test_descriptors_not_16b_aligned(dev, F):
    # F % 4 == 0 but desc only 4-B aligned: the padded workspace copy is gathered instead of the
    # caller's rows (include/trips.h, trips_project)
    sc = scenes.tiny_scene(7, n=600, F=F, W=61, H=45, n_layers=4)
    G = grads_for(sc, sc.cams[0], seed=F + 50)
    got = gpu_run(sc, dev, G=G, desc_misalign=True)
    check_forward(sc, got)
    check_backward(sc, got, G)


def test_dense_tiles_multi_chunk_and_long_lists(dev):
    """Many points in few tiles: several 512-pair chunks per tile, lists >> 16."""
    sc = scenes.tiny_scene(11, n=30000, F=4, W=40, H=24, n_layers=3)
    G = grads_for(sc, sc.cams[0], seed=3)
    got = gpu_run(sc, dev, G=G)
    check_forward(sc, got)
    check_backward(sc, got, G)
    assert got["stats"]["max_list"] > 100


def test_empty_and_all_culled(dev):
    sc = scenes.tiny_scene(1, n=10)
    sc.pos[:, :] = np.float32(np.nan)
    got = gpu_run(sc, dev)
    assert not got["pyr"].any() and got["stats"]["n_culled"] == 10
    sc0 = scenes.tiny_scene(2, n=1)
    sc0.pos, sc0.sw, sc0.alpha, sc0.desc = sc0.pos[:0], sc0.sw[:0], sc0.alpha[:0], sc0.desc[:0]
    got = gpu_run(sc0, dev)
    assert not got["pyr"].any() and not got["counts"].any()


def test_forward_is_deterministic(dev):
    sc = scenes.tiny_scene(4, n=5000, W=64, H=48)
    a = gpu_run(sc, dev)
    b = gpu_run(sc, dev)
    assert np.array_equal(a["pyr"].view(np.uint32), b["pyr"].view(np.uint32))


def test_multi_view_accumulation(dev):
    """Gradients of several views accumulate (+=) into one packed buffer (reading Q21)."""
    from paper_2401_06003_b200 import Rasterizer
    sc = scenes.make_config("C4", n=20000, n_views=3)
    cams = [scenes.look_at(-c.R.T.astype(np.float64) @ c.t.astype(np.float64), [0, 0, 0], 160, 96, 100.0)
            for c in sc.cams]
    r = Rasterizer(160, 96, 4, sc.F, max_points=sc.n, device=dev)
    pos, sw, al, de = (T(a, dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
    grad = r.new_grad(sc.n)
    acc, accm = None, None
    for v, cam in enumerate(cams):
        G = scenes.grad_pyramid(r.pyramid_floats, seed=v)
        r.project(cam, pos, sw, al, de)
        r.forward(save=True)
        r.backward(T(G, dev), grad)
        acc, accm = oracle.backward(cam, 4, sc.pos, sc.sw, sc.alpha, sc.desc, G, grad=acc, grad_mag=accm)
    got = r.grad_rows(grad).cpu().numpy()
    assert np.all(np.abs(got - acc) <= GRAD_TOL * accm + 1e-30)


def test_batch_step_over_two_streams(dev):
    """dist.cuda_batch_step: views spread over 2 streams / 2 workspaces accumulate the same
    gradient sum as the oracle (reading Q21), concurrent reductions included."""
    from paper_2401_06003_b200 import Rasterizer
    from paper_2401_06003_b200 import dist as tdist
    sc = scenes.make_config("C4", n=20000, n_views=5)
    cams = [scenes.look_at(-c.R.T.astype(np.float64) @ c.t.astype(np.float64), [0, 0, 0], 160, 96, 100.0)
            for c in sc.cams]
    rasts = [Rasterizer(160, 96, 4, sc.F, max_points=sc.n, device=dev) for _ in range(2)]
    pos, sw, al, de = (T(a, dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
    Gs = [scenes.grad_pyramid(rasts[0].pyramid_floats, seed=v) for v in range(5)]
    Gd = [T(g, dev) for g in Gs]
    grad = torch.full((rasts[0].grad_floats(sc.n),), 7.0, device=dev)       # zeroed by the step
    tdist.cuda_batch_step(rasts, cams, pos, sw, al, de, lambda v: Gd[v], range(5), grad)
    torch.cuda.synchronize()
    acc, accm = None, None
    for v, cam in enumerate(cams):
        acc, accm = oracle.backward(cam, 4, sc.pos, sc.sw, sc.alpha, sc.desc, Gs[v], grad=acc, grad_mag=accm)
    got = rasts[0].grad_rows(grad, sc.n).cpu().numpy()
    assert np.all(np.abs(got - acc) <= GRAD_TOL * accm + 1e-30)


def test_streamed_steps_pipeline(dev):
    """dist.ShardedStreamedSteps (the bench's e2e path, world 1): double-buffered host -> device
    -> host steps through the flat input buffer give every step's exact gradients (same as a
    synchronous step) in host memory."""
    from paper_2401_06003_b200 import Rasterizer
    from paper_2401_06003_b200 import dist as tdist
    sc = scenes.make_config("C4", n=20000, n_views=3)
    cams = [scenes.look_at(-c.R.T.astype(np.float64) @ c.t.astype(np.float64), [0, 0, 0], 160, 96, 100.0)
            for c in sc.cams]
    rasts = [Rasterizer(160, 96, 4, sc.F, max_points=sc.n, device=dev) for _ in range(2)]
    G = T(scenes.grad_pyramid(rasts[0].pyramid_floats, seed=3), dev)
    dv = {k: T(v, dev) for k, v in (("pos", sc.pos), ("sw", sc.sw), ("alpha", sc.alpha), ("desc", sc.desc))}
    nf = rasts[0].grad_floats(sc.n)
    ref = torch.zeros(nf, device=dev)
    tdist.cuda_batch_step(rasts, cams, dv["pos"], dv["sw"], dv["alpha"], dv["desc"], G, range(3), ref)
    torch.cuda.synchronize()
    ref = ref.cpu().numpy()

    flat, n, F = tdist.flat_inputs(dv["pos"], dv["sw"], dv["alpha"], dv["desc"])
    host_flat = flat.cpu().pin_memory()
    pipe = tdist.ShardedStreamedSteps(host_flat, nf, dev)
    assert pipe.h2d_bytes == host_flat.numel() * 4 and pipe.d2h_bytes == nf * 4
    out = [torch.zeros(nf).pin_memory() for _ in range(2)]

    def step(dev_flat, g, o):
        pos, sw, al, de = tdist.input_views(dev_flat, n, F)
        tdist.cuda_batch_step(rasts, cams, pos, sw, al, de, G, range(3), g, reduce="reduce_scatter", out=o)

    pipe.run(5, step, out)
    torch.cuda.synchronize()
    for o in out:
        got = o.numpy()
        assert np.allclose(got, ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max())


def test_autograd_render(dev):
    from paper_2401_06003_b200 import Rasterizer
    sc = scenes.c1()
    cam = sc.cams[0]
    r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
    ps = [T(a, dev).requires_grad_() for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
    layers = r.render(cam, *ps)
    G = scenes.grad_pyramid(r.pyramid_floats, seed=7)
    flat = torch.cat([L.reshape(-1) for L in layers])
    (flat * T(G, dev)).sum().backward()
    g, gm = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G)
    got = np.concatenate([ps[0].grad.cpu().numpy(), ps[1].grad.cpu().numpy()[:, None],
                          ps[2].grad.cpu().numpy()[:, None], ps[3].grad.cpu().numpy()], 1)
    assert np.all(np.abs(got - g) <= GRAD_TOL * gm + 1e-30)


# ------------------------------------------------------------------ ABI error paths

def test_abi_error_paths(dev):
    from paper_2401_06003_b200 import _abi as A
    sc = scenes.c1()
    cam = sc.cams[0]
    plan = A.trips_plan_create(sc.n_layers, sc.F, cam.width, cam.height, sc.n)
    try:
        ws = torch.empty(A.trips_workspace_bytes(plan), dtype=torch.uint8, device=dev)
        ws2 = torch.empty(A.trips_workspace_bytes(plan), dtype=torch.uint8, device=dev)
        pyr = torch.empty(A.trips_pyramid_floats(plan), device=dev)
        grad = torch.zeros(sc.n * (5 + sc.F), device=dev)
        gps, gde, gop = grad.data_ptr(), grad.data_ptr() + 16 * sc.n, grad.data_ptr() + 4 * (4 + sc.F) * sc.n
        pos, sw, al, de = (T(a, dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
        args = (pos.data_ptr(), sw.data_ptr(), al.data_ptr(), de.data_ptr())
        assert A.trips_splat_forward(plan, ws.data_ptr(), pyr.data_ptr(), 1) == A.TRIPS_ERR_STATE
        assert A.trips_project(plan, ws.data_ptr(), cam, sc.n + 1, *args) == A.TRIPS_ERR_CAPACITY
        assert A.trips_project(plan, ws.data_ptr() + 16, cam, sc.n, *args) == A.TRIPS_ERR_ALIGN
        assert A.trips_project(plan, ws.data_ptr(), cam, -1, *args) == A.TRIPS_ERR_ARG
        assert A.trips_project(plan, ws.data_ptr(), cam, sc.n, None, *args[1:]) == A.TRIPS_ERR_ARG
        assert A.trips_project(plan, ws.data_ptr(), cam, sc.n, *args) == A.TRIPS_OK
        assert A.trips_splat_forward(plan, ws2.data_ptr(), pyr.data_ptr(), 1) == A.TRIPS_ERR_STATE
        assert A.trips_splat_forward(plan, ws.data_ptr(), pyr.data_ptr(), 0) == A.TRIPS_OK
        assert A.trips_splat_backward(plan, ws.data_ptr(), pyr.data_ptr(), gps, gop, gde) == A.TRIPS_ERR_STATE
        assert A.trips_splat_forward(plan, ws.data_ptr(), pyr.data_ptr(), 1) == A.TRIPS_ERR_STATE  # needs project
        assert A.trips_project(plan, ws.data_ptr(), cam, sc.n, *args) == A.TRIPS_OK
        assert A.trips_splat_forward(plan, ws.data_ptr(), pyr.data_ptr(), 1) == A.TRIPS_OK
        assert A.trips_splat_backward(plan, ws.data_ptr(), pyr.data_ptr(), gps + 4, gop, gde) == A.TRIPS_ERR_ALIGN
        assert A.trips_splat_backward(plan, ws.data_ptr(), pyr.data_ptr(), gps, gop + 2, gde) == A.TRIPS_ERR_ALIGN
        assert A.trips_splat_backward(plan, ws.data_ptr(), pyr.data_ptr(), None, gop, gde) == A.TRIPS_ERR_ARG
        assert A.trips_splat_backward(plan, ws.data_ptr(), pyr.data_ptr(), gps, gop, gde) == A.TRIPS_OK
        torch.cuda.synchronize()
    finally:
        A.trips_plan_destroy(plan)


# ------------------------------------------------------------------ full-size configs

def _sample_mask(cam, n_layers, seed, n_random=3000):
    P = oracle.num_pixels(cam.width, cam.height, n_layers)
    rng = np.random.default_rng(seed)
    mask = np.zeros(P, np.uint8)
    mask[rng.choice(P, n_random, replace=False)] = 1
    # plus two full 16x16 blocks in layer 0 and everything in the coarsest layer
    W = cam.width
    for (y0, x0) in ((cam.height // 2 - 8, W // 2 - 8), (cam.height - 20, 40)):
        for y in range(y0, y0 + 16):
            mask[y * W + x0:y * W + x0 + 16] = 1
    dims = oracle.layer_dims(cam.width, cam.height, n_layers)
    mask[P - dims[-1][0] * dims[-1][1]:] = 1
    return mask


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_full_size_sampled(dev, name):
    """Full-size configs in the bench launch configuration; the oracle computes sampled
    pixels (lists restricted to a pixel mask), gradients of a loss on those pixels."""
    sc = scenes.make_config(name)
    cam = sc.cams[0]
    mask = _sample_mask(cam, sc.n_layers, seed=len(name))
    G = None if sc.forward_only else grads_for(sc, cam, seed=1, mask=mask)
    got = gpu_run(sc, dev, G=G, save=True)
    check_forward(sc, got, mask=mask)
    st = got["stats"]
    assert st["n_visible"] + st["n_culled"] == sc.n
    assert st["n_kept"] <= st["n_frag"] and int(got["counts"].sum()) == st["n_frag"]
    assert np.minimum(got["counts"], 16).sum() == st["n_kept"]
    if G is not None:
        check_backward(sc, got, G, mask=mask)


def test_c2_whole_frame_forward(dev):
    """C2 (5M points, 1080p, forward only) compared on EVERY pyramid pixel: counts, kept lists,
    statistics bit-exact and all features within tolerance (no pixel sampling)."""
    sc = scenes.make_config("C2")
    got = gpu_run(sc, dev, save=True)
    check_forward(sc, got)


def test_c4_full_size_bench_layout(dev):
    """C4 at full size in the bench launch layout: 8M points in Morton order,
    views spread over two CUDA streams with one plan + workspace each, gradients of two views
    accumulated into one flat buffer by dist.cuda_batch_step.  The oracle (full lists, every pixel)
    checks view 0's counts, kept lists and features bit-exact / within tolerance, and EVERY point's
    gradient summed over both views (full-frame upstream gradients)."""
    from paper_2401_06003_b200 import Rasterizer
    from paper_2401_06003_b200 import dist as tdist
    sc = scenes.make_config("C4", order="morton")        # generator-side Morton layout (no CUDA-made input)
    views = [0, 17]
    cam0 = sc.cams[0]
    rasts = [Rasterizer(cam0.width, cam0.height, sc.n_layers, sc.F, max_points=sc.n, device=dev) for _ in range(2)]
    streams = [torch.cuda.current_stream(), torch.cuda.Stream(device=dev)]
    pos, sw, al, de = (T(a, dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
    Gs = {v: scenes.grad_pyramid(rasts[0].pyramid_floats, seed=200 + v) for v in views}
    Gd = {v: T(g, dev) for v, g in Gs.items()}
    grad = rasts[0].new_grad(sc.n)
    tdist.cuda_batch_step(rasts, sc.cams, pos, sw, al, de, lambda v: Gd[v], views, grad, streams=streams)
    torch.cuda.synchronize()
    got_grad = rasts[0].grad_rows(grad).cpu().numpy().astype(np.float64)
    # view 0's forward state (the forward is deterministic, so this is the step's view 0)
    got = gpu_run(sc, dev, cam=sc.cams[0], save=True)
    check_forward(sc, got, cam=sc.cams[0])
    acc, accm = None, None
    for v in views:
        acc, accm = oracle.backward(sc.cams[v], sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, Gs[v], grad=acc,
                                    grad_mag=accm)
    err = np.abs(got_grad - acc)
    bad = err > GRAD_TOL * accm + 1e-30
    assert not bad.any(), f"{bad.sum()} of {bad.size} gradient entries out of tolerance"
    assert np.linalg.norm(got_grad - acc) / np.linalg.norm(acc) < 1e-4
    assert np.count_nonzero(acc[:, 5]) > 0.5 * sc.n          # most points received a gradient


def test_2k_relation_full_size(dev):
    """P5 at full scale, GPU only: doubling (fx, fy, cx, cy, f, W, H) and adding a layer maps
    layer l of the original onto layer l+1 bit for bit (counts, kept lists, features)."""
    sc = scenes.make_config("C2", n=2_000_000)
    cam = sc.cams[0]
    cam.cx, cam.cy = 959.0, 539.0                      # make 2*c exact and the relation exact
    cam2 = scenes.Camera(fx=2 * cam.fx, fy=2 * cam.fy, cx=2 * cam.cx, cy=2 * cam.cy, f=2 * cam.f, R=cam.R, t=cam.t,
                         width=2 * cam.width, height=2 * cam.height, near=cam.near)
    a = gpu_run(sc, dev, cam=cam)
    sc.n_layers += 1
    b = gpu_run(sc, dev, cam=cam2)
    sc.n_layers -= 1
    da = oracle.layer_dims(cam.width, cam.height, sc.n_layers)
    db = oracle.layer_dims(cam2.width, cam2.height, sc.n_layers + 1)
    pa = np.cumsum([0] + [h * w for h, w in da])
    pb = np.cumsum([0] + [h * w for h, w in db])
    F1 = sc.F + 1
    for l in range(1, sc.n_layers):
        assert np.array_equal(a["counts"][pa[l]:pa[l + 1]], b["counts"][pb[l + 1]:pb[l + 2]])
        assert np.array_equal(a["kept"][pa[l]:pa[l + 1]], b["kept"][pb[l + 1]:pb[l + 2]])
        assert np.array_equal(a["pyr"][pa[l] * F1:pa[l + 1] * F1], b["pyr"][pb[l + 1] * F1:pb[l + 2] * F1])


# ------------------------------------------------------------------ data-layout utility

def test_morton_order_permutation(dev):
    """trips_morton_order returns a permutation whose 30-bit Morton codes (recomputed here in
    numpy over the same bounding box) are non-decreasing; rendering the permuted cloud gives
    the same pyramid (no depth ties in this scene)."""
    from paper_2401_06003_b200 import Rasterizer, morton_order
    sc = scenes.make_config("C4", n=200_000, n_views=1)
    pos = T(sc.pos, dev)
    perm = morton_order(pos).cpu().numpy()
    assert np.array_equal(np.sort(perm), np.arange(sc.n))
    p = sc.pos.astype(np.float32)
    lo, hi = p.min(0), p.max(0)
    ext = np.maximum(hi - lo, np.float32(1e-30))
    q = np.clip(((p - lo) / ext * np.float32(1023.0)), 0, 1023).astype(np.uint32)

    def spread(v):
        v = v & 0x3FF
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        v = (v | (v << 2)) & 0x09249249
        return v
    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    c = code[perm].astype(np.int64)
    # float rounding of the quantisation may differ by one cell at cell borders
    assert (np.diff(c) < 0).mean() < 1e-3
    a = gpu_run(sc, dev)
    sc2 = scenes.Scene("C4p", sc.pos[perm], sc.sw[perm], sc.alpha[perm], sc.desc[perm], sc.cams, sc.n_layers)
    b = gpu_run(sc2, dev)
    assert np.array_equal(a["counts"], b["counts"])
    kb = np.where(b["kept"] >= 0, perm[np.maximum(b["kept"], 0)], -1)
    differ = (a["kept"] != kb).any(1)
    # only exact depth ties may reorder (the tie-break is the point index, reading Q12)
    z = a["proj"][:, 2]
    for p in np.nonzero(differ)[0]:
        ka = a["kept"][p][a["kept"][p] >= 0]
        kk = kb[p][kb[p] >= 0]
        assert np.array_equal(z[ka], z[kk]) and len(set(z[ka])) < len(ka)
    assert differ.mean() < 1e-4
    F1 = sc.F + 1
    same_pix = np.nonzero(~differ)[0]
    sel = pixel_float_index(sc.cams[0], sc.n_layers, F1, same_pix)
    assert np.array_equal(a["pyr"][sel], b["pyr"][sel])
    del Rasterizer


# ------------------------------------------------------------------ camera gradient (8(f) row 1)

def _camera_grad_case(sc, dev, mask=None, seed=3):
    from paper_2401_06003_b200 import Rasterizer
    cam = sc.cams[0]
    G = grads_for(sc, cam, seed=seed, mask=mask)
    r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=max(sc.n, 1), device=dev)
    pos, sw, al, de = (T(a, dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
    r.project(cam, pos, sw, al, de)
    r.forward(save=True)
    gcam = torch.zeros(17, device=dev)
    grad = r.backward(T(G, dev), grad_camera=gcam)
    grad_nocam = r.backward(T(G, dev))                  # the CAM=false kernel gives the same point grads
    torch.cuda.synchronize()
    gc = np.zeros(17)
    gcm = np.zeros(17)
    g, gm = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, mask=mask, grad_cam=gc,
                            grad_cam_mag=gcm)
    got = gcam.cpu().numpy().astype(np.float64)
    err = np.abs(got - gc)
    bad = err > GRAD_TOL * gcm + 1e-30
    assert not bad.any(), [(oracle.CAMERA_GRAD_NAMES[k], got[k], gc[k], gcm[k]) for k in np.nonzero(bad)[0]]
    a = r.grad_rows(grad).cpu().numpy()
    b = r.grad_rows(grad_nocam).cpu().numpy()
    assert np.all(np.abs(a - b) <= 1e-3 * np.abs(b) + 1e-6 * np.abs(b).max())


@pytest.mark.parametrize("t_min", [0.05, 0.4])
def test_tmin_variant(dev, t_min):
    """T_min early termination -- identical cut lists (the cut is an fp32
    decision taken the same way on both sides), features and gradients within tolerance."""
    for sc in (scenes.c1(), scenes.tiny_scene(11, n=30000, F=4, W=40, H=24, n_layers=3)):
        cam = sc.cams[0]
        G = grads_for(sc, cam, seed=2)
        got = gpu_run(sc, dev, G=G, t_min=t_min)
        ref = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, t_min=t_min)
        assert np.array_equal(got["kept"], ref["kept"])
        assert np.array_equal(got["counts"], ref["counts"])
        err = np.abs(got["pyr"].astype(np.float64) - ref["pyramid"])
        assert np.all(err <= FEAT_TOL * ref["mag"] + 1e-30)
        g, gm = oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, t_min=t_min)
        assert np.all(np.abs(got["grad"] - g) <= GRAD_TOL * gm + 1e-30)
        full = oracle.forward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc)
        assert (ref["kept"] >= 0).sum() < (full["kept"] >= 0).sum()          # the variant does cut


def test_camera_gradient_c1(dev):
    _camera_grad_case(scenes.c1(), dev)


@pytest.mark.parametrize("seed", range(6))
def test_camera_gradient_random(dev, seed):
    _camera_grad_case(scenes.tiny_scene(seed), dev, seed=seed)


def test_camera_gradient_adversarial_and_full_size(dev):
    _camera_grad_case(scenes.adversarial_scene(), dev)
    sc = scenes.make_config("C3", n=1_000_000)
    _camera_grad_case(sc, dev, mask=_sample_mask(sc.cams[0], sc.n_layers, seed=9))


# ------------------------------------------------------------------ coarse-layer inclusion

def _coarse_cases():
    yield "c1", scenes.c1(), 3
    yield "adv", scenes.adversarial_scene(), 1
    yield "dense", scenes.tiny_scene(11, n=30000, F=4, W=40, H=24, n_layers=3), 2
    yield "f6", scenes.tiny_scene(3, n=800, F=6, W=50, H=37, n_layers=5), 4
    for seed in range(6):
        yield f"tiny{seed}", scenes.tiny_scene(seed), 1 + seed % 3


@pytest.mark.parametrize("case", range(10))
def test_coarse_inclusion(dev, case):
    """SURVEY.md 8(f) row 3 / reading Q22: bit-exact own counts, merged kept lists and their
    layer offsets; features and gradients within the north-star tolerances."""
    name, sc, c = list(_coarse_cases())[case]
    G = grads_for(sc, sc.cams[0], seed=case)
    got = gpu_run(sc, dev, G=G, coarse_layers=c)
    check_forward(sc, got, coarse_layers=c)
    check_backward(sc, got, G, coarse_layers=c)
    if sc.n_layers > 1 and got["stats"]["n_frag"] > 100:
        assert (got["kept_layer"] > 0).any(), name                  # coarse fragments were merged


def test_coarse_with_tmin_and_camera_gradient(dev):
    from paper_2401_06003_b200 import Rasterizer
    sc = scenes.tiny_scene(11, n=30000, F=4, W=40, H=24, n_layers=3)
    cam = sc.cams[0]
    G = grads_for(sc, cam, seed=8)
    got = gpu_run(sc, dev, G=G, coarse_layers=2, t_min=0.1)
    check_forward(sc, got, coarse_layers=2, t_min=0.1)
    check_backward(sc, got, G, coarse_layers=2, t_min=0.1)
    r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=sc.n, device=dev, coarse_layers=2)
    pos, sw, al, de = (T(a, dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc))
    r.project(cam, pos, sw, al, de)
    r.forward(save=True)
    gc = torch.zeros(17, device=dev)
    r.backward(T(G, dev), grad_camera=gc)
    ref, refm = np.zeros(17), np.zeros(17)
    oracle.backward(cam, sc.n_layers, sc.pos, sc.sw, sc.alpha, sc.desc, G, grad_cam=ref, grad_cam_mag=refm,
                    coarse=2)
    assert np.all(np.abs(gc.cpu().numpy() - ref) <= GRAD_TOL * refm + 1e-30)


def test_coarse_full_size_c3_sampled(dev):
    """C3 (6M points, 8 layers, wide sizes) in the bench launch configuration with every
    coarser layer included; oracle on sampled pixels (their ancestors' lists are built)."""
    sc = scenes.make_config("C3")
    cam = sc.cams[0]
    mask = _sample_mask(cam, sc.n_layers, seed=33, n_random=1500)
    G = grads_for(sc, cam, seed=2, mask=mask)
    got = gpu_run(sc, dev, G=G, coarse_layers=7)
    check_forward(sc, got, mask=mask, coarse_layers=7)
    check_backward(sc, got, G, mask=mask, coarse_layers=7)
    plain = gpu_run(sc, dev, export=True)
    assert np.array_equal(plain["counts"], got["counts"])          # counts stay the own lists


def test_large_plan_global_binning(dev):
    """A plan with more tiles than the per-CTA shared-memory counters hold (4096 x 3072, 3 layers:
    64 512 tiles > 49 152) bins with global counters (k_count<.., true>, k_gscan_*, k_emit<true>);
    forward + backward on sampled pixels against the oracle."""
    import dataclasses
    base = scenes.make_config("C2", n=300_000)
    cam = scenes._orbit_cam(0.6, W=4096, H=3072, fx=2453.0)
    sc = dataclasses.replace(base, cams=[cam], n_layers=3, forward_only=False)
    mask = _sample_mask(cam, sc.n_layers, seed=9)
    G = grads_for(sc, cam, seed=2, mask=mask)
    got = gpu_run(sc, dev, G=G, save=True)
    check_forward(sc, got, mask=mask)
    check_backward(sc, got, G, mask=mask)


def test_forced_global_binning_small_scenes(dev, monkeypatch):
    """The global-counter binning path on the small parity scenes (forced by the plan-time switch
    TRIPS_FORCE_GLOBAL_BINNING): bit-exact counts / kept lists, forward and backward in tolerance."""
    monkeypatch.setenv("TRIPS_FORCE_GLOBAL_BINNING", "1")
    for sc in (scenes.c1(), scenes.adversarial_scene(), scenes.tiny_scene(11, n=30000, F=4, W=40, H=24, n_layers=3)):
        G = grads_for(sc, sc.cams[0], seed=4)
        got = gpu_run(sc, dev, G=G, save=True)
        check_forward(sc, got)
        check_backward(sc, got, G)
