#!/usr/bin/env python
"""Benchmark of the B200 TRIPS rasterizer (BASELINE.json metric: forward+backward frames/s
and splatted points/s at 1080p, HBM GB/s vs peak, 1/2/4/8-GPU scaling).

Workload (BASELINE.json configs[3], "C4"): a batch of 32 camera views of an 8M-point
Tanks&Temples-like synthetic cloud at 1920x1080, 4 pyramid layers, F = 4.  One step =
for every view of this rank: project -> splat forward (saved) -> splat backward into
one flat gradient buffer; then one NCCL reduction (SUM) of that buffer across ranks,
issued asynchronously so that step k's reduction overlaps step k+1's views (double-
buffered gradients).  Views are sharded r::N over ranks (strong scaling: the batch is fixed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Rank 0 prints ONE JSON line.  Besides the contract keys it carries a per-kernel table
(`kernels`), the dominant kernel's `roofline` (chosen by serialised time) with its gradient
reductions against the measured reduction ceiling (`roofline.atomics`), the other configs
C2/C3/C5 (`configs`) and the CPU oracle timed on all host cores (`cpu_baseline`).
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same workload
(the one other place bench.py may execute oracle/).
"""
import argparse
import concurrent.futures as cf
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd frames/s and splatted points/s at 1080p; HBM GB/s vs peak; 1/2/4/8 GPU scaling"
UNIT = "frames/s"
N_POINTS = 8_000_000
N_VIEWS = 32
STRIP = 32                     # oracle sample: horizontal strips of 32 pixel rows
# timing stages of libtrips (trips_read_stage_ms) and the kernel each one brackets
KERNEL_OF = {"count": "k_count", "tscan": "k_tscan", "emit": "k_emit", "raster": "k_raster",
             "backward": "k_backward_pairs"}
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "dram_traffic_r02.json")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_peaks():
    """MEASURED_PEAKS.json as a dict (empty when absent)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "model": model, "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS")}


def dram_traffic():
    try:
        with open(TRAFFIC_FILE) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.first = 0

    def _rows(self):
        with open(self.f.name) as g:
            return [r for r in g.read().splitlines() if r.strip()]

    def live(self):
        """nvidia-smi has produced its first sample (it takes a few hundred ms to start)."""
        return self.p is not None and len(self._rows()) > 0

    def mark(self):
        """Samples from here on belong to the timed region."""
        self.first = len(self._rows()) if self.p is not None else 0

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        allrows = self._rows()
        os.unlink(self.f.name)
        timed = allrows[self.first:]
        # the timed region can be shorter than the sampling period: then the samples of the
        # warm-up steps just before it (same kernels, same load) stand in, and say so
        rows = [r.split(",") for r in (timed if timed else allrows[-3:])]
        self.in_timed = bool(timed)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for k, nm in enumerate(names):
                    if r[4 + k].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "window": "timed region" if self.in_timed else "warm-up steps just before it"}


# ------------------------------------------------------------------ algorithmic bytes

def alg_bytes(st, n, F, P, backward=True):
    """Algorithmic bytes per view (SURVEY.md 8(d) per-unit figures, DESIGN.md "Algorithmic
    bytes"), attributed to the kernel whose stage consumes / produces them:
      forward : 16 N (pos, s_w) | (4+4F) N_vis (alpha, tau) | 16 N_frag ((z, i) lists written
                and read) | 8 P (counts, offsets) | 4 (F+1) P (pyramid) | 4 N_kept (saved list)
      backward: 4 (F+1) P (grad pyramid) | 4 N_kept + 4 P (saved list, offsets) |
                (20+4F) N_vis (record, alpha, tau) | 2 * 4 (5+F) N_vis (gradient accumulation) |
                4 (5+F) N (world gradients)
    st: trips stats of the view (n_visible, n_frag, n_kept)."""
    nv, nf, nk = st["n_visible"], st["n_frag"], st["n_kept"]
    k = {"count": 16 * n, "tscan": 0, "emit": 8 * nf,
         "raster": (4 + 4 * F) * nv + 8 * nf + 8 * P + 4 * (F + 1) * P + (4 * nk if backward else 0)}
    k["backward"] = (4 * (F + 1) * P + 4 * nk + 4 * P + (20 + 4 * F) * nv + 8 * (5 + F) * nv
                     + 4 * (5 + F) * n) if backward else 0
    return k


# ------------------------------------------------------------------ CPU oracle sample

def oracle_strip_tasks(sc, cams, n_tasks, seed=100, phase=0):
    """Inputs of n_tasks oracle runs, each the forward+backward of one STRIP-row strip of a view
    (a crop camera with the same intrinsics, cy shifted by a multiple of 2^(n-1) so that every
    layer's pixel grid is the full image's) over the points that can reach it (a generous numpy
    pre-filter: sample selection only, not timed).  One view per call (cams[phase]); the strips
    walk its image bands."""
    from oracle import oracle
    from synth import scenes
    tasks = []
    cam = cams[phase % len(cams)]
    H = cam.height
    align = 1 << (sc.n_layers - 1)
    bands = H // STRIP
    p = sc.pos.astype(np.float64) @ cam.R.astype(np.float64).T + cam.t.astype(np.float64)
    with np.errstate(all="ignore"):
        u = cam.fx * p[:, 0] / p[:, 2] + cam.cx
        v = cam.fy * p[:, 1] / p[:, 2] + cam.cy
        margin = 64 + 2 * cam.f * sc.sw / p[:, 2]
        ok = (p[:, 2] > cam.near) & (u > -margin) & (u < cam.width + margin)
    del p, u
    for t in range(n_tasks):
        y0 = ((phase * 7 + t * 13) % bands) * STRIP // align * align
        crop = scenes.Camera(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy - y0, f=cam.f, R=cam.R, t=cam.t,
                             width=cam.width, height=STRIP, near=cam.near)
        with np.errstate(all="ignore"):
            keep = ok & (v - y0 > -margin) & (v - y0 < STRIP + margin)
        idx = np.nonzero(keep)[0]
        P = oracle.num_pixels(crop.width, crop.height, sc.n_layers)
        tasks.append((crop, sc.n_layers, sc.pos[idx], sc.sw[idx], sc.alpha[idx], sc.desc[idx],
                      scenes.grad_pyramid(P * (sc.F + 1), seed=seed + t)))
    return tasks


def _oracle_task(task):
    from oracle import oracle
    crop, nl, pos, sw, al, de, G = task
    oracle.forward(crop, nl, pos, sw, al, de, want_kept=False)
    oracle.backward(crop, nl, pos, sw, al, de, G)


def oracle_frames_per_s(tasks, threads, H):
    """The oracle as it stands, on `threads` host threads (one task each at a time; the ctypes
    calls release the GIL): frames/s = (strip rows processed / H) / wall seconds."""
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(_oracle_task, tasks))
    wall = time.perf_counter() - t0
    return len(tasks) * STRIP / H / wall, wall


def cpu_threads():
    return max(1, int(os.environ.get("OMP_NUM_THREADS") or os.cpu_count() or 1))


def run_reference(args, rank, world):
    from synth import scenes
    if rank != 0:
        return
    # lib-morton: the same Morton layout, computed by the generator (the oracle has no GPU)
    sc = scenes.make_config("C4", n=N_POINTS, n_views=N_VIEWS,
                            order="morton" if args.order == "lib-morton" else args.order)
    H = sc.cams[0].height
    thr = cpu_threads()
    per_step = 2 * thr
    for w in range(args.warmup):
        oracle_frames_per_s(oracle_strip_tasks(sc, sc.cams, thr, phase=1000 + w), thr, H)
    vals, walls = [], []
    for k in range(args.steps):
        v, wall = oracle_frames_per_s(oracle_strip_tasks(sc, sc.cams, per_step, phase=k * per_step), thr, H)
        vals.append(v)
        walls.append(wall)
    value = len(vals) / sum(1.0 / v for v in vals)
    sample = (f"per step: {per_step} strips of {STRIP} pixel rows of C4 views (8M points, 1920x1080, n=4, F=4; "
              f"crop cameras over the points that can reach them), oracle forward+backward, {thr} host threads; "
              f"frames/s = rows processed / 1080 / wall seconds")
    info = host_info()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": "C4: 32 views x 8M points, 1920x1080, 4 layers, F=4",
                                             "point_order": args.order},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle", "sample": sample,
                             "host": info},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ CUDA arm

def stage_ms_per_view(torch, r, cam, inputs, views_n, backward=True, gp=None, gbuf=None):
    """Single-stream per-stage device ms per view (libtrips' CUDA events on the launching stream),
    after 2 warm-up views; also the view's stats."""
    def one():
        r.project(cam, *inputs)
        r.forward(save=backward)
        if backward:
            r.backward(gp, gbuf)
    for _ in range(2):
        one()
    torch.cuda.synchronize()
    r.stage_ms(reset=True)
    r.set_profiling(True)
    for _ in range(views_n):
        one()
    torch.cuda.synchronize()
    st = r.stage_ms(reset=True)
    r.set_profiling(False)
    return {k: st[k][0] / views_n for k in KERNEL_OF}, r.stats()


def kernel_table(ms_alone, ms_step, bytes_, traffic, peak):
    """Per-kernel algorithmic bytes, ncu DRAM bytes, times and roofline fractions (per launch)."""
    out = {}
    for k, kern in KERNEL_OF.items():
        t = ms_alone.get(k)
        if not t:
            continue
        row = {"kernel": kern, "alg_bytes": bytes_[k], "ms_alone": t,
               "alg_GBps_alone": bytes_[k] / (t * 1e-3) / 1e9, "alg_frac_alone": bytes_[k] / (t * 1e-3) / 1e9 / peak}
        if ms_step and ms_step.get(k):
            row["ms_in_step"] = ms_step[k]
            row["alg_frac_in_step"] = bytes_[k] / (ms_step[k] * 1e-3) / 1e9 / peak
        d = (traffic or {}).get(kern)
        if d:
            row["dram_bytes"] = d
            row["dram_GBps_alone"] = d / (t * 1e-3) / 1e9
            row["dram_frac_alone"] = d / (t * 1e-3) / 1e9 / peak
        out[k] = row
    return out


def run_configs(torch, dev, peak, traffic, views_n=8):
    """C2 (forward only), C3, C5 (forward + backward) at full size, one stream, library Morton
    layout: per-view stage times, frames/s, points/s, algorithmic and DRAM fractions."""
    from paper_2401_06003_b200 import Rasterizer, morton_order
    from synth import scenes
    out = {}
    for name in ("C2", "C3", "C5"):
        sc = scenes.make_config(name)
        cam = sc.cams[0]
        d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sc.pos, sc.sw, sc.alpha, sc.desc)]
        perm = morton_order(d[0])
        d = [a[perm].contiguous() for a in d]
        r = Rasterizer(cam.width, cam.height, sc.n_layers, sc.F, max_points=sc.n, device=dev)
        bwd = not sc.forward_only
        gp = torch.from_numpy(scenes.grad_pyramid(r.pyramid_floats, seed=100)).to(dev) if bwd else None
        gb = r.new_grad(sc.n) if bwd else None
        ms, st = stage_ms_per_view(torch, r, cam, d, views_n, backward=bwd, gp=gp, gbuf=gb)
        ms_view = sum(ms.values())
        by = alg_bytes(st, sc.n, sc.F, r.P, backward=bwd)
        tot = sum(by.values())
        row = {"workload": f"{name}: {sc.n / 1e6:g}M points, {cam.width}x{cam.height}, {sc.n_layers} layers, F={sc.F}, "
                           + ("fwd+bwd" if bwd else "forward only"),
               "ms_per_view": ms_view, "frames_per_s": 1e3 / ms_view, "points_per_s": sc.n * 1e3 / ms_view,
               "stage_ms": ms, "alg_bytes_per_view": tot, "alg_frac": tot / (ms_view * 1e-3) / 1e9 / peak,
               "kernels": kernel_table(ms, None, by, (traffic or {}).get(name), peak), "view_stats": st,
               "timing": f"CUDA events per stage, one stream, mean of {views_n} views after 2 warm-up"}
        dr = sum(v.get("dram_bytes", 0) for v in row["kernels"].values())
        if dr:
            row["dram_GBps"] = dr / (ms_view * 1e-3) / 1e9
            row["dram_frac"] = row["dram_GBps"] / peak
        out[name] = row
        del r, d, gp, gb
        torch.cuda.empty_cache()
    return out


def microbench(torch, dev):
    """Measured ceilings of 16-byte reductions (trips_microbench; tools/microbench.py has more)."""
    from paper_2401_06003_b200 import _abi as A
    buf = torch.zeros((2 << 30) // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    for name, op in (("red_v4_f32", 0), ("red_f32", 1), ("atomic_add_u32", 2)):
        for sname, nbytes in (("l2_32MB", 32 << 20), ("dram_2GB", 2 << 30)):
            for pat, pname in ((0, "random"), (1, "coherent")):
                A.trips_microbench(op, pat, buf.data_ptr(), nbytes, 16, 1 << 25, st)
                best = min(A.trips_microbench(op, pat, buf.data_ptr(), nbytes, 16, 1 << 28, st)[0] for _ in range(2))
                res[f"{name}|{sname}|{pname}"] = (1 << 28) / (best * 1e-3) / 1e9
    del buf
    torch.cuda.empty_cache()
    return res


def run_cuda(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2401_06003_b200 import Rasterizer, _abi
    from paper_2401_06003_b200 import dist as tdist
    from synth import scenes

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    sc = scenes.make_config("C4", n=N_POINTS, n_views=N_VIEWS,
                            order="random" if args.order == "lib-morton" else args.order)
    n, F = sc.n, sc.F
    W, H = sc.cams[0].width, sc.cams[0].height
    # views of a step are spread over args.streams CUDA streams, one plan + workspace each
    rasts = [Rasterizer(W, H, sc.n_layers, F, max_points=n, device=dev) for _ in range(args.streams)]
    rast = rasts[0]
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream(device=dev) for _ in range(args.streams - 1)]
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
         for k, v in (("pos", sc.pos), ("sw", sc.sw), ("alpha", sc.alpha), ("desc", sc.desc))}
    Gp = torch.from_numpy(scenes.grad_pyramid(rast.pyramid_floats, seed=100)).to(dev)
    # flat gradient buffers, padded so that they split into `world` equal shards
    gnum = tdist.padded_numel(rast.grad_floats(n), world)
    grads = [torch.zeros(gnum, dtype=torch.float32, device=dev) for _ in range(2)]
    shards = [torch.empty(gnum // world, dtype=torch.float32, device=dev) for _ in range(2)] \
        if args.reduce == "reduce_scatter" and world > 1 else [None, None]
    my_views = tdist.shard_views(N_VIEWS, rank, world)
    stream = torch.cuda.current_stream()

    def step(dv, g, out=None):
        return tdist.cuda_batch_step(rasts, sc.cams, dv["pos"], dv["sw"], dv["alpha"], dv["desc"], Gp, my_views, g,
                                     world=world, streams=streams, reduce=args.reduce, out=out, async_op=world > 1)

    def timed_ms(dv, steps):
        """device ms per step (CUDA events on the launching stream), max over ranks"""
        pipe = tdist.PipelinedSteps(grads)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        pipe.run(steps, lambda g, k: step(dv, g, shards[k % 2]))
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    random_order = None
    if args.order == "lib-morton":
        if not args.no_random_order:
            # side measurement: the same workload in the generator's (random) point order
            for _ in range(2):
                step(d, grads[0])
            ms_r = timed_ms(d, 3)
            random_order = {"value": N_VIEWS / (ms_r * 1e-3), "ms_per_step": ms_r, "steps": 3, "warmup": 2}
        # one-time data layout at load: the library's Morton permutation applied to every
        # per-point array (the cloud then lives in this order for the whole run)
        from paper_2401_06003_b200 import morton_order
        perm = morton_order(d["pos"])
        d = {k: v[perm].contiguous() for k, v in d.items()}

    # per-view statistics (deterministic; read outside the timed region)
    view_stats = []
    for v in my_views:
        rast.project(sc.cams[v], d["pos"], d["sw"], d["alpha"], d["desc"])
        rast.forward(save=True)
        view_stats.append(rast.stats())
    torch.cuda.synchronize()

    # nvidia-smi clock sampling starts with the warm-up; extra warm-up steps run until it reports,
    # so that it samples the timed region itself
    clocks = ClockSampler(local_rank)
    t_w = time.time()
    for _ in range(args.warmup):
        step(d, grads[0])
    torch.cuda.synchronize()
    while not clocks.live() and time.time() - t_w < 5.0:
        step(d, grads[0])
        torch.cuda.synchronize()

    # ---- device-timed region: inputs resident in HBM
    for r_ in rasts:
        r_.stage_ms(reset=True)
        r_.set_profiling(True)
    l0 = _abi.trips_launch_count()
    clocks.mark()
    ms_max = timed_ms(d, args.steps) * args.steps
    clk = clocks.stop()
    launches = _abi.trips_launch_count() - l0
    stage = {}
    for r_ in rasts:
        r_.set_profiling(False)
        for k_, (ms_, la_) in r_.stage_ms(reset=True).items():
            a_ = stage.get(k_, (0.0, 0))
            stage[k_] = (a_[0] + ms_, a_[1] + la_)

    # ---- every kernel alone (one stream): serialised per-launch times, the dominant kernel
    inputs = (d["pos"], d["sw"], d["alpha"], d["desc"])
    gb = rast.new_grad(n)
    alone, _ = stage_ms_per_view(torch, rast, sc.cams[my_views[0]], inputs, 8, True, Gp, gb)

    # ---- side measurement: backward with the camera gradient
    gcam = torch.zeros(17, dtype=torch.float32, device=dev)
    cam_ms = {}
    for with_cam in (False, True):
        rast.stage_ms(reset=True)
        rast.set_profiling(True)
        for v in my_views[:8]:
            rast.project(sc.cams[v], *inputs)
            rast.forward(save=True)
            rast.backward(Gp, gb, grad_camera=gcam if with_cam else None)
        torch.cuda.synchronize()
        st_ = rast.stage_ms(reset=True)
        rast.set_profiling(False)
        cam_ms["with_camera_grad" if with_cam else "without"] = st_["backward"][0] / max(st_["backward"][1], 1)

    # ---- side measurement: blend variants and feature counts, per view
    def per_view_ms(r, desc, views):
        gp = torch.from_numpy(scenes.grad_pyramid(r.pyramid_floats, seed=100)).to(dev)
        g = r.new_grad(n)
        for v in views[:2]:                                          # warm-up
            r.project(sc.cams[v], d["pos"], d["sw"], d["alpha"], desc)
            r.forward(save=True)
            r.backward(gp, g)
        torch.cuda.synchronize()
        r.stage_ms(reset=True)
        r.set_profiling(True)
        for v in views:
            r.project(sc.cams[v], d["pos"], d["sw"], d["alpha"], desc)
            r.forward(save=True)
            r.backward(gp, g)
        torch.cuda.synchronize()
        st_ = r.stage_ms(reset=True)
        r.set_profiling(False)
        out = {k: st_[k][0] / len(views) for k in KERNEL_OF}
        out["total"] = sum(out.values())
        return out

    variants = {}
    side_views = my_views[:8]
    variants["plain"] = per_view_ms(rast, d["desc"], side_views)
    for name, kw in (("t_min_0.01", {"t_min": 0.01}), ("coarse_all_layers", {"coarse_layers": sc.n_layers - 1})):
        rv = Rasterizer(W, H, sc.n_layers, F, max_points=n, device=dev, **kw)
        variants[name] = per_view_ms(rv, d["desc"], side_views)
        del rv
    for Fv in (6, 8):
        gen = torch.Generator(device=dev).manual_seed(Fv)
        dv8 = (torch.randn(n, Fv, generator=gen, device=dev) * 0.5).contiguous()
        rv = Rasterizer(W, H, sc.n_layers, Fv, max_points=n, device=dev)
        variants[f"F{Fv}"] = per_view_ms(rv, dv8, side_views)
        del rv, dv8
    torch.cuda.empty_cache()

    # ---- side measurement: 4-NN point-size initialisation of the cloud
    from paper_2401_06003_b200 import knn_sizes
    knn_sizes(d["pos"])
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(3):
        knn_sizes(d["pos"])
    k1.record(stream)
    torch.cuda.synchronize()
    knn_ms = k0.elapsed_time(k1) / 3

    # ---- side measurement: the gated-conv decoder on this bench's pyramid
    # geometry (1080p, 4 layers, F = 4 -> 3 channels), tcgen05 implicit-GEMM convolutions
    from paper_2401_06003_b200 import Decoder
    dec = Decoder(rast, 3)
    gen = torch.Generator(device=dev).manual_seed(3)
    dec_prm = (torch.randn(dec.param_count, generator=gen, device=dev) * 0.1).contiguous()
    dec_pyr = (torch.randn(rast.pyramid_floats, generator=gen, device=dev) * 0.5).contiguous()
    dec_out = dec(dec_prm, dec_pyr)
    torch.cuda.synchronize()
    k0.record(stream)
    for _ in range(10):
        dec(dec_prm, dec_pyr, dec_out)
    k1.record(stream)
    torch.cuda.synchronize()
    dec_ms = k0.elapsed_time(k1) / 10
    dec_flops = 2.0 * H * W * 32 * 3                     # output projection
    for l in range(sc.n_layers):
        hl, wl, _ = _abi.trips_layer_dims(rast.plan, l)
        C = F + 1 if l == sc.n_layers - 1 else 32 + F + 1
        dec_flops += 2.0 * hl * wl * (2 * 32 * C * 9 + 32 * C)   # Wf, Wg (3x3) and Wb (1x1)
    tc_peak = measured_peaks().get("bf16_tflops")
    decoder = {"workload": f"{W}x{H}, {sc.n_layers} layers, F={F} -> 3 channels (fp16 operands, fp32 accumulate)",
               "ms_per_frame": dec_ms, "frames_per_s": 1e3 / dec_ms,
               "alg_tflops": dec_flops / (dec_ms * 1e-3) / 1e12, "alg_flops_per_frame": dec_flops,
               "bound": "tensor", "peak_tflops": tc_peak,
               "peak_source": "MEASURED_PEAKS.json bf16_tflops (fp16 runs at the bf16 rate)" if tc_peak else None}
    if tc_peak:
        decoder["frac"] = decoder["alg_tflops"] / tc_peak
    del dec, dec_prm, dec_pyr, dec_out
    torch.cuda.empty_cache()

    # ---- end to end through the public API: pinned host inputs in, gradients out.  Each rank
    # uploads its 1/N slice of the flat input buffer (+ NCCL all-gather) and downloads its 1/N
    # shard of the reduce-scattered gradients (dist.ShardedStreamedSteps; at N = 1 the whole
    # buffers, double-buffered, copies on their own streams overlapping the kernels)
    flat_in, _, _ = tdist.flat_inputs(d["pos"], d["sw"], d["alpha"], d["desc"], world)
    host_flat = flat_in.cpu().pin_memory()
    del flat_in
    pipe = tdist.ShardedStreamedSteps(host_flat, gnum, dev, world, rank)
    out_host = [torch.empty(pipe.ghi - pipe.glo, dtype=torch.float32).pin_memory() for _ in range(2)]

    def e2e_step(dev_flat, g, out):
        pos, sw, al, de = tdist.input_views(dev_flat, n, F)
        tdist.cuda_batch_step(rasts, sc.cams, pos, sw, al, de, Gp, my_views, g, world=world, streams=streams,
                              reduce="reduce_scatter", out=out)

    pipe.run(2, e2e_step, out_host)                                  # warm the pipeline buffers
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    pipe.run(args.steps, e2e_step, out_host)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    del pipe
    torch.cuda.empty_cache()

    # ---- measured reduction ceilings, the other configs
    mb = microbench(torch, dev) if rank == 0 else {}
    peak, peak_src = peaks()
    traffic = dram_traffic()
    configs = run_configs(torch, dev, peak, traffic) if (rank == 0 and not args.no_configs) else None

    if rank != 0:
        return
    # ---- roofline: dominant kernel by serialised time
    per_view_bytes = [alg_bytes(s, n, F, rast.P) for s in view_stats]
    mean_bytes = {k: sum(b[k] for b in per_view_bytes) / len(per_view_bytes) for k in KERNEL_OF}
    step_ms = ms_max / args.steps
    in_step = {k: stage[k][0] / max(stage[k][1], 1) for k in KERNEL_OF if k in stage}
    kernels = kernel_table(alone, in_step, mean_bytes, traffic.get("C4"), peak)
    dom = max(("count", "emit", "raster", "backward"), key=lambda k: alone[k])
    kd = kernels[dom]
    step_bytes = sum(sum(b.values()) for b in per_view_bytes)
    value = N_VIEWS / (step_ms * 1e-3)
    kp = float(np.mean([s["n_kept_pairs"] for s in view_stats]))
    reds = 3 * kp                          # per kept pair: pos_size v4 + desc v4 + opacity f32
    red_peak = max(v for k, v in mb.items() if k.startswith("red_v4_f32")) if mb else None
    atomics = {"kernel": "k_backward_pairs", "reductions_per_launch": reds,
               "per": "3 per kept (point, tile) pair: red.global.add.v4.f32 (pos, s_w), .v4.f32 (tau), .f32 (alpha)",
               "achieved_G_per_s_alone": reds / (alone["backward"] * 1e-3) / 1e9}
    if red_peak:
        atomics.update({"peak_G_per_s": red_peak, "frac_alone": atomics["achieved_G_per_s_alone"] / red_peak,
                        "peak_source": "trips_microbench: best red.global.add.v4.f32 rate over L2-resident / "
                                       "DRAM-sized x random / warp-coherent addresses", "microbench": mb})
    roof = {"bound": "hbm", "kernel": KERNEL_OF[dom], "achieved": kd["alg_bytes"] / (in_step[dom] * 1e-3) / 1e9,
            "peak": peak, "unit": "GB/s", "peak_source": peak_src,
            "traffic": kd.get("dram_bytes"), "alg_bytes_per_launch": kd["alg_bytes"], "launch_ms": in_step[dom],
            "dominant_by": "serialised (single-stream) per-launch time; achieved uses the launch time inside "
                           f"the timed step ({args.streams} concurrent streams)",
            "alone": {"launch_ms": alone[dom], "achieved": kd["alg_GBps_alone"], "frac": kd["alg_frac_alone"],
                      "dram_frac": kd.get("dram_frac_alone")},
            "atomics": atomics}
    roof["frac"] = roof["achieved"] / peak
    ctraffic = traffic.get("C4") or {}
    dram_view = sum(ctraffic.get(KERNEL_OF[k], 0) for k in KERNEL_OF) if ctraffic else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C4: batch of 32 views x 8M points (T&T-like), 1920x1080, 4 layers, F=4, "
                               "fwd+bwd, view-parallel + NCCL reduction of point gradients",
                   "global_batch": N_VIEWS, "points": n, "resolution": [W, H], "layers": sc.n_layers,
                   "features": F, "parallelism": f"views{world}", "point_order": args.order,
                   "streams_per_gpu": args.streams, "reduction": args.reduce + (" (async, overlapped)" if world > 1
                                                                                else " (none at 1 GPU)"),
                   "l2": "inputs larger than L2 (288 MB of point data, 288 MB gradients per step)"},
        "points_per_s": N_VIEWS * n / (step_ms * 1e-3),
        "fragments_per_s": sum(s["n_frag"] for s in view_stats) * world / (step_ms * 1e-3),
        "alg_GBps_step": step_bytes * world / (step_ms * 1e-3) / 1e9,
        "alg_frac_step": step_bytes * world / (step_ms * 1e-3) / 1e9 / peak,
        "roofline": roof,
        "kernels": kernels,
        "stage_ms_per_step": {k: v[0] / args.steps for k, v in stage.items()},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "e2e": {"value": N_VIEWS / (e2e_ms / args.steps * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": host_flat.numel() * 4 // world,
                "d2h_bytes_per_step": out_host[0].numel() * 4,
                "note": "per rank: 1/N slice of the flat input buffer up (+ all-gather), 1/N shard of the "
                        "reduce-scattered gradients down, every step"},
        "view_stats_mean": {k: float(np.mean([s[k] for s in view_stats])) for k in view_stats[0]},
    }
    if dram_view:
        line["dram_frac_view_alone"] = dram_view / (sum(alone.values()) * 1e-3) / 1e9 / peak
    if clk is not None:
        line["clocks"] = clk
    if random_order is not None:
        line["random_point_order"] = random_order
    line["backward_ms_per_view"] = cam_ms
    line["variants_ms_per_view"] = variants
    line["knn4_size_init"] = {"ms": knn_ms, "points_per_s": n / (knn_ms * 1e-3)}
    line["decoder"] = decoder
    if configs:
        line["configs"] = configs
    if world == 1 and not args.no_cpu_baseline:
        thr = cpu_threads()
        tasks = oracle_strip_tasks(sc, sc.cams, 2 * thr, phase=3)
        v, wall = oracle_frames_per_s(tasks, thr, H)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle", "wall_s": wall,
                                "host": host_info(),
                                "sample": f"{2 * thr} strips of {STRIP} pixel rows of C4 views (8M points, crop "
                                          f"cameras over the points that can reach them), oracle forward+backward "
                                          f"on {thr} host threads; frames/s = rows / 1080 / wall s"}
        qs = np.random.default_rng(0).choice(n, 64, replace=False)
        from oracle import oracle as _o
        t0 = time.perf_counter()
        _o.knn4(sc.pos, queries=qs)
        line["knn4_size_init"]["cpu_baseline"] = {"points_per_s": len(qs) / (time.perf_counter() - t0), "cores": 1,
                                                  "kind": "oracle",
                                                  "sample": "64 query points, brute force over all 8M points"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--order", default="lib-morton", choices=["random", "morton", "lib-morton"],
                    help="point order: as generated (random), numpy Morton sort, or the library's "
                         "trips_morton_order applied once at load (outside the timed region)")
    ap.add_argument("--reduce", default="allreduce", choices=["allreduce", "reduce_scatter"],
                    help="cross-rank gradient reduction of the timed step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2/C3/C5 side measurements")
    ap.add_argument("--streams", type=int, default=2,
                    help="CUDA streams (one plan + workspace each) the views of a step are spread over")
    ap.add_argument("--no-random-order", action="store_true", help="skip the random-order side measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    from paper_2401_06003_b200 import dist as tdist
    rank, world, local_rank = tdist.init_from_env("nccl")
    run_cuda(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
