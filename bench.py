#!/usr/bin/env python
"""Benchmark of the B200 TRIPS rasterizer (BASELINE.json metric: forward+backward frames/s
and splatted points/s at 1080p, HBM GB/s vs peak, 1/2/4/8-GPU scaling).

Workload (BASELINE.json configs[3], "C4"): a batch of 32 camera views of an 8M-point
Tanks&Temples-like synthetic cloud at 1920x1080, 4 pyramid layers, F = 4.  One step =
for every view of this rank: project -> splat forward (saved) -> splat backward into
one packed gradient buffer; then one NCCL all-reduce (SUM) of that buffer across ranks.
Views are sharded r::N over ranks (strong scaling: the batch is fixed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (oracle/) on a
bounded sample of the same workload (the one other place bench.py may execute oracle/).
"""
import argparse
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
SAMPLE_ROWS = 4          # oracle sample: 4 strips of 32 rows (one per 1/4 band), time scaled x1080/128


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


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
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
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
                "samples": len(sm)}


# ------------------------------------------------------------------ algorithmic bytes

def alg_bytes(st, n, F, P):
    """Algorithmic bytes per view (SURVEY.md 8(d) per-unit figures), attributed to the kernel
    whose stage consumes / produces them:
      forward : 16 N (pos, s_w) | (4+4F) N_vis (alpha, tau) | 16 N_frag ((z, i) lists written
                and read) | 8 P (counts, offsets) | 4 (F+1) P (pyramid) | 4 N_kept (saved list)
      backward: 4 (F+1) P (grad pyramid) | 4 N_kept + 4 P (saved list, offsets) |
                (20+4F) N_vis (record, alpha, tau) | 2 * 4 (5+F) N_vis (gradient accumulation) |
                4 (5+F) N (world gradients)
    st: trips stats of the view (n_visible, n_frag, n_kept)."""
    nv, nf, nk = st["n_visible"], st["n_frag"], st["n_kept"]
    k = {}
    k["count"] = 16 * n
    k["emit"] = 8 * nf
    k["raster"] = (4 + 4 * F) * nv + 8 * nf + 8 * P + 4 * (F + 1) * P + 4 * nk
    k["backward"] = (4 * (F + 1) * P + 4 * nk + 4 * P + (20 + 4 * F) * nv + 8 * (5 + F) * nv
                     + 4 * (5 + F) * n)
    k["sort"] = 0
    return k


# ------------------------------------------------------------------ CPU oracle sample

def oracle_sample(sc, cam, rows=SAMPLE_ROWS, phase=0, seed=100, strip=32):
    """One view forward+backward of the oracle on `rows` horizontal strips of `strip` pixel rows,
    one strip per 1/`rows` band of the image, each a crop camera (same intrinsics, cy shifted by
    a multiple of 2^(n-1) so every layer's pixel grid is the full image's) over the points that
    can reach it (a generous numpy pre-filter; sample selection only).  Returns the oracle's
    seconds scaled by H / (rows * strip), the pixel fraction."""
    from oracle import oracle
    from synth import scenes
    H = cam.height
    band = H // rows
    align = 1 << (sc.n_layers - 1)
    p = sc.pos.astype(np.float64) @ cam.R.astype(np.float64).T + cam.t.astype(np.float64)
    total = 0.0
    for b in range(rows):
        y0 = (b * band + (phase * 37) % max(band - strip, 1)) // align * align
        crop = scenes.Camera(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy - y0, f=cam.f, R=cam.R, t=cam.t,
                             width=cam.width, height=strip, near=cam.near)
        with np.errstate(all="ignore"):
            u = cam.fx * p[:, 0] / p[:, 2] + cam.cx
            v = cam.fy * p[:, 1] / p[:, 2] + crop.cy
            margin = 64 + 2 * cam.f * sc.sw / p[:, 2]
            keep = (p[:, 2] > cam.near) & (u > -margin) & (u < cam.width + margin) & (v > -margin) & \
                (v < strip + margin)
        idx = np.nonzero(keep)[0]
        pos, sw, al, de = sc.pos[idx], sc.sw[idx], sc.alpha[idx], sc.desc[idx]
        P = oracle.num_pixels(crop.width, crop.height, sc.n_layers)
        G = scenes.grad_pyramid(P * (sc.F + 1), seed=seed + b)
        t0 = time.perf_counter()
        oracle.forward(crop, sc.n_layers, pos, sw, al, de, want_kept=False)
        oracle.backward(crop, sc.n_layers, pos, sw, al, de, G)
        total += time.perf_counter() - t0
    return total * H / (rows * strip)


def run_reference(args, rank, world):
    from synth import scenes
    if rank != 0:
        return
    # lib-morton: the same Morton layout, computed by the generator (the oracle has no GPU)
    sc = scenes.make_config("C4", n=N_POINTS, n_views=N_VIEWS,
                            order="morton" if args.order == "lib-morton" else args.order)
    for w in range(args.warmup):
        oracle_sample(sc, sc.cams[w % N_VIEWS], phase=w)
    times = [oracle_sample(sc, sc.cams[(args.warmup + k) % N_VIEWS], phase=k) for k in range(args.steps)]
    t_view = sum(times) / len(times)                  # seconds per full view (scaled)
    value = 1.0 / t_view
    sample = ("per step: 1 view of C4 (8M points, 1920x1080, n=4, F=4), oracle forward+backward on 4 strips "
              "of 32 pixel rows (one per 1/4 band; crop cameras over the points that can reach them), "
              "time x1080/128; single thread")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_view * 1e3 * N_VIEWS,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": "C4: 32 views x 8M points, 1920x1080, 4 layers, F=4",
                                             "point_order": args.order},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ CUDA arm

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
    rast = Rasterizer(W, H, sc.n_layers, F, max_points=n, device=dev)
    # views of the step are spread over args.streams CUDA streams, one plan + workspace each
    rasts = [rast] + [Rasterizer(W, H, sc.n_layers, F, max_points=n, device=dev) for _ in range(args.streams - 1)]
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream(device=dev) for _ in range(args.streams - 1)]
    host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
            for k, v in (("pos", sc.pos), ("sw", sc.sw), ("alpha", sc.alpha), ("desc", sc.desc))}
    d = {k: v.to(dev, non_blocking=True) for k, v in host.items()}
    Gp = torch.from_numpy(scenes.grad_pyramid(rast.pyramid_floats, seed=100)).to(dev)
    grad = rast.new_grad(n)
    my_views = tdist.shard_views(N_VIEWS, rank, world)
    stream = torch.cuda.current_stream()

    def step(dv, grad_buf):
        tdist.cuda_batch_step(rasts, sc.cams, dv["pos"], dv["sw"], dv["alpha"], dv["desc"], Gp, my_views, grad_buf,
                              world=world, streams=streams)

    def timed_ms(dv, steps):
        """device ms per step (CUDA events on the launching stream), max over ranks"""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            step(dv, grad)
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
                step(d, grad)
            ms_r = timed_ms(d, 3)
            random_order = {"value": N_VIEWS / (ms_r * 1e-3), "ms_per_step": ms_r, "steps": 3, "warmup": 2}
        # one-time data layout at load: the library's Morton permutation applied to every
        # per-point array (the cloud then lives in this order for the whole run)
        from paper_2401_06003_b200 import morton_order
        perm = morton_order(d["pos"])
        d = {k: v[perm].contiguous() for k, v in d.items()}
        host = {k: v.cpu().pin_memory() for k, v in d.items()}

    # per-view statistics (deterministic; read outside the timed region)
    view_stats = []
    for v in my_views:
        rast.project(sc.cams[v], d["pos"], d["sw"], d["alpha"], d["desc"])
        rast.forward(save=True)
        view_stats.append(rast.stats())
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(d, grad)
    torch.cuda.synchronize()

    # ---- device-timed region: inputs resident in HBM
    for r_ in rasts:
        r_.stage_ms(reset=True)
        r_.set_profiling(True)
    l0 = _abi.trips_launch_count()
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(d, grad)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = _abi.trips_launch_count() - l0
    stage = {}
    for r_ in rasts:
        r_.set_profiling(False)
        for k_, (ms_, la_) in r_.stage_ms(reset=True).items():
            a_ = stage.get(k_, (0.0, 0))
            stage[k_] = (a_[0] + ms_, a_[1] + la_)
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # ---- side measurement: backward with the camera gradient
    gcam = torch.zeros(17, dtype=torch.float32, device=dev)
    cam_ms = {}
    for with_cam in (False, True):
        rast.stage_ms(reset=True)
        rast.set_profiling(True)
        for v in my_views[:8]:
            rast.project(sc.cams[v], d["pos"], d["sw"], d["alpha"], d["desc"])
            rast.forward(save=True)
            rast.backward(Gp, grad, grad_camera=gcam if with_cam else None)
        torch.cuda.synchronize()
        st_ = rast.stage_ms(reset=True)
        rast.set_profiling(False)
        cam_ms["with_camera_grad" if with_cam else "without"] = st_["backward"][0] / max(st_["backward"][1], 1)

    # ---- side measurement: blend variants and feature counts, per view
    def per_view_ms(r, desc, views):
        gp = torch.from_numpy(scenes.grad_pyramid(r.pyramid_floats, seed=100)).to(dev)
        gb = r.new_grad(n)
        for v in views[:2]:                                          # warm-up
            r.project(sc.cams[v], d["pos"], d["sw"], d["alpha"], desc)
            r.forward(save=True)
            r.backward(gp, gb)
        torch.cuda.synchronize()
        r.stage_ms(reset=True)
        r.set_profiling(True)
        for v in views:
            r.project(sc.cams[v], d["pos"], d["sw"], d["alpha"], desc)
            r.forward(save=True)
            r.backward(gp, gb)
        torch.cuda.synchronize()
        st_ = r.stage_ms(reset=True)
        r.set_profiling(False)
        out = {k: st_[k][0] / len(views) for k in ("count", "emit", "raster", "backward")}
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

    # ---- end to end through the public API: pinned host inputs in, gradients out
    # (dist.StreamedSteps: double-buffered, copies on their own streams overlap the kernels)
    out_host = [torch.empty(rast.grad_floats(n), dtype=torch.float32).pin_memory() for _ in range(2)]
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = out_host[0].numel() * out_host[0].element_size()
    pipe = tdist.StreamedSteps(host, grad, dev)
    pipe.run(2, step, out_host)                                      # warm the pipeline buffers
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    pipe.run(args.steps, step, out_host)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # ---- roofline of the dominant kernel (stage events are on the launching stream)
    peak, peak_src = peaks()
    per_view_bytes = [alg_bytes(s, n, F, rast.P) for s in view_stats]
    stage_ms = {k: v[0] for k, v in stage.items()}
    stage_launch = {k: v[1] for k, v in stage.items()}
    dom = max(("raster", "backward"), key=lambda k: stage_ms[k])     # single-kernel stages
    dom_launch_ms = stage_ms[dom] / max(stage_launch[dom], 1)
    dom_bytes = sum(b[dom] for b in per_view_bytes) / len(per_view_bytes)
    achieved = dom_bytes / (dom_launch_ms * 1e-3) / 1e9
    step_bytes = sum(sum(b.values()) for b in per_view_bytes)
    step_ms = ms_max / args.steps

    traffic = None
    tf = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(dom)
        except Exception:
            traffic = None

    if rank == 0:
        value = N_VIEWS / (step_ms * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C4: batch of 32 views x 8M points (T&T-like), 1920x1080, 4 layers, F=4, "
                                   "fwd+bwd, view-parallel + NCCL all-reduce of point gradients",
                       "global_batch": N_VIEWS, "points": n, "resolution": [W, H], "layers": sc.n_layers,
                       "features": F, "parallelism": f"views{world}", "point_order": args.order,
                       "streams_per_gpu": args.streams,
                       "l2": "inputs larger than L2 (288 MB of point data, 288 MB gradients per step)"},
            "points_per_s": N_VIEWS * n / (step_ms * 1e-3),
            "fragments_per_s": sum(s["n_frag"] for s in view_stats) * world / (step_ms * 1e-3),
            "alg_GBps_step": step_bytes * world / (step_ms * 1e-3) / 1e9,
            "alg_frac_step": step_bytes * world / (step_ms * 1e-3) / 1e9 / peak,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": dom_bytes, "launch_ms": dom_launch_ms,
                         "note": f"launch_ms measured inside the timed step, {args.streams} concurrent streams"},
            "stage_ms_per_step": {k: v / args.steps for k, v in stage_ms.items()},
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / args.steps,
            "e2e": {"value": N_VIEWS / (e2e_ms / args.steps * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "view_stats_mean": {k: float(np.mean([s[k] for s in view_stats])) for k in view_stats[0]},
        }
        alone_ms = (variants.get("plain") or {}).get(dom)
        if alone_ms:
            # the same kernel timed alone on one stream (side measurement, CUDA events on its
            # stream): its own roofline fraction without the other stream's kernels sharing the SMs
            line["roofline"]["alone"] = {"launch_ms": alone_ms, "achieved": dom_bytes / (alone_ms * 1e-3) / 1e9,
                                         "frac": dom_bytes / (alone_ms * 1e-3) / 1e9 / peak}
        if clk is not None:
            line["clocks"] = clk
        if random_order is not None:
            line["random_point_order"] = random_order
        line["backward_ms_per_view"] = cam_ms
        line["variants_ms_per_view"] = variants
        knn = {"ms": knn_ms, "points_per_s": n / (knn_ms * 1e-3)}
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as _o
            qs = np.random.default_rng(0).choice(n, 64, replace=False)
            t0 = time.perf_counter()
            _o.knn4(sc.pos, queries=qs)
            dt = time.perf_counter() - t0
            knn["cpu_baseline"] = {"points_per_s": len(qs) / dt, "cores": 1, "kind": "oracle",
                                   "sample": "64 query points, brute force over all 8M points"}
        line["knn4_size_init"] = knn
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as _o  # noqa: F401  (cpu_baseline leg only)
            t = [oracle_sample(sc, sc.cams[k], phase=k + 3) for k in range(2)]
            v = 1.0 / (sum(t) / len(t))
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                                    "sample": "2 views of C4 (8M points), oracle fwd+bwd on 4 strips of 32 pixel "
                                              "rows each (one per 1/4 band, crop cameras), time x1080/128; "
                                              "single thread"}
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
