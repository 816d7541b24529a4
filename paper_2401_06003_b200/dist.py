"""View-parallel multi-GPU plumbing: the point cloud is replicated, every
rank renders a disjoint subset of a batch of camera views (forward + backward, gradients
accumulated into one packed buffer), and a single all-reduce (SUM, reading Q21) combines
the point gradients.  One process per GPU; NCCL over NVLink/NVSwitch on GPUs, gloo on CPU
(tests).  There is no per-view exchange: views are independent given the cloud.
"""
import torch
import torch.distributed as dist


def shard_views(n_views, rank, world):
    """Views of this rank: v = rank, rank + world, ... (every view exactly once overall)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n_views, world))


def batch_step(render_view, views, grad, world=1, group=None, zero=True):
    """One step of the batch: grad <- sum over `views` of render_view(v, grad) (which must
    ACCUMULATE into grad), then all-reduce(SUM) over the group.  Returns grad."""
    if zero:
        grad.zero_()
    for v in views:
        render_view(v, grad)
    if world > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


def cuda_view_renderer(rast, cams, pos, world_size, opacity, desc, grad_pyramid):
    """render_view for batch_step on the CUDA path: project -> forward (saved) -> backward."""
    def render_view(v, grad):
        rast.project(cams[v], pos, world_size, opacity, desc)
        rast.forward(save=True)
        rast.backward(grad_pyramid(v) if callable(grad_pyramid) else grad_pyramid, grad)
    return render_view


def cuda_batch_step(rasts, cams, pos, world_size, opacity, desc, grad_pyramid, views, grad, world=1, group=None,
                    zero=True, streams=None):
    """batch_step on the CUDA path with the views spread round-robin over len(rasts) CUDA
    streams, one Rasterizer (plan + workspace) per stream, so that one view's memory-streaming
    binning kernels overlap another view's latency-bound raster/backward kernels.  Gradients
    of all views accumulate into `grad` (vector reductions are atomic, so concurrent backward
    passes are safe); the streams join the current stream before the all-reduce."""
    main = torch.cuda.current_stream()
    if streams is None:
        streams = [main] + [torch.cuda.Stream(device=grad.device) for _ in range(len(rasts) - 1)]
    if zero:
        grad.zero_()
    start = torch.cuda.Event()
    start.record(main)
    for s in streams:
        if s != main:
            s.wait_event(start)
    for j, v in enumerate(views):
        k = j % len(rasts)
        with torch.cuda.stream(streams[k]):
            r = rasts[k]
            r.project(cams[v], pos, world_size, opacity, desc)
            r.forward(save=True)
            r.backward(grad_pyramid(v) if callable(grad_pyramid) else grad_pyramid, grad)
    for s in streams:
        if s != main:
            e = torch.cuda.Event()
            e.record(s)
            main.wait_event(e)
    if world > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


def init_from_env(backend=None):
    """torch.distributed init from torchrun's env (RANK, WORLD_SIZE, LOCAL_RANK, MASTER_*).
    Returns (rank, world, local_rank); world == 1 without a launcher."""
    import os
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local
