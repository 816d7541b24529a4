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


class StreamedSteps:
    """End-to-end step pipeline from pinned host memory: every step copies its inputs host ->
    device, runs `step_fn(device_inputs, grad)` and copies the gradient buffer device -> host.
    Inputs and gradients are double-buffered and the copies run on their own streams, so step
    k+1's upload and step k-1's download overlap step k's kernels (the copy engines are
    separate from the SMs); event edges keep every buffer reuse ordered.

        pipe = StreamedSteps(host_inputs, grad_like, device)
        pipe.run(steps, step_fn, host_out)        # host_out[k % 2] holds step k's gradients
    """

    def __init__(self, host_inputs, grad_like, device):
        self.host = host_inputs
        self.dev_in = [{k: torch.empty_like(v, device=device) for k, v in host_inputs.items()} for _ in range(2)]
        self.grads = [grad_like, torch.empty_like(grad_like)]
        self.up = torch.cuda.Stream(device=device)
        self.down = torch.cuda.Stream(device=device)

    def run(self, steps, step_fn, host_out):
        main = torch.cuda.current_stream()
        done = [None, None]      # compute of the step that last used buffer b finished
        out = [None, None]       # download of gradient buffer b finished
        for k in range(steps):
            b = k % 2
            with torch.cuda.stream(self.up):
                if done[b] is not None:
                    self.up.wait_event(done[b])
                for key, v in self.host.items():
                    self.dev_in[b][key].copy_(v, non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(self.up)
            main.wait_event(ready)
            if out[b] is not None:
                main.wait_event(out[b])
            step_fn(self.dev_in[b], self.grads[b])
            done[b] = torch.cuda.Event()
            done[b].record(main)
            with torch.cuda.stream(self.down):
                self.down.wait_event(done[b])
                host_out[b].copy_(self.grads[b], non_blocking=True)
                out[b] = torch.cuda.Event()
                out[b].record(self.down)
        for e in out:
            if e is not None:
                main.wait_event(e)


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
