"""View-parallel multi-GPU plumbing: the point cloud is replicated, every
rank renders a disjoint subset of a batch of camera views (forward + backward, gradients
accumulated into one flat buffer), and a single reduction (SUM, reading Q21) combines the
point gradients.  One process per GPU; NCCL over NVLink/NVSwitch on GPUs, gloo on CPU
(tests).  There is no per-view exchange: views are independent given the cloud.

The same `batch_step` drives the CPU tests (an oracle-backed renderer, gloo) and the GPU bench
(CudaViewRenderer, NCCL); only the renderer differs.

Reduction modes of `batch_step`:
  "allreduce"       every rank ends with the full gradient sum (one all-reduce)
  "reduce_scatter"  rank r ends with shard r of the sum (half the bytes of an all-reduce; the
                    natural choice when an optimizer owns point shards)
Both can be issued asynchronously (async_op=True): NCCL runs on its own stream, so step k's
reduction overlaps step k+1's rendering when the caller double-buffers the gradients
(`PipelinedSteps`).
"""
import torch
import torch.distributed as dist


def shard_views(n_views, rank, world):
    """Views of this rank: v = rank, rank + world, ... (every view exactly once overall)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n_views, world))


def shard_range(numel, rank, world):
    """[lo, hi) of rank's equal shard of a buffer whose size is a multiple of world."""
    if numel % world:
        raise ValueError(f"buffer of {numel} elements does not split into {world} equal shards")
    s = numel // world
    return rank * s, (rank + 1) * s


def padded_numel(numel, world, align=4):
    """Smallest size >= numel that splits into `world` shards of a multiple of `align` elements."""
    q = world * align
    return (numel + q - 1) // q * q


def reduce_grads(grad, world=1, group=None, reduce="allreduce", out=None, async_op=False):
    """Cross-rank SUM of the flat gradient buffer.  reduce_scatter writes rank r's shard into
    `out` (grad.numel() // world elements).  Returns the work handle (async_op) or None."""
    if world <= 1:
        if reduce == "reduce_scatter" and out is not None and out.data_ptr() != grad.data_ptr():
            out.copy_(grad)
        return None
    if reduce == "allreduce":
        return dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    if reduce == "reduce_scatter":
        if out is None or out.numel() * world != grad.numel():
            raise ValueError("reduce_scatter needs out with grad.numel() // world elements")
        return dist.reduce_scatter_tensor(out, grad, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    raise ValueError(f"unknown reduction {reduce!r}")


def batch_step(render_view, views, grad, world=1, group=None, zero=True, reduce="allreduce", out=None,
               async_op=False):
    """One step of the batch: grad <- sum over `views` of render_view(v, grad) (which must
    ACCUMULATE into grad), then the cross-rank reduction (reduce_grads).  A renderer may define
    begin() / end() hooks (stream fan-out / join).  Returns the reduction's work handle
    (async_op) or None."""
    if zero:
        grad.zero_()
    begin = getattr(render_view, "begin", None)
    end = getattr(render_view, "end", None)
    if begin is not None:
        begin()
    for v in views:
        render_view(v, grad)
    if end is not None:
        end()
    return reduce_grads(grad, world, group, reduce, out, async_op)


class CudaViewRenderer:
    """render_view for batch_step on the CUDA path: project -> forward (saved) -> backward of
    view v, with the views of a step spread round-robin over len(rasts) CUDA streams (one
    Rasterizer = plan + workspace per stream), so that one view's memory-streaming binning
    kernels overlap another view's latency-bound raster/backward kernels.  Gradients of all
    views accumulate into the same buffer (vector reductions are atomic, so concurrent backward
    passes are safe); end() joins the streams into the current stream before the reduction.
    `grad_pyramid` is a tensor or a callable v -> tensor."""

    def __init__(self, rasts, cams, pos, world_size, opacity, desc, grad_pyramid, streams=None):
        self.rasts = list(rasts)
        self.cams = cams
        self.inputs = (pos, world_size, opacity, desc)
        self.grad_pyramid = grad_pyramid
        self.streams = streams
        self.j = 0

    def begin(self):
        self.main = torch.cuda.current_stream()
        if self.streams is None:
            self.streams = [self.main] + [torch.cuda.Stream(device=self.main.device)
                                          for _ in range(len(self.rasts) - 1)]
        start = torch.cuda.Event()
        start.record(self.main)
        for s in self.streams:
            if s != self.main:
                s.wait_event(start)
        self.j = 0

    def __call__(self, v, grad):
        k = self.j % len(self.rasts)
        self.j += 1
        with torch.cuda.stream(self.streams[k]):
            r = self.rasts[k]
            r.project(self.cams[v], *self.inputs)
            r.forward(save=True)
            gp = self.grad_pyramid(v) if callable(self.grad_pyramid) else self.grad_pyramid
            r.backward(gp, grad)

    def end(self):
        for s in self.streams:
            if s != self.main:
                e = torch.cuda.Event()
                e.record(s)
                self.main.wait_event(e)


def cuda_batch_step(rasts, cams, pos, world_size, opacity, desc, grad_pyramid, views, grad, world=1, group=None,
                    zero=True, streams=None, reduce="allreduce", out=None, async_op=False):
    """batch_step with a CudaViewRenderer (the bench's step)."""
    render = CudaViewRenderer(rasts, cams, pos, world_size, opacity, desc, grad_pyramid, streams)
    return batch_step(render, views, grad, world, group, zero, reduce, out, async_op)


class PipelinedSteps:
    """Steps whose cross-rank reduction overlaps the next step: gradients are double-buffered,
    step k reduces buffer k % 2 asynchronously and step k + 1 renders into the other buffer; a
    buffer is reused only after its reduction completed.  step_fn(grad, k) -> work handle."""

    def __init__(self, grads):
        self.grads = list(grads)
        self.pending = [None] * len(self.grads)

    def run(self, steps, step_fn):
        for k in range(steps):
            b = k % len(self.grads)
            if self.pending[b] is not None:
                self.pending[b].wait()
                self.pending[b] = None
            self.pending[b] = step_fn(self.grads[b], k)
        self.drain()

    def drain(self):
        for b, h in enumerate(self.pending):
            if h is not None:
                h.wait()
            self.pending[b] = None


def flat_inputs(pos, world_size, opacity, desc, world=1):
    """One flat float32 buffer [pos 3n | s_w n | alpha n | desc F n | zero padding] whose size
    splits into `world` equal shards; desc starts 16-B aligned when n % 4 == 0.  Returns
    (flat, n, F)."""
    n, F = pos.shape[0], desc.shape[1]
    parts = [pos.reshape(-1), world_size.reshape(-1), opacity.reshape(-1), desc.reshape(-1)]
    tot = (5 + F) * n
    pad = padded_numel(tot, world) - tot
    if pad:
        parts.append(torch.zeros(pad, dtype=pos.dtype, device=pos.device))
    return torch.cat(parts), n, F


def input_views(flat, n, F):
    """(pos [n,3], s_w [n], alpha [n], desc [n,F]) views of a flat input buffer."""
    return (flat[:3 * n].view(n, 3), flat[3 * n:4 * n], flat[4 * n:5 * n], flat[5 * n:(5 + F) * n].view(n, F))


class ShardedStreamedSteps:
    """End-to-end steps from pinned host memory with sharded transfers: each step, rank r copies
    only its 1/N slice of the flat input buffer host -> device and an all-gather assembles the
    cloud on every rank; after the step's reduce-scatter rank r copies only its 1/N shard of the
    gradient sum device -> host.  Per rank and step that is (5+F) n / N floats each way instead
    of (5+F) n (otherwise PCIe caps the end-to-end rate past a few GPUs).  At
    world = 1 this is the plain streamed step.  Inputs and gradients are double-buffered; the
    copies run on their own streams and overlap the neighbouring steps' kernels.

        pipe = ShardedStreamedSteps(host_flat, grad_numel, device, world, rank, group)
        pipe.run(steps, step_fn, host_out)   # step_fn(dev_flat, grad, out_shard) -> None
    host_flat: pinned float32 [padded (5+F) n]; host_out: two pinned [shard] buffers.
    """

    def __init__(self, host_flat, grad_numel, device, world=1, rank=0, group=None):
        self.host = host_flat
        self.world, self.rank, self.group = world, rank, group
        self.lo, self.hi = shard_range(host_flat.numel(), rank, world)
        self.glo, self.ghi = shard_range(grad_numel, rank, world)
        self.dev_in = [torch.empty(host_flat.numel(), dtype=host_flat.dtype, device=device) for _ in range(2)]
        self.grads = [torch.zeros(grad_numel, dtype=torch.float32, device=device) for _ in range(2)]
        if world > 1:
            self.dev_shard = [torch.empty(self.hi - self.lo, dtype=host_flat.dtype, device=device) for _ in range(2)]
            self.shards = [torch.empty(self.ghi - self.glo, dtype=torch.float32, device=device) for _ in range(2)]
        else:                    # one rank: upload straight into the input buffer, download the gradients
            self.dev_shard = self.dev_in
            self.shards = self.grads
        self.up = torch.cuda.Stream(device=device)
        self.down = torch.cuda.Stream(device=device)

    @property
    def h2d_bytes(self):
        return (self.hi - self.lo) * self.host.element_size()

    @property
    def d2h_bytes(self):
        return (self.ghi - self.glo) * 4

    def run(self, steps, step_fn, host_out):
        main = torch.cuda.current_stream()
        done = [None, None]      # compute of the step that last used buffer b finished
        out = [None, None]       # download of shard b finished
        for k in range(steps):
            b = k % 2
            with torch.cuda.stream(self.up):
                if done[b] is not None:
                    self.up.wait_event(done[b])
                self.dev_shard[b][:self.hi - self.lo].copy_(self.host[self.lo:self.hi], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(self.up)
            main.wait_event(ready)
            if self.world > 1:
                dist.all_gather_into_tensor(self.dev_in[b], self.dev_shard[b], group=self.group)
            if out[b] is not None:
                main.wait_event(out[b])
            step_fn(self.dev_in[b], self.grads[b], self.shards[b])
            done[b] = torch.cuda.Event()
            done[b].record(main)
            with torch.cuda.stream(self.down):
                self.down.wait_event(done[b])
                host_out[b].copy_(self.shards[b], non_blocking=True)
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
