"""PyTorch-facing wrapper of the C ABI: device memory, streams and autograd plumbing only.

    r = Rasterizer(width=1920, height=1080, num_layers=4, num_features=4, max_points=N)
    layers = r.render(cam, pos, world_size, opacity, desc)   # list of (F+1, H_l, W_l)
    loss(layers).backward()                                 # grads of pos, s_w, alpha, tau

All arithmetic runs in libtrips.so on torch.cuda.current_stream().
"""
import torch

from . import _abi as A


def _stream_handle():
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _check_input(name, t, shape_tail=()):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{name} must be a CUDA float32 tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if tuple(t.shape[1:]) != tuple(shape_tail):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected (n, {', '.join(map(str, shape_tail))})")


class Rasterizer:
    """One plan + one workspace (one in-flight view).  Not thread-safe."""

    def __init__(self, width, height, num_layers=4, num_features=4, max_points=1 << 20, device=None, t_min=0.0,
                 coarse_layers=0):
        self.width, self.height = int(width), int(height)
        self.num_layers, self.F = int(num_layers), int(num_features)
        self.max_points = int(max_points)
        self.device = torch.device(device if device is not None else "cuda")
        A.lib()
        self.t_min = float(t_min)
        self.coarse_layers = int(coarse_layers)
        self.plan = A.trips_plan_create(self.num_layers, self.F, self.width, self.height, self.max_points,
                                        self.t_min, self.coarse_layers)
        self.ws = torch.empty(A.trips_workspace_bytes(self.plan), dtype=torch.uint8, device=self.device)
        self.P = A.trips_num_pixels(self.plan)
        self.pyramid_floats = A.trips_pyramid_floats(self.plan)
        self.G = A.trips_grad_stride(self.plan)
        self.dims = [A.trips_layer_dims(self.plan, l) for l in range(self.num_layers)]
        self.generation = 0
        self.n = 0

    def __del__(self):
        plan = getattr(self, "plan", None)
        if plan:
            try:
                A.trips_plan_destroy(plan)
            except Exception:
                pass
            self.plan = None

    # ---- the three ABI stages ------------------------------------------------------
    def project(self, cam, pos, world_size, opacity, desc, level_out=None, proj_out=None):
        n = pos.shape[0]
        _check_input("pos", pos, (3,))
        _check_input("world_size", world_size.view(n, 1) if world_size.dim() == 1 else world_size, (1,))
        _check_input("opacity", opacity.view(n, 1) if opacity.dim() == 1 else opacity, (1,))
        _check_input("desc", desc, (self.F,))
        self.generation += 1
        self.n = n
        A.check(A.trips_project(self.plan, self.ws.data_ptr(), cam, n, pos.data_ptr(), world_size.data_ptr(),
                                opacity.data_ptr(), desc.data_ptr(), _ptr(level_out), _ptr(proj_out),
                                _stream_handle()), "trips_project")

    def forward(self, save=True, out=None):
        if out is None:
            out = torch.empty(self.pyramid_floats, dtype=torch.float32, device=self.device)
        flags = A.TRIPS_FWD_SAVE_FOR_BACKWARD if save else 0
        A.check(A.trips_splat_forward(self.plan, self.ws.data_ptr(), out.data_ptr(), flags, _stream_handle()),
                "trips_splat_forward")
        return out

    def backward(self, grad_pyramid, grad=None, grad_camera=None):
        """Accumulates into grad [n, G] (packed rows: dx, dy, dz, ds_w, dalpha, dtau[F], pad) and,
        if given, into grad_camera [17] (dR row-major, dt, dfx, dfy, dcx, dcy, df)."""
        if grad is None:
            grad = torch.zeros(self.n, self.G, dtype=torch.float32, device=self.device)
        if not grad_pyramid.is_contiguous() or grad_pyramid.numel() != self.pyramid_floats:
            raise ValueError("grad_pyramid must be contiguous with trips_pyramid_floats elements")
        if grad_camera is not None and (grad_camera.numel() != 17 or grad_camera.dtype != torch.float32
                                        or not grad_camera.is_contiguous()):
            raise ValueError("grad_camera must be a contiguous float32 tensor of 17 elements")
        A.check(A.trips_splat_backward(self.plan, self.ws.data_ptr(), grad_pyramid.data_ptr(), grad.data_ptr(),
                                       _ptr(grad_camera), _stream_handle()), "trips_splat_backward")
        return grad

    # ---- views / introspection ------------------------------------------------------
    def layers(self, flat):
        out = []
        for (h, w, off) in self.dims:
            out.append(flat[off:off + (self.F + 1) * h * w].view(self.F + 1, h, w))
        return out

    def unpack_grad(self, grad):
        return grad[:, 0:3], grad[:, 3], grad[:, 4], grad[:, 5:5 + self.F]

    def stats(self):
        return A.trips_read_stats(self.plan, self.ws.data_ptr(), _stream_handle())

    def export_counts(self):
        dst = torch.empty(self.P, dtype=torch.int32, device=self.device)
        A.check(A.trips_debug_export(self.plan, self.ws.data_ptr(), A.TRIPS_EXPORT_COUNTS, dst.data_ptr(),
                                     _stream_handle()), "trips_debug_export")
        return dst

    def export_kept(self):
        dst = torch.empty(self.P * 16, dtype=torch.int32, device=self.device)
        A.check(A.trips_debug_export(self.plan, self.ws.data_ptr(), A.TRIPS_EXPORT_KEPT, dst.data_ptr(),
                                     _stream_handle()), "trips_debug_export")
        return dst.view(self.P, 16)

    def export_kept_layer(self):
        """Layer offset d of each kept entry (coarse-layer inclusion), -1 padded."""
        dst = torch.empty(self.P * 16, dtype=torch.int32, device=self.device)
        A.check(A.trips_debug_export(self.plan, self.ws.data_ptr(), A.TRIPS_EXPORT_KEPT_LAYER, dst.data_ptr(),
                                     _stream_handle()), "trips_debug_export")
        return dst.view(self.P, 16)

    def set_profiling(self, enable=True):
        A.trips_set_profiling(self.plan, enable)

    def stage_ms(self, reset=False):
        return A.trips_read_stage_ms(self.plan, reset)

    # ---- autograd ------------------------------------------------------------------
    def render(self, cam, pos, world_size, opacity, desc):
        flat = _TripsFunction.apply(self, cam, pos, world_size, opacity, desc)
        return self.layers(flat)


class _TripsFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, rast, cam, pos, world_size, opacity, desc):
        rast.project(cam, pos.detach(), world_size.detach(), opacity.detach(), desc.detach())
        out = rast.forward(save=True)
        ctx.rast = rast
        ctx.gen = rast.generation
        return out

    @staticmethod
    def backward(ctx, grad_out):
        rast = ctx.rast
        if rast.generation != ctx.gen:
            raise RuntimeError("TRIPS workspace was reused by another render before backward; "
                               "use one Rasterizer per in-flight view")
        g = rast.backward(grad_out.contiguous())
        gpos, gsw, galpha, gdesc = rast.unpack_grad(g)
        return None, None, gpos, gsw, galpha, gdesc


def morton_order(pos):
    """Permutation (int64 CUDA tensor) putting the cloud in 3-D Morton order
    (trips_morton_order).  Apply once to every per-point array: x[perm]."""
    _check_input("pos", pos, (3,))
    n = pos.shape[0]
    ws = torch.empty(max(A.trips_morton_workspace_bytes(n), 256), dtype=torch.uint8, device=pos.device)
    perm = torch.empty(n, dtype=torch.int32, device=pos.device)
    A.check(A.trips_morton_order(ws.data_ptr(), n, pos.data_ptr(), perm.data_ptr(), _stream_handle()),
            "trips_morton_order")
    return perm.long()


def knn_sizes(pos, return_neighbors=False):
    """Initial world sizes s_w = mean distance to the 4 nearest neighbours,
    computed on the GPU (trips_knn_sizes).  Returns size [n] (and neighbours [n, 4])."""
    _check_input("pos", pos, (3,))
    n = pos.shape[0]
    ws = torch.empty(max(A.trips_knn_workspace_bytes(n), 256), dtype=torch.uint8, device=pos.device)
    size = torch.empty(n, dtype=torch.float32, device=pos.device)
    nbr = torch.empty(n, 4, dtype=torch.int32, device=pos.device) if return_neighbors else None
    A.check(A.trips_knn_sizes(ws.data_ptr(), n, pos.data_ptr(), size.data_ptr(), _ptr(nbr), _stream_handle()),
            "trips_knn_sizes")
    return (size, nbr) if return_neighbors else size


def render(rast, cam, pos, world_size, opacity, desc):
    return rast.render(cam, pos, world_size, opacity, desc)
