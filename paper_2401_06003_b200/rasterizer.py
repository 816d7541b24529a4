"""PyTorch-facing wrapper of the C ABI: device memory, streams and autograd plumbing only.

    r = Rasterizer(width=1920, height=1080, num_layers=4, num_features=4, max_points=N)
    layers = r.render(cam, pos, world_size, opacity, desc)   # list of (F+1, H_l, W_l)
    loss(layers).backward()                                 # grads of pos, s_w, alpha, tau

All arithmetic runs in libtrips.so on the device's current stream.

Gradient buffer (trips_splat_backward): one flat float32 tensor of (5 + F) * n floats laid out
[pos_size: n x 4 | desc: n x F | opacity: n], i.e. 36 B per point at F = 4 -- the buffer a
multi-GPU step all-reduces once per batch.  `new_grad`, `grad_parts` and `unpack_grad` build
and view it.
"""
import torch

from . import _abi as A


def _ptr(t):
    return None if t is None else t.data_ptr()


def _check_input(name, t, shape_tail=(), device=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{name} must be a CUDA float32 tensor")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, the rasterizer on {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if tuple(t.shape[1:]) != tuple(shape_tail):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected (n, {', '.join(map(str, shape_tail))})")


def _vector(name, t, n, device):
    """(n,) or (n, 1) float32 CUDA tensor -> contiguous (n,) view."""
    if not isinstance(t, torch.Tensor) or t.numel() != n or t.dim() not in (1, 2) or (t.dim() == 2 and t.shape[1] != 1):
        raise ValueError(f"{name} must have shape (n,) or (n, 1) with n = {n}")
    _check_input(name, t.reshape(n, 1), (1,), device)
    return t.reshape(n)


class Rasterizer:
    """One plan + one workspace (one in-flight view).  Not thread-safe."""

    def __init__(self, width, height, num_layers=4, num_features=4, max_points=1 << 20, device=None, t_min=0.0,
                 coarse_layers=0):
        self.width, self.height = int(width), int(height)
        self.num_layers, self.F = int(num_layers), int(num_features)
        self.max_points = int(max_points)
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        A.lib()
        self.t_min = float(t_min)
        self.coarse_layers = int(coarse_layers)
        self.plan = A.trips_plan_create(self.num_layers, self.F, self.width, self.height, self.max_points,
                                        self.t_min, self.coarse_layers)
        self.ws = torch.empty(A.trips_workspace_bytes(self.plan), dtype=torch.uint8, device=self.device)
        self.P = A.trips_num_pixels(self.plan)
        self.pyramid_floats = A.trips_pyramid_floats(self.plan)
        self.dims = [A.trips_layer_dims(self.plan, l) for l in range(self.num_layers)]
        self.generation = 0
        self.n = 0
        self._desc = None          # descriptors of the current frame (gathered in place by the kernels)
        self._last_gpyr = None     # grad_pyramid of the last backward (SCREEN_GRADS export)

    def __del__(self):
        plan = getattr(self, "plan", None)
        if plan:
            try:
                A.trips_plan_destroy(plan)
            except Exception:
                pass
            self.plan = None

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    # ---- gradient buffer ------------------------------------------------------------
    def grad_floats(self, n=None):
        return (5 + self.F) * (self.n if n is None else int(n))

    def new_grad(self, n=None):
        """Zeroed flat gradient buffer [(5 + F) n] (layout in the module docstring)."""
        return torch.zeros(self.grad_floats(n), dtype=torch.float32, device=self.device)

    def grad_parts(self, flat, n=None):
        """(pos_size [n, 4], desc [n, F], opacity [n]) views of a flat gradient buffer."""
        n = self.n if n is None else int(n)
        if flat.numel() < self.grad_floats(n):
            raise ValueError(f"gradient buffer has {flat.numel()} floats, expected >= (5 + F) n = {self.grad_floats(n)}")
        return (flat[:4 * n].view(n, 4), flat[4 * n:(4 + self.F) * n].view(n, self.F),
                flat[(4 + self.F) * n:(5 + self.F) * n])

    def unpack_grad(self, flat, n=None):
        """(d pos [n, 3], d s_w [n], d alpha [n], d tau [n, F]) views of a flat gradient buffer."""
        ps, de, op = self.grad_parts(flat, n)
        return ps[:, 0:3], ps[:, 3], op, de

    def grad_rows(self, flat, n=None):
        """[n, 5 + F] copy in the oracle's row order (d pos, d s_w, d alpha, d tau)."""
        gp, gs, ga, gd = self.unpack_grad(flat, n)
        return torch.cat([gp, gs[:, None], ga[:, None], gd], 1)

    # ---- the three ABI stages ------------------------------------------------------
    def project(self, cam, pos, world_size, opacity, desc, level_out=None, proj_out=None):
        """Stage 1.  When F % 4 == 0 and desc is 16-B aligned the kernels of this frame read the
        descriptor rows in place: desc must stay allocated and unmodified until the frame's last
        backward (the Rasterizer keeps a reference; autograd's render() also version-checks it)."""
        n = pos.shape[0]
        _check_input("pos", pos, (3,), self.device)
        world_size = _vector("world_size", world_size, n, self.device)
        opacity = _vector("opacity", opacity, n, self.device)
        _check_input("desc", desc, (self.F,), self.device)
        self.generation += 1
        self.n = n
        self._desc = desc
        self._last_gpyr = None
        with torch.cuda.device(self.device):
            A.check(A.trips_project(self.plan, self.ws.data_ptr(), cam, n, pos.data_ptr(), world_size.data_ptr(),
                                    opacity.data_ptr(), desc.data_ptr(), _ptr(level_out), _ptr(proj_out),
                                    self._stream()), "trips_project")

    def forward(self, save=True, out=None):
        if out is None:
            out = torch.empty(self.pyramid_floats, dtype=torch.float32, device=self.device)
        elif (not out.is_cuda or out.dtype != torch.float32 or out.device != self.device or not out.is_contiguous()
              or out.numel() != self.pyramid_floats):
            raise ValueError("out must be a contiguous CUDA float32 tensor of trips_pyramid_floats elements")
        flags = A.TRIPS_FWD_SAVE_FOR_BACKWARD if save else 0
        with torch.cuda.device(self.device):
            A.check(A.trips_splat_forward(self.plan, self.ws.data_ptr(), out.data_ptr(), flags, self._stream()),
                    "trips_splat_forward")
        return out

    def backward(self, grad_pyramid, grad=None, grad_camera=None):
        """Accumulates into the flat gradient buffer `grad` [>= (5 + F) n] (allocated zeroed if None)
        and, if given, into grad_camera [17] (dR row-major, dt, dfx, dfy, dcx, dcy, df)."""
        if grad is None:
            grad = self.new_grad()
        for name, t, numel in (("grad_pyramid", grad_pyramid, self.pyramid_floats), ("grad", grad, self.grad_floats()),
                               ("grad_camera", grad_camera, 17)):
            if t is None and name == "grad_camera":
                continue
            # the flat gradient buffer may carry trailing padding (sharded reductions), never less
            ok_n = t.numel() >= numel if (name == "grad" and isinstance(t, torch.Tensor)) else \
                (isinstance(t, torch.Tensor) and t.numel() == numel)
            if (not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 or t.device != self.device
                    or not t.is_contiguous() or not ok_n):
                raise ValueError(f"{name} must be a contiguous float32 tensor of {numel} elements on {self.device}")
        ps, de, op = self.grad_parts(grad)
        self._last_gpyr = grad_pyramid
        with torch.cuda.device(self.device):
            A.check(A.trips_splat_backward(self.plan, self.ws.data_ptr(), grad_pyramid.data_ptr(), ps.data_ptr(),
                                           op.data_ptr(), de.data_ptr(), _ptr(grad_camera), self._stream()),
                    "trips_splat_backward")
        return grad

    # ---- views / introspection ------------------------------------------------------
    def layers(self, flat):
        out = []
        for (h, w, off) in self.dims:
            out.append(flat[off:off + (self.F + 1) * h * w].view(self.F + 1, h, w))
        return out

    def stats(self):
        with torch.cuda.device(self.device):
            return A.trips_read_stats(self.plan, self.ws.data_ptr(), self._stream())

    def _export(self, what, dst):
        with torch.cuda.device(self.device):
            A.check(A.trips_debug_export(self.plan, self.ws.data_ptr(), what, dst.data_ptr(), self._stream()),
                    "trips_debug_export")
        return dst

    def export_counts(self):
        return self._export(A.TRIPS_EXPORT_COUNTS, torch.empty(self.P, dtype=torch.int32, device=self.device))

    def export_kept(self):
        return self._export(A.TRIPS_EXPORT_KEPT, torch.empty(self.P * 16, dtype=torch.int32,
                                                             device=self.device)).view(self.P, 16)

    def export_kept_layer(self):
        """Layer offset d of each kept entry (coarse-layer inclusion), -1 padded."""
        return self._export(A.TRIPS_EXPORT_KEPT_LAYER, torch.empty(self.P * 16, dtype=torch.int32,
                                                                   device=self.device)).view(self.P, 16)

    def export_screen_grads(self):
        """[n, 4 + F] screen-space gradients (d x, d y, d s, d alpha, d tau) of the last backward's
        grad_pyramid, before the projection chain (SURVEY.md 8(b) SCREEN_GRADS)."""
        return self._export(A.TRIPS_EXPORT_SCREEN_GRADS, torch.empty(self.n * (4 + self.F), dtype=torch.float32,
                                                                     device=self.device)).view(self.n, 4 + self.F)

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
        ctx.shapes = (world_size.shape, opacity.shape)
        # the kernels read the descriptor rows again in the backward: keep them alive (a computed,
        # non-leaf desc would otherwise be freed and reused) and let autograd's version counter
        # reject in-place edits between forward and backward
        ctx.save_for_backward(desc)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        (desc,) = ctx.saved_tensors
        rast = ctx.rast
        if rast.generation != ctx.gen:
            raise RuntimeError("TRIPS workspace was reused by another render before backward; "
                               "use one Rasterizer per in-flight view")
        del desc
        g = rast.backward(grad_out.contiguous())
        gpos, gsw, galpha, gdesc = rast.unpack_grad(g)
        return None, None, gpos, gsw.reshape(ctx.shapes[0]), galpha.reshape(ctx.shapes[1]), gdesc


def morton_order(pos):
    """Permutation (int64 CUDA tensor) putting the cloud in 3-D Morton order
    (trips_morton_order).  Apply once to every per-point array: x[perm]."""
    _check_input("pos", pos, (3,))
    n = pos.shape[0]
    ws = torch.empty(max(A.trips_morton_workspace_bytes(n), 256), dtype=torch.uint8, device=pos.device)
    perm = torch.empty(n, dtype=torch.int32, device=pos.device)
    with torch.cuda.device(pos.device):
        A.check(A.trips_morton_order(ws.data_ptr(), n, pos.data_ptr(), perm.data_ptr(),
                                     torch.cuda.current_stream(pos.device).cuda_stream), "trips_morton_order")
    return perm.long()


def knn_sizes(pos, return_neighbors=False):
    """Initial world sizes s_w = mean distance to the 4 nearest neighbours,
    computed on the GPU (trips_knn_sizes).  Returns size [n] (and neighbours [n, 4])."""
    _check_input("pos", pos, (3,))
    n = pos.shape[0]
    ws = torch.empty(max(A.trips_knn_workspace_bytes(n), 256), dtype=torch.uint8, device=pos.device)
    size = torch.empty(n, dtype=torch.float32, device=pos.device)
    nbr = torch.empty(n, 4, dtype=torch.int32, device=pos.device) if return_neighbors else None
    with torch.cuda.device(pos.device):
        A.check(A.trips_knn_sizes(ws.data_ptr(), n, pos.data_ptr(), size.data_ptr(), _ptr(nbr),
                                  torch.cuda.current_stream(pos.device).cuda_stream), "trips_knn_sizes")
    return (size, nbr) if return_neighbors else size


def render(rast, cam, pos, world_size, opacity, desc):
    return rast.render(cam, pos, world_size, opacity, desc)
