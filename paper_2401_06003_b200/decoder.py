"""PyTorch-facing wrapper of trips_decode (the gated-convolution decoder over the pyramid,
SURVEY.md 8(f) row 2): device memory and streams only -- the weight packing,
upsampling, convolutions and activations all run in libtrips.so.

    dec = Decoder(rasterizer, out_channels=3)          # shares the rasterizer's pyramid geometry
    image = dec(params, pyramid_flat)                   # (out_channels, H, W) float32

`params` is the flat float32 parameter vector of include/trips.h (trips_decode); its length is
`dec.param_count`.
"""
import torch

from . import _abi as A


class Decoder:
    def __init__(self, rasterizer, out_channels=3):
        self.r = rasterizer
        self.out_channels = int(out_channels)
        self.param_count = A.trips_decoder_param_count(rasterizer.plan, self.out_channels)
        self.ws = torch.empty(A.trips_decoder_workspace_bytes(rasterizer.plan), dtype=torch.uint8,
                              device=rasterizer.device)

    def __call__(self, params, pyramid, out=None):
        dev = self.r.device
        for name, t, n in (("params", params, self.param_count), ("pyramid", pyramid, self.r.pyramid_floats)):
            if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 or t.device != dev:
                raise TypeError(f"{name} must be a float32 tensor on {dev}")
            if not t.is_contiguous() or t.numel() != n:
                raise ValueError(f"{name} must be contiguous with {n} elements")
        shape = (self.out_channels, self.r.height, self.r.width)
        if out is None:
            out = torch.empty(shape, dtype=torch.float32, device=dev)
        elif out.shape != shape or out.dtype != torch.float32 or out.device != dev or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous float32 {shape} tensor on {dev}")
        with torch.cuda.device(dev):
            A.trips_decode(self.r.plan, self.ws.data_ptr(), params.data_ptr(), self.out_channels, pyramid.data_ptr(),
                           out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
        return out
