"""B200-native TRIPS trilinear point-splatting rasterizer (arXiv 2401.06003).

The product is the C-ABI library libtrips.so (include/trips.h; hand-written CUDA for
sm_100a in csrc/).  This package is its thin Python binding:

  _abi        ctypes marshalling, same names as include/trips.h
  rasterizer  Rasterizer (plan + workspace on torch memory/streams) and autograd
  dist        view-parallel multi-GPU step (replicated points, one gradient all-reduce)

There is no CPU fallback: importing the binding loads libtrips.so or raises.
"""
from . import _abi  # noqa: F401
from .rasterizer import Rasterizer, knn_sizes, morton_order, render  # noqa: F401
from .decoder import Decoder  # noqa: F401

__all__ = ["Rasterizer", "render", "morton_order", "knn_sizes", "Decoder"]
