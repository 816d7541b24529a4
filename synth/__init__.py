"""Seeded synthetic inputs (point clouds, cameras, gradient pyramids).

Shared by the oracle side (tests) and the CUDA side (tests, bench).  Holds NONE of
the method's arithmetic: no projection, layer selection, footprint or blending --
only random numbers, scene geometry and camera poses.
"""
from .scenes import Camera, Scene, look_at, make_config, tiny_scene, adversarial_scene, grad_pyramid  # noqa: F401
