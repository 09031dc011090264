"""Degenerate cameras and images shared by the CPU (port vs reference) and GPU
(pipeline vs reference) edge-case tests."""
import numpy as np


def _cam(pos, target, near=0.1, far=40.0, w=128, h=128, fov=45.0, up=(0.0, 1.0, 0.0)):
    return np.array([*pos, *target, *up, fov, near, far, w, h], np.float32)


EDGE = [
    # name, camera, what it exercises
    ("C1", _cam((0, 0, -6), (0, 0, -12)), "looking away: no fragments at all"),
    ("C1", _cam((0, 0, -6), (0, 0, 0), far=3.0), "whole scene beyond the far plane"),
    ("C2", _cam((0.1, 0.05, 0.0), (0.1, 0.05, 5.0), w=96, h=64), "camera inside the volumes (near clipping)"),
    ("csg", _cam((0, 0, -6), (0, 0, 0), w=1, h=1), "a 1x1 image"),
    ("csg", _cam((0, 0, -6), (0, 0, 0), w=7, h=3), "an image smaller than one tile"),
    ("C2", _cam((0.0, 0.0, -7.5), (0.0, -0.15, 0.0), w=1, h=97), "a one-pixel-wide column"),
    ("stack:120", _cam((0, 0, -6), (0, 0, 0), w=64, h=64), "overlap saturation (maxOverlap 96, parameter cache spills)"),
    ("slab", _cam((0, 0, -6), (0, 0, 0), fov=170.0, w=64, h=48), "extreme field of view"),
]
