"""blobtree-b200: B200-native synchronized tracing of blobtree implicit
surfaces (arXiv 2304.09673), behind the reference's C++ API.

The product is libblobtree_b200.so (include/blobtree/*.hpp drop-in C++ API
and the include/bt_cuda.h C-ABI over hand-written sm_100a kernels).  This
Python package is a thin ctypes mirror used by the tests and bench.py.
"""
from ._capi import BtError, LIB_PATH, load  # noqa: F401
from .pipeline import GBuffer, Renderer, RenderConfig, Scene  # noqa: F401

__all__ = ["BtError", "GBuffer", "LIB_PATH", "Renderer", "RenderConfig", "Scene", "load"]
