"""ctypes binding of the C-ABI in include/bt_cuda.h (libblobtree_b200.so).

This module is plumbing for the Python side (tests, bench): it declares the
POD structs with the exact C layouts and the function prototypes.  There is
no Python fallback: importing it without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libblobtree_b200.so")
SCENES_PATH = os.path.join(LIB_DIR, "libbt_scenes.so")


class BtError(RuntimeError):
    """Raised when a bt_* entry point returns a non-zero status."""


class bt_node(C.Structure):
    _fields_ = [("word", C.c_uint32), ("parentWord", C.c_uint32), ("leftChild", C.c_int32),
                ("rightChild", C.c_int32), ("isPrimitive", C.c_uint8), ("nodeOp", C.c_uint8),
                ("pad_", C.c_uint8 * 2)]


class bt_camera(C.Structure):
    _fields_ = [("position", C.c_float * 3), ("forward", C.c_float * 3), ("right", C.c_float * 3),
                ("up", C.c_float * 3), ("tanHalf", C.c_float), ("aspect", C.c_float),
                ("invNear", C.c_float), ("invDepthRange", C.c_float), ("nearZ", C.c_float),
                ("farZ", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class bt_render_config(C.Structure):
    _fields_ = [("lipschitz", C.c_float), ("relax", C.c_float), ("minStep", C.c_float),
                ("hitEpsilon", C.c_float), ("maxOverlap", C.c_uint32), ("maxNewPerFetch", C.c_uint32),
                ("fetchWindow", C.c_float), ("normalsMode", C.c_int32), ("threads", C.c_uint32)]


class bt_voi(C.Structure):
    _fields_ = [("family", C.c_uint8), ("pad_", C.c_uint8 * 3), ("primitiveWord", C.c_uint32),
                ("center", C.c_float * 3), ("radius", C.c_float), ("halfExtents", C.c_float * 3),
                ("rotation", C.c_float * 4), ("axisEnd", C.c_float * 3)]


class bt_fragment(C.Structure):
    _fields_ = [("primitiveWord", C.c_uint32), ("zEntry", C.c_float), ("zExit", C.c_float)]


class bt_ipc_handles(C.Structure):
    _fields_ = [("plane", (C.c_ubyte * 64) * 7), ("width", C.c_int32), ("height", C.c_int32)]


class bt_stats(C.Structure):
    _fields_ = [("fieldEvals", C.c_uint64), ("retainedNodeVisits", C.c_uint64),
                ("primitiveEvals", C.c_uint64), ("treeNodeCount", C.c_uint64),
                ("maxOverlap", C.c_uint32), ("maxCacheBytes", C.c_uint32), ("fieldFlops", C.c_uint64),
                ("fragments", C.c_uint64), ("candidatePairs", C.c_uint64), ("tileErrors", C.c_uint64),
                ("normalFallbacks", C.c_uint64), ("warpSteps", C.c_uint64)]


class bt_gbuffer_view(C.Structure):
    _fields_ = [("hit", C.c_void_p), ("depth", C.c_void_p), ("normal", C.c_void_p),
                ("evalCount", C.c_void_p), ("tileMaxOverlap", C.c_void_p), ("tileCacheBytes", C.c_void_p),
                ("tileError", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("tilesX", C.c_int32), ("tilesY", C.c_int32)]


P = C.POINTER
vp = C.c_void_p
u32, i32, f32, u64 = C.c_uint32, C.c_int32, C.c_float, C.c_uint64

# name -> (argtypes); every function returns int status
PROTOTYPES = {
    "bt_ctx_create": [C.c_int, P(vp)],
    "bt_ctx_destroy": [vp],
    "bt_sync": [vp],
    "bt_set_stream": [vp, vp],
    "bt_device_info": [vp, P(C.c_int), P(C.c_int)],
    "bt_tree_upload": [vp, vp, u32, vp, u32, vp, u32, u32],
    "bt_params_update": [vp, vp, vp, vp, u32, u32],
    "bt_params_update_device": [vp, vp, vp, vp, u32, u32],
    "bt_tree_download": [vp, vp, u32],
    "bt_tree_compile": [vp, vp, u32, u32, C.c_int],
    "bt_tree_info": [vp, vp, vp, vp],
    "bt_tree_nodes_download": [vp, vp, u32, vp, u32],
    "bt_tree_fast_indices": [vp],
    "bt_roi": [vp, vp, u32],
    "bt_roi_upload": [vp, vp, u32],
    "bt_voi_build": [vp, f32],
    "bt_voi_upload": [vp, vp, u32],
    "bt_voi_download": [vp, vp, u32],
    "bt_abuffer_build": [vp, P(bt_camera), u32, u32],
    "bt_abuffer_info": [vp, P(u64), P(i32), P(i32)],
    "bt_abuffer_download": [vp, vp, vp, u64],
    "bt_abuffer_upload": [vp, P(bt_camera), vp, vp],
    "bt_trace": [vp, P(bt_camera), P(bt_render_config), u32, u32, C.c_int],
    "bt_normals": [vp, P(bt_camera), C.c_int, C.c_int],
    "bt_normals_rows": [vp, P(bt_camera), C.c_int, C.c_int, u32, u32],
    "bt_oracle_render": [vp, P(bt_camera), P(bt_render_config), C.c_int],
    "bt_render_frame": [vp, P(bt_camera), P(bt_render_config), u32, u32, C.c_int, C.c_int],
    "bt_gbuffer_download": [vp, vp, vp, vp, vp, vp, vp, vp],
    "bt_gbuffer_download_async": [vp, vp, vp, vp, vp, vp, vp, vp],
    "bt_download_wait": [vp],
    "bt_gbuffer_layout": [vp, P(C.c_size_t), P(C.c_size_t)],
    "bt_gbuffer_download_async_slab": [vp, vp],
    "bt_set_tile_order": [vp, vp, u32],
    "bt_gbuffer_export": [vp, vp],
    "bt_gbuffer_import": [vp, vp],
    "bt_gbuffer_import_release": [vp],
    "bt_set_scheduling": [vp, C.c_int],
    "bt_set_step_bound": [vp, C.c_int],
    "bt_set_depth_slabs": [vp, C.c_int],
    "bt_gbuffer_device": [vp, P(bt_gbuffer_view)],
    "bt_gbuffer_upload": [vp, P(bt_camera), vp, vp],
    "bt_stats_download": [vp, P(bt_stats)],
    "bt_stats_reset": [vp],
    "bt_profile_enable": [vp, C.c_int],
    "bt_profile_read": [vp, vp, vp],
    "bt_profile_read_ex": [vp, vp, vp, C.c_uint32],
    "bt_fp32_peak": [C.c_int, P(f32), P(f32)],
    "bt_graph_kernel_count": [vp, P(u32), P(u32)],
}

_lib = None


def load() -> C.CDLL:
    """Load libblobtree_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()) first; "
                          "there is no CPU fallback for the blobtree-b200 hot path")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    lenient = os.environ.get("BT_CAPI_LENIENT") == "1"  # A/B timing against older builds (scripts/ab_multi.sh)
    for name, args in PROTOTYPES.items():
        if lenient and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.bt_last_error.argtypes = []
    lib.bt_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().bt_last_error().decode(errors="replace")
        raise BtError(f"{what} failed (status {rc}): {msg}")


def exported_symbols() -> list[str]:
    return list(PROTOTYPES) + ["bt_last_error"]
