"""Python mirror of the reference's per-frame pipeline over the C-ABI.

The reference composes a frame as (proj/tests/test_tracer.cpp:25-31)::

    rois    = propagate_roi(tree)                          # (a)
    volumes = build_volumes_of_interest(tree, rois, eps)   # (a)
    abuffer = rasterize_volumes(volumes, frame)            # (b)
    g       = render_tiles(tree, abuffer, frame, cfg)      # (c)
    compute_normals(tree, g, frame, cfg.normalsMode)

`Renderer` exposes the same stages (same names, argument meaning and
error behaviour: invalid configs raise before touching the device) on a
device-resident context, plus `render_frame` for the fused, CUDA-graph
replayed frame.  Everything runs in libblobtree_b200.so; this module only
moves numpy buffers across the boundary.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi as capi
from ._capi import bt_camera, bt_fragment, bt_node, bt_render_config, bt_stats, bt_voi, check

_scenes = None


def _scenes_lib() -> C.CDLL:
    global _scenes
    if _scenes is None:
        capi.load()
        lib = C.CDLL(capi.SCENES_PATH)
        lib.sc_scene_new.argtypes = [C.c_char_p, C.c_uint32, C.c_int, C.c_int]
        lib.sc_scene_new.restype = C.c_void_p
        lib.sc_scene_error.restype = C.c_char_p
        lib.sc_scene_free.argtypes = [C.c_void_p]
        lib.sc_scene_info.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        lib.sc_scene_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.sc_scene_camera.argtypes = [C.c_void_p, C.c_void_p]
        lib.sc_scene_device_camera.argtypes = [C.c_void_p, C.POINTER(bt_camera)]
        lib.sc_scene_perturb.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.sc_scene_set_camera.argtypes = [C.c_void_p, C.c_void_p]
        lib.sc_scene_perturb.restype = C.c_uint32
        _scenes = lib
    return _scenes


def ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(0)


NODE_DTYPE = np.dtype([("word", "<u4"), ("parentWord", "<u4"), ("leftChild", "<i4"), ("rightChild", "<i4"),
                       ("isPrimitive", "u1"), ("nodeOp", "u1"), ("pad", "u1", 2)])
VOI_DTYPE = np.dtype([("family", "u1"), ("pad", "u1", 3), ("primitiveWord", "<u4"), ("center", "<f4", 3),
                      ("radius", "<f4"), ("halfExtents", "<f4", 3), ("rotation", "<f4", 4), ("axisEnd", "<f4", 3)])
FRAG_DTYPE = np.dtype([("primitiveWord", "<u4"), ("zEntry", "<f4"), ("zExit", "<f4")])
# bt_scene_node: one node of a scene graph for the GPU compile (bt_tree_compile)
GRAPH_DTYPE = np.dtype([("isPrimitive", "u1"), ("kind", "u1"), ("pad", "u1", 2), ("left", "<i4"), ("right", "<i4"),
                        ("params", "<f4", 17)])
assert GRAPH_DTYPE.itemsize == 80
assert NODE_DTYPE.itemsize == C.sizeof(bt_node) == 20
assert VOI_DTYPE.itemsize == C.sizeof(bt_voi) == 64
assert FRAG_DTYPE.itemsize == C.sizeof(bt_fragment) == 12


@dataclass
class RenderConfig:
    """RenderConfig (reference include/blobtree/tracer.hpp:11-26)."""
    lipschitz: float = 1.45
    relax: float = 1.7
    minStep: float = 0.005
    hitEpsilon: float = float(np.float32(0.5) * np.float32(0.005) * np.float32(1.45))
    maxOverlap: int = 96
    maxNewPerFetch: int = 6
    fetchWindow: float = 0.0
    normalsMode: int = 0  # 0 depth-differential, 1 central difference
    threads: int = 0

    def validate(self) -> None:
        """validate_config (reference src/tracer.cpp:10-19)."""
        if not (1.0 <= self.relax < 2.0):
            raise ValueError("relaxation factor must lie in [1, 2)")
        if not self.lipschitz >= 1.0:
            raise ValueError("lipschitz bound must be at least 1")
        if not self.minStep > 0.0:
            raise ValueError("min step must be > 0")
        if not self.hitEpsilon > 0.0:
            raise ValueError("hit epsilon must be > 0")
        if self.maxOverlap == 0 or self.maxOverlap > 96:
            raise ValueError("max overlap must lie in [1, 96]")

    def to_c(self) -> bt_render_config:
        self.validate()
        return bt_render_config(self.lipschitz, self.relax, self.minStep, self.hitEpsilon, self.maxOverlap,
                                self.maxNewPerFetch, self.fetchWindow, self.normalsMode, self.threads)


@dataclass
class Scene:
    """A synthetic workload built by libbt_scenes.so through the C++ API."""
    name: str
    seed: int
    handle: int
    data: np.ndarray          # float32 [nwords*4]
    nodes: np.ndarray         # NODE_DTYPE [nnodes]
    prims: np.ndarray         # uint32 [nprims]
    root_word: int
    width: int
    height: int
    camera14: np.ndarray      # position, target, up, fov, near, far, w, h
    device_camera: bt_camera = field(repr=False, default=None)

    @classmethod
    def build(cls, name: str, seed: int = 0, width: int = 0, height: int = 0) -> "Scene":
        lib = _scenes_lib()
        h = lib.sc_scene_new(name.encode(), seed, width, height)
        if not h:
            raise ValueError(f"scene {name!r}: {lib.sc_scene_error().decode()}")
        nw, nn, npr, rw, w, hh = (C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_int32(), C.c_int32())
        lib.sc_scene_info(h, C.byref(nw), C.byref(nn), C.byref(npr), C.byref(rw), C.byref(w), C.byref(hh))
        data = np.zeros(nw.value * 4, np.float32)
        nodes = np.zeros(nn.value, NODE_DTYPE)
        prims = np.zeros(npr.value, np.uint32)
        lib.sc_scene_tree(h, ptr(data), ptr(nodes), ptr(prims))
        cam = np.zeros(14, np.float32)
        lib.sc_scene_camera(h, ptr(cam))
        dc = bt_camera()
        lib.sc_scene_device_camera(h, C.byref(dc))
        return cls(name, seed, h, data, nodes, prims, rw.value, w.value, hh.value, cam, dc)

    def graph(self, seed: int | None = None) -> tuple[np.ndarray, int]:
        """The scene graph this tree was compiled from (GRAPH_DTYPE), nodes in
        a random order when `seed` is given; returns (graph, root index)."""
        n = len(self.nodes)
        perm = np.arange(n) if seed is None else np.random.default_rng(seed).permutation(n)
        where = np.empty(n, np.int64)
        where[perm] = np.arange(n)  # ordinal -> graph index
        g = np.zeros(n, GRAPH_DTYPE)
        words = self.data.reshape(-1, 4)
        for o, rec in enumerate(self.nodes):
            e = g[where[o]]
            e["isPrimitive"] = rec["isPrimitive"]
            e["kind"] = rec["nodeOp"]
            if rec["isPrimitive"]:
                cnt = 7 + (1, 3, 2, 3, 3, 10)[rec["nodeOp"]]  # transform + shape floats
                e["left"] = e["right"] = -1
                e["params"][:cnt] = words[rec["word"] + 1:].reshape(-1)[:cnt]
            else:
                e["left"] = where[rec["leftChild"]]
                e["right"] = where[rec["rightChild"]]
                if rec["nodeOp"] > 5:
                    e["params"][:2] = words[rec["word"] + 1][:2]
        return g, int(where[n - 1])

    @property
    def tiles(self) -> tuple[int, int]:
        return (self.width + 7) // 8, (self.height + 7) // 8

    def set_camera(self, camera14) -> None:
        """Replace the camera: position[3] target[3] up[3] fov near far width height."""
        v = np.ascontiguousarray(camera14, np.float32)
        lib = _scenes_lib()
        if lib.sc_scene_set_camera(self.handle, ptr(v)) != 0:
            raise ValueError(f"camera: {lib.sc_scene_error().decode()}")
        lib.sc_scene_camera(self.handle, ptr(self.camera14))
        self.width, self.height = int(v[12]), int(v[13])
        dc = bt_camera()
        lib.sc_scene_device_camera(self.handle, C.byref(dc))
        self.device_camera = dc

    def perturb(self, frame: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """C3/C4 per-frame perturbation; returns (words, params[n,17], counts)."""
        n = len(self.prims)
        words = np.zeros(n, np.uint32)
        params = np.zeros((n, 17), np.float32)
        counts = np.zeros(n, np.uint32)
        _scenes_lib().sc_scene_perturb(self.handle, frame, ptr(words), ptr(params), ptr(counts))
        self.data[:] = 0  # refresh the host copy of the tree words
        _scenes_lib().sc_scene_tree(self.handle, ptr(self.data), ptr(self.nodes), ptr(self.prims))
        return words, params, counts

    def close(self) -> None:
        if self.handle:
            _scenes_lib().sc_scene_free(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class GBuffer:
    """GBuffer (reference include/blobtree/tracer.hpp:30-43) as numpy planes."""
    width: int
    height: int
    hit: np.ndarray
    depth: np.ndarray
    normal: np.ndarray
    evalCount: np.ndarray
    tileMaxOverlap: np.ndarray
    tileCacheBytes: np.ndarray
    tileError: np.ndarray

    @classmethod
    def empty(cls, w: int, h: int) -> "GBuffer":
        tx, ty = (w + 7) // 8, (h + 7) // 8
        return cls(w, h, np.zeros(w * h, np.uint8), np.zeros(w * h, np.float32), np.zeros((w * h, 3), np.float32),
                   np.zeros(w * h, np.uint32), np.zeros(tx * ty, np.uint32), np.zeros(tx * ty, np.uint32),
                   np.zeros(tx * ty, np.uint8))


class Renderer:
    """Device-resident context (one per GPU) over include/bt_cuda.h."""

    def __init__(self, device: int = 0):
        self.lib = capi.load()
        self.ctx = C.c_void_p()
        check(self.lib.bt_ctx_create(device, C.byref(self.ctx)), "bt_ctx_create")
        self.scene: Scene | None = None

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        if self.ctx:
            self.lib.bt_ctx_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self) -> None:
        check(self.lib.bt_sync(self.ctx), "bt_sync")

    def set_stream(self, stream_ptr: int) -> None:
        check(self.lib.bt_set_stream(self.ctx, C.c_void_p(stream_ptr)), "bt_set_stream")

    def device_info(self) -> tuple[int, int]:
        sm, clk = C.c_int(), C.c_int()
        check(self.lib.bt_device_info(self.ctx, C.byref(sm), C.byref(clk)), "bt_device_info")
        return sm.value, clk.value

    # -- tree ----------------------------------------------------------------
    def upload(self, scene: Scene) -> None:
        self.scene = scene
        check(self.lib.bt_tree_upload(self.ctx, ptr(scene.data), len(scene.data) // 4, ptr(scene.nodes),
                                      len(scene.nodes), ptr(scene.prims), len(scene.prims), scene.root_word),
              "bt_tree_upload")

    def compile_tree(self, graph: np.ndarray, root: int, on_device: bool = False) -> None:
        """GPU compile of a scene graph (GRAPH_DTYPE, any node order) into the
        context's tree (bt_tree_compile); `graph` may be a device address
        (int) with `on_device`."""
        if on_device:
            addr, n = graph
            check(self.lib.bt_tree_compile(self.ctx, C.c_void_p(addr), n, root, 1), "bt_tree_compile")
        else:
            g = np.ascontiguousarray(graph, GRAPH_DTYPE)
            check(self.lib.bt_tree_compile(self.ctx, ptr(g), len(g), root, 0), "bt_tree_compile")

    def fast_indices(self) -> None:
        """compute_fast_indices on the device (bt_tree_fast_indices)."""
        check(self.lib.bt_tree_fast_indices(self.ctx), "bt_tree_fast_indices")

    def tree_arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(words float32 [nwords*4], node records, primitive words) of the context's tree."""
        nw, nn, npr = C.c_uint32(), C.c_uint32(), C.c_uint32()
        check(self.lib.bt_tree_info(self.ctx, C.byref(nw), C.byref(nn), C.byref(npr)), "bt_tree_info")
        data = np.zeros(nw.value * 4, np.float32)
        nodes = np.zeros(nn.value, NODE_DTYPE)
        prims = np.zeros(npr.value, np.uint32)
        check(self.lib.bt_tree_download(self.ctx, ptr(data), nw.value), "bt_tree_download")
        check(self.lib.bt_tree_nodes_download(self.ctx, ptr(nodes), nn.value, ptr(prims), npr.value),
              "bt_tree_nodes_download")
        return data, nodes, prims

    def update_params(self, words: np.ndarray, params: np.ndarray, counts: np.ndarray) -> None:
        check(self.lib.bt_params_update(self.ctx, ptr(words), ptr(params), ptr(counts), len(words), 17),
              "bt_params_update")

    def update_params_device(self, d_words: int, d_params: int, d_counts: int, n: int) -> None:
        check(self.lib.bt_params_update_device(self.ctx, C.c_void_p(d_words), C.c_void_p(d_params),
                                               C.c_void_p(d_counts), n, 17), "bt_params_update_device")

    def tree_words(self) -> np.ndarray:
        out = np.zeros_like(self.scene.data)
        check(self.lib.bt_tree_download(self.ctx, ptr(out), len(out) // 4), "bt_tree_download")
        return out

    # -- (a) -----------------------------------------------------------------
    def propagate_roi(self) -> np.ndarray:
        out = np.zeros(len(self.scene.nodes), np.float32)
        check(self.lib.bt_roi(self.ctx, ptr(out), len(out)), "bt_roi")
        return out

    def build_volumes_of_interest(self, margin: float, roi: np.ndarray | None = None) -> np.ndarray:
        if roi is None:
            check(self.lib.bt_roi(self.ctx, None, 0), "bt_roi")
        else:
            roi = np.ascontiguousarray(roi, np.float32)
            check(self.lib.bt_roi_upload(self.ctx, ptr(roi), len(roi)), "bt_roi_upload")
        check(self.lib.bt_voi_build(self.ctx, margin), "bt_voi_build")
        out = np.zeros(len(self.scene.prims), VOI_DTYPE)
        check(self.lib.bt_voi_download(self.ctx, ptr(out), len(out)), "bt_voi_download")
        return out

    def upload_volumes(self, vois: np.ndarray) -> None:
        vois = np.ascontiguousarray(vois, VOI_DTYPE)
        check(self.lib.bt_voi_upload(self.ctx, ptr(vois), len(vois)), "bt_voi_upload")

    # -- (b) -----------------------------------------------------------------
    def rasterize_volumes(self, cam: bt_camera, tile0: int = 0, tile1: int = 0) -> tuple[np.ndarray, np.ndarray]:
        check(self.lib.bt_abuffer_build(self.ctx, C.byref(cam), tile0, tile1), "bt_abuffer_build")
        return self.download_abuffer()

    def download_abuffer(self) -> tuple[np.ndarray, np.ndarray]:
        total, tx, ty = C.c_uint64(), C.c_int32(), C.c_int32()
        check(self.lib.bt_abuffer_info(self.ctx, C.byref(total), C.byref(tx), C.byref(ty)), "bt_abuffer_info")
        offsets = np.zeros(tx.value * ty.value + 1, np.uint32)
        frags = np.zeros(total.value, FRAG_DTYPE)
        check(self.lib.bt_abuffer_download(self.ctx, ptr(offsets), ptr(frags), total.value), "bt_abuffer_download")
        return offsets, frags

    def upload_abuffer(self, cam: bt_camera, offsets: np.ndarray, frags: np.ndarray) -> None:
        offsets = np.ascontiguousarray(offsets, np.uint32)
        frags = np.ascontiguousarray(frags, FRAG_DTYPE)
        check(self.lib.bt_abuffer_upload(self.ctx, C.byref(cam), ptr(offsets), ptr(frags)), "bt_abuffer_upload")

    # -- (c) -----------------------------------------------------------------
    def render_tiles(self, cam: bt_camera, cfg: RenderConfig, exact: bool = True, tile0: int = 0,
                     tile1: int = 0) -> None:
        c = cfg.to_c()
        check(self.lib.bt_trace(self.ctx, C.byref(cam), C.byref(c), tile0, tile1, int(exact)), "bt_trace")

    def compute_normals(self, cam: bt_camera, mode: int = 0, exact: bool = True) -> None:
        check(self.lib.bt_normals(self.ctx, C.byref(cam), mode, int(exact)), "bt_normals")

    def set_step_bound(self, mode: int) -> None:
        """0: the reference's global Lipschitz bound; 1: a bound per interval
        view (1-Lipschitz views march with L = 1; bt_set_step_bound)."""
        check(self.lib.bt_set_step_bound(self.ctx, int(mode)), "bt_set_step_bound")

    def set_depth_slabs(self, slabs: int) -> None:
        """1: the reference's single pass; n > 1: frames rendered in n depth
        slabs, front to back (bt_set_depth_slabs)."""
        check(self.lib.bt_set_depth_slabs(self.ctx, int(slabs)), "bt_set_depth_slabs")

    def compute_normals_rows(self, cam: bt_camera, tile0: int, tile1: int, mode: int = 0, exact: bool = True) -> None:
        """Normals of the tile rows covering [tile0, tile1) only (a sharded
        rank; into the root's planes when a G-buffer is imported)."""
        check(self.lib.bt_normals_rows(self.ctx, C.byref(cam), mode, int(exact), tile0, tile1), "bt_normals_rows")

    def oracle_render(self, cam: bt_camera, cfg: RenderConfig, exact: bool = True) -> None:
        c = cfg.to_c()
        check(self.lib.bt_oracle_render(self.ctx, C.byref(cam), C.byref(c), int(exact)), "bt_oracle_render")

    def render_frame(self, cam: bt_camera, cfg: RenderConfig, exact: bool = False, graph: bool = True,
                     tile0: int = 0, tile1: int = 0, normals: bool = True) -> None:
        c = cfg.to_c()
        flags = (1 if graph else 0) | (0 if normals else 2)
        check(self.lib.bt_render_frame(self.ctx, C.byref(cam), C.byref(c), tile0, tile1, int(exact), flags),
              "bt_render_frame")

    def download_gbuffer(self, out: GBuffer | None = None) -> GBuffer:
        s = self.scene
        w, h = int(self._view().width), int(self._view().height)
        g = out if out is not None else GBuffer.empty(w, h)
        check(self.lib.bt_gbuffer_download(self.ctx, ptr(g.hit), ptr(g.depth), ptr(g.normal), ptr(g.evalCount),
                                           ptr(g.tileMaxOverlap), ptr(g.tileCacheBytes), ptr(g.tileError)),
              "bt_gbuffer_download")
        return g

    def upload_gbuffer(self, cam: bt_camera, hit: np.ndarray, depth: np.ndarray) -> None:
        hit = np.ascontiguousarray(hit, np.uint8)
        depth = np.ascontiguousarray(depth, np.float32)
        check(self.lib.bt_gbuffer_upload(self.ctx, C.byref(cam), ptr(hit), ptr(depth)), "bt_gbuffer_upload")

    def _view(self) -> capi.bt_gbuffer_view:
        v = capi.bt_gbuffer_view()
        check(self.lib.bt_gbuffer_device(self.ctx, C.byref(v)), "bt_gbuffer_device")
        return v

    def gbuffer_device(self) -> capi.bt_gbuffer_view:
        return self._view()

    def stats(self) -> bt_stats:
        s = bt_stats()
        check(self.lib.bt_stats_download(self.ctx, C.byref(s)), "bt_stats_download")
        return s

    def reset_stats(self) -> None:
        check(self.lib.bt_stats_reset(self.ctx), "bt_stats_reset")

    def profile(self, on: bool) -> None:
        check(self.lib.bt_profile_enable(self.ctx, int(on)), "bt_profile_enable")

    def profile_read(self) -> tuple[np.ndarray, np.ndarray]:
        ms = np.zeros(4, np.float32)
        n = np.zeros(4, np.uint32)
        check(self.lib.bt_profile_read(self.ctx, ptr(ms), ptr(n)), "bt_profile_read")
        return ms, n

    def profile_read_ex(self) -> tuple[np.ndarray, np.ndarray]:
        """[roi_voi, abuffer, trace, normals, views, march] device ms and launch counts."""
        ms = np.zeros(6, np.float32)
        n = np.zeros(6, np.uint32)
        check(self.lib.bt_profile_read_ex(self.ctx, ptr(ms), ptr(n), 6), "bt_profile_read_ex")
        return ms, n
