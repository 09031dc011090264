"""ctypes access to the CPU checkers (TEST INFRASTRUCTURE ONLY).

* oracle/_ref/libbt_ref.so  -- the unmodified reference library compiled from
  /root/reference/proj/src with -Dblobtree=blobtree_ref (oracle/Makefile),
  plus oracle/ref_bridge.cpp and the shared scene recipes.
* oracle/_port/libbt_port.so -- the C restatement (oracle/port/bt_port.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load these.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from paper_2304_09673_b200.pipeline import FRAG_DTYPE, NODE_DTYPE, VOI_DTYPE, GBuffer, RenderConfig, ptr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libbt_ref.so")
PORT_LIB = os.path.join(ROOT, "oracle", "_port", "libbt_port.so")

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_LIB)
        vp = C.c_void_p
        lib.ref_scene_new.argtypes = [C.c_char_p, C.c_uint32, C.c_int, C.c_int]
        lib.ref_scene_new.restype = vp
        lib.ref_scene_error.restype = C.c_char_p
        lib.ref_error.restype = C.c_char_p
        lib.ref_scene_free.argtypes = [vp]
        lib.ref_scene_info.argtypes = [vp] + [vp] * 6
        lib.ref_scene_tree.argtypes = [vp, vp, vp, vp]
        lib.ref_scene_camera.argtypes = [vp, vp]
        lib.ref_scene_perturb.argtypes = [vp, C.c_uint32, vp, vp, vp]
        lib.ref_scene_set_camera.argtypes = [vp, vp]
        lib.ref_scene_perturb.restype = C.c_uint32
        lib.ref_roi.argtypes = [vp, vp]
        lib.ref_vois.argtypes = [vp, C.c_float, vp]
        lib.ref_rasterize.argtypes = [vp, vp, C.c_uint32, vp, vp, C.c_uint64, vp, vp]
        lib.ref_render_tiles.argtypes = [vp, vp, C.c_uint32, vp, vp, C.c_int] + [vp] * 9
        lib.ref_frame.argtypes = [vp, vp, C.c_uint32] + [vp] * 10
        lib.ref_oracle.argtypes = [vp, vp, C.c_uint32, vp, vp, vp, vp]
        lib.ref_compare.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp, C.c_float, vp]
        lib.ref_eval_primitive_raw.argtypes = [C.c_uint8, vp, C.c_float, C.c_float, C.c_float]
        lib.ref_eval_primitive_raw.restype = C.c_float
        lib.ref_eval_operator_raw.argtypes = [C.c_uint8, vp, C.c_float, C.c_float]
        lib.ref_eval_operator_raw.restype = C.c_float
        lib.ref_eval_full.argtypes = [vp, C.c_float, C.c_float, C.c_float]
        lib.ref_eval_full.restype = C.c_float
        _ref = lib
    return _ref


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("reference: " + ref_lib().ref_error().decode())


@dataclass
class RefStats:
    fieldEvals: int
    retainedNodeVisits: int
    primitiveEvals: int
    treeNodeCount: int
    maxOverlap: int
    maxCacheBytes: int


class RefScene:
    """The same scene recipe built through the REFERENCE C++ API."""

    def __init__(self, name: str, seed: int = 0, width: int = 0, height: int = 0):
        lib = ref_lib()
        self.h = lib.ref_scene_new(name.encode(), seed, width, height)
        if not self.h:
            raise ValueError(lib.ref_scene_error().decode())
        nw, nn, npr, rw, w, hh = (C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_int32(), C.c_int32())
        lib.ref_scene_info(self.h, C.byref(nw), C.byref(nn), C.byref(npr), C.byref(rw), C.byref(w), C.byref(hh))
        self.nwords, self.nnodes, self.nprims = nw.value, nn.value, npr.value
        self.width, self.height = w.value, hh.value
        self.root_word = rw.value

    def tree(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        data = np.zeros(self.nwords * 4, np.float32)
        nodes = np.zeros(self.nnodes, NODE_DTYPE)
        prims = np.zeros(self.nprims, np.uint32)
        ref_lib().ref_scene_tree(self.h, ptr(data), ptr(nodes), ptr(prims))
        return data, nodes, prims

    def set_camera(self, camera14) -> None:
        v = np.ascontiguousarray(camera14, np.float32)
        if ref_lib().ref_scene_set_camera(self.h, ptr(v)) != 0:
            raise ValueError(ref_lib().ref_scene_error().decode())
        self.width, self.height = int(v[12]), int(v[13])

    def camera14(self) -> np.ndarray:
        c = np.zeros(14, np.float32)
        ref_lib().ref_scene_camera(self.h, ptr(c))
        return c

    @property
    def tiles(self) -> tuple[int, int]:
        return (self.width + 7) // 8, (self.height + 7) // 8

    def perturb(self, frame: int) -> None:
        ref_lib().ref_scene_perturb(self.h, frame, None, None, None)

    def roi(self) -> np.ndarray:
        out = np.zeros(self.nnodes, np.float32)
        _check(ref_lib().ref_roi(self.h, ptr(out)))
        return out

    def vois(self, margin: float) -> np.ndarray:
        out = np.zeros(self.nprims, VOI_DTYPE)
        _check(ref_lib().ref_vois(self.h, C.c_float(margin), ptr(out)))
        return out

    def rasterize(self, vois: np.ndarray) -> tuple[np.ndarray, np.ndarray, float]:
        vois = np.ascontiguousarray(vois, VOI_DTYPE)
        tx, ty = self.tiles
        offsets = np.zeros(tx * ty + 1, np.uint32)
        total = C.c_uint64()
        ms = C.c_double()
        _check(ref_lib().ref_rasterize(self.h, ptr(vois), len(vois), ptr(offsets), None, 0, C.byref(total),
                                       C.byref(ms)))
        frags = np.zeros(total.value, FRAG_DTYPE)
        _check(ref_lib().ref_rasterize(self.h, ptr(vois), len(vois), ptr(offsets), ptr(frags), total.value,
                                       C.byref(total), C.byref(ms)))
        return offsets, frags, ms.value

    def render_tiles(self, cfg: RenderConfig, offsets: np.ndarray, frags: np.ndarray, threads: int = 0,
                     normals: bool = True) -> tuple[GBuffer, RefStats, np.ndarray]:
        g = GBuffer.empty(self.width, self.height)
        st = np.zeros(6, np.uint64)
        ms = np.zeros(2, np.float64)
        c = cfg.to_c()
        offsets = np.ascontiguousarray(offsets, np.uint32)
        frags = np.ascontiguousarray(frags, FRAG_DTYPE)
        _check(ref_lib().ref_render_tiles(self.h, C.byref(c), threads, ptr(offsets), ptr(frags), int(normals), ptr(g.hit),
                                          ptr(g.depth), ptr(g.normal), ptr(g.evalCount), ptr(g.tileMaxOverlap),
                                          ptr(g.tileCacheBytes), ptr(g.tileError), ptr(st), ptr(ms)))
        return g, RefStats(*[int(v) for v in st]), ms

    def frame(self, cfg: RenderConfig, threads: int = 0) -> tuple[GBuffer, RefStats, np.ndarray, int]:
        g = GBuffer.empty(self.width, self.height)
        st = np.zeros(6, np.uint64)
        ms = np.zeros(4, np.float64)
        nf = C.c_uint64()
        c = cfg.to_c()
        _check(ref_lib().ref_frame(self.h, C.byref(c), threads, ptr(g.hit), ptr(g.depth), ptr(g.normal),
                                   ptr(g.evalCount), ptr(g.tileMaxOverlap), ptr(g.tileCacheBytes), ptr(g.tileError),
                                   ptr(st), ptr(ms), C.byref(nf)))
        return g, RefStats(*[int(v) for v in st]), ms, nf.value

    def oracle(self, cfg: RenderConfig, threads: int = 0) -> tuple[GBuffer, RefStats]:
        g = GBuffer.empty(self.width, self.height)
        st = np.zeros(6, np.uint64)
        c = cfg.to_c()
        _check(ref_lib().ref_oracle(self.h, C.byref(c), threads, ptr(g.hit), ptr(g.depth), ptr(g.evalCount),
                                    ptr(st)))
        return g, RefStats(*[int(v) for v in st])

    def eval_full(self, p) -> float:
        return ref_lib().ref_eval_full(self.h, *[C.c_float(float(v)) for v in p])

    def close(self):
        if self.h:
            ref_lib().ref_scene_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def compare_gbuffers(a: GBuffer, b: GBuffer, tol: float) -> dict:
    """compare_gbuffers of the reference (image_io.cpp:175-209)."""
    out = np.zeros(5, np.float64)
    ref_lib().ref_compare(a.width, a.height, ptr(a.hit), ptr(a.depth), ptr(b.hit), ptr(b.depth), C.c_float(tol),
                          ptr(out))
    return {"hitAgreement": out[0], "depthRms": out[1], "depthMax": out[2], "depthOutliers": int(out[3]),
            "hitMismatches": int(out[4])}


# ---------------------------------------------------------------------------
# C restatement (oracle/port/bt_port.c)

_port = None


class port_tree(C.Structure):
    _fields_ = [("data", C.c_void_p), ("nwords", C.c_uint32), ("nodes", C.c_void_p), ("nnodes", C.c_uint32),
                ("prims", C.c_void_p), ("nprims", C.c_uint32)]


def port_available() -> bool:
    return os.path.exists(PORT_LIB)


def port_lib() -> C.CDLL:
    global _port
    if _port is None:
        lib = C.CDLL(PORT_LIB)
        vp = C.c_void_p
        T = C.POINTER(port_tree)
        lib.port_roi.argtypes = [T, vp]
        lib.port_vois.argtypes = [T, vp, C.c_float, vp]
        lib.port_rasterize.argtypes = [vp, C.c_uint32, vp, vp, vp, C.c_uint64, vp]
        lib.port_render_tiles.argtypes = [T, vp, vp, vp, vp, C.c_int] + [vp] * 7
        lib.port_normals.argtypes = [T, vp, C.c_int, vp, vp, vp]
        lib.port_oracle.argtypes = [T, vp, vp, C.c_int, vp, vp, vp, vp]
        lib.port_eval_primitive.argtypes = [C.c_uint32, vp, C.c_float, C.c_float, C.c_float]
        lib.port_eval_primitive.restype = C.c_float
        lib.port_eval_operator.argtypes = [C.c_uint32, vp, C.c_float, C.c_float]
        lib.port_eval_operator.restype = C.c_float
        lib.port_eval_full.argtypes = [T, C.c_float, C.c_float, C.c_float]
        lib.port_eval_full.restype = C.c_float
        _port = lib
    return _port


class Port:
    """The C restatement driven with a scene's compiled arrays."""

    def __init__(self, data: np.ndarray, nodes: np.ndarray, prims: np.ndarray, device_camera, width: int,
                 height: int):
        self.data, self.nodes, self.prims = data, nodes, prims  # keep alive
        self.t = port_tree(data.ctypes.data, len(data) // 4, nodes.ctypes.data, len(nodes), prims.ctypes.data,
                           len(prims))
        self.cam = device_camera
        self.width, self.height = width, height

    @classmethod
    def from_scene(cls, scene) -> "Port":
        return cls(scene.data.copy(), scene.nodes.copy(), scene.prims.copy(), scene.device_camera, scene.width,
                   scene.height)

    def roi(self) -> np.ndarray:
        out = np.zeros(len(self.nodes), np.float32)
        port_lib().port_roi(C.byref(self.t), ptr(out))
        return out

    def vois(self, margin: float) -> np.ndarray:
        out = np.zeros(len(self.prims), VOI_DTYPE)
        roi = self.roi()
        port_lib().port_vois(C.byref(self.t), ptr(roi), C.c_float(margin), ptr(out))
        return out

    def rasterize(self, vois: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        vois = np.ascontiguousarray(vois, VOI_DTYPE)
        tx, ty = (self.width + 7) // 8, (self.height + 7) // 8
        offsets = np.zeros(tx * ty + 1, np.uint32)
        total = C.c_uint64()
        port_lib().port_rasterize(ptr(vois), len(vois), C.byref(self.cam), ptr(offsets), None, 0, C.byref(total))
        frags = np.zeros(total.value, FRAG_DTYPE)
        port_lib().port_rasterize(ptr(vois), len(vois), C.byref(self.cam), ptr(offsets), ptr(frags), total.value,
                                  C.byref(total))
        return offsets, frags

    def render_tiles(self, cfg: RenderConfig, offsets, frags, threads: int = 1) -> tuple[GBuffer, np.ndarray]:
        g = GBuffer.empty(self.width, self.height)
        st = np.zeros(6, np.uint64)
        c = cfg.to_c()
        offsets = np.ascontiguousarray(offsets, np.uint32)
        frags = np.ascontiguousarray(frags, FRAG_DTYPE)
        port_lib().port_render_tiles(C.byref(self.t), C.byref(self.cam), C.byref(c), ptr(offsets), ptr(frags),
                                     threads, ptr(g.hit), ptr(g.depth),
                                     ptr(g.evalCount), ptr(g.tileMaxOverlap), ptr(g.tileCacheBytes),
                                     ptr(g.tileError), ptr(st))
        return g, st

    def normals(self, g: GBuffer, mode: int = 0) -> None:
        port_lib().port_normals(C.byref(self.t), C.byref(self.cam), mode, ptr(g.hit), ptr(g.depth), ptr(g.normal))

    def frame(self, cfg: RenderConfig, threads: int = 1) -> tuple[GBuffer, np.ndarray, np.ndarray, np.ndarray]:
        v = self.vois(cfg.hitEpsilon)
        off, fr = self.rasterize(v)
        g, st = self.render_tiles(cfg, off, fr, threads)
        self.normals(g, cfg.normalsMode)
        return g, st, off, fr

    def oracle(self, cfg: RenderConfig, threads: int = 1) -> tuple[GBuffer, np.ndarray]:
        g = GBuffer.empty(self.width, self.height)
        st = np.zeros(6, np.uint64)
        c = cfg.to_c()
        port_lib().port_oracle(C.byref(self.t), C.byref(self.cam), C.byref(c), threads, ptr(g.hit), ptr(g.depth),
                               ptr(g.evalCount), ptr(st))
        return g, st
