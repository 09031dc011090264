"""The C-ABI boundary: the library builds for sm_100a, loads, exports every
symbol include/bt_cuda.h declares, keeps the reference's struct layouts, and
fails loudly (no CPU fallback) when there is no GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2304_09673_b200 import _capi as capi
from paper_2304_09673_b200.pipeline import FRAG_DTYPE, NODE_DTYPE, VOI_DTYPE

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bt_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"BT_API\s+[\w\s\*]+?\b(bt_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("bt_ctx_create", "bt_tree_upload", "bt_params_update", "bt_roi", "bt_voi_build",
                 "bt_abuffer_build", "bt_trace", "bt_normals", "bt_oracle_render", "bt_render_frame",
                 "bt_gbuffer_download", "bt_stats_download"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bt_\w+)", out))
    missing = [n for n in declared_symbols() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    for n in declared_symbols():
        getattr(lib, n)
    assert set(capi.exported_symbols()) >= set(declared_symbols())


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_the_reference():
    # NodeRecord 20 B, VolumeOfInterest 64 B, Fragment 12 B (linear_tree.hpp, abuffer.hpp)
    assert NODE_DTYPE.itemsize == 20 and C.sizeof(capi.bt_node) == 20
    assert VOI_DTYPE.itemsize == 64 and C.sizeof(capi.bt_voi) == 64
    assert FRAG_DTYPE.itemsize == 12 and C.sizeof(capi.bt_fragment) == 12
    assert capi.bt_voi.center.offset == 8 and capi.bt_voi.rotation.offset == 36
    assert C.sizeof(capi.bt_camera) == 80
    assert C.sizeof(capi.bt_render_config) == 36


def test_scene_library_exports():
    out = subprocess.run(["nm", "-D", "--defined-only", capi.SCENES_PATH], capture_output=True, text=True).stdout
    for n in ("sc_scene_new", "sc_scene_tree", "sc_scene_perturb", "sc_scene_device_camera"):
        assert n in out


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    lib = capi.load()
    ctx = C.c_void_p()
    rc = lib.bt_ctx_create(0, C.byref(ctx))
    assert rc == 2  # BT_ECUDA
    assert b"CUDA" in lib.bt_last_error()
    from paper_2304_09673_b200.pipeline import Renderer
    with pytest.raises(capi.BtError):
        Renderer(0)


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(capi, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(capi, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        capi.load()
