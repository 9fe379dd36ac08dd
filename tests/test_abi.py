"""The C-ABI library builds, loads and exports every symbol include/fdgs.h
declares; argument checks that need no GPU (-m "not gpu")."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fdgs.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fdgs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2503_16422_b200 import build
    build.build_lib()
    from paper_2503_16422_b200 import _lib
    return _lib.lib()


def test_every_declared_symbol_is_exported(lib):
    from paper_2503_16422_b200 import _lib
    declared = _declared()
    assert len(declared) >= 15
    assert sorted(_lib.EXPORTS) == declared
    so = os.path.join(ROOT, "paper_2503_16422_b200", "libfdgs.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (fdgs_[a-z0-9_]+)$", out, flags=re.M))
    assert set(declared) <= exported
    for name in declared:
        assert getattr(lib, name) is not None


def test_library_is_sm100a(lib):
    so = os.path.join(ROOT, "paper_2503_16422_b200", "libfdgs.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(lib):
    from paper_2503_16422_b200 import _lib as _lib_mod
    assert lib.fdgs_abi_version() == 2 == _lib_mod.ABI_VERSION
    assert lib.fdgs_status_string(0) == b"ok"
    assert lib.fdgs_status_string(4) == b"tile-entry capacity exceeded"


def test_host_side_argument_errors_without_gpu(lib):
    from paper_2503_16422_b200 import _lib
    cam = _lib.FdgsCamera()
    cam.width = cam.height = 64
    cam.fx = cam.fy = 64.0
    # NULL scene -> INVALID_ARG before any CUDA call
    st = lib.fdgs_render(None, None, None, C.byref(cam), 0.0, None, None, None, 0, 0, None, None)
    assert st == _lib.FDGS_ERR_INVALID_ARG
    assert b"scene" in lib.fdgs_last_error()
    sc = _lib.FdgsScene()
    sc.n = 0
    # bad camera (R = 0 is not a rotation)
    out = C.c_float()
    st = lib.fdgs_render(C.byref(sc), None, None, C.byref(cam), 0.0, C.byref(out), None, None, 0, 0, None, None)
    assert st == _lib.FDGS_ERR_INVALID_ARG and b"camera" in lib.fdgs_last_error()
    # stv score: NULL scene / opts / cameras and a bad percentile fail on the host
    assert lib.fdgs_stv_score(None, None, 0, None, 0, None, None, None, None, None, 0, None, None) == \
        _lib.FDGS_ERR_INVALID_ARG
    cams = (_lib.FdgsCamera * 1)(cam)
    opts = _lib.FdgsStvOpts(1.5, 0, 0, 1024)
    ts = (C.c_float * 1)(0.5)
    st = lib.fdgs_stv_score(C.byref(sc), cams, 1, ts, 1, C.byref(opts), None, None, None, None, 0, None, None)
    assert st == _lib.FDGS_ERR_INVALID_ARG and b"percentile" in lib.fdgs_last_error()
    opts = _lib.FdgsStvOpts(0.9, 7, 0, 1024)
    st = lib.fdgs_stv_score(C.byref(sc), cams, 1, ts, 1, C.byref(opts), None, None, None, None, 0, None, None)
    assert st == _lib.FDGS_ERR_INVALID_ARG and b"combine" in lib.fdgs_last_error()
    opts = _lib.FdgsStvOpts(0.9, 0, 5, 1024)
    st = lib.fdgs_stv_score(C.byref(sc), cams, 1, ts, 1, C.byref(opts), None, None, None, None, 0, None, None)
    assert st == _lib.FDGS_ERR_INVALID_ARG and b"variant" in lib.fdgs_last_error()


def test_workspace_sizes(lib):
    from paper_2503_16422_b200 import _lib
    a = lib.fdgs_render_workspace_bytes(200_000, 1352, 1014, 12_800_000)
    b = lib.fdgs_render_workspace_bytes(200_000, 1352, 1014, 25_600_000)
    assert a > 200_000 * 48 and b - a >= 4 * 12_800_000
    assert lib.fdgs_render_workspace_bytes(-1, 10, 10, 0) == 0
    assert lib.fdgs_mask_compact_workspace_bytes(1000) >= 4 * (32 + 4)
    cam = _lib.FdgsCamera()
    cam.width, cam.height = 1352, 1014
    cams = (_lib.FdgsCamera * 2)(cam, cam)
    s1 = lib.fdgs_stv_workspace_bytes(200_000, cams, 2, 12_800_000)
    assert s1 >= lib.fdgs_render_workspace_bytes(200_000, 1352, 1014, 12_800_000) + 4 * 8 * 200_000
    assert lib.fdgs_stv_workspace_bytes(10, None, 0, 0) == 0


def test_graph_entry_points_host_errors(lib):
    from paper_2503_16422_b200 import _lib
    h = C.c_void_p()
    assert lib.fdgs_render_graph_create(None, 64, 64, None, 0, 0, C.byref(h)) == _lib.FDGS_ERR_INVALID_ARG
    assert lib.fdgs_render_graph_launch(None, None, None, None, None, 0.0, None, None, None) == \
        _lib.FDGS_ERR_INVALID_ARG
    assert lib.fdgs_render_graph_destroy(None) == _lib.FDGS_OK
