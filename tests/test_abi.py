"""CPU-side checks of the boundary: libxrt.so builds, loads and exports every symbol that
include/xrt.h declares; argument validation answers without touching a GPU."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2006_00686_b200 as xrt
from paper_2006_00686_b200 import _lib, build
from paper_2006_00686_b200.plan import _geometry_struct


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "xrt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xrt_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 12
    assert sorted(_lib.EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n


def test_version(lib):
    assert xrt.version() == (0, 1)


def test_struct_layout_matches_header(lib):
    # offsets of the C struct as the compiler lays it out (x86-64 SysV): check a few anchors
    assert ctypes.sizeof(_lib.XrtGeometry) == 4 + 4 + 24 + 24 + 24 + 8 + 8 + 8 + 8 + 16 + 16 + 8 * 5
    assert _lib.XrtGeometry.angles.offset == 88


def _geom(**kw):
    g = dict(beam="cone", n=(8, 8, 8), spacing=(1, 1, 1), center=(0, 0, 0), angles=np.zeros(3),
             det_cols=4, det_rows=4, det_spacing=(1, 1), det_offset=(0, 0), sod=10.0, sdd=20.0)
    g.update(kw)
    return g


@pytest.mark.parametrize("bad", [
    dict(n=(0, 8, 8)), dict(spacing=(1, -1, 1)), dict(spacing=(1, math.nan, 1)), dict(angles=np.zeros(0)),
    dict(angles=np.array([math.inf])), dict(det_cols=0), dict(det_spacing=(0, 1)), dict(sod=0.0),
    dict(sdd=5.0), dict(beam="par2d", n=(8, 8, 2), det_rows=1), dict(beam="fan2d", n=(8, 8, 1), det_rows=3),
    dict(beam="par3d", tilt=2.0), dict(center=(0, math.inf, 0)),
    dict(beam="par3d", det_curved=True), dict(det_curved=True, det_cols=200, det_spacing=(1, 1)),
])
def test_invalid_geometry_rejected(lib, bad):
    s, keep = _geometry_struct(_geom(**bad))
    h = ctypes.c_void_p()
    st = lib.xrt_plan_create(ctypes.byref(s), 0, ctypes.byref(h))
    assert st == _lib.XRT_ERR_INVALID_ARG
    assert h.value is None
    assert lib.xrt_last_error()


def test_unknown_flags_rejected(lib):
    s, keep = _geometry_struct(_geom())
    s.flags = 6
    h = ctypes.c_void_p()
    assert lib.xrt_plan_create(ctypes.byref(s), 0, ctypes.byref(h)) == _lib.XRT_ERR_INVALID_ARG
    assert b"flags" in lib.xrt_last_error()


def test_null_arguments(lib):
    h = ctypes.c_void_p()
    assert lib.xrt_plan_create(None, 0, ctypes.byref(h)) == _lib.XRT_ERR_INVALID_ARG
    assert lib.xrt_forward(None, None, None, None) == _lib.XRT_ERR_INVALID_ARG
    assert lib.xrt_plan_destroy(None) == _lib.XRT_OK
    assert lib.xrt_plan_launch_count(None) == -1


@pytest.mark.parametrize("bad", [dict(dim=4), dict(n_rays=0), dict(nan=True), dict(flags=1), dict(n=(0, 4, 4))])
def test_ray_list_rejected(lib, bad):
    """xrt_plan_create_rays validates before touching a device."""
    r = _lib.XrtRayList()
    r.dim = bad.get("dim", 3)
    r.flags = bad.get("flags", 0)
    for a in range(3):
        r.n[a] = bad.get("n", (4, 4, 4))[a]
        r.spacing[a] = 1.0
        r.center[a] = 0.0
    params = np.zeros((2, 4))
    if bad.get("nan"):
        params[1, 2] = math.nan
    r.n_rays = bad.get("n_rays", 2)
    r.params = params.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    h = ctypes.c_void_p()
    assert lib.xrt_plan_create_rays(ctypes.byref(r), 0, ctypes.byref(h)) == _lib.XRT_ERR_INVALID_ARG
    assert h.value is None
