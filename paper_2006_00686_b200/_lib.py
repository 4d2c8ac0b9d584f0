"""ctypes declarations of include/xrt.h (argument marshalling only).

The native library is ``paper_2006_00686_b200/libxrt.so`` built in-tree by
``paper_2006_00686_b200.build``.  There is no fallback: if the library is missing or
fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libxrt.so")

XRT_OK, XRT_ERR_INVALID_ARG, XRT_ERR_UNSUPPORTED, XRT_ERR_CUDA, XRT_ERR_OOM, XRT_ERR_CAPACITY = range(6)
STATUS_NAMES = {0: "XRT_OK", 1: "XRT_ERR_INVALID_ARG", 2: "XRT_ERR_UNSUPPORTED", 3: "XRT_ERR_CUDA",
                4: "XRT_ERR_OOM", 5: "XRT_ERR_CAPACITY"}
BEAMS = {"par2d": 0, "fan2d": 1, "par3d": 2, "cone": 3, "helical": 4, "rays": 5}
OP_FORWARD, OP_ADJOINT = 0, 1
DET_CURVED = 1
ALGO_AUTO, ALGO_RAY, ALGO_COLUMN, ALGO_GATHER = 0, 1, 2, 3
ALGOS = {"auto": 0, "ray": 1, "column": 2, "gather": 3}

# every symbol include/xrt.h declares (checked by tests/test_abi.py)
EXPORTS = ("xrt_plan_create", "xrt_plan_create_rays", "xrt_plan_destroy", "xrt_plan_query", "xrt_plan_set_algorithm",
           "xrt_plan_launch_count", "xrt_forward", "xrt_adjoint", "xrt_forward_host",
           "xrt_adjoint_host", "xrt_forward_f64", "xrt_adjoint_f64",
           "xrt_forward_mixed", "xrt_adjoint_mixed",
           "xrt_forward_attenuated", "xrt_adjoint_attenuated", "xrt_ray_units", "xrt_last_error", "xrt_version",
           "xrt_adjoint_stages", "xrt_adjoint_stage")


class XrtGeometry(ctypes.Structure):
    _fields_ = [
        ("beam", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("n", ctypes.c_int64 * 3), ("spacing", ctypes.c_double * 3), ("center", ctypes.c_double * 3),
        ("n_views", ctypes.c_int64), ("angles", ctypes.POINTER(ctypes.c_double)),
        ("det_cols", ctypes.c_int64), ("det_rows", ctypes.c_int64),
        ("det_spacing", ctypes.c_double * 2), ("det_offset", ctypes.c_double * 2),
        ("sod", ctypes.c_double), ("sdd", ctypes.c_double),
        ("pitch", ctypes.c_double), ("z0", ctypes.c_double), ("tilt", ctypes.c_double),
    ]


class XrtRayList(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("n", ctypes.c_int64 * 3), ("spacing", ctypes.c_double * 3), ("center", ctypes.c_double * 3),
        ("n_rays", ctypes.c_int64), ("params", ctypes.POINTER(ctypes.c_double)),
    ]


class XrtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lock = threading.Lock()
_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libxrt.so (no fallback: raises if absent).  XRT_LIB overrides the path (A/B builds)."""
    global _lib
    if path is None:
        path = os.environ.get("XRT_LIB", LIB_PATH)
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(f"native library {path} is missing: run `python -m paper_2006_00686_b200.build` "
                               "(there is no CPU or Python fallback)")
        lib = ctypes.CDLL(path)
        vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        sig = {
            "xrt_plan_create": (i32, [ctypes.POINTER(XrtGeometry), ctypes.c_int, ctypes.POINTER(vp)]),
            "xrt_plan_destroy": (i32, [vp]),
            "xrt_plan_create_rays": (i32, [ctypes.POINTER(XrtRayList), ctypes.c_int, ctypes.POINTER(vp)]),
            "xrt_plan_query": (i32, [vp, ip, ip]),
            "xrt_plan_set_algorithm": (i32, [vp, i32, i32]),
            "xrt_plan_launch_count": (i64, [vp]),
            "xrt_forward": (i32, [vp, vp, vp, vp]),
            "xrt_adjoint": (i32, [vp, vp, vp, vp]),
            "xrt_forward_host": (i32, [vp, vp, vp, vp]),
            "xrt_forward_f64": (i32, [vp, vp, vp, vp]),
            "xrt_adjoint_f64": (i32, [vp, vp, vp, vp]),
            "xrt_forward_mixed": (i32, [vp, vp, vp, vp]),
            "xrt_adjoint_mixed": (i32, [vp, vp, vp, vp]),
            "xrt_forward_attenuated": (i32, [vp, vp, vp, vp, vp]),
            "xrt_adjoint_attenuated": (i32, [vp, vp, vp, vp, vp]),
            "xrt_adjoint_host": (i32, [vp, vp, vp, vp]),
            "xrt_ray_units": (i32, [vp, i64, i64, vp, vp, vp, i64, ip, vp]),
            "xrt_last_error": (ctypes.c_char_p, []),
            "xrt_version": (i32, []),
            "xrt_adjoint_stages": (i32, [vp, ctypes.POINTER(i32), ip, ip]),
            "xrt_adjoint_stage": (i32, [vp, vp, vp, i32, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    if status != XRT_OK:
        msg = load().xrt_last_error()
        raise XrtError(status, msg.decode() if msg else "")
