"""The paper's O(N)-per-ray enumeration on the host cores: a fair CPU baseline
beside the brute-force oracle.  Independent of both the product (CUDA) and the oracle; rays are
passed in physical coordinates (p, theta).  Tests pin it to the oracle; bench.py's cpu_baseline leg
reports its throughput next to the oracle's."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "xrt_cpu.c")
LIB = os.path.join(HERE, "_xrt_cpu.so")
_lock = threading.Lock()
_lib = None


class CpuGrid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64 * 3), ("d", ctypes.c_double * 3),
                ("x_lo", ctypes.c_double), ("y_hi", ctypes.c_double), ("z_hi", ctypes.c_double)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(LIB)
            P = ctypes.POINTER
            lib.xrt_cpu_forward.argtypes = [P(CpuGrid), ctypes.c_int64, P(ctypes.c_double), P(ctypes.c_double),
                                            P(ctypes.c_float), ctypes.c_double, P(ctypes.c_double),
                                            P(ctypes.c_int64)]
            lib.xrt_cpu_forward.restype = None
            lib.xrt_cpu_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _grid(c: dict) -> CpuGrid:
    g = CpuGrid()
    nx, ny, nz = c["n"]
    dx, dy, dz = c["spacing"]
    cx, cy, cz = c.get("center", (0.0, 0.0, 0.0))
    for a, (n, d) in enumerate(zip((nx, ny, nz), (dx, dy, dz))):
        g.n[a] = int(n)
        g.d[a] = float(d)
    g.x_lo = cx - nx * dx / 2.0
    g.y_hi = cy + ny * dy / 2.0
    g.z_hi = cz + nz * dz / 2.0
    return g


def forward(c: dict, img, p, th, with_counts: bool = False):
    """fp64 forward of the rays (p, theta) [n, 3] over the fp32 image (flat [N_z*N_y*N_x])."""
    lib = _load()
    P = ctypes.POINTER
    img = np.ascontiguousarray(np.asarray(img, dtype=np.float32).reshape(-1))
    p = np.ascontiguousarray(p, dtype=np.float64)
    th = np.ascontiguousarray(th, dtype=np.float64)
    n = p.shape[0]
    out = np.zeros(n)
    counts = np.zeros(n, dtype=np.int64) if with_counts else None
    g = _grid(c)
    tau = 1e-9 * min(g.d[0], g.d[1], g.d[2])
    lib.xrt_cpu_forward(ctypes.byref(g), n, p.ctypes.data_as(P(ctypes.c_double)),
                        th.ctypes.data_as(P(ctypes.c_double)), img.ctypes.data_as(P(ctypes.c_float)), tau,
                        out.ctypes.data_as(P(ctypes.c_double)),
                        counts.ctypes.data_as(P(ctypes.c_int64)) if with_counts else None)
    return (out, counts) if with_counts else out


def threads() -> int:
    return int(_load().xrt_cpu_threads())
