"""ctypes wrapper of oracle/brute.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from . import geometry

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "brute.c")
LIB = os.path.join(HERE, "_brute.so")

# drop threshold tau = TAU_FACTOR * min spacing (reading 4)
TAU_FACTOR = 1e-9

_lock = threading.Lock()
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile oracle/brute.c with gcc (-O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class OracleGrid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64 * 3), ("d", ctypes.c_double * 3),
                ("x_lo", ctypes.c_double), ("y_hi", ctypes.c_double), ("z_hi", ctypes.c_double)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build_oracle()
            lib = ctypes.CDLL(LIB)
            P = ctypes.POINTER
            dp = P(ctypes.c_double)
            ip = P(ctypes.c_int64)
            g = P(OracleGrid)
            for name, extra in (("oracle_count", [ip]), ("oracle_fill", [ip, ip, dp]),
                                ("oracle_forward", [P(ctypes.c_float), dp]),
                                ("oracle_adjoint", [dp, dp])):
                fn = getattr(lib, name)
                fn.restype = ctypes.c_int
                fn.argtypes = [g, ctypes.c_int64, dp, dp, ctypes.c_double, ctypes.c_int] + extra
            lib.oracle_threads.restype = ctypes.c_int
            lib.oracle_set_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def threads() -> int:
    return _load().oracle_threads()


def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def grid_of(c: dict) -> OracleGrid:
    x_lo, y_hi, z_hi = geometry.grid_bounds(c)
    g = OracleGrid()
    for a in range(3):
        g.n[a] = int(c["n"][a])
        g.d[a] = float(c["spacing"][a])
    g.x_lo, g.y_hi, g.z_hi = x_lo, y_hi, z_hi
    return g


def _tau(c):
    return TAU_FACTOR * min(c["spacing"])


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def _prep(c, p, th):
    p = np.ascontiguousarray(p, dtype=np.float64).reshape(-1, 3)
    th = np.ascontiguousarray(th, dtype=np.float64).reshape(-1, 3)
    return p, th


def rows(c: dict, p, th, mode: int = 1):
    """CSR (row_ptr int64[n+1], cols int64[nnz], lens f64[nnz]); rows ascending in flat index."""
    lib = _load()
    p, th = _prep(c, p, th)
    n = p.shape[0]
    g = grid_of(c)
    counts = np.zeros(n, dtype=np.int64)
    if lib.oracle_count(ctypes.byref(g), n, _ptr(p, ctypes.c_double), _ptr(th, ctypes.c_double),
                        _tau(c), mode, _ptr(counts, ctypes.c_int64)) != 0:
        raise MemoryError("oracle_count")
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    cols = np.zeros(max(nnz, 1), dtype=np.int64)
    lens = np.zeros(max(nnz, 1), dtype=np.float64)
    if lib.oracle_fill(ctypes.byref(g), n, _ptr(p, ctypes.c_double), _ptr(th, ctypes.c_double),
                       _tau(c), mode, _ptr(row_ptr, ctypes.c_int64), _ptr(cols, ctypes.c_int64),
                       _ptr(lens, ctypes.c_double)) != 0:
        raise MemoryError("oracle_fill")
    return row_ptr, cols[:nnz], lens[:nnz]


def forward(c: dict, img, p, th, mode: int = 1) -> np.ndarray:
    """fp64 sum_I f_I l_I per ray; ``img`` is the fp32 image in flat-index order."""
    lib = _load()
    p, th = _prep(c, p, th)
    f = np.ascontiguousarray(np.asarray(img, dtype=np.float32).reshape(-1))
    assert f.size == int(np.prod(c["n"]))
    out = np.zeros(p.shape[0], dtype=np.float64)
    g = grid_of(c)
    if lib.oracle_forward(ctypes.byref(g), p.shape[0], _ptr(p, ctypes.c_double), _ptr(th, ctypes.c_double),
                          _tau(c), mode, _ptr(f, ctypes.c_float), _ptr(out, ctypes.c_double)) != 0:
        raise MemoryError("oracle_forward")
    return out


def adjoint(c: dict, y, p, th, mode: int = 1) -> np.ndarray:
    """fp64 A^T y over the given rays only (flat-index image of size N_x N_y N_z)."""
    lib = _load()
    p, th = _prep(c, p, th)
    yy = np.ascontiguousarray(np.asarray(y, dtype=np.float64).reshape(-1))
    assert yy.size == p.shape[0]
    img = np.zeros(int(np.prod(c["n"])), dtype=np.float64)
    g = grid_of(c)
    if lib.oracle_adjoint(ctypes.byref(g), p.shape[0], _ptr(p, ctypes.c_double), _ptr(th, ctypes.c_double),
                          _tau(c), mode, _ptr(yy, ctypes.c_double), _ptr(img, ctypes.c_double)) != 0:
        raise MemoryError("oracle_adjoint")
    return img
