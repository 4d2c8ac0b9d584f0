"""Thin Python binding of the C ABI (include/xrt.h): same names, argument marshalling only.

Every step of the X-ray transform runs in libxrt.so's CUDA kernels; torch provides
device memory and streams.  Geometry dicts use the field names of ``xrt_geometry``
(see ``workloads/configs.py`` for the five BASELINE configurations).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check


def _geometry_struct(g: dict) -> tuple[_lib.XrtGeometry, np.ndarray]:
    angles = np.ascontiguousarray(np.asarray(g["angles"], dtype=np.float64))
    s = _lib.XrtGeometry()
    s.beam = _lib.BEAMS[g["beam"]] if isinstance(g["beam"], str) else int(g["beam"])
    s.flags = _lib.DET_CURVED if g.get("det_curved", False) else 0
    for a in range(3):
        s.n[a] = int(g["n"][a])
        s.spacing[a] = float(g["spacing"][a])
        s.center[a] = float(g.get("center", (0.0, 0.0, 0.0))[a])
    s.n_views = int(angles.shape[0])
    s.angles = angles.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    s.det_cols = int(g["det_cols"])
    s.det_rows = int(g.get("det_rows", 1))
    for a in range(2):
        s.det_spacing[a] = float(g["det_spacing"][a])
        s.det_offset[a] = float(g.get("det_offset", (0.0, 0.0))[a])
    s.sod = float(g.get("sod", 0.0))
    s.sdd = float(g.get("sdd", 0.0))
    s.pitch = float(g.get("pitch", 0.0))
    s.z0 = float(g.get("z0", 0.0))
    s.tilt = float(g.get("tilt", 0.0))
    return s, angles


def _ray_list_struct(g: dict):
    """xrt_ray_list of a {"beam": "rays", "dim": 2|3, "n", "spacing", "center", "ray_params"} dict;
    ray_params [n_rays][4]: (s, phi, 0, 0) in 2D, (s1, s2, phi1, phi2) in 3D."""
    params = np.ascontiguousarray(np.asarray(g["ray_params"], dtype=np.float64).reshape(-1, 4))
    r = _lib.XrtRayList()
    r.dim = int(g["dim"])
    r.flags = 0
    for a in range(3):
        r.n[a] = int(g["n"][a])
        r.spacing[a] = float(g["spacing"][a])
        r.center[a] = float(g.get("center", (0.0, 0.0, 0.0))[a])
    r.n_rays = int(params.shape[0])
    r.params = params.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    return r, params


def _stream_handle(stream, device: int) -> int:
    """The raw cudaStream_t of ``stream`` (default: the current torch stream of the plan's device)."""
    if stream is None:
        stream = torch.cuda.current_stream(device)
    elif stream.device.index != device:
        raise ValueError(f"stream is on cuda:{stream.device.index}, plan on cuda:{device}")
    return int(stream.cuda_stream)


class Plan:
    """xrt_plan: a validated acquisition geometry with its device tables on one GPU."""

    def __init__(self, geometry: dict, device: int | None = None):
        lib = _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.geometry = dict(geometry)
        h = ctypes.c_void_p()
        if geometry.get("beam") == "rays":
            # explicit ray list: xrt_plan_create_rays (Remark 3.5)
            r, self._angles = _ray_list_struct(geometry)
            check(lib.xrt_plan_create_rays(ctypes.byref(r), self.device, ctypes.byref(h)))
            s, _ = _geometry_struct(dict(geometry, beam="par2d" if r.dim == 2 else "par3d",
                                         angles=np.zeros(1), det_cols=r.n_rays, det_rows=1,
                                         det_spacing=(1.0, 1.0)))
        else:
            s, self._angles = _geometry_struct(geometry)
            check(lib.xrt_plan_create(ctypes.byref(s), self.device, ctypes.byref(h)))
        self._h = h
        self._lib = lib
        n = ctypes.c_int64()
        check(lib.xrt_plan_query(h, ctypes.byref(n), None))
        self.n_rays = int(n.value)
        self.n_views = int(s.n_views)
        self.det_rows, self.det_cols = int(s.det_rows), int(s.det_cols)
        is2d = s.beam in (0, 1)
        self.image_shape = (1 if is2d else int(s.n[2]), int(s.n[1]), int(s.n[0]))
        self.sino_shape = (self.n_views, self.det_rows, self.det_cols)

    # -------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._lib.xrt_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- queries
    @property
    def n_units(self) -> int:
        """Exact nnz of the projection matrix (fp64 enumeration; synchronous, cached)."""
        n = ctypes.c_int64()
        check(self._lib.xrt_plan_query(self._h, None, ctypes.byref(n)))
        return int(n.value)

    @property
    def launch_count(self) -> int:
        return int(self._lib.xrt_plan_launch_count(self._h))

    def set_algorithm(self, op: str, algo: str) -> None:
        o = {"forward": _lib.OP_FORWARD, "adjoint": _lib.OP_ADJOINT}[op]
        check(self._lib.xrt_plan_set_algorithm(self._h, o, _lib.ALGOS[algo]))

    # -------------------------------------------------------------- operators
    def _check_dev(self, t: torch.Tensor, shape, name, dtype=torch.float32):
        if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous {dtype} CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"{name} is on cuda:{t.device.index}, plan on cuda:{self.device}")
        if t.numel() != int(np.prod(shape)):
            raise ValueError(f"{name} has {t.numel()} elements, expected {shape}")

    def forward(self, img: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_forward: sino[m] = sum_I img[I] l_I(ray m)."""
        self._check_dev(img, self.image_shape, "img")
        if out is None:
            out = torch.empty(self.sino_shape, dtype=torch.float32, device=img.device)
        self._check_dev(out, self.sino_shape, "sino")
        check(self._lib.xrt_forward(self._h, img.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def adjoint(self, sino: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_adjoint: img[I] = sum_m sino[m] l_I(ray m)."""
        self._check_dev(sino, self.sino_shape, "sino")
        if out is None:
            out = torch.empty(self.image_shape, dtype=torch.float32, device=sino.device)
        self._check_dev(out, self.image_shape, "img")
        check(self._lib.xrt_adjoint(self._h, sino.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def adjoint_stages(self) -> list[tuple[int, int]]:
        """xrt_adjoint_stages: per stage s, the image rows [k0, k1) final after stage s."""
        n = ctypes.c_int32()
        check(self._lib.xrt_adjoint_stages(self._h, ctypes.byref(n), None, None))
        kb = (ctypes.c_int64 * n.value)()
        ke = (ctypes.c_int64 * n.value)()
        check(self._lib.xrt_adjoint_stages(self._h, ctypes.byref(n), kb, ke))
        return [(int(kb[i]), int(ke[i])) for i in range(n.value)]

    def adjoint_stage(self, sino: torch.Tensor, out: torch.Tensor, stage: int, stream=None) -> torch.Tensor:
        """xrt_adjoint_stage: stage `stage` of the staged adjoint (writes out's final rows of that stage)."""
        self._check_dev(sino, self.sino_shape, "sino")
        self._check_dev(out, self.image_shape, "img")
        check(self._lib.xrt_adjoint_stage(self._h, sino.data_ptr(), out.data_ptr(), int(stage),
                                          _stream_handle(stream, self.device)))
        return out

    def forward64(self, img: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_forward_f64: the same operator in fp64 (P:725's double option)."""
        self._check_dev(img, self.image_shape, "img", torch.float64)
        if out is None:
            out = torch.empty(self.sino_shape, dtype=torch.float64, device=img.device)
        self._check_dev(out, self.sino_shape, "sino", torch.float64)
        check(self._lib.xrt_forward_f64(self._h, img.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def adjoint64(self, sino: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_adjoint_f64."""
        self._check_dev(sino, self.sino_shape, "sino", torch.float64)
        if out is None:
            out = torch.empty(self.image_shape, dtype=torch.float64, device=sino.device)
        self._check_dev(out, self.image_shape, "img", torch.float64)
        check(self._lib.xrt_adjoint_f64(self._h, sino.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def forward_mixed(self, img: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_forward_mixed: fp32 lengths, fp64 products and sums (fp64 buffers)."""
        self._check_dev(img, self.image_shape, "img", torch.float64)
        if out is None:
            out = torch.empty(self.sino_shape, dtype=torch.float64, device=img.device)
        self._check_dev(out, self.sino_shape, "sino", torch.float64)
        check(self._lib.xrt_forward_mixed(self._h, img.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def adjoint_mixed(self, sino: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_adjoint_mixed."""
        self._check_dev(sino, self.sino_shape, "sino", torch.float64)
        if out is None:
            out = torch.empty(self.image_shape, dtype=torch.float64, device=sino.device)
        self._check_dev(out, self.image_shape, "img", torch.float64)
        check(self._lib.xrt_adjoint_mixed(self._h, sino.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def forward_attenuated(self, img: torch.Tensor, mu: torch.Tensor, out: torch.Tensor | None = None,
                           stream=None) -> torch.Tensor:
        """xrt_forward_attenuated: sino[m] = sum_I img[I] exp(-A_mI) (1 - exp(-mu_I l_mI)) / mu_I
        (SPECT weight of P:36-40; A_mI = attenuation of the units after I along the ray)."""
        self._check_dev(img, self.image_shape, "img")
        self._check_dev(mu, self.image_shape, "mu")
        if out is None:
            out = torch.empty(self.sino_shape, dtype=torch.float32, device=img.device)
        self._check_dev(out, self.sino_shape, "sino")
        check(self._lib.xrt_forward_attenuated(self._h, img.data_ptr(), mu.data_ptr(), out.data_ptr(),
                                               _stream_handle(stream, self.device)))
        return out

    def adjoint_attenuated(self, sino: torch.Tensor, mu: torch.Tensor, out: torch.Tensor | None = None,
                           stream=None) -> torch.Tensor:
        """xrt_adjoint_attenuated: the transpose of forward_attenuated."""
        self._check_dev(sino, self.sino_shape, "sino")
        self._check_dev(mu, self.image_shape, "mu")
        if out is None:
            out = torch.empty(self.image_shape, dtype=torch.float32, device=sino.device)
        self._check_dev(out, self.image_shape, "img")
        check(self._lib.xrt_adjoint_attenuated(self._h, sino.data_ptr(), mu.data_ptr(), out.data_ptr(),
                                               _stream_handle(stream, self.device)))
        return out

    @staticmethod
    def _check_host(t: torch.Tensor, shape, name):
        """The C side copies exactly prod(shape) floats through the raw pointer: check it all."""
        if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous float32 CPU tensor")
        if t.numel() != int(np.prod(shape)):
            raise ValueError(f"{name} has {t.numel()} elements, expected {shape}")

    def forward_host(self, img: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_forward_host: host (ideally pinned) fp32 buffers, copies inside the call."""
        self._check_host(img, self.image_shape, "img")
        if out is None:
            out = torch.empty(self.sino_shape, dtype=torch.float32, pin_memory=True)
        self._check_host(out, self.sino_shape, "sino")
        check(self._lib.xrt_forward_host(self._h, img.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def adjoint_host(self, sino: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """xrt_adjoint_host: host buffers, copies inside the call."""
        self._check_host(sino, self.sino_shape, "sino")
        if out is None:
            out = torch.empty(self.image_shape, dtype=torch.float32, pin_memory=True)
        self._check_host(out, self.image_shape, "img")
        check(self._lib.xrt_adjoint_host(self._h, sino.data_ptr(), out.data_ptr(), _stream_handle(stream, self.device)))
        return out

    def ray_unit_counts(self, ray_begin: int, ray_end: int, stream=None) -> torch.Tensor:
        """xrt_ray_units count-only (cols = lens = NULL): |index set| of every ray in the range, int64
        CUDA tensor (the fp64 enumeration's drop threshold applies)."""
        n = int(ray_end) - int(ray_begin)
        row_ptr = torch.empty(max(n, 0) + 1, dtype=torch.int64, device=torch.device("cuda", self.device))
        nnz = ctypes.c_int64()
        check(self._lib.xrt_ray_units(self._h, int(ray_begin), int(ray_end), row_ptr.data_ptr(), None, None,
                                      0, ctypes.byref(nnz), _stream_handle(stream, self.device)))
        return row_ptr[1:] - row_ptr[:-1]

    def ray_units(self, ray_begin: int, ray_end: int, stream=None):
        """xrt_ray_units (two-phase): CSR (row_ptr, cols, lens) as CUDA tensors (int64, int64, fp64)."""
        n = int(ray_end) - int(ray_begin)
        dev = torch.device("cuda", self.device)
        row_ptr = torch.empty(max(n, 0) + 1, dtype=torch.int64, device=dev)
        nnz = ctypes.c_int64()
        sh = _stream_handle(stream, self.device)
        check(self._lib.xrt_ray_units(self._h, int(ray_begin), int(ray_end), row_ptr.data_ptr(), None, None,
                                      0, ctypes.byref(nnz), sh))
        cols = torch.empty(max(nnz.value, 1), dtype=torch.int64, device=dev)
        lens = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
        check(self._lib.xrt_ray_units(self._h, int(ray_begin), int(ray_end), row_ptr.data_ptr(), cols.data_ptr(),
                                      lens.data_ptr(), cols.numel(), ctypes.byref(nnz), sh))
        return row_ptr, cols[:nnz.value], lens[:nnz.value]


def version() -> tuple[int, int]:
    v = _lib.load().xrt_version()
    return v >> 16, v & 0xFFFF
