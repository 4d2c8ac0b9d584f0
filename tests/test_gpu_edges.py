"""Rays on grid lines / planes and through corners, on full 3D geometries, through the kernels AUTO
runs (COLUMN for the 3D beams, the slice kernels for the 2D adjoint), against the oracle.

* The tie rule (reading 2: half-open units, the bigger 1D index) is exercised by:
  - par3d on a unit grid with an odd unit-spacing detector: at phi1 in {0, pi/2, pi, 3pi/2} every
    ray lies on an in-plane grid line AND on a z plane (s1, s2 integers); at pi/4 with spacing
    sqrt(2)/2 every ray passes through in-plane cell corners (the Section 4.1 examples, P:680-689,
    generalised to a whole detector);
  - cone / helical with odd detectors: the central column of views 0, pi/2, ... lies on the plane
    x = 0 or y = 0 between two cells, the central row (h = 0) on the plane z = 0 (helical: on
    z = H(phi') whenever H is a multiple of d_z);
  - the 32 constructed 2D rays through every 2D adjoint kernel.
* Reading 9 on the GPU: the point phantoms of test_oracle_detector.py land in the same bins.
Index sets bit-exact (fp64 CSR), forward <= 1e-5 of max|sino| (oracle scale), adjoint <= 1e-4 rel L2.
"""
import math

import numpy as np
import pytest
import torch

import workloads
from paper_2006_00686_b200 import Plan, XrtError
from paper_2006_00686_b200 import _lib

import helpers as H
import test_oracle_detector as TD

pytestmark = pytest.mark.gpu


def _plan(c, fwd=None, adj=None):
    p = Plan(c, device=0)
    try:
        if fwd:
            p.set_algorithm("forward", fwd)
        if adj:
            p.set_algorithm("adjoint", adj)
    except XrtError as e:
        if e.status == _lib.XRT_ERR_UNSUPPORTED:
            pytest.skip(f"{fwd}/{adj} does not serve {c['beam']}")
        raise
    return p


def _edge_par3d(angles, du):
    c = workloads.config(3)
    c.update(n=(48, 48, 48), spacing=(1.0, 1.0, 1.0), angles=np.asarray(angles, dtype=np.float64),
             n_views=len(angles), det_cols=71, det_rows=55, det_spacing=(du, 1.0))
    return c


def _edge_cone(beam):
    c = workloads.config(4 if beam == "cone" else 5)
    angles = np.array([0.0, math.pi / 2, math.pi, 1.5 * math.pi, 0.37, 2.9])
    c.update(n=(48, 48, 48), spacing=(0.5, 0.5, 0.5), angles=angles, n_views=len(angles),
             det_cols=97, det_rows=71, det_offset=(0.0, 0.0))
    c["det_spacing"] = (2 * 0.5 * 48 * 1.5 / 97, 2 * 0.5 * 48 * 1.2 / 71)   # covers the box at M = 2
    if beam == "helical":
        # H(phi') = pitch phi' / (2 pi): a multiple of d_z at every listed right-angle view
        c.update(sod=600.0, sdd=1200.0, pitch=8 * 0.5, z0=0.0)
    return c


EDGE_GEOMS = {
    "par3d_axes": lambda: _edge_par3d([0.0, math.pi / 2, math.pi, 1.5 * math.pi], 1.0),
    "par3d_diag": lambda: _edge_par3d([math.pi / 4, 3 * math.pi / 4], math.sqrt(2.0) / 2),
    "cone": lambda: _edge_cone("cone"),
    "helical": lambda: _edge_cone("helical"),
}


@pytest.mark.parametrize("name", list(EDGE_GEOMS))
def test_edge_csr_every_ray(cuda_ok, name):
    c = EDGE_GEOMS[name]()
    p = _plan(c)
    ids = H.ray_ids_all(c)
    M = len(ids)
    cuts = np.linspace(0, M, 5).astype(int)
    for a, b in zip(cuts[:-1], cuts[1:]):
        H.compare_csr(p.ray_units(int(a), int(b)), H.oracle_csr(c, ids[a:b]), f"{name} [{a},{b})")


@pytest.mark.parametrize("fwd", [None, "ray"])
@pytest.mark.parametrize("name", list(EDGE_GEOMS))
def test_edge_forward_every_ray(cuda_ok, name, fwd):
    c = EDGE_GEOMS[name]()
    p = _plan(c, fwd=fwd)
    img = workloads.make_image(c, device="cuda")
    sino = p.forward(img)
    ref = H.oracle_forward(c, img.cpu(), H.ray_ids_all(c))
    assert H.fwd_err(sino.cpu().numpy().ravel(), ref) <= H.FWD_TOL
    # a ray on a face between two cells sees the bigger-index cell only: constant image -> the
    # chord of the half-open box (exact up to fp32), never the doubled or the missing face
    ones = torch.ones_like(img)
    ch = p.forward(ones)
    refc = H.oracle_forward(c, ones.cpu(), H.ray_ids_all(c))
    assert H.fwd_err(ch.cpu().numpy().ravel(), refc) <= H.FWD_TOL


@pytest.mark.parametrize("adj", [None, "ray", "gather"])
@pytest.mark.parametrize("name", list(EDGE_GEOMS))
def test_edge_adjoint(cuda_ok, name, adj):
    c = EDGE_GEOMS[name]()
    p = _plan(c, adj=adj)
    M = p.n_rays
    rng = np.random.Generator(np.random.PCG64(4242))
    y = rng.uniform(-1, 1, size=M).astype(np.float32)
    back = p.adjoint(torch.from_numpy(y).reshape(p.sino_shape).cuda())
    ref = H.oracle_adjoint(c, y.astype(np.float64), H.ray_ids_all(c))
    assert H.rel_l2(back.cpu().numpy().ravel(), ref) <= H.ADJ_TOL


@pytest.mark.parametrize("adj", [None, "ray", "column", "gather"])
def test_constructed_rays_adjoint(cuda_ok, adj):
    """The 32 constructed cfg-1 rays (edges, corners, outer faces) through every 2D adjoint kernel
    (AUTO = the lockstep slice kernel) and the 2D slice forward."""
    for g, _ in H.constructed_plans():
        p = _plan(g, adj=adj)
        y = np.random.Generator(np.random.PCG64(31)).uniform(-1, 1, size=p.n_rays).astype(np.float32)
        back = p.adjoint(torch.from_numpy(y).reshape(p.sino_shape).cuda())
        ref = H.oracle_adjoint(g, y.astype(np.float64), H.ray_ids_all(g))
        assert H.rel_l2(back.cpu().numpy().ravel(), ref) <= H.ADJ_TOL, g["angles"][0]


def test_constructed_rays_slice_forward(cuda_ok):
    img = workloads.make_image(workloads.config(1), device="cuda")
    for g, _ in H.constructed_plans():
        p = _plan(g, fwd="column")
        sino = p.forward(img)
        ref = H.oracle_forward(g, img.cpu(), H.ray_ids_all(g))
        assert H.fwd_err(sino.cpu().numpy().ravel(), ref, scale=64.0) <= H.FWD_TOL


@pytest.mark.parametrize("fwd", [None, "ray"])
@pytest.mark.parametrize("beam", ["par2d", "fan2d", "par3d", "cone", "helical"])
def test_point_phantom_bins(cuda_ok, beam, fwd):
    """Reading 9 on the GPU: a point at the origin projects to the centre bin in every view, points
    at +y / +z to bins right of / above centre -- the same bins as the pinned oracle."""
    angles = np.arange(8) * (2 * math.pi / 8) + 0.1
    c = TD._geometry(beam, angles)
    p = _plan(c, fwd=fwd)
    cases = [(0.0, 0.0, 0.0), (0.0, 3.0, 0.0)] + ([(0.0, 0.0, 3.0)] if c["det_rows"] > 1 else [])
    for pt in cases:
        img_np = TD._point_image(c, *pt)
        img = torch.from_numpy(img_np).reshape(p.image_shape).cuda()
        sino = p.forward(img).cpu().numpy()
        ref = H.oracle_forward(c, torch.from_numpy(img_np), H.ray_ids_all(c)).reshape(sino.shape)
        assert H.fwd_err(sino.ravel(), ref.ravel()) <= H.FWD_TOL
        for v in range(len(angles)):
            g = np.unravel_index(int(np.argmax(sino[v])), sino[v].shape)
            o = np.unravel_index(int(np.argmax(ref[v])), ref[v].shape)
            assert g == o, (beam, pt, v, g, o)
        if pt == (0.0, 0.0, 0.0):
            for v in range(len(angles)):
                assert np.unravel_index(int(np.argmax(sino[v])), sino[v].shape) == \
                    ((c["det_rows"] - 1) // 2, (c["det_cols"] - 1) // 2)
