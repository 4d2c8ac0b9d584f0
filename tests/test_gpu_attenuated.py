"""Attenuated transform (xrt_forward_attenuated / xrt_adjoint_attenuated) through the
C ABI vs the fp64 oracle (oracle/attenuated.py) on the same seeded inputs.

Bars (reading 23): forward within 1e-5 per ray relative to max|sino| (the north_star
forward bar), adjoint within 1e-4 relative L2 (sparse-y parity), dot-product test to 1e-5; the
hand-worked golden rays exactly as printed (to fp32 rounding).
"""
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import geometry as G
import workloads
from paper_2006_00686_b200 import Plan

import helpers as H
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


ALGOS = ["auto", "ray"]   # auto: the column kernels on the 3D beams; ray: one thread per ray


def _plan(c, algo):
    p = Plan(c, device=0)
    if algo != "auto":
        p.set_algorithm("forward", algo)
        p.set_algorithm("adjoint", algo)
    return p


def _inputs(c):
    return workloads.make_image(c, device="cuda"), workloads.make_attenuation(c, device="cuda")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_forward_sampled_parity(cuda_ok, idx, algo):
    c = H.small_config(idx)
    p = _plan(c, algo)
    img, mu = _inputs(c)
    sino = p.forward_attenuated(img, mu).cpu().numpy().ravel()
    ids = workloads.sample_rays(c, 300, seed=700 + idx)
    pp, th = G.rays(c, ids)
    ref = oracle.forward_attenuated(c, img.cpu().numpy().ravel(), mu.cpu().numpy().ravel(), pp, th)
    assert H.fwd_err(sino[ids], ref) <= H.FWD_TOL
    # the weight really attenuates on these inputs (not a disguised plain transform)
    plain = oracle.forward(c, img.cpu().numpy().ravel(), pp, th)
    assert np.max(np.abs(plain - ref)) > 1e-2 * np.max(np.abs(ref))


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("idx", [2, 4])
def test_mu_zero_matches_forward(cuda_ok, idx, algo):
    c = H.small_config(idx)
    p = _plan(c, algo)
    img, _ = _inputs(c)
    a = p.forward_attenuated(img, torch.zeros_like(img)).cpu().numpy()
    b = p.forward(img).cpu().numpy()
    assert np.max(np.abs(a - b)) <= 1e-6 * np.max(np.abs(b))


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_adjoint_sparse_parity(cuda_ok, idx, algo):
    c = H.small_config(idx)
    p = _plan(c, algo)
    _, mu = _inputs(c)
    ids = workloads.sample_rays(c, 300, seed=800 + idx)
    y_full = workloads.make_sino_input(c).numpy().ravel()
    y = np.zeros_like(y_full)
    y[ids] = y_full[ids]
    back = p.adjoint_attenuated(torch.from_numpy(y).reshape(p.sino_shape).cuda(), mu).cpu().numpy().ravel()
    pp, th = G.rays(c, ids)
    ref = oracle.adjoint_attenuated(c, y[ids], mu.cpu().numpy().ravel(), pp, th)
    assert H.rel_l2(back, ref) <= H.ADJ_TOL


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_dot_product(cuda_ok, idx, algo):
    c = H.small_config(idx)
    p = _plan(c, algo)
    img, mu = _inputs(c)
    y = workloads.make_sino_input(c, device="cuda")
    Rx = p.forward_attenuated(img, mu).double()
    Rty = p.adjoint_attenuated(y, mu).double()
    lhs = float((Rx * y.double()).sum())
    rhs = float((img.double() * Rty).sum())
    # relative to ||Rx|| ||y|| + ||x|| ||R^T y|| (fp64 sums of fp32 outputs)
    scale = float(Rx.norm() * y.double().norm() + img.double().norm() * Rty.norm())
    assert abs(lhs - rhs) <= H.DOT_TOL * scale, (lhs, rhs)


def _golden():
    out = []
    with open(os.path.join(GOLDEN, "attenuated.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, g, r, fv, mv, ex = [x.strip() for x in line.split("|")]
            out.append((name, [int(x) for x in g.split()], r.split(), [float(x) for x in fv.split()],
                        [float(x) for x in mv.split()], float(ex)))
    return out


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c[0])
def test_golden_rays(cuda_ok, case):
    """The hand-worked rays of tests/golden/attenuated.txt through explicit ray-list plans."""
    name, n, r, f, mu, expected = case
    q = [float(x) for x in r[1:]]
    params = [q[0], q[1], 0.0, 0.0] if r[0] == "par2d" else q
    c = dict(beam="rays", dim=2 if r[0] == "par2d" else 3, n=tuple(n), spacing=(1.0, 1.0, 1.0),
             center=(0.0, 0.0, 0.0), ray_params=[params])
    p = Plan(c, device=0)
    img = torch.tensor(f, dtype=torch.float32, device="cuda").reshape(p.image_shape)
    m = torch.tensor(mu, dtype=torch.float32, device="cuda").reshape(p.image_shape)
    got = p.forward_attenuated(img, m).item()
    assert abs(got - expected) <= 1e-6 * max(1.0, abs(expected)), (name, got, expected)
    back = p.adjoint_attenuated(torch.ones(p.sino_shape, device="cuda"), m).cpu().numpy().ravel()
    assert abs(float(np.dot(back, f)) - expected) <= 1e-6 * max(1.0, abs(expected)), name


@pytest.mark.parametrize("idx", [3, 4, 5])
def test_column_matches_ray(cuda_ok, idx):
    """The column and RAY attenuated kernels agree on the whole oracle-sized sinogram / image."""
    c = H.small_config(idx)
    pc, pr = _plan(c, "auto"), _plan(c, "ray")
    img, mu = _inputs(c)
    y = workloads.make_sino_input(c, device="cuda")
    a, b = pc.forward_attenuated(img, mu).cpu().numpy(), pr.forward_attenuated(img, mu).cpu().numpy()
    assert H.fwd_err(a.ravel(), b.ravel()) <= H.FWD_TOL
    ba, bb = pc.adjoint_attenuated(y, mu).cpu().numpy(), pr.adjoint_attenuated(y, mu).cpu().numpy()
    assert H.rel_l2(ba, bb) <= H.ADJ_TOL


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("idx", [3, 4])
def test_strong_attenuation(cuda_ok, idx, algo):
    """mu x 40 (total attenuation of a central ray ~ 100, units with mu l > 1/8: the exact weights
    instead of the Taylor series) against the oracle on a ray sample."""
    c = H.small_config(idx)
    p = _plan(c, algo)
    img, mu = _inputs(c)
    mu = mu * 40.0
    sino = p.forward_attenuated(img, mu).cpu().numpy().ravel()
    ids = workloads.sample_rays(c, 300, seed=900 + idx)
    pp, th = G.rays(c, ids)
    ref = oracle.forward_attenuated(c, img.cpu().numpy().ravel(), mu.cpu().numpy().ravel(), pp, th)
    assert H.fwd_err(sino[ids], ref) <= H.FWD_TOL


@pytest.mark.parametrize("beam", ["par2d", "fan2d", "par3d", "cone", "helical"])
def test_random_geometries(cuda_ok, beam):
    """The seeded random small geometries of test_gpu_parity (non-cubic, anisotropic, off-centre,
    curved detectors, tilted parallel beams, single rows / views): attenuated forward and adjoint of
    every kernel family that serves the geometry against the oracle on every ray."""
    from test_gpu_parity import _random_geometry
    from paper_2006_00686_b200 import XrtError
    rng = np.random.Generator(np.random.PCG64({"par2d": 21, "fan2d": 22, "par3d": 23, "cone": 24, "helical": 25}[beam]))
    for trial in range(4):
        g = _random_geometry(rng, beam)
        p = Plan(g, device=0)
        ids = H.ray_ids_all(g)
        pp, th = G.rays(g, ids)
        img = workloads.make_image(g, device="cuda")
        mu = (img.abs() * float(rng.uniform(0.02, 0.6))).contiguous()
        ref = oracle.forward_attenuated(g, img.cpu().numpy().ravel(), mu.cpu().numpy().ravel(), pp, th)
        y = np.random.Generator(np.random.PCG64(trial)).uniform(-1, 1, p.n_rays).astype(np.float32)
        refb = oracle.adjoint_attenuated(g, y.astype(np.float64), mu.cpu().numpy().ravel(), pp, th)
        for algo in ("ray", "column"):
            try:
                p.set_algorithm("forward", algo)
                p.set_algorithm("adjoint", algo)
            except XrtError:
                continue
            sino = p.forward_attenuated(img, mu).cpu().numpy().ravel()
            assert H.fwd_err(sino, ref) <= H.FWD_TOL, (beam, trial, algo)
            back = p.adjoint_attenuated(torch.from_numpy(y).reshape(p.sino_shape).cuda(), mu).cpu().numpy().ravel()
            if np.linalg.norm(refb) > 0:
                assert H.rel_l2(back, refb) <= H.ADJ_TOL, (beam, trial, algo)


@pytest.mark.parametrize("idx", [4, 5])
def test_view_sharding_equivalence(cuda_ok, idx):
    """Attenuated operators on view shards (the per-rank plans of dist.ShardedPlan, run here on one
    GPU): forward slabs bitwise equal to the unsharded sinogram, adjoint partials sum to it."""
    from paper_2006_00686_b200.dist import shard_geometry
    c = H.small_config(idx)
    img, mu = _inputs(c)
    full = Plan(c, device=0)
    y = workloads.make_sino_input(c, device="cuda")
    ref_f = full.forward_attenuated(img, mu)
    ref_b = full.adjoint_attenuated(y, mu)
    acc = torch.zeros_like(ref_b)
    for r in range(3):
        g = shard_geometry(c, r, 3)
        v0, v1 = g["view_block"]
        p = Plan(g, device=0)
        assert torch.equal(p.forward_attenuated(img, mu), ref_f[v0:v1])
        acc += p.adjoint_attenuated(y[v0:v1].contiguous(), mu)
    assert H.rel_l2(acc.cpu().numpy(), ref_b.cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("tile", ["16", "8"])
@pytest.mark.parametrize("idx", [4, 5])
def test_tiled_pieces_combine(cuda_ok, idx, tile, monkeypatch):
    """Forced xy tiling (XRT_COLUMN_TILE at plan creation): the attenuated forward runs per tile
    piece, (sigma, S_t, A_t), and combines the pieces in path order -- against the oracle and the
    RAY kernel (no tiling) on the whole sinogram.  Tile 8 gives 36 / 64 tiles, more than the
    combine's 16 piece slots: the attenuated operators then run untiled (att_tiled), still exact."""
    c = H.small_config(idx)
    monkeypatch.setenv("XRT_COLUMN_TILE", tile)
    pt = Plan(c, device=0)
    monkeypatch.delenv("XRT_COLUMN_TILE")
    pr = _plan(c, "ray")
    img, mu = _inputs(c)
    for scale in (1.0, 40.0):
        m = (mu * scale).contiguous()
        a = pt.forward_attenuated(img, m).cpu().numpy().ravel()
        if scale == 1.0:   # (at x40 both kernels sit near the bar from opposite sides: oracle only)
            b = pr.forward_attenuated(img, m).cpu().numpy().ravel()
            assert H.fwd_err(a, b) <= H.FWD_TOL, scale
        ids = workloads.sample_rays(c, 200, seed=950 + idx)
        pp, th = G.rays(c, ids)
        ref = oracle.forward_attenuated(c, img.cpu().numpy().ravel(), m.cpu().numpy().ravel(), pp, th)
        assert H.fwd_err(a[ids], ref) <= H.FWD_TOL, scale
    # the tiled adjoint (pieces' suffix attenuation) against the oracle's scatter on a ray sample
    ids = workloads.sample_rays(c, 300, seed=960 + idx)
    y_full = workloads.make_sino_input(c).numpy().ravel()
    y = np.zeros_like(y_full)
    y[ids] = y_full[ids]
    pp, th = G.rays(c, ids)
    for scale in (1.0, 40.0):
        m = (mu * scale).contiguous()
        back = pt.adjoint_attenuated(torch.from_numpy(y).reshape(pt.sino_shape).cuda(), m).cpu().numpy().ravel()
        refb = oracle.adjoint_attenuated(c, y[ids], m.cpu().numpy().ravel(), pp, th)
        assert H.rel_l2(back, refb) <= H.ADJ_TOL, scale
