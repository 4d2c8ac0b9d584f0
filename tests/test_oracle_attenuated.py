"""Pins of the attenuated-transform oracle (oracle/attenuated.py, DESIGN reading 23).

* mu = 0: the weight is 1 and the transform is the X-ray transform -> oracle.forward (brute.c, a
  separate code) on the same rays;
* f = mu (any mu): int mu(t) exp(-int_t^inf mu) dt = 1 - exp(-int mu) (fundamental theorem of
  calculus) -> 1 - exp(-oracle.forward(mu));
* constant f and mu on the image box: (1 - exp(-mu L)) / mu with L the chord (one slab clip,
  written here);
* hand-worked rays of tests/golden/attenuated.txt (the orientation of the weight along theta);
* midpoint quadrature of the continuous integral along the ray (a different algorithm: point
  lookups of f and mu, cumulative attenuation) to its O(1/K) error;
* adjoint identity <R x, y> = <x, R^T y>.
"""
import math
import os

import numpy as np
import pytest

import oracle
from oracle import geometry as G
from conftest import GOLDEN

RNG = np.random.Generator(np.random.PCG64(2323))


def grid(n, d=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0)):
    return dict(n=tuple(n), spacing=tuple(d), center=tuple(center))


def ray2d(s, phi):
    th, perp = G.par2d_basis(phi)
    return np.array([[s * perp[0], s * perp[1], 0.0]]), G._snap(np.array([[th[0], th[1], 0.0]]))


def ray3d(s1, s2, phi1, phi2):
    th, t1, t2 = G.par3d_basis(phi1, phi2)
    return (s1 * t1 + s2 * t2)[None, :], G._snap(th[None, :])


def random_rays(c, k, rng, dim=3):
    ext = np.array(c["n"]) * np.array(c["spacing"])
    ctr = np.array(c["center"])
    th = rng.normal(size=(k, 3))
    if dim == 2:
        th[:, 2] = 0
    th /= np.linalg.norm(th, axis=1, keepdims=True)
    p = ctr + rng.uniform(-0.55, 0.55, size=(k, 3)) * ext
    if dim == 2:
        p[:, 2] = ctr[2]
    return p, th


def chord(c, p, th):
    """|{p + t th} inside the image box| (slab clip, written here)."""
    lo = np.array(c["center"]) - np.array(c["n"]) * np.array(c["spacing"]) / 2
    hi = lo + np.array(c["n"]) * np.array(c["spacing"])
    t0, t1 = -np.inf, np.inf
    for a in range(3):
        if th[a] == 0.0:
            if not (lo[a] <= p[a] < hi[a]):
                return 0.0
            continue
        u, v = (lo[a] - p[a]) / th[a], (hi[a] - p[a]) / th[a]
        t0, t1 = max(t0, min(u, v)), min(t1, max(u, v))
    return max(0.0, t1 - t0)


CASES3 = [grid((7, 6, 5), (1.0, 0.8, 1.3), (0.2, -0.1, 0.3)), grid((8, 8, 8))]
CASES2 = [grid((9, 7, 1), (1.0, 1.2, 1.0), (0.3, 0.0, 0.0))]


@pytest.mark.parametrize("c,dim", [(c, 3) for c in CASES3] + [(c, 2) for c in CASES2])
def test_mu_zero_is_xray_transform(c, dim):
    p, th = random_rays(c, 60, RNG, dim)
    f = RNG.uniform(-1, 1, size=int(np.prod(c["n"]))).astype(np.float32).astype(np.float64)  # oracle.forward reads fp32
    ref = oracle.forward(c, f, p, th)
    got = oracle.forward_attenuated(c, f, np.zeros_like(f), p, th)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("c,dim", [(c, 3) for c in CASES3] + [(c, 2) for c in CASES2])
def test_f_equals_mu_closed_form(c, dim):
    p, th = random_rays(c, 60, RNG, dim)
    mu = RNG.uniform(0.0, 0.4, size=int(np.prod(c["n"]))).astype(np.float32).astype(np.float64)
    total = oracle.forward(c, mu, p, th)
    got = oracle.forward_attenuated(c, mu, mu, p, th)
    assert np.max(np.abs(got - (1.0 - np.exp(-total)))) <= 1e-12


def test_constant_chord_closed_form():
    c = CASES3[0]
    p, th = random_rays(c, 60, RNG, 3)
    n = int(np.prod(c["n"]))
    for m in (0.0, 0.05, 0.7):
        got = oracle.forward_attenuated(c, np.ones(n), np.full(n, m), p, th)
        L = np.array([chord(c, p[i], th[i]) for i in range(len(p))])
        ref = L if m == 0.0 else (1.0 - np.exp(-m * L)) / m
        assert np.max(np.abs(got - ref)) <= 1e-11, m


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
def test_golden(case):
    name, n, r, f, mu, expected = case
    c = grid(n)
    q = [float(x) for x in r[1:]]
    p, th = ray2d(*q) if r[0] == "par2d" else ray3d(*q)
    got = oracle.forward_attenuated(c, np.array(f), np.array(mu), p, th)[0]
    assert abs(got - expected) <= 1e-12, (name, got, expected)


def quadrature(c, f, mu, p, th, K=40000):
    """Midpoint rule of int f(x(t)) exp(-int_t^inf mu) dt over the chord, with point lookups of the
    half-open unit containing each sample and the inner integral as a reversed cumulative sum."""
    lo = np.array(c["center"]) - np.array(c["n"]) * np.array(c["spacing"]) / 2
    hi = lo + np.array(c["n"]) * np.array(c["spacing"])
    t0, t1 = -np.inf, np.inf
    for a in range(3):
        if th[a] == 0.0:
            continue
        u, v = (lo[a] - p[a]) / th[a], (hi[a] - p[a]) / th[a]
        t0, t1 = max(t0, min(u, v)), min(t1, max(u, v))
    if not t1 > t0:
        return 0.0
    h = (t1 - t0) / K
    t = t0 + (np.arange(K) + 0.5) * h
    x = p[None, :] + t[:, None] * th[None, :]
    nx, ny, nz = c["n"]
    dx, dy, dz = c["spacing"]
    i = np.floor((x[:, 0] - lo[0]) / dx).astype(int)
    j = np.floor((hi[1] - x[:, 1]) / dy).astype(int)
    k = np.floor((hi[2] - x[:, 2]) / dz).astype(int)
    ok = (i >= 0) & (i < nx) & (j >= 0) & (j < ny) & (k >= 0) & (k < nz)
    idx = np.where(ok, (k * ny + j) * nx + i, 0)
    fv = np.where(ok, f[idx], 0.0)
    mv = np.where(ok, mu[idx], 0.0)
    after = (np.cumsum(mv[::-1])[::-1] - 0.5 * mv) * h      # int_t^inf mu at each midpoint
    return float(np.sum(fv * np.exp(-after)) * h)


def test_quadrature_agrees():
    c = grid((6, 5, 4), (1.0, 1.1, 0.9), (0.1, 0.2, -0.1))
    rng = np.random.Generator(np.random.PCG64(99))
    n = int(np.prod(c["n"]))
    f = rng.uniform(0, 1, size=n)
    mu = rng.uniform(0, 0.8, size=n)
    p, th = random_rays(c, 25, rng, 3)
    got = oracle.forward_attenuated(c, f, mu, p, th)
    ref = np.array([quadrature(c, f, mu, p[m], th[m]) for m in range(len(p))])
    # O(h) per discontinuity (<= ~15 unit faces per chord), h = chord / 40000
    assert np.max(np.abs(got - ref)) <= 5e-4 * max(1.0, np.max(np.abs(ref)))   # measured 5.4e-5
    # and the orientation matters: the reversed rays give clearly different values
    rev = oracle.forward_attenuated(c, f, mu, p, -th)
    assert np.max(np.abs(rev - got)) > 1e-2


@pytest.mark.parametrize("c,dim", [(CASES3[0], 3), (CASES2[0], 2)])
def test_adjoint_identity(c, dim):
    p, th = random_rays(c, 50, RNG, dim)
    n = int(np.prod(c["n"]))
    x = RNG.uniform(-1, 1, size=n)
    mu = RNG.uniform(0.0, 0.5, size=n)
    y = RNG.uniform(-1, 1, size=len(p))
    lhs = np.dot(oracle.forward_attenuated(c, x, mu, p, th), y)
    rhs = np.dot(x, oracle.adjoint_attenuated(c, y, mu, p, th))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
