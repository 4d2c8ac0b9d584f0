"""Oracle for the attenuated X-ray transform -- TEST INFRASTRUCTURE (see oracle/__init__.py).

The generalized transform of eq:generalizedRadontransform,
    R_Phi f(theta, x) = int Phi(theta, x, t) f(x + t theta) dt,
with the SPECT weight Phi(theta, x, t) = exp(-int_t^inf mu(x + s theta) ds) (the attenuated Radon
transform the paper names at P:38-39; reading 23), for f and mu in the unit basis of
eq:f_represent.  Both are constant on each unit, so the integral over unit I (entered
at t_lo, left at t_hi = t_lo + l) is exact in closed form:
    f_I int_{t_lo}^{t_hi} exp(-(mu_I (t_hi - t) + A_I)) dt = f_I exp(-A_I) (1 - exp(-mu_I l)) / mu_I
(= f_I exp(-A_I) l for mu_I = 0), with A_I = sum of mu_J l_J over the units J entered after I.

Plain definition, written out: every unit box is clipped against the ray (slab test, the same
definition as brute.c but coded separately here because the attenuation needs each unit's
position t along the ray, which the CSR rows do not carry), the units with l > tau are ordered by
their entry t, and the sum above is evaluated in fp64.  Rays are {p + t theta} from
oracle.geometry.rays (theta from the source towards the detector for divergent beams; the
paper's theta for parallel beams).  Pinned in tests/test_oracle_attenuated.py: mu = 0 reduces to
oracle.forward; f = mu gives 1 - exp(-X mu) (fundamental theorem of calculus); the hand-worked
two-pixel rays of tests/golden/attenuated.txt (orientation); midpoint quadrature of the
continuous integral along the ray; the adjoint identity.
"""
from __future__ import annotations

import numpy as np

from .core import TAU_FACTOR
from .geometry import grid_bounds


def _axis_intervals(u0: float, w: float, n: int):
    """Entry / exit t of every slab [i, i+1) of one axis (index space u = u0 + t w).  A fixed axis
    (w = 0) keeps only the half-open cell floor(u0) (reading 2), over all t."""
    if w == 0.0:
        lo = np.full(n, np.inf)
        hi = np.full(n, -np.inf)
        if 0.0 <= u0 < n:
            k = int(np.floor(u0))
            lo[k], hi[k] = -np.inf, np.inf
        return lo, hi
    i = np.arange(n, dtype=np.float64)
    t0 = (i - u0) / w
    t1 = (i + 1.0 - u0) / w
    return np.minimum(t0, t1), np.maximum(t0, t1)


def ray_units_t(c: dict, p, th):
    """(flat index, t_lo, t_hi) of the units ray {p + t th} crosses with l = t_hi - t_lo > tau,
    ordered by t_lo (along theta)."""
    nx, ny, nz = (int(v) for v in c["n"])
    dx, dy, dz = (float(v) for v in c["spacing"])
    x_lo, y_hi, z_hi = grid_bounds(c)
    # index-space frame: u_x = (x - x_lo)/dx, u_y = (y_hi - y)/dy, u_z = (z_hi - z)/dz
    lx, hx = _axis_intervals((p[0] - x_lo) / dx, th[0] / dx, nx)
    ly, hy = _axis_intervals((y_hi - p[1]) / dy, -th[1] / dy, ny)
    lz, hz = _axis_intervals((z_hi - p[2]) / dz, -th[2] / dz, nz)
    lo = np.maximum(np.maximum(lz[:, None, None], ly[None, :, None]), lx[None, None, :])
    hi = np.minimum(np.minimum(hz[:, None, None], hy[None, :, None]), hx[None, None, :])
    tau = TAU_FACTOR * min(dx, dy, dz)
    with np.errstate(invalid="ignore"):
        keep = (hi - lo) > tau
    idx = np.flatnonzero(keep)          # flat index (k N_y + j) N_x + i of the C-ordered [z][y][x] array
    t_lo, t_hi = lo.ravel()[idx], hi.ravel()[idx]
    order = np.argsort(t_lo, kind="stable")
    return idx[order], t_lo[order], t_hi[order]


def _weights(mu_u: np.ndarray, l: np.ndarray) -> np.ndarray:
    """exp(-A_I) (1 - exp(-mu_I l_I)) / mu_I for units in path order (A_I: attenuation after I)."""
    a = mu_u * l
    after = np.cumsum(a[::-1])[::-1] - a          # sum over the units after I
    with np.errstate(invalid="ignore", divide="ignore"):
        g = np.where(mu_u == 0.0, l, -np.expm1(-a) / np.where(mu_u == 0.0, 1.0, mu_u))
    return np.exp(-after) * g


def forward_attenuated(c: dict, img, mu, p, th) -> np.ndarray:
    """sino[m] = sum_I f_I exp(-A_mI) (1 - exp(-mu_I l_mI)) / mu_I for rays (p[m], th[m]); fp64."""
    f = np.asarray(img, dtype=np.float64).ravel()
    m_ = np.asarray(mu, dtype=np.float64).ravel()
    out = np.zeros(len(p))
    for r in range(len(p)):
        idx, lo, hi = ray_units_t(c, p[r], th[r])
        if idx.size:
            out[r] = np.dot(f[idx], _weights(m_[idx], hi - lo))
    return out


def adjoint_attenuated(c: dict, y, mu, p, th) -> np.ndarray:
    """img[I] = sum_m y_m exp(-A_mI) (1 - exp(-mu_I l_mI)) / mu_I over the given rays; fp64."""
    nx, ny, nz = (int(v) for v in c["n"])
    m_ = np.asarray(mu, dtype=np.float64).ravel()
    y = np.asarray(y, dtype=np.float64).ravel()
    out = np.zeros(nx * ny * nz)
    for r in range(len(p)):
        if y[r] == 0.0:
            continue
        idx, lo, hi = ray_units_t(c, p[r], th[r])
        if idx.size:
            np.add.at(out, idx, y[r] * _weights(m_[idx], hi - lo))
    return out
