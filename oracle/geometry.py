"""Oracle ray geometry: the paper's transformation formulas, written out literally (fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of the product's
plan builder: the product builds rays as source + detector-frame vectors, the
oracle builds them through the paper's parallel-beam parameters.

Every function cites the passage it follows (P:n = /root/reference/PAPER.md line n).
The conventions the paper leaves open are DESIGN.md readings 7-11; they are
restated at each use.
"""
from __future__ import annotations

import math

import numpy as np

SNAP = 1e-12  # |theta_a| <= SNAP -> exactly 0 (reading 2/5)


# ---------------------------------------------------------------- 2D (Section 2.2)
def par2d_basis(phi):
    """theta = (cos phi, sin phi), theta_perp = (-sin phi, cos phi): eq:direction_normal P:134-137."""
    phi = np.asarray(phi, dtype=np.float64)
    theta = np.stack([np.cos(phi), np.sin(phi)], axis=-1)
    perp = np.stack([-np.sin(phi), np.cos(phi)], axis=-1)
    return theta, perp


def fan_equiangular_to_parallel(D, alpha, gamma):
    """s = D sin(gamma), phi = gamma + alpha - pi/2: eq:2Dparalleltofan P:263-265."""
    return D * np.sin(gamma), gamma + alpha - math.pi / 2


def fan_equispaced_to_parallel(D, alpha, t):
    """s = D t / sqrt(D^2 + t^2), phi = arctan(t/D) + alpha - pi/2: eq:2Dparalleltofan_2 P:269-271."""
    return D * t / np.sqrt(D * D + t * t), np.arctan(t / D) + alpha - math.pi / 2


def canonicalize_2d(s, phi):
    """(s, phi + 2n pi) == (s, phi); (s, phi + pi) == (-s, phi) -> phi in [0, pi): P:166."""
    s = np.asarray(s, dtype=np.float64).copy()
    phi = np.mod(np.asarray(phi, dtype=np.float64), 2 * math.pi)
    flip = phi >= math.pi
    phi = np.where(flip, phi - math.pi, phi)
    s = np.where(flip, -s, s)
    return s, phi


# ---------------------------------------------------------------- 3D (Section 3.2)
def par3d_basis(phi1, phi2):
    """theta, theta_1, theta_2 of eq:3Dparallel_direction / eq:theta_1 / eq:theta_2."""
    phi1 = np.asarray(phi1, dtype=np.float64)
    phi2 = np.asarray(phi2, dtype=np.float64)
    c1, s1, c2, s2 = np.cos(phi1), np.sin(phi1), np.cos(phi2), np.sin(phi2)
    theta = np.stack([c2 * c1, c2 * s1, s2], axis=-1)
    th1 = np.stack([-s1, c1, np.zeros_like(c1)], axis=-1)
    th2 = np.stack([-s2 * c1, -s2 * s1, c2], axis=-1)
    return theta, th1, th2


def euler_R(phi1, phi2, phi3=0.0):
    """The three Eulerian rotations of eq:Eulerian_rotations, P:326-367 (rows = x', y', z')."""
    R3 = np.array([[math.cos(phi3), math.sin(phi3), 0], [-math.sin(phi3), math.cos(phi3), 0], [0, 0, 1]])
    R2 = np.array([[math.cos(phi2), 0, math.sin(phi2)], [0, 1, 0], [-math.sin(phi2), 0, math.cos(phi2)]])
    R1 = np.array([[math.cos(phi1), math.sin(phi1), 0], [-math.sin(phi1), math.cos(phi1), 0], [0, 0, 1]])
    return R3 @ R2 @ R1


def cone_equiangular_to_parallel(D, phi1p, alpha, beta):
    """phi1 = phi1' + alpha, phi2 = beta, s1 = D sin(alpha), s2 = D cos(alpha) sin(beta):
    eq:equiangular_cone_beam P:619-624."""
    return D * np.sin(alpha), D * np.cos(alpha) * np.sin(beta), phi1p + alpha, beta


def cone_equispaced_to_parallel(D, phi1p, t, h):
    """alpha = arctan(t/D), beta = arctan(h / sqrt(D^2 + t^2)); phi1 = phi1' + alpha, phi2 = beta,
    s1 = D sin(alpha), s2 = h cos^2(alpha) cos(beta): eq:equispaced_cone_beam P:631-640."""
    alpha = np.arctan(t / D)
    beta = np.arctan(h / np.sqrt(D * D + t * t))
    return D * np.sin(alpha), h * np.cos(alpha) ** 2 * np.cos(beta), phi1p + alpha, beta


def helical_equiangular_to_parallel(D, phi1p, alpha, beta, H):
    """As the equiangular cone with s2 = D cos(alpha) sin(beta) + H cos(beta):
    eq:Helical_cone_beam_equiangular P:652-654."""
    s1, s2, p1, p2 = cone_equiangular_to_parallel(D, phi1p, alpha, beta)
    return s1, s2 + H * np.cos(beta), p1, p2


def helical_equispaced_to_parallel(D, phi1p, t, h, H):
    """As the equispaced cone with s2 = h cos^2(alpha) cos(beta) + H cos(beta):
    eq:Helical_cone_beam_equispaced P:659-661."""
    s1, s2, p1, p2 = cone_equispaced_to_parallel(D, phi1p, t, h)
    return s1, s2 + H * np.cos(p2), p1, p2


def canonicalize_3d(s1, s2, phi1, phi2):
    """Reduce to (phi1, phi2) in [0, 2pi) x [0, pi/2] with the three equivalences of P:443:
    2pi periodicity; (s1, s2, phi1, phi2 + pi) == (s1, -s2, phi1, phi2);
    (-s1, s2, phi1 + pi, -phi2) == (s1, s2, phi1, phi2)."""
    s1 = float(s1); s2 = float(s2)
    phi1 = math.fmod(float(phi1), 2 * math.pi)
    phi2 = math.fmod(float(phi2), 2 * math.pi)
    if phi2 < 0:
        phi2 += 2 * math.pi
    if phi2 >= math.pi:                   # phi2 + pi equivalence
        phi2 -= math.pi
        s2 = -s2
    if phi2 > math.pi / 2:                # phi2 in (pi/2, pi): use (-s1, s2, phi1 + pi, -phi2) then +pi
        phi1, phi2, s1 = phi1 + math.pi, -phi2, -s1
        phi2 += math.pi
        s2 = -s2
    phi1 = math.fmod(phi1, 2 * math.pi)
    if phi1 < 0:
        phi1 += 2 * math.pi
    return s1, s2, phi1, phi2


# ---------------------------------------------------------------- rays of a config
def _snap(theta):
    theta = np.array(theta, dtype=np.float64)
    theta[np.abs(theta) <= SNAP] = 0.0
    return theta


def det_u(c: dict, cols):
    """Detector column position u_c = (c - (N_cols - 1)/2) du + offset_u (reading 9)."""
    return (np.asarray(cols, dtype=np.float64) - (c["det_cols"] - 1) / 2.0) * c["det_spacing"][0] + c["det_offset"][0]


def det_v(c: dict, rows):
    """Detector row position v_r = (r - (N_rows - 1)/2) dv + offset_v, +v = +z (reading 9)."""
    return (np.asarray(rows, dtype=np.float64) - (c["det_rows"] - 1) / 2.0) * c["det_spacing"][1] + c["det_offset"][1]


def rays(c: dict, ids) -> tuple[np.ndarray, np.ndarray]:
    """(p, theta) in PHYSICAL coordinates, shape [n, 3] fp64, for ray ids m = (v*rows + r)*cols + col.

    The ray is {p + t theta}, theta a unit vector, p the paper's foot point
    s theta_perp (2D) or s1 theta_1 + s2 theta_2 (3D).  2D rays live in
    the plane z = 0 with theta_z = 0 (the image is one slab thick).
    """
    ids = np.asarray(ids, dtype=np.int64)
    if c["beam"] == "rays":
        # explicit paper parameters per ray (Remark 3.5)
        q = np.asarray(c["ray_params"], dtype=np.float64).reshape(-1, 4)[ids]
        n = ids.shape[0]
        p = np.zeros((n, 3))
        th = np.zeros((n, 3))
        if int(c["dim"]) == 2:
            theta, perp = par2d_basis(q[:, 1])
            p[:, :2] = q[:, 0:1] * perp                      # s theta_perp
            th[:, :2] = theta
        else:
            theta, th1, th2 = par3d_basis(q[:, 2], q[:, 3])
            p = q[:, 0:1] * th1 + q[:, 1:2] * th2            # s1 theta_1 + s2 theta_2
            th = theta
        return p, _snap(th)
    C, R = c["det_cols"], c["det_rows"]
    col = ids % C
    row = (ids // C) % R
    view = ids // (C * R)
    ang = np.asarray(c["angles"], dtype=np.float64)[view]
    u = det_u(c, col)
    v = det_v(c, row)
    beam = c["beam"]
    n = ids.shape[0]
    p = np.zeros((n, 3))
    th = np.zeros((n, 3))
    if beam in ("par2d", "fan2d"):
        if beam == "par2d":
            s, phi = u, ang                                   # ray (s, phi)
        elif c.get("det_curved", False):
            # cylindrical detector of radius sdd: equiangular fan angle gamma = u / sdd
            s, phi = fan_equiangular_to_parallel(c["sod"], ang, u / c["sdd"])
        else:
            D = c["sod"]
            t = u * c["sod"] / c["sdd"]                       # flat detector scaled to the iso plane (reading 8)
            s, phi = fan_equispaced_to_parallel(D, ang, t)    # P:269-271; alpha = source angle (reading 7)
        theta, perp = par2d_basis(phi)
        p[:, :2] = s[:, None] * perp                          # x = t theta + s theta_perp
        th[:, :2] = theta
    else:
        if beam == "par3d":
            s1, s2, phi1, phi2 = u, v, ang, np.full(n, c.get("tilt", 0.0))
        elif beam in ("cone", "helical") and c.get("det_curved", False):
            # cylindrical detector: alpha = u / sdd (equiangular columns), tan(beta) = v / sdd (flat
            # rows); the equiangular transforms P:619-624 / P:652-654
            alpha, beta = u / c["sdd"], np.arctan(v / c["sdd"])
            if beam == "cone":
                s1, s2, phi1, phi2 = cone_equiangular_to_parallel(c["sod"], ang, alpha, beta)
            else:
                H = c["z0"] + c["pitch"] * ang / (2 * math.pi)
                s1, s2, phi1, phi2 = helical_equiangular_to_parallel(c["sod"], ang, alpha, beta, H)
        elif beam == "cone":
            t = u * c["sod"] / c["sdd"]
            h = v * c["sod"] / c["sdd"]
            s1, s2, phi1, phi2 = cone_equispaced_to_parallel(c["sod"], ang, t, h)
        elif beam == "helical":
            t = u * c["sod"] / c["sdd"]
            h = v * c["sod"] / c["sdd"]
            H = c["z0"] + c["pitch"] * ang / (2 * math.pi)    # source height (reading 11)
            s1, s2, phi1, phi2 = helical_equispaced_to_parallel(c["sod"], ang, t, h, H)
        else:
            raise ValueError(beam)
        theta, th1, th2 = par3d_basis(phi1, phi2)
        p = s1[:, None] * th1 + s2[:, None] * th2             # x = t theta + s1 theta_1 + s2 theta_2
        th = theta
    return p, _snap(th)


def grid_bounds(c: dict):
    """x_lo, y_hi, z_hi of the image box [c - N d / 2, c + N d / 2]."""
    nx, ny, nz = c["n"]
    dx, dy, dz = c["spacing"]
    cx, cy, cz = c["center"]
    return cx - nx * dx / 2.0, cy + ny * dy / 2.0, cz + nz * dz / 2.0


