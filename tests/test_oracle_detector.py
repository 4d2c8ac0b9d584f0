"""Pins of the detector-bin convention (reading 9), with point phantoms.

The paper fixes where a ray of parameter s / (s1, s2) / gamma / (alpha, beta) goes, not how bins
are numbered.  Reading 9 numbers them u_c = (c - (N_c - 1) / 2) du + off_u, v_r = (r - (N_r - 1) / 2)
dv + off_v, with +u the +gamma direction and +v = +z.  Two facts of the paper pin that rule:

* centring -- the central ray of every beam passes through the origin: s = 0,
  gamma = 0 <=> s = D sin(gamma) = 0, alpha = beta = 0 <=> s1 = s2 = 0.  So a
  point phantom at the origin projects to the centre bin of an odd detector in EVERY view;
* orientation -- the foot point of ray (s, phi) is s theta_perp with theta_perp = (-sin phi, cos phi)
  (P:132-138), of (s1, s2, phi1, phi2) s1 theta_1 + s2 theta_2; a point at (0, +y) seen at
  phi = 0 therefore lies on the ray s = +y, i.e. in a bin right of centre, and a point at +z on a row
  above centre.  For the divergent beams the same follows from the source positions of reading 7 and
  the transforms (gamma > 0 on the +e_u side of the central ray).

Each check builds a one-voxel phantom, projects it with the oracle and locates the brightest bin:
an error in the centring, a flipped sign of u or v, or a swapped row / column fails here.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import geometry as G
import workloads

NPIX = 21            # odd grid: voxel (10, 10, 10) is centred on the origin
NCOL, NROW = 31, 31  # odd detector: bin 15 is the central ray


def _geometry(beam, angles, du_iso=1.0):
    """An NPIX^d unit grid and an odd detector whose bins are du_iso apart at the isocentre."""
    c = workloads.config({"par2d": 1, "fan2d": 2, "par3d": 3, "cone": 4, "helical": 5}[beam])
    is2d = beam in ("par2d", "fan2d")
    c.update(n=(NPIX, NPIX, 1 if is2d else NPIX), spacing=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0),
             angles=np.asarray(angles, dtype=np.float64), n_views=len(angles), det_cols=NCOL,
             det_rows=1 if is2d else NROW, det_offset=(0.0, 0.0), tilt=0.0)
    mag = c["sdd"] / c["sod"] if beam in ("fan2d", "cone", "helical") else 1.0
    c["det_spacing"] = (du_iso * mag, du_iso * mag)
    if beam == "helical":
        c.update(pitch=0.0, z0=0.0)   # H = 0: the helix reduces to the circular cone
    return c


def _point_image(c, x, y, z=0.0):
    """f = 1 in the voxel containing the physical point (x, y, z), 0 elsewhere (flat index
    (k N_y + j) N_x + i, j down from +y, k down from +z: readings 1-2)."""
    nx, ny, nz = c["n"]
    img = np.zeros(nx * ny * nz, dtype=np.float32)
    i = int(math.floor(x + nx / 2))
    j = int(math.floor(ny / 2 - y))
    k = int(math.floor(nz / 2 - z)) if nz > 1 else 0
    img[(k * ny + j) * nx + i] = 1.0
    return img


def _brightest(c, img, view):
    """(row, col) of the largest oracle value in one view."""
    per = c["det_rows"] * c["det_cols"]
    ids = np.arange(view * per, (view + 1) * per, dtype=np.int64)
    p, th = G.rays(c, ids)
    s = oracle.forward(c, img, p, th, mode=1).reshape(c["det_rows"], c["det_cols"])
    r, col = np.unravel_index(int(np.argmax(s)), s.shape)
    # the maximum must be unique (a ray through a voxel's interior, neighbours miss or graze it)
    assert np.sum(s >= s[r, col] - 1e-12) == 1, s
    return int(r), int(col)


@pytest.mark.parametrize("beam", ["par2d", "fan2d", "par3d", "cone", "helical"])
def test_origin_projects_to_centre_bin(beam):
    angles = np.arange(16) * (2 * math.pi / 16) + 0.1
    c = _geometry(beam, angles)
    img = _point_image(c, 0.0, 0.0, 0.0)
    cr = 0 if c["det_rows"] == 1 else (NROW - 1) // 2
    for v in range(len(angles)):
        assert _brightest(c, img, v) == (cr, (NCOL - 1) // 2), (beam, v)


@pytest.mark.parametrize("beam", ["par2d", "par3d"])
def test_parallel_orientation(beam):
    """phi = 0: theta_perp = (0, 1) -> the point (0, +3) is on the ray s = +3 (bin 15 + 3);
    phi = pi/2: theta_perp = (-1, 0) -> the point (-3, 0) is on s = +3; +z rows above centre."""
    c = _geometry(beam, [0.0, math.pi / 2])
    z = 2.0 if beam == "par3d" else 0.0
    rz = 0 if beam == "par2d" else (NROW - 1) // 2 + 2
    assert _brightest(c, _point_image(c, 0.0, 3.0, z), 0) == (rz, (NCOL - 1) // 2 + 3)
    assert _brightest(c, _point_image(c, -3.0, 0.0, z), 1) == (rz, (NCOL - 1) // 2 + 3)
    assert _brightest(c, _point_image(c, 0.0, -3.0, -z), 0) == (0 if beam == "par2d" else (NROW - 1) // 2 - 2,
                                                              (NCOL - 1) // 2 - 3)


def test_fan_orientation():
    """alpha = 0: source S = D(-sin 0, cos 0) = (0, D) (reading 7); the line from S to (+3, 0) has
    gamma > 0, so the point is right of centre (about 3 iso bins: the source sits far away)."""
    c = _geometry("fan2d", [0.0, math.pi / 2])
    r, col = _brightest(c, _point_image(c, 3.0, 0.0), 0)
    assert col > (NCOL - 1) // 2 and abs(col - ((NCOL - 1) // 2 + 3)) <= 1
    # alpha = pi/2: S = (-D, 0); the +gamma side is (0, +1) rotated... e_u = (cos a, sin a) = (0, 1)
    r, col = _brightest(c, _point_image(c, 0.0, 3.0), 1)
    assert col > (NCOL - 1) // 2


@pytest.mark.parametrize("beam", ["cone", "helical"])
def test_cone_orientation(beam):
    """phi1' = 0: source (-D, 0, 0) (reading 7), e_u = (0, 1, 0): a point at +y lies right of centre,
    a point at +z on a row above centre (beta > 0 <=> h > 0)."""
    c = _geometry(beam, [0.0])
    r, col = _brightest(c, _point_image(c, 0.0, 3.0, 0.0), 0)
    assert r == (NROW - 1) // 2 and col > (NCOL - 1) // 2 and abs(col - ((NCOL - 1) // 2 + 3)) <= 1
    r, col = _brightest(c, _point_image(c, 0.0, 0.0, 3.0), 0)
    assert col == (NCOL - 1) // 2 and r > (NROW - 1) // 2 and abs(r - ((NROW - 1) // 2 + 3)) <= 1
