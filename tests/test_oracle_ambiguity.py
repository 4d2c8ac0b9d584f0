"""Pins of the oracle's tie-break (reading 2) and of edge/corner-grazing rays.

Expected rows are derived by hand from the geometry (closed forms), not from the
oracle: a ray on a grid line belongs to the unit with the bigger 1D index; a
diagonal through lattice corners crosses 64 - |m| pixels with length sqrt(2).
"""
import math
import os

import numpy as np
import pytest

import oracle
from oracle import geometry as G
from conftest import GOLDEN


def grid(n, d=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0)):
    return dict(n=tuple(n), spacing=tuple(d), center=tuple(center))


def ray2d(s, phi):
    th, perp = G.par2d_basis(phi)
    return np.array([[s * perp[0], s * perp[1], 0.0]]), G._snap(np.array([[th[0], th[1], 0.0]]))


def ray3d(s1, s2, phi1, phi2):
    th, t1, t2 = G.par3d_basis(phi1, phi2)
    return (s1 * t1 + s2 * t2)[None, :], G._snap(th[None, :])


def row(c, p, th, mode=1):
    _, cols, lens = oracle.rows(c, p, th, mode=mode)
    return cols.tolist(), lens.tolist()


def _ambiguity_cases():
    out = []
    with open(os.path.join(GOLDEN, "ambiguity.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, g, r, idx, ln = [x.strip() for x in line.split("|")]
            out.append((name, [int(x) for x in g.split()], r.split(), [int(x) for x in idx.split()], float(ln)))
    return out


@pytest.mark.parametrize("case", _ambiguity_cases(), ids=lambda c: c[0])
@pytest.mark.parametrize("mode", [0, 1])
def test_section41_examples(case, mode):
    name, n, r, idx, ln = case
    vals = [float(x) for x in r[1:]]
    p, th = ray2d(*vals) if r[0] == "par2d" else ray3d(*vals)
    cols, lens = row(grid(n), p, th, mode)
    assert cols == idx
    assert all(abs(l - ln) < 1e-12 for l in lens)


N = 64


@pytest.mark.parametrize("s", [32, 31, 16, 1, 0, -1, -31, -32])
def test_constructed_horizontal(s):
    """phi = 0: y = s.  u_y = 32 - s; row j = 32 - s if 0 <= 32 - s < 64 else empty (reading 2)."""
    cols, lens = row(grid((N, N, 1)), *ray2d(float(s), 0.0))
    j = 32 - s
    exp = [j * N + i for i in range(N)] if 0 <= j < N else []
    assert cols == exp and all(abs(l - 1.0) < 1e-12 for l in lens)


@pytest.mark.parametrize("s", [32, 31, 16, 1, 0, -1, -31, -32])
def test_constructed_vertical(s):
    """phi = pi/2 (theta_x snapped to 0): x = -s.  u_x = 32 - s; column i = 32 - s if in range."""
    cols, lens = row(grid((N, N, 1)), *ray2d(float(s), math.pi / 2))
    i = 32 - s
    exp = [j * N + i for j in range(N)] if 0 <= i < N else []
    assert cols == exp and all(abs(l - 1.0) < 1e-12 for l in lens)


@pytest.mark.parametrize("m", [0, 1, -1, 31, -31, 63, -63, 64])
def test_constructed_diagonal(m):
    """phi = pi/4, s = m/sqrt2: line u_x + u_y = 64 - m through lattice corners; crosses the
    pixels with i + j = 63 - m along their anti-diagonal (length sqrt 2): 64 - |m| of them."""
    cols, lens = row(grid((N, N, 1)), *ray2d(m / math.sqrt(2.0), math.pi / 4))
    exp = sorted(j * N + i for j in range(N) for i in range(N) if i + j == 63 - m)
    assert len(exp) == max(0, 64 - abs(m))
    assert cols == exp and all(abs(l - math.sqrt(2.0)) < 1e-9 for l in lens)


@pytest.mark.parametrize("m", [0, 1, -1, 31, -31, 63, -63, 64])
def test_constructed_antidiagonal(m):
    """phi = 3pi/4, s = m/sqrt2: line u_x - u_y = -m; pixels with i - j = -m, length sqrt 2."""
    cols, lens = row(grid((N, N, 1)), *ray2d(m / math.sqrt(2.0), 3 * math.pi / 4))
    exp = sorted(j * N + i for j in range(N) for i in range(N) if i - j == -m)
    assert len(exp) == max(0, 64 - abs(m))
    assert cols == exp and all(abs(l - math.sqrt(2.0)) < 1e-9 for l in lens)


def test_constructed_3d_axis_rays():
    """3D Case 3/4: axis-parallel rays through a 5x4x6 (non-cubic) grid.
    Ray along x at y = 0.5, z = -1 (grid y in [-2,2], z in [-3,3]): u_y = 1.5 -> j = 1,
    u_z = 4 -> k = 4 (on a plane: bigger index, reading 2); I = (k*4 + j)*5 + i (reading 1)."""
    c = grid((5, 4, 6))
    p = np.array([[0.0, 0.5, -1.0]]); th = np.array([[1.0, 0.0, 0.0]])
    cols, lens = row(c, p, th)
    assert cols == [(4 * 4 + 1) * 5 + i for i in range(5)] and all(l == 1.0 for l in lens)
    # along -z at x = -2.5 (outer face: included, u_x = 0), y = 2 (top outer face: included, j = 0)
    p = np.array([[-2.5, 2.0, 0.0]]); th = np.array([[0.0, 0.0, -1.0]])
    cols, lens = row(c, p, th)
    assert cols == [(k * 4 + 0) * 5 + 0 for k in range(6)] and all(l == 1.0 for l in lens)
    # on the bottom / right outer faces: empty (the face belongs to a unit outside the grid)
    for p, th in (([2.5, 0.3, 0.1], [0, 0, 1.0]), ([0.2, -2.0, 0.1], [0, 0, 1.0]),
                  ([0.2, 0.3, -3.0], [1.0, 0, 0])):
        cols, _ = row(c, np.array([p]), np.array([th]))
        assert cols == []


def test_plane_ray_case2():
    """3D Case 2: ray in the plane y = 0.25 at 45 deg in x-z on a 4^3 grid: every
    crossed voxel has j = 1 and the lengths telescope to the x-z chord."""
    c = grid((4, 4, 4))
    p, th = ray3d(0.25, 0.0, 0.0, math.pi / 4)   # theta_1 = (0,1,0): y = s1
    cols, lens = row(c, p, th)
    js = {(I // 4) % 4 for I in cols}
    assert js == {1}
    assert abs(sum(lens) - 4 * math.sqrt(2.0)) < 1e-12
