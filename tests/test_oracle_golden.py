"""Pins of the CPU oracle against the paper's printed results (Tables 1-5).

Each test rebuilds the paper's single ray from its printed parameters with the
paper's own transformation formulas (oracle/geometry.py) and compares the oracle's
row to (a) the float32-printed table (+-5e-6) and (b) the exact closed forms
the paper derives (<= 1e-12).
"""
import math

import numpy as np
import pytest

import oracle
from oracle import geometry as G
from conftest import read_table

SQ2, SQ3 = math.sqrt(2.0), math.sqrt(3.0)


def grid(n):
    return dict(n=tuple(n), spacing=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0))


def ray2d(s, phi):
    th, perp = G.par2d_basis(phi)
    return np.array([[s * perp[0], s * perp[1], 0.0]]), np.array([[th[0], th[1], 0.0]])


def ray3d(s1, s2, phi1, phi2):
    th, t1, t2 = G.par3d_basis(phi1, phi2)
    return (s1 * t1 + s2 * t2)[None, :], th[None, :]


def row(c, p, th, mode=1):
    rp, cols, lens = oracle.rows(c, p, th, mode=mode)
    assert rp.shape == (2,)
    return dict(zip(cols.tolist(), lens.tolist()))


def check_table(r, name):
    tab = read_table(name)
    assert sorted(r) == [i for i, _ in tab], (name, sorted(r))
    for i, v in tab:
        assert abs(r[i] - v) <= 5e-6 * max(1.0, abs(v)), (name, i, r[i], v)


@pytest.mark.parametrize("mode", [0, 1])
def test_table1_par2d(mode):
    """Test suite 1: 3x3, ray (1, pi/4) -> Table 1; closed forms P:732."""
    r = row(grid((3, 3, 1)), *ray2d(1.0, math.pi / 4), mode=mode)
    check_table(r, "table1.txt")
    assert abs(r[0] - (2 - SQ2)) < 1e-12
    assert abs(r[1] - (2 * SQ2 - 2)) < 1e-12
    assert abs(r[3] - (2 * SQ2 - 2)) < 1e-12


def test_table2_fan_equiangular():
    """Test suite 2: D=4, alpha=pi/2, gamma=-pi/6 -> (s,phi)=(-2,-pi/6) == (2, 5pi/6)."""
    s, phi = G.fan_equiangular_to_parallel(4.0, math.pi / 2, -math.pi / 6)
    assert abs(s - (-2.0)) < 1e-12 and abs(phi - (-math.pi / 6)) < 1e-12
    sc, phic = G.canonicalize_2d(s, phi)
    assert abs(sc - 2.0) < 1e-12 and abs(phic - 5 * math.pi / 6) < 1e-12  # "it indicates the ray (2, 5pi/6)"
    r = row(grid((4, 4, 1)), *ray2d(float(s), float(phi)))
    check_table(r, "table2.txt")
    assert abs(r[12] - 2 * SQ3 / 3) < 1e-12 and abs(r[13] - (4 - 2 * SQ3)) < 1e-12
    # the canonical representative gives the same row (rays are undirected lines)
    r2 = row(grid((4, 4, 1)), *ray2d(float(sc), float(phic)))
    assert r2.keys() == r.keys() and all(abs(r2[k] - r[k]) < 1e-12 for k in r)


@pytest.mark.parametrize("mode", [0, 1])
def test_table3_par3d(mode):
    """Test suite 3: 3x3x3, ray (0, 0, pi/4, pi/4) -> Table 3; closed forms P:791."""
    r = row(grid((3, 3, 3)), *ray3d(0.0, 0.0, math.pi / 4, math.pi / 4), mode=mode)
    check_table(r, "table3.txt")
    exact = {2: 3 * SQ2 / 2 - 1, 4: 1 - SQ2 / 2, 13: SQ2, 22: 1 - SQ2 / 2, 24: 3 * SQ2 / 2 - 1}
    for k, v in exact.items():
        assert abs(r[k] - v) < 1e-12


def _cone_row(H):
    D, p1, a, b = 4.0, math.pi / 4, math.pi / 12, math.pi / 12
    if H is None:
        s1, s2, phi1, phi2 = G.cone_equiangular_to_parallel(D, p1, a, b)
    else:
        s1, s2, phi1, phi2 = G.helical_equiangular_to_parallel(D, p1, a, b, H)
    return (s1, s2, phi1, phi2), row(grid((4, 4, 4)), *ray3d(s1, s2, phi1, phi2))


def test_table4_cone():
    """Test suite 4: printed parallel parameters, Table 4, closed forms P:828-836."""
    (s1, s2, phi1, phi2), r = _cone_row(None)
    t = math.tan(math.pi / 12)
    assert abs(phi1 - math.pi / 3) < 1e-15 and abs(phi2 - math.pi / 12) < 1e-15
    assert abs(s1 - 4 * math.sin(math.pi / 12)) < 1e-15
    assert abs(s2 - 4 * math.sin(math.pi / 12) * math.cos(math.pi / 12)) < 1e-15
    check_table(r, "table4.txt")
    c12, s12 = math.cos(math.pi / 12), math.sin(math.pi / 12)
    K = (4 - SQ2) * t * math.sin(5 * math.pi / 12) / math.sin(math.pi / 3)
    # voxel (k, j, i) -> I = 16k + 4j + i
    exact = {
        16 + 12 + 0: 2 * (1 - K) / c12,                                  # (1,3,0)
        16 + 8 + 0: 2 * SQ3 / (3 * c12),                                 # (1,2,0)
        16 + 4 + 0: 2 * (K - SQ3 / 3) / c12,                             # (1,1,0)
        0 + 0 + 1: 2 * SQ3 / (3 * c12),                                  # (0,0,1)
        16 + 4 + 1: (1 - (4 * SQ2 - 2) * t) / s12,                       # (1,1,1)
        0 + 4 + 1: (((4 - SQ2) * (SQ2 - 2 * t * math.sin(5 * math.pi / 12) / math.sin(math.pi / 3))
                     + 4 * SQ3 / 3) * t - 1) / s12,                      # (0,1,1)
    }
    assert sorted(exact) == sorted(r)
    for k, v in exact.items():
        assert abs(r[k] - v) < 1e-12, (k, r[k], v)


def test_table5_helical():
    """Test suite 5: H=0 reproduces Table 4 bitwise; H=0.5 -> printed s2,
    Table 5, and the closed forms P:868-876 with the (0,3,0)/(1,3,0) labels swapped (reading 18)."""
    prm0, r0 = _cone_row(0.0)
    prmc, rc = _cone_row(None)
    assert prm0 == prmc and r0 == rc                       # bitwise: H cos(beta) = 0 exactly
    (s1, s2, phi1, phi2), r = _cone_row(0.5)
    c12, s12 = math.cos(math.pi / 12), math.sin(math.pi / 12)
    assert abs(s2 - (4 * c12 * s12 + c12 / 2)) < 1e-15
    check_table(r, "table5.txt")
    t = math.tan(math.pi / 12)
    K = (4 - SQ2) * t * math.sin(5 * math.pi / 12) / math.sin(math.pi / 3)
    A = (0.5 - (4 * SQ2 - 4) * t) / s12                    # printed for voxel (0,3,0)
    B = 2 * (1 - K) / c12 - A                              # printed for voxel (1,3,0)
    exact = {
        8: 2 * SQ3 / (3 * c12),                            # (0,2,0)
        4: 2 * (K - SQ3 / 3) / c12,                        # (0,1,0)
        1: 2 * SQ3 / (3 * c12),                            # (0,0,1)
        5: (2 - (8 - 2 * SQ2) * t * math.sin(5 * math.pi / 12)) / (math.cos(math.pi / 6) * c12),  # (0,1,1)
        12: B,                                             # (0,3,0): the expression printed for (1,3,0)
        28: A,                                             # (1,3,0): the expression printed for (0,3,0)
    }
    assert sorted(exact) == sorted(r)
    for k, v in exact.items():
        assert abs(r[k] - v) < 1e-12, (k, r[k], v)
