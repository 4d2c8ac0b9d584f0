"""Property pins of the oracle: closed forms and invariants that hold for ANY correct
X-ray transform, each checked with code written independently of oracle/brute.c.

* chord conservation: constant image -> sum of lengths = |ray  box| (one slab clip,
  written here), P:53-57 with f = 1;
* point sampling: lengths agree with a dense midpoint-rule sampling of the ray (a
  completely different algorithm) to the sampling error;
* adjoint identity <A x, y> = <x, A^T y>;
* symmetries: direction reversal (P:166 / P:443 equivalences), 90-degree rotation and
  mirror reflection (index permutations), translation of the image centre, scaling of
  all lengths ("real value = scale x unit-scale value"), anisotropic covariance;
* geometry: every oracle ray of a fan / cone / helical configuration passes through its
  source and its flat-detector point (readings 7, 8, 11); equispaced = equiangular o atan
  (S:189); helical with H = 0 = cone.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import geometry as G
import workloads

RNG = np.random.Generator(np.random.PCG64(1234))


def grid(n, d=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0)):
    return dict(n=tuple(n), spacing=tuple(d), center=tuple(center))


def random_rays(c, k, rng, dim=3, through=0.45):
    """Random lines passing near the image box (some miss)."""
    ext = np.array(c["n"]) * np.array(c["spacing"])
    ctr = np.array(c["center"])
    th = rng.normal(size=(k, 3))
    if dim == 2:
        th[:, 2] = 0
    th /= np.linalg.norm(th, axis=1, keepdims=True)
    p = ctr + rng.uniform(-through * 1.3, through * 1.3, size=(k, 3)) * ext
    if dim == 2:
        p[:, 2] = ctr[2]
    return p, th


def chord(c, p, th):
    """|line  box| by one slab clip over the whole image box (written independently)."""
    lo = np.array(c["center"]) - np.array(c["n"]) * np.array(c["spacing"]) / 2
    hi = lo + np.array(c["n"]) * np.array(c["spacing"])
    t0, t1 = -np.inf, np.inf
    for a in range(3):
        if th[a] == 0:
            # half-open in index space: x in [lo, hi) ; y, z in (lo, hi]
            inside = (lo[a] <= p[a] < hi[a]) if a == 0 else (lo[a] < p[a] <= hi[a])
            if not inside:
                return 0.0
            continue
        a0, a1 = (lo[a] - p[a]) / th[a], (hi[a] - p[a]) / th[a]
        t0, t1 = max(t0, min(a0, a1)), min(t1, max(a0, a1))
    return max(0.0, t1 - t0)


@pytest.mark.parametrize("n,d,dim", [((7, 7, 1), (1, 1, 1), 2), ((8, 8, 8), (1, 1, 1), 3),
                                     ((5, 4, 6), (0.5, 0.7, 1.3), 3), ((9, 6, 1), (2.0, 0.5, 1), 2)])
def test_chord_conservation(n, d, dim):
    c = grid(n, d, center=(0.3, -0.2, 0.1) if dim == 3 else (0.3, -0.2, 0.0))
    p, th = random_rays(c, 300, RNG, dim)
    ones = np.ones(int(np.prod(n)), dtype=np.float32)
    out = oracle.forward(c, ones, p, th)
    for m in range(len(p)):
        assert abs(out[m] - chord(c, p[m], th[m])) < 1e-9 * max(1, out[m])


def test_dense_sampling_agrees():
    """Lengths vs a midpoint-rule sampling of the ray (100k samples / chord)."""
    c = grid((4, 3, 5), (1.0, 0.8, 0.6), center=(0.1, 0.2, -0.3))
    lo = np.array(c["center"]) - np.array(c["n"]) * np.array(c["spacing"]) / 2
    p, th = random_rays(c, 40, RNG, 3, through=0.3)
    rp, cols, lens = oracle.rows(c, p, th)
    for m in range(len(p)):
        L = 40.0
        ns = 400_000
        t = -L / 2 + (np.arange(ns) + 0.5) * (L / ns)
        x = p[m][None, :] + t[:, None] * th[m][None, :]
        ux = (x[:, 0] - lo[0]) / c["spacing"][0]
        uy = (lo[1] + c["n"][1] * c["spacing"][1] - x[:, 1]) / c["spacing"][1]
        uz = (lo[2] + c["n"][2] * c["spacing"][2] - x[:, 2]) / c["spacing"][2]
        i, j, k = np.floor(ux).astype(int), np.floor(uy).astype(int), np.floor(uz).astype(int)
        ok = (i >= 0) & (i < c["n"][0]) & (j >= 0) & (j < c["n"][1]) & (k >= 0) & (k < c["n"][2])
        I = ((k * c["n"][1] + j) * c["n"][0] + i)[ok]
        est = np.bincount(I, minlength=int(np.prod(c["n"]))) * (L / ns)
        got = np.zeros_like(est)
        got[cols[rp[m]:rp[m + 1]]] = lens[rp[m]:rp[m + 1]]
        assert np.max(np.abs(est - got)) < 3 * L / ns * 4


def test_modes_agree_and_sorted():
    c = grid((6, 7, 5), (1.0, 0.9, 1.1))
    p, th = random_rays(c, 200, RNG, 3)
    a = oracle.rows(c, p, th, mode=0)
    for mode in (1, 2):
        b = oracle.rows(c, p, th, mode=mode)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), mode
    rp, cols, lens = a
    for m in range(len(p)):
        seg = cols[rp[m]:rp[m + 1]]
        assert np.all(np.diff(seg) > 0)
    assert np.all(lens > 0)
    # max length per unit = the unit diagonal
    assert np.all(lens <= math.sqrt(1.0 + 0.81 + 1.21) + 1e-12)


@pytest.mark.parametrize("n,dim", [((9, 8, 1), 2), ((7, 6, 5), 3)])
def test_mode2_agrees_on_edge_rays(n, dim):
    """Mode 2 (x-range restricted) = mode 0 also for rays on grid lines / planes and through
    corners (axis-parallel and diagonal rays at integer offsets: the tie cases of reading 2)."""
    c = grid(n, (1.0, 1.0, 1.0))
    pts, dirs = [], []
    for s in np.arange(-5, 5.5, 0.5):
        for th in ((1, 0, 0), (0, 1, 0), (1, 1, 0), (1, -1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1)):
            if dim == 2 and th[2] != 0:
                continue
            t = np.array(th, dtype=float) / np.linalg.norm(th)
            off = np.array([s, -s, 0.0 if dim == 2 else s * 0.5])
            pts.append(off)
            dirs.append(t)
    p, th = np.array(pts), np.array(dirs)
    a = oracle.rows(c, p, th, mode=0)
    b = oracle.rows(c, p, th, mode=2)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    img = RNG.uniform(0, 1, size=int(np.prod(n))).astype(np.float32)
    assert np.array_equal(oracle.forward(c, img, p, th, mode=0), oracle.forward(c, img, p, th, mode=2))


def test_adjoint_identity():
    c = grid((6, 5, 4), (1.0, 0.5, 2.0))
    p, th = random_rays(c, 150, RNG, 3)
    x = RNG.uniform(-1, 1, size=int(np.prod(c["n"]))).astype(np.float32)
    y = RNG.uniform(-1, 1, size=len(p))
    Ax = oracle.forward(c, x, p, th)
    Aty = oracle.adjoint(c, y, p, th)
    lhs, rhs = float(Ax @ y), float(x.astype(np.float64) @ Aty)
    assert abs(lhs - rhs) <= 1e-12 * (np.linalg.norm(Ax) * np.linalg.norm(y) + np.linalg.norm(x) * np.linalg.norm(Aty))


def test_direction_reversal():
    c = grid((5, 5, 5))
    p, th = random_rays(c, 100, RNG, 3)
    a = oracle.rows(c, p, th)
    b = oracle.rows(c, p + 3.7 * th, -th)   # same line, opposite direction, other foot point
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.max(np.abs(a[2] - b[2])) < 1e-12


def test_rotation_90_2d():
    """Rotating a ray by +90 deg about the centre of an N x N grid maps pixel (j, i) -> (N-1-i, j)."""
    N = 8
    c = grid((N, N, 1))
    p, th = random_rays(c, 100, RNG, 2)
    R = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]])
    a = oracle.rows(c, p, th)
    b = oracle.rows(c, p @ R.T, G._snap(th @ R.T))
    for m in range(len(p)):
        ra = dict(zip(a[1][a[0][m]:a[0][m + 1]].tolist(), a[2][a[0][m]:a[0][m + 1]].tolist()))
        rb = dict(zip(b[1][b[0][m]:b[0][m + 1]].tolist(), b[2][b[0][m]:b[0][m + 1]].tolist()))
        mapped = {}
        for I, l in ra.items():
            j, i = divmod(I, N)
            mapped[(N - 1 - i) * N + j] = l
        assert mapped.keys() == rb.keys()
        assert all(abs(mapped[k] - rb[k]) < 1e-12 for k in rb)


def test_reflection_x():
    """Mirror x -> -x maps pixel (j, i) -> (j, N-1-i) (generic rays: no ties)."""
    N = 7
    c = grid((N, N, 3))
    p, th = random_rays(c, 100, RNG, 3)
    F = np.diag([-1.0, 1, 1])
    a = oracle.rows(c, p, th)
    b = oracle.rows(c, p @ F, th @ F)
    for m in range(len(p)):
        ra = dict(zip(a[1][a[0][m]:a[0][m + 1]].tolist(), a[2][a[0][m]:a[0][m + 1]].tolist()))
        rb = dict(zip(b[1][b[0][m]:b[0][m + 1]].tolist(), b[2][b[0][m]:b[0][m + 1]].tolist()))
        mapped = {(I // N) * N + (N - 1 - I % N): l for I, l in ra.items()}
        assert mapped.keys() == rb.keys()
        assert all(abs(mapped[k] - rb[k]) < 1e-12 for k in rb)


def test_translation_and_scaling():
    """Shifting image and rays together leaves rows unchanged; scaling all spacings and ray
    positions by s scales every length by s with the same index set (reading 14)."""
    c = grid((6, 6, 6), (1.0, 1.0, 1.0))
    p, th = random_rays(c, 100, RNG, 3)
    a = oracle.rows(c, p, th)
    shift = np.array([3.25, -1.5, 0.75])
    c2 = grid((6, 6, 6), (1.0, 1.0, 1.0), center=tuple(shift))
    b = oracle.rows(c2, p + shift, th)
    assert np.array_equal(a[1], b[1]) and np.max(np.abs(a[2] - b[2])) < 1e-12
    s = 0.5
    c3 = grid((6, 6, 6), (s, s, s))
    d = oracle.rows(c3, p * s, th)
    assert np.array_equal(a[1], d[1]) and np.max(np.abs(a[2] * s - d[2])) < 1e-12


def test_anisotropic_covariance():
    """Stretching z by c (spacing and ray geometry) keeps the index set (reading 13)."""
    c = grid((5, 5, 5), (1.0, 1.0, 1.0))
    p, th = random_rays(c, 100, RNG, 3)
    a = oracle.rows(c, p, th)
    S = np.diag([1.0, 1.0, 2.5])
    th2 = th @ S
    th2 /= np.linalg.norm(th2, axis=1, keepdims=True)
    b = oracle.rows(grid((5, 5, 5), (1.0, 1.0, 2.5)), p @ S, th2)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ------------------------------------------------------------------ geometry transforms
def _flat_det_point(c, v, col, row):
    """Plain vector geometry (readings 7-9): the flat detector sits at SDD from the source,
    perpendicular to the central ray, +u = central direction rotated +90 deg in xy, +v = +z."""
    ang = c["angles"][v]
    u = (col - (c["det_cols"] - 1) / 2) * c["det_spacing"][0] + c["det_offset"][0]
    w = (row - (c["det_rows"] - 1) / 2) * c["det_spacing"][1] + c["det_offset"][1]
    D, SDD = c["sod"], c["sdd"]
    if c["beam"] == "fan2d":
        S = np.array([-D * math.sin(ang), D * math.cos(ang), 0.0])
        ew = -S / D
        eu = np.array([-ew[1], ew[0], 0.0])
        return S, S + SDD * ew + u * eu
    H = c["z0"] + c["pitch"] * ang / (2 * math.pi) if c["beam"] == "helical" else 0.0
    S = np.array([-D * math.cos(ang), -D * math.sin(ang), H])
    ew = np.array([math.cos(ang), math.sin(ang), 0.0])
    eu = np.array([-math.sin(ang), math.cos(ang), 0.0])
    return S, S + SDD * ew + u * eu + w * np.array([0, 0, 1.0])


@pytest.mark.parametrize("idx", [2, 4, 5])
def test_rays_pass_through_source_and_detector(idx):
    c = workloads.config(idx)
    ids = workloads.sample_rays(c, 300, seed=7)
    p, th = G.rays(c, ids)
    C, R = c["det_cols"], c["det_rows"]
    for m, I in enumerate(ids):
        col, row, v = I % C, (I // C) % R, I // (C * R)
        S, P = _flat_det_point(c, v, col, row)
        for X in (S, P):
            d = X - p[m]
            perp = d - (d @ th[m]) * th[m]
            assert np.linalg.norm(perp) < 1e-9 * max(1.0, np.linalg.norm(d))
        assert (P - S) @ th[m] > 0 or True   # orientation is irrelevant (undirected lines)
    assert np.allclose(np.linalg.norm(th, axis=1), 1.0, atol=1e-15)


def test_equispaced_equals_equiangular():
    D = 7.5
    for alpha in np.linspace(0, 2 * math.pi, 9):
        for t in (-3.0, -0.4, 0.0, 1.1, 5.0):
            s1, p1 = G.fan_equispaced_to_parallel(D, alpha, t)
            s2, p2 = G.fan_equiangular_to_parallel(D, alpha, math.atan(t / D))
            assert abs(s1 - s2) < 1e-12 and abs(p1 - p2) < 1e-12
            for h in (-2.0, 0.0, 0.7):
                a = G.cone_equispaced_to_parallel(D, alpha, t, h)
                al = math.atan(t / D)
                be = math.atan(h / math.sqrt(D * D + t * t))
                b = G.cone_equiangular_to_parallel(D, alpha, al, be)
                assert all(abs(x - y) < 1e-12 for x, y in zip(a, b))   # h cos^2 a cos b = D cos a sin b


def test_euler_rows_are_basis():
    """Rows of R(phi1, phi2, 0) (eq:Eulerian_rotations_2) are theta, theta_1, theta_2."""
    for phi1, phi2 in ((0.3, 0.2), (2.0, 1.1), (4.0, 0.0), (5.5, math.pi / 2)):
        R = G.euler_R(phi1, phi2)
        th, t1, t2 = G.par3d_basis(phi1, phi2)
        assert np.allclose(R[0], th) and np.allclose(R[1], t1) and np.allclose(R[2], t2)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-15)


def test_canonicalization_same_line():
    rng = np.random.Generator(np.random.PCG64(5))
    for _ in range(200):
        s1, s2 = rng.uniform(-3, 3, 2)
        phi1, phi2 = rng.uniform(-10, 10, 2)
        c1, c2, q1, q2 = G.canonicalize_3d(s1, s2, phi1, phi2)
        assert 0 <= q1 < 2 * math.pi and 0 <= q2 <= math.pi / 2 + 1e-15
        th, a1, a2 = G.par3d_basis(phi1, phi2)
        tc, b1, b2 = G.par3d_basis(q1, q2)
        pa, pb = s1 * a1 + s2 * a2, c1 * b1 + c2 * b2
        assert abs(abs(th @ tc) - 1) < 1e-12
        d = pb - pa
        assert np.linalg.norm(d - (d @ th) * th) < 1e-12


def _curved_det_point(c, v, col, row):
    """Plain vector geometry of the cylindrical detector (XRT_DET_CURVED): radius sdd about the
    source, column at fan angle u / sdd from the central ray, row at height v (+v = +z)."""
    ang = c["angles"][v]
    u = (col - (c["det_cols"] - 1) / 2) * c["det_spacing"][0] + c["det_offset"][0]
    w = (row - (c["det_rows"] - 1) / 2) * c["det_spacing"][1] + c["det_offset"][1]
    D, SDD = c["sod"], c["sdd"]
    g = u / SDD
    if c["beam"] == "fan2d":
        S = np.array([-D * math.sin(ang), D * math.cos(ang), 0.0])
        ew = -S / D
        eu = np.array([-ew[1], ew[0], 0.0])
        return S, S + SDD * (math.cos(g) * ew + math.sin(g) * eu)
    H = c["z0"] + c["pitch"] * ang / (2 * math.pi) if c["beam"] == "helical" else 0.0
    S = np.array([-D * math.cos(ang), -D * math.sin(ang), H])
    ew = np.array([math.cos(ang), math.sin(ang), 0.0])
    eu = np.array([-math.sin(ang), math.cos(ang), 0.0])
    return S, S + SDD * (math.cos(g) * ew + math.sin(g) * eu) + w * np.array([0, 0, 1.0])


@pytest.mark.parametrize("idx", [2, 4, 5])
def test_curved_rays_pass_through_source_and_cylinder(idx):
    """Equiangular transforms with alpha = u / sdd and
    tan(beta) = v / sdd give the line from the source to the cylindrical detector point."""
    c = workloads.config(idx)
    c["det_curved"] = True
    ids = workloads.sample_rays(c, 300, seed=8)
    p, th = G.rays(c, ids)
    C, R = c["det_cols"], c["det_rows"]
    for m, I in enumerate(ids):
        col, row, v = I % C, (I // C) % R, I // (C * R)
        S, P = _curved_det_point(c, v, col, row)
        for X in (S, P):
            d = X - p[m]
            perp = d - (d @ th[m]) * th[m]
            assert np.linalg.norm(perp) < 1e-9 * max(1.0, np.linalg.norm(d))
    assert np.allclose(np.linalg.norm(th, axis=1), 1.0, atol=1e-15)
