"""Shared helpers for the GPU parity tests (CUDA path vs oracle on the same seeded inputs)."""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle
from oracle import geometry as G
import workloads

FWD_TOL = 1e-5      # north_star: per-ray |err| / max|sino| <= 1e-5
ADJ_TOL = 1e-4      # north_star: relative L2 of the adjoint
DOT_TOL = 1e-5      # north_star: dot-product test
LEN_TOL = 1e-9      # fp64 CSR lengths vs fp64 oracle (different rounding order only)

# oracle-sized versions of the five configs: several tiles, ragged tails (detector sizes that are
# not multiples of the 32-lane warp or the 256-thread block)
SMALL = {
    1: dict(),
    2: dict(n=(96, 96, 1), n_views=36, det_cols=147),
    3: dict(n=(40, 40, 40), n_views=12, det_cols=61, det_rows=45),
    4: dict(n=(48, 48, 48), n_views=10, det_cols=97, det_rows=71),
    5: dict(n=(64, 64, 32), n_views=24, det_cols=93, det_rows=37),
}


def small_config(idx: int) -> dict:
    return workloads.scaled(idx, **SMALL[idx])


def ray_ids_all(c):
    return np.arange(workloads.configs.n_rays(c), dtype=np.int64)


def oracle_csr(c, ids, mode=2):
    p, th = G.rays(c, ids)
    return oracle.rows(c, p, th, mode=mode)


def oracle_forward(c, img_cpu, ids, mode=2):
    p, th = G.rays(c, ids)
    return oracle.forward(c, img_cpu.numpy().reshape(-1), p, th, mode=mode)


def stratified_ranges(c, n_ranges: int, width: int, seed: int):
    """Reading 21: n_ranges ranges of `width` consecutive ray ids, one per stratum of the ray-id
    space (uniform over (view, row, column)); returns the list of (begin, end)."""
    M = workloads.configs.n_rays(c)
    rng = np.random.Generator(np.random.PCG64(seed))
    edges = np.linspace(0, M - width, n_ranges + 1).astype(np.int64)
    out = []
    for a, b in zip(edges[:-1], edges[1:]):
        s = int(rng.integers(a, max(a + 1, b)))
        out.append((s, s + width))
    return out


def oracle_adjoint(c, y, ids, mode=2):
    p, th = G.rays(c, ids)
    return oracle.adjoint(c, y, p, th, mode=mode)


def compare_csr(gpu, ref, ids_desc=""):
    """Index sets bit-exact per row; lengths to LEN_TOL."""
    rp_g, cols_g, lens_g = [t.cpu().numpy() if torch.is_tensor(t) else t for t in gpu]
    rp_o, cols_o, lens_o = ref
    assert rp_g.shape == rp_o.shape, ids_desc
    if not np.array_equal(rp_g, rp_o):
        bad = np.nonzero(np.diff(rp_g) != np.diff(rp_o))[0]
        raise AssertionError(f"{ids_desc}: row sizes differ in {len(bad)} rows, first {bad[:5]}: "
                             f"gpu {np.diff(rp_g)[bad[:5]]} oracle {np.diff(rp_o)[bad[:5]]}")
    assert np.array_equal(cols_g, cols_o), ids_desc
    if lens_o.size:
        err = np.max(np.abs(lens_g - lens_o) / np.maximum(1.0, np.abs(lens_o)))
        assert err <= LEN_TOL, (ids_desc, err)


def fwd_err(gpu_vals, ref_vals, scale=None):
    ref = np.asarray(ref_vals, dtype=np.float64)
    g = np.asarray(gpu_vals, dtype=np.float64)
    s = scale if scale is not None else max(np.max(np.abs(ref)), 1e-30)
    return float(np.max(np.abs(g - ref)) / s)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def constructed_plans():
    """The 32 constructed cfg-1 rays as auxiliary par2d plans on the 64^2 grid:
    (geometry, {bin: expected row size}) where s lands exactly on the listed values."""
    base = workloads.config(1)
    out = []
    for phi, ncols, du, svals in ((0.0, 65, 1.0, [32, 31, 16, 1, 0, -1, -31, -32]),
                                  (math.pi / 2, 65, 1.0, [32, 31, 16, 1, 0, -1, -31, -32]),
                                  (math.pi / 4, 129, math.sqrt(2.0) / 2, [0, 1, -1, 31, -31, 63, -63, 64]),
                                  (3 * math.pi / 4, 129, math.sqrt(2.0) / 2, [0, 1, -1, 31, -31, 63, -63, 64])):
        g = dict(base)
        g.update(n_views=1, angles=np.array([phi]), det_cols=ncols, det_spacing=(du, 1.0))
        half = (ncols - 1) // 2
        if phi in (0.0, math.pi / 2):
            expect = {half + s: (64 if 0 <= 32 - s <= 63 else 0) for s in svals}
        else:
            expect = {half + m: max(0, 64 - abs(m)) for m in svals}
        out.append((g, expect))
    return out
