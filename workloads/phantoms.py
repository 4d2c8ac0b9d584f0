"""Seeded phantoms, adjoint inputs and ray samples (input data only).

Recipe (DESIGN.md §4 "Inputs"), following BASELINE.json ``configs``:

* ``uniform``: f_I ~ U[0, 1) drawn in flat-index order from PCG64(seed) (cfg 1).
* ``ellipses`` / ``ellipsoids``: ``count`` shapes, centres uniform in the inner 80 %
  of the field (|c_a| <= 0.4 W_a), semi-axes uniform in [0.05, 0.4] W_a, densities
  uniform in [-0.5, 1], orientation uniform (2D: angle in [0, pi); 3D: normalised
  Gaussian quaternion), overlaps additive, value = sum of densities of the shapes
  containing the unit CENTRE (reading 19).  W_a = N_a * d_a is the field width.
  Evaluated in fp64, stored as fp32.
* adjoint input y ~ U[-1, 1) per ray from PCG64(adj_seed).
* attenuation map mu (the attenuated transform): the config's phantom with its
  densities' absolute values, |f_I|, scaled by 2 / W_max (W_max the widest field width), so a
  chord through the densest region attenuates by exp(-O(1)) as in SPECT; fp32.

Unit centres are the paper's shifted by the image centre and
scaled by the spacing: x_i = x_lo + (i + 1/2) d_x, y_j = y_hi - (j + 1/2) d_y,
z_k = z_hi - (k + 1/2) d_z.  This is input construction, not the transform.
"""
from __future__ import annotations

import numpy as np
import torch


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _shape_params(count: int, widths, seed: int, dim: int):
    rng = _rng(seed)
    w = np.asarray(widths[:dim], dtype=np.float64)
    centers = rng.uniform(-0.4, 0.4, size=(count, dim)) * w
    axes = rng.uniform(0.05, 0.4, size=(count, dim)) * w
    rho = rng.uniform(-0.5, 1.0, size=count)
    if dim == 2:
        psi = rng.uniform(0.0, np.pi, size=count)
        rots = np.stack([np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]]) for a in psi])
    else:
        q = rng.normal(size=(count, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        rots = []
        for a, b, c, d in q:
            rots.append(np.array([
                [a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
                [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
                [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]]))
        rots = np.stack(rots)
    return centers, axes, rho, rots


def make_image(c: dict, device: str | torch.device = "cpu") -> torch.Tensor:
    """fp32 image, C-contiguous [N_z][N_y][N_x] (2D: [1][N_y][N_x]) on ``device``."""
    nx, ny, nz = c["n"]
    dx, dy, dz = c["spacing"]
    cx, cy, cz = c["center"]
    spec = c["image"]
    kind = spec["kind"]
    if kind == "uniform":
        vals = _rng(spec["seed"]).random(nx * ny * nz)  # flat-index order
        return torch.from_numpy(vals.astype(np.float32)).reshape(nz, ny, nx).to(device)
    if kind == "zeros":
        return torch.zeros((nz, ny, nx), dtype=torch.float32, device=device)
    if kind == "ones":
        return torch.ones((nz, ny, nx), dtype=torch.float32, device=device)
    dim = 2 if kind == "ellipses" else 3
    widths = (nx * dx, ny * dy, nz * dz)
    centers, axes, rho, rots = _shape_params(spec["count"], widths, spec["seed"], dim)
    dev = torch.device(device)
    f64 = torch.float64
    xs = (cx - nx * dx / 2) + (torch.arange(nx, dtype=f64, device=dev) + 0.5) * dx
    ys = (cy + ny * dy / 2) - (torch.arange(ny, dtype=f64, device=dev) + 0.5) * dy
    zs = (cz + nz * dz / 2) - (torch.arange(nz, dtype=f64, device=dev) + 0.5) * dz
    img = torch.zeros((nz, ny, nx), dtype=f64, device=dev)
    if dim == 2:
        zs = torch.tensor([cz], dtype=f64, device=dev)
    for s in range(spec["count"]):
        ctr = np.zeros(3)
        ctr[:dim] = centers[s]
        ctr += np.array([cx, cy, cz])
        r = float(np.max(axes[s]))
        # bounding box in index ranges (conservative: radius = largest semi-axis)
        ix = torch.nonzero((xs >= ctr[0] - r) & (xs <= ctr[0] + r)).flatten()
        iy = torch.nonzero((ys >= ctr[1] - r) & (ys <= ctr[1] + r)).flatten()
        if dim == 3:
            iz = torch.nonzero((zs >= ctr[2] - r) & (zs <= ctr[2] + r)).flatten()
        else:
            iz = torch.zeros(1, dtype=torch.long, device=dev)
        if ix.numel() == 0 or iy.numel() == 0 or iz.numel() == 0:
            continue
        x0, x1 = int(ix[0]), int(ix[-1]) + 1
        y0, y1 = int(iy[0]), int(iy[-1]) + 1
        z0, z1 = int(iz[0]), int(iz[-1]) + 1
        R = torch.from_numpy(rots[s]).to(dev)
        ax = torch.from_numpy(axes[s]).to(dev)
        X = (xs[x0:x1] - ctr[0]).view(1, 1, -1)
        Y = (ys[y0:y1] - ctr[1]).view(1, -1, 1)
        if dim == 2:
            # body coordinates q = R^T (p - c)
            q0 = R[0, 0] * X + R[1, 0] * Y
            q1 = R[0, 1] * X + R[1, 1] * Y
            inside = (q0 / ax[0]) ** 2 + (q1 / ax[1]) ** 2 <= 1.0
        else:
            for zc in range(z0, z1, 64):  # chunk z to bound memory
                ze = min(z1, zc + 64)
                Z = (zs[zc:ze] - ctr[2]).view(-1, 1, 1)
                q0 = R[0, 0] * X + R[1, 0] * Y + R[2, 0] * Z
                q1 = R[0, 1] * X + R[1, 1] * Y + R[2, 1] * Z
                q2 = R[0, 2] * X + R[1, 2] * Y + R[2, 2] * Z
                inside = (q0 / ax[0]) ** 2 + (q1 / ax[1]) ** 2 + (q2 / ax[2]) ** 2 <= 1.0
                img[zc:ze, y0:y1, x0:x1] += inside.to(f64) * float(rho[s])
            continue
        img[z0:z1, y0:y1, x0:x1] += inside.to(f64) * float(rho[s])
    return img.to(torch.float32).contiguous()


def make_sino_input(c: dict, device="cpu", seed: int | None = None) -> torch.Tensor:
    """Adjoint input y ~ U[-1, 1) in ray order, shaped [V][rows][cols] fp32."""
    s = c["adj_seed"] if seed is None else seed
    V, R, C = c["n_views"], c["det_rows"], c["det_cols"]
    gen = torch.Generator(device="cpu").manual_seed(int(s))
    y = torch.rand((V, R, C), generator=gen, dtype=torch.float32) * 2 - 1
    return y.to(device)


def make_attenuation(c: dict, device="cpu") -> torch.Tensor:
    """Attenuation map mu >= 0 on the image grid (fp32, same shape as make_image), 1/length."""
    w = max(float(c["n"][a]) * float(c["spacing"][a]) for a in range(3) if int(c["n"][a]) > 1)
    return (make_image(c).abs() * (2.0 / w)).to(device)


def sample_rays(c: dict, count: int, seed: int) -> np.ndarray:
    """Seeded stratified sample of ray ids m = (v*rows + r)*cols + c, sorted, unique.

    Stratified over views: each view block gets count/V (or one draw per view
    chosen at random when count < V), uniform over (row, col) within a view.
    """
    V, R, C = c["n_views"], c["det_rows"], c["det_cols"]
    M = V * R * C
    rng = _rng(seed)
    if count >= M:
        return np.arange(M, dtype=np.int64)
    views = rng.integers(0, V, size=count) if count < V else np.repeat(np.arange(V), count // V + 1)[:count]
    rows = rng.integers(0, R, size=count)
    cols = rng.integers(0, C, size=count)
    ids = np.unique((views.astype(np.int64) * R + rows) * C + cols)
    return ids
