"""View-sharded multi-GPU X-ray transform (rays are independent).

One process per GPU.  Rank r of G owns the contiguous view block
[V r / G, V (r + 1) / G) and builds its own plan from that slice of the angle array
(helical source heights are angle based, so shards stay consistent).

* forward: every rank projects its block into its own sinogram slab -- no exchange when x
  is already replicated; ``forward`` can broadcast x from ``src`` first (NCCL).
* adjoint: every rank backprojects its slab into a partial image; the partials are summed
  with one NCCL all_reduce (the path's only real exchange step).

The process group is torch.distributed's (backend "nccl" on GPUs; "gloo" for the CPU tests
of the sharding logic).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def view_block(n_views: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced block of views for ``rank`` (sizes differ by at most 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    return n_views * rank // world, n_views * (rank + 1) // world


def shard_geometry(geometry: dict, rank: int, world: int) -> dict:
    """The sub-geometry of rank ``rank``: same image and detector, its block of view angles."""
    angles = np.asarray(geometry["angles"], dtype=np.float64)
    v0, v1 = view_block(angles.shape[0], rank, world)
    if v1 <= v0:
        raise ValueError(f"rank {rank} of {world} gets no views (n_views={angles.shape[0]})")
    g = dict(geometry)
    g["angles"] = angles[v0:v1]
    g["n_views"] = v1 - v0
    g["view_block"] = (v0, v1)
    return g


class ShardedPlan:
    """A plan over this rank's view block plus the collectives that make it the full operator."""

    def __init__(self, geometry: dict, rank: int | None = None, world: int | None = None,
                 device: int | None = None, group=None, plan_factory=None):
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank, self.world, self.group = rank, world, group
        self.geometry = shard_geometry(geometry, rank, world)
        self.view_block = self.geometry["view_block"]
        if plan_factory is None:
            from .plan import Plan  # local import: the sharding logic is testable without the library
            plan_factory = Plan
        self.plan = plan_factory(self.geometry, device=device)

    def forward(self, img: torch.Tensor, out: torch.Tensor | None = None, broadcast_src: int | None = None):
        """This rank's sinogram slab [views in block][rows][cols] of A img."""
        if broadcast_src is not None and self.world > 1:
            dist.broadcast(img, src=broadcast_src, group=self.group)
        return self.plan.forward(img, out=out)

    def adjoint(self, sino_slab: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """A^T y of the FULL sinogram (replicated on every rank): local partial + all_reduce(sum)."""
        part = self.plan.adjoint(sino_slab, out=out)
        if self.world > 1:
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group)
        return part

    def forward_attenuated(self, img: torch.Tensor, mu: torch.Tensor, out: torch.Tensor | None = None,
                           broadcast_src: int | None = None):
        """This rank's slab of the attenuated transform: rays are independent, so
        the view split is the same as for A; img and mu replicated (broadcast from src if asked)."""
        if broadcast_src is not None and self.world > 1:
            dist.broadcast(img, src=broadcast_src, group=self.group)
            dist.broadcast(mu, src=broadcast_src, group=self.group)
        return self.plan.forward_attenuated(img, mu, out=out)

    def adjoint_attenuated(self, sino_slab: torch.Tensor, mu: torch.Tensor,
                           out: torch.Tensor | None = None) -> torch.Tensor:
        """R_mu^T y of the full sinogram: local partial over this rank's views + all_reduce(sum)."""
        part = self.plan.adjoint_attenuated(sino_slab, mu, out=out)
        if self.world > 1:
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group)
        return part


def gather_sinogram(slab: torch.Tensor, n_views_total: int, rank: int, world: int, group=None) -> torch.Tensor:
    """Assemble the full sinogram on every rank (testing / I/O helper; not on the hot path)."""
    rows, cols = slab.shape[1], slab.shape[2]
    full = torch.zeros((n_views_total, rows, cols), dtype=slab.dtype, device=slab.device)
    v0, v1 = view_block(n_views_total, rank, world)
    full[v0:v1] = slab
    if world > 1:
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


# --------------------------------------------------------------------- z-slab sharding (par3d)
def zslab_partition(geometry: dict, world: int) -> list[tuple[int, int, int, int]]:
    """Zero-communication partition of a 3D parallel beam WITHOUT tilt (every ray horizontal:
    z = v_r, fixed z cell k(r) = floor((z_hi - v_r) / d_z), DESIGN reading 5): rank r owns the
    image slab k in [k0, k1) and exactly the detector rows whose rays lie in it, [r0, r1).
    Rows outside the image in z (no unit) go to the nearest slab.  Returns [(k0, k1, r0, r1)].
    (the forward and adjoint of a slab need no exchange at all.)"""
    if geometry["beam"] != "par3d" or abs(float(geometry.get("tilt", 0.0))) != 0.0:
        raise ValueError("z-slab sharding needs a 3D parallel beam with tilt 0")
    nz = int(geometry["n"][2])
    dz = float(geometry["spacing"][2])
    z_hi = float(geometry.get("center", (0, 0, 0))[2]) + nz * dz / 2.0
    R = int(geometry["det_rows"])
    dv = float(geometry["det_spacing"][1])
    off = float(geometry.get("det_offset", (0.0, 0.0))[1])
    v = (np.arange(R) - (R - 1) / 2.0) * dv + off
    kr = np.clip(np.floor((z_hi - v * np.cos(0.0)) / dz), 0, nz - 1).astype(np.int64)   # as ray_z
    if world < 1 or world > nz:
        raise ValueError(f"world {world} must be in [1, N_z={nz}]")
    out = []
    for r in range(world):
        k0, k1 = nz * r // world, nz * (r + 1) // world
        rows = np.nonzero((kr >= k0) & (kr < k1))[0]
        r0, r1 = (int(rows.min()), int(rows.max()) + 1) if rows.size else (0, 0)
        out.append((k0, k1, r0, r1))
    return out


def zslab_geometry(geometry: dict, k0: int, k1: int, r0: int, r1: int) -> dict:
    """Sub-geometry of one slab: image rows k0..k1 (same x, y; centre moved in z) and detector rows
    r0..r1 (same physical row positions: the detector offset absorbs the shift).  The slab box
    z_hi - k0 d_z is exact when d_z and z_hi are dyadic (cfg 3: 1.0, 128); otherwise a row lying
    exactly on a z plane may round into the neighbouring cell (DESIGN reading 2 ties)."""
    g = dict(geometry)
    nx, ny, nz = geometry["n"]
    dz = float(geometry["spacing"][2])
    cx, cy, cz = geometry.get("center", (0.0, 0.0, 0.0))
    z_hi = cz + nz * dz / 2.0
    g["n"] = (nx, ny, k1 - k0)
    g["center"] = (cx, cy, z_hi - (k0 + k1) * dz / 2.0)        # slab [z_hi - k1 dz, z_hi - k0 dz]
    R = int(geometry["det_rows"])
    dv = float(geometry["det_spacing"][1])
    off_u, off_v = geometry.get("det_offset", (0.0, 0.0))
    Rn = r1 - r0
    g["det_rows"] = Rn
    g["det_offset"] = (off_u, off_v + (r0 - (R - 1) / 2.0 + (Rn - 1) / 2.0) * dv)
    g["zslab"] = (k0, k1, r0, r1)
    return g


class ZSlabShardedPlan:
    """3D parallel beam without tilt, sharded by z slabs with NO exchange (zslab_partition): rank r
    owns the image slab x[k0:k1] and the detector rows [r0, r1) of every view; forward maps the slab
    to those sinogram rows, adjoint maps them back to the slab.  Results stay distributed; gather
    helpers assemble them (tests / I/O, not the hot path)."""

    def __init__(self, geometry: dict, rank: int | None = None, world: int | None = None,
                 device: int | None = None, group=None, plan_factory=None):
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank, self.world, self.group = rank, world, group
        self.parts = zslab_partition(geometry, world)
        k0, k1, r0, r1 = self.parts[rank]
        self.slab, self.rows = (k0, k1), (r0, r1)
        self.geometry = zslab_geometry(geometry, k0, k1, r0, r1)
        if plan_factory is None:
            from .plan import Plan
            plan_factory = Plan
        self.plan = plan_factory(self.geometry, device=device)

    def forward(self, img_slab: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Sinogram rows [views][r0:r1][cols] of A x from this rank's slab x[k0:k1] alone."""
        return self.plan.forward(img_slab, out=out)

    def adjoint(self, sino_rows: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Slab [k0:k1] of A^T y from this rank's sinogram rows alone."""
        return self.plan.adjoint(sino_rows, out=out)

    def forward_attenuated(self, img_slab: torch.Tensor, mu_slab: torch.Tensor,
                           out: torch.Tensor | None = None) -> torch.Tensor:
        """Attenuated transform (N4) of the slab: a horizontal ray never leaves its slab, so its
        attenuation along the whole ray is the slab's -- no exchange either."""
        return self.plan.forward_attenuated(img_slab, mu_slab, out=out)

    def adjoint_attenuated(self, sino_rows: torch.Tensor, mu_slab: torch.Tensor,
                           out: torch.Tensor | None = None) -> torch.Tensor:
        return self.plan.adjoint_attenuated(sino_rows, mu_slab, out=out)

    def gather_image(self, slab: torch.Tensor, nz: int) -> torch.Tensor:
        full = torch.zeros((nz,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=slab.device)
        full[self.slab[0]:self.slab[1]] = slab
        if self.world > 1:
            dist.all_reduce(full, op=dist.ReduceOp.SUM, group=self.group)
        return full
