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


def gather_sinogram(slab: torch.Tensor, n_views_total: int, rank: int, world: int, group=None) -> torch.Tensor:
    """Assemble the full sinogram on every rank (testing / I/O helper; not on the hot path)."""
    rows, cols = slab.shape[1], slab.shape[2]
    full = torch.zeros((n_views_total, rows, cols), dtype=slab.dtype, device=slab.device)
    v0, v1 = view_block(n_views_total, rank, world)
    full[v0:v1] = slab
    if world > 1:
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full
