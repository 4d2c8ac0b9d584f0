"""View-sharded multi-GPU X-ray transform (rays are independent).

One process per GPU.  Rank r of G owns the contiguous view block
[V r / G, V (r + 1) / G) and builds its own plan from that slice of the angle array
(helical source heights are angle based, so shards stay consistent).

* forward: every rank projects its block into its own sinogram slab -- no exchange when x
  is already replicated; ``forward`` can broadcast x from ``src`` first (NCCL).
* adjoint: every rank backprojects its slab into a partial image; the partials are summed
  with NCCL all_reduce (the path's only real exchange step).  With the staged adjoint
  (xrt_adjoint_stages / xrt_adjoint_stage) each z slab of the image is reduced as soon as no later
  band of detector rows can reach it, overlapping the reduction with the remaining bands.
* helical (cfg 5): a contiguous view block sees only a z window of the image (the source rises
  with the angle), so ``adjoint_windowed`` exchanges only the overlaps of neighbouring windows
  (P2P) and ``forward`` needs x only on the window -- traffic ~ overlap, not image size.

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
        self.full_geometry = geometry
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

    def adjoint(self, sino_slab: torch.Tensor, out: torch.Tensor | None = None, overlap: bool = True) -> torch.Tensor:
        """A^T y of the FULL sinogram (replicated on every rank): local partial + all_reduce(sum).
        overlap: run the staged adjoint and all-reduce each final z slab asynchronously while the
        next band computes (same result up to fp32 reassociation of the reduction)."""
        if self.world == 1 or not overlap or not hasattr(self.plan, "adjoint_stages"):
            part = self.plan.adjoint(sino_slab, out=out)
            if self.world > 1:
                dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group)
            return part
        if out is None:
            out = torch.empty(self.plan.image_shape, dtype=sino_slab.dtype, device=sino_slab.device)
        works = []
        for s, (k0, k1) in enumerate(self.plan.adjoint_stages()):
            self.plan.adjoint_stage(sino_slab, out, s)
            if k1 > k0:
                works.append(dist.all_reduce(out[k0:k1], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        for w in works:
            w.wait()
        return out

    # ---------------------------------------------------------------- helical z windows
    def window(self, rank: int | None = None) -> tuple[int, int]:
        """Image rows [k0, k1) that the rays of ``rank``'s view block can reach (conservative)."""
        r = self.rank if rank is None else rank
        return zwindow(shard_geometry(self.full_geometry, r, self.world))

    def adjoint_windowed(self, sino_slab: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """A^T y restricted to this rank's z window: the local partial plus the overlapping rows of
        the other ranks' partials (P2P, only the overlaps travel).  Rows outside the window hold this
        rank's partial (zero: no ray of the block reaches them)."""
        part = self.plan.adjoint(sino_slab, out=out)
        if self.world == 1:
            return part
        k0, k1 = self.window()
        ops, bufs = [], []
        for q in range(self.world):
            if q == self.rank:
                continue
            a0, a1 = self.window(q)
            lo, hi = max(k0, a0), min(k1, a1)
            if hi <= lo:
                continue
            buf = torch.empty_like(part[lo:hi])
            ops.append((True, part[lo:hi].contiguous(), q))
            ops.append((False, buf, q))
            bufs.append((lo, hi, buf))
        self._p2p(ops)
        for lo, hi, buf in bufs:
            part[lo:hi] += buf
        return part

    def _p2p(self, ops) -> None:
        """One batch of point-to-point transfers, ops = [(is_send, tensor, peer)].  With the gloo
        backend (CPU tests; the functional N > 1 check of bench.py on fewer GPUs than ranks) CUDA
        tensors are staged through host memory, which gloo's send / recv require."""
        if not ops:
            return
        stage = dist.get_backend(self.group) == "gloo" and ops[0][1].is_cuda
        work = [(snd, t.cpu() if stage else t, q) for snd, t, q in ops]
        p2p = [dist.P2POp(dist.isend if snd else dist.irecv, t, q, group=self.group) for snd, t, q in work]
        for w in dist.batch_isend_irecv(p2p):
            w.wait()
        if stage:
            for (snd, t, _), (_, th, _) in zip(ops, work):
                if not snd:
                    t.copy_(th)

    def scatter_windows(self, img: torch.Tensor, src: int = 0) -> torch.Tensor:
        """Send every rank the rows of ``img`` (valid on ``src``) in its z window (P2P): the
        windowed counterpart of broadcasting x before the forward."""
        if self.world == 1:
            return img
        ops = []
        if self.rank == src:
            for q in range(self.world):
                if q != src:
                    a0, a1 = self.window(q)
                    ops.append((True, img[a0:a1].contiguous(), q))
        else:
            k0, k1 = self.window()
            buf = torch.empty_like(img[k0:k1])
            ops.append((False, buf, src))
        self._p2p(ops)
        if self.rank != src:
            img[k0:k1] = buf
        return img

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


def zwindow(g: dict) -> tuple[int, int]:
    """Image rows [k0, k1) (of [N_z][N_y][N_x]) that any ray of geometry ``g`` can reach: z of a ray
    at in-plane distance rho from the source is affine in the row coordinate v (cone / helical:
    z = H + v rho / sdd, P:631-661 with reading 8), so the extreme rows, the extreme rho over the image
    square and the extreme source heights of the views bound it; parallel beams: v / cos(tilt) +-
    R tan(tilt).  Two-cell margin (conservative; rows outside receive nothing)."""
    nx, ny, nz = (int(v) for v in g["n"])
    dx, dy, dz = (float(v) for v in g["spacing"])
    cx, cy, cz = g.get("center", (0.0, 0.0, 0.0))
    if g["beam"] in ("par2d", "fan2d"):
        return 0, 1
    R = float(np.hypot(nx * dx / 2 + abs(cx), ny * dy / 2 + abs(cy)))
    rows = int(g["det_rows"])
    dv = float(g["det_spacing"][1])
    off = float(g.get("det_offset", (0.0, 0.0))[1])
    v = np.array([-(rows - 1) / 2.0, (rows - 1) / 2.0]) * dv + off
    ang = np.asarray(g["angles"], dtype=np.float64)
    if g["beam"] == "par3d":
        t = float(g.get("tilt", 0.0))
        z = np.concatenate([v / np.cos(t) - R * abs(np.tan(t)), v / np.cos(t) + R * abs(np.tan(t))])
    else:
        sod, sdd = float(g["sod"]), float(g["sdd"])
        rho = np.array([max(0.0, sod - R), sod + R])
        H = np.zeros(1)
        if g["beam"] == "helical":
            H = float(g["z0"]) + float(g["pitch"]) * ang / (2 * np.pi)
        zz = np.outer(v, rho).ravel() / sdd
        z = np.concatenate([zz + H.min(), zz + H.max()])
    z_hi = float(cz) + nz * dz / 2.0
    k0 = int(np.floor((z_hi - z.max()) / dz)) - 2
    k1 = int(np.floor((z_hi - z.min()) / dz)) + 3
    return max(0, k0), min(nz, max(k1, 0))


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
        self.full_rows = int(geometry["det_rows"])
        self.full_off_v = float(geometry.get("det_offset", (0.0, 0.0))[1])
        self.full_z_hi = float(geometry.get("center", (0, 0, 0))[2]) + int(geometry["n"][2]) * float(geometry["spacing"][2]) / 2.0
        self.slab, self.rows = (k0, k1), (r0, r1)
        self.geometry = zslab_geometry(geometry, k0, k1, r0, r1)
        if plan_factory is None:
            from .plan import Plan
            plan_factory = Plan
        self.plan = plan_factory(self.geometry, device=device)
        if hasattr(self.plan, "ray_units"):
            self.check_row_cells()

    def check_row_cells(self) -> None:
        """Assert that the kernel's fixed z cell of every row of this slab (its fp64 floor decision,
        read back through xrt_ray_units on the central column of view 0) is the cell
        zslab_partition assigned from numpy -- a disagreement at a tie would silently drop a row."""
        g = self.geometry
        k0, k1 = self.slab
        nxy = int(g["n"][0]) * int(g["n"][1])
        cols = int(g["det_cols"])
        c_mid = (cols - 1) // 2
        v_full = (np.arange(self.rows[0], self.rows[1]) - (int(self.full_rows) - 1) / 2.0) * float(g["det_spacing"][1]) \
            + float(self.full_off_v)
        z_hi = float(self.full_z_hi)
        dz = float(g["spacing"][2])
        want = np.floor((z_hi - v_full) / dz).astype(np.int64)
        for i in range(self.rows[1] - self.rows[0]):
            if not (k0 <= want[i] < k1):
                continue                     # rows outside the image: no unit either way
            rp, colsI, _ = self.plan.ray_units(i * cols + c_mid, i * cols + c_mid + 1)
            ks = np.unique(colsI.cpu().numpy() // nxy) + k0
            if ks.size and not (ks.size == 1 and ks[0] == want[i]):
                raise AssertionError(f"z-slab row {self.rows[0] + i}: kernel cells {ks}, partition cell {want[i]}")

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
