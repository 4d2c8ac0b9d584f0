"""The five BASELINE.json workloads as plain geometry dicts (input data only).

Every field maps 1:1 onto ``xrt_geometry`` in ``include/xrt.h``.  The readings of
the paper / BASELINE.json that fix these numbers are listed in DESIGN.md §3
("Readings"); the ones that matter here:

* views "evenly over [0, R)" -> angle_v = v * R / V, endpoint excluded (reading 10).
* cfg 5 "pitch 1.0 detector heights per turn" -> table feed per turn
  = 1.0 * det_rows * dv * sod / sdd (isocentre collimation), source height
  H(phi') = z0 + pitch * phi' / (2 pi) with z0 chosen so the helix is centred
  on the volume (reading 11).
* cfg 5 "curved-row detector treated as flat" -> flat detector (reading 12).
* phantom details (orientation, overlap, ellipsoid count 12 for cfg 4/5) -> reading 19.
"""
from __future__ import annotations

import copy
import math

import numpy as np

BEAMS = ("par2d", "fan2d", "par3d", "cone", "helical")

_CFG5_FEED = 1.0 * 64 * 1.0 * 570.0 / 1040.0  # mm of table feed per 2*pi turn

CONFIGS = {
    1: dict(
        name="cfg1_par2d_64", beam="par2d",
        n=(64, 64, 1), spacing=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0),
        n_views=90, angle_range=math.pi, angle_start=0.0,
        det_cols=96, det_rows=1, det_spacing=(1.0, 1.0), det_offset=(0.0, 0.0),
        sod=0.0, sdd=0.0, pitch=0.0, z0=0.0, tilt=0.0,
        image=dict(kind="uniform", seed=1), adj_seed=101,
    ),
    2: dict(
        name="cfg2_fan2d_512", beam="fan2d",
        n=(512, 512, 1), spacing=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0),
        n_views=720, angle_range=2 * math.pi, angle_start=0.0,
        det_cols=768, det_rows=1, det_spacing=(1.2, 1.0), det_offset=(0.0, 0.0),
        sod=1000.0, sdd=1500.0, pitch=0.0, z0=0.0, tilt=0.0,
        image=dict(kind="ellipses", count=10, seed=2), adj_seed=102,
    ),
    3: dict(
        name="cfg3_par3d_256", beam="par3d",
        n=(256, 256, 256), spacing=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0),
        n_views=180, angle_range=math.pi, angle_start=0.0,
        det_cols=384, det_rows=384, det_spacing=(1.0, 1.0), det_offset=(0.0, 0.0),
        sod=0.0, sdd=0.0, pitch=0.0, z0=0.0, tilt=0.0,
        image=dict(kind="ellipsoids", count=12, seed=3), adj_seed=103,
    ),
    4: dict(
        name="cfg4_cone_512", beam="cone",
        n=(512, 512, 512), spacing=(0.5, 0.5, 0.5), center=(0.0, 0.0, 0.0),
        n_views=720, angle_range=2 * math.pi, angle_start=0.0,
        det_cols=1024, det_rows=768, det_spacing=(0.8, 0.8), det_offset=(0.0, 0.0),
        sod=600.0, sdd=1200.0, pitch=0.0, z0=0.0, tilt=0.0,
        image=dict(kind="ellipsoids", count=12, seed=4), adj_seed=104,
    ),
    5: dict(
        name="cfg5_helical_512x256", beam="helical",
        n=(512, 512, 256), spacing=(0.5, 0.5, 1.0), center=(0.0, 0.0, 0.0),
        n_views=1440, angle_range=4 * math.pi, angle_start=0.0,
        det_cols=736, det_rows=64, det_spacing=(1.0, 1.0), det_offset=(0.0, 0.0),
        sod=570.0, sdd=1040.0, pitch=_CFG5_FEED, z0=-_CFG5_FEED * 719.5 / 720.0, tilt=0.0,
        image=dict(kind="ellipsoids", count=12, seed=5), adj_seed=105,
    ),
}


def config(idx: int) -> dict:
    """Deep copy of configuration ``idx`` (1..5) with its view angles attached."""
    c = copy.deepcopy(CONFIGS[idx])
    c["angles"] = view_angles(c)
    return c


def view_angles(c: dict) -> np.ndarray:
    """angle_v = start + v * range / V, v = 0..V-1 (fp64, endpoint excluded)."""
    v = np.arange(c["n_views"], dtype=np.float64)
    return c["angle_start"] + v * c["angle_range"] / c["n_views"]


def scaled(idx: int, n_views: int | None = None, det_cols: int | None = None,
           det_rows: int | None = None, n: tuple | None = None) -> dict:
    """A reduced copy of config ``idx`` for oracle-sized parity tests.

    Shrinking keeps the geometry family, spacing ratios and detector coverage:
    detector spacing is scaled so the detector still covers the same field.
    """
    c = config(idx)
    if n is not None:
        f = [c["n"][a] * c["spacing"][a] / n[a] for a in range(3)]
        c["spacing"] = tuple(f)
        c["n"] = tuple(n)
    if det_cols is not None:
        c["det_spacing"] = (c["det_spacing"][0] * c["det_cols"] / det_cols, c["det_spacing"][1])
        c["det_cols"] = det_cols
    if det_rows is not None and c["beam"] in ("par3d", "cone", "helical"):
        c["det_spacing"] = (c["det_spacing"][0], c["det_spacing"][1] * c["det_rows"] / det_rows)
        c["det_rows"] = det_rows
    if n_views is not None:
        c["n_views"] = n_views
    if c["beam"] == "helical":
        # keep the same source-height trajectory over the (possibly fewer) views
        nv = c["n_views"]
        c["z0"] = -c["pitch"] * (c["angle_range"] / (2 * math.pi)) * ((nv - 1) / 2.0) / nv
    c["angles"] = view_angles(c)
    return c


def n_rays(c: dict) -> int:
    return int(c["n_views"]) * int(c["det_rows"]) * int(c["det_cols"])
