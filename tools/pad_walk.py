"""Share of the column walk's ray-segments that lie inside the z range of the volume (cfg 4 cone),
and what a per-band sigma clip would remove.  Analytic (in-plane chord lengths; ray z linear in sigma):
    python tools/pad_walk.py"""
import numpy as np

sod, sdd, h = 600., 1200., 128.          # cfg 4: source-iso / source-detector (mm), half volume (mm)
du = dv = 0.8; cols, rows = 1024, 768; band = 128
u = (np.arange(cols) - (cols - 1) / 2) * du
v = (np.arange(rows) - (rows - 1) / 2) * dv
walk = inside_tot = band_tot = 0.
for phi in np.linspace(0, np.pi / 4, 7):
    c, s = np.cos(phi), np.sin(phi)
    S = np.array([-sod * c, -sod * s])
    for uu in u[::8]:
        D = np.array([(sdd - sod) * c - uu * s, (sdd - sod) * s + uu * c])
        d = D - S; L = np.linalg.norm(d); e = d / L
        lo, hi = -np.inf, np.inf
        for a in range(2):
            if abs(e[a]) < 1e-12:
                if abs(S[a]) > h: lo, hi = 1., 0.
                continue
            t0, t1 = (-h - S[a]) / e[a], (h - S[a]) / e[a]
            lo, hi = max(lo, min(t0, t1)), min(hi, max(t0, t1))
        if hi <= lo:
            continue
        with np.errstate(divide="ignore"):
            zl = np.where(v != 0, h * L / np.abs(v), np.inf)   # |z(sigma)| = |v| sigma / L <= h
        a0 = np.maximum(lo, -zl); b0 = np.minimum(hi, zl)
        inside = np.clip(b0 - a0, 0, None)
        walk += (hi - lo) * rows; inside_tot += inside.sum()
        for r0 in range(0, rows, band):
            m = inside[r0:r0 + band] > 0
            if m.any():
                band_tot += (b0[r0:r0 + band][m].max() - a0[r0:r0 + band][m].min()) * band
print({"inside_over_walked": round(inside_tot / walk, 4), "band_clipped_over_walked": round(band_tot / walk, 4)})
