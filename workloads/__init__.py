"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds INPUT DATA ONLY: the five BASELINE.json configurations as plain
parameter dicts (including the view-angle arrays handed to ``xrt_plan_create``),
the seeded phantom generators (ellipses / ellipsoids, uniform images), seeded
adjoint inputs and seeded ray samples.  It contains none of the X-ray-transform
arithmetic (no ray construction, no detector-bin positions, no intersection
lengths), so the oracle (``oracle/``) and the product
(``paper_2006_00686_b200/``) can both consume it without sharing any of the
method's code.
"""
from .configs import CONFIGS, config, view_angles, scaled  # noqa: F401
from .phantoms import make_image, make_sino_input, make_attenuation, sample_rays  # noqa: F401
