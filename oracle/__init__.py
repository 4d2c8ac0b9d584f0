"""CPU oracle for the discrete X-ray transform (arXiv 2006.00686) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` and
``--impl reference`` legs may import, call, link or execute anything under
``oracle/``.  The product path (``paper_2006_00686_b200``) never touches it and
shares no code with it.

* ``oracle/brute.c``   fp64 brute force: every ray clipped against every unit box
  (the plain definition, Eq. (1.4) P:53-57 with the per-unit length of
  eq:condition_nonzero / eq:condition_nonzero_3D, P:157-164 / P:433-441).
* ``oracle/geometry.py`` the paper's beam -> parallel-beam transforms, literally
  (P:260-272).
* ``oracle/core.py``   ctypes wrapper: rows (CSR), forward, adjoint.
* ``oracle/attenuated.py`` the attenuated transform (SPECT weight of P:36-40),
  numpy fp64, units ordered along the ray.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): Tables 1-5 (tests/golden/),
closed forms, the Section 4.1 ambiguity examples, constructed edge / diagonal
rays, chord conservation, adjoint identity, symmetry and scaling identities, the
geometry transforms against the source / detector points.  Nothing here is
"parity unpinned" except the detector-bin convention (reading 9),
which is a convention both sides implement from the written rule.
"""
from .core import (  # noqa: F401
    TAU_FACTOR, OracleGrid, grid_of, rows, forward, adjoint, threads, set_threads, build_oracle,
)
from . import geometry  # noqa: F401
from .attenuated import forward_attenuated, adjoint_attenuated, ray_units_t  # noqa: F401
