"""ORACLE — test infrastructure only (NOT product code).

A plain, slow, obviously-correct fp64 CPU implementation of what the FDA
matvec approximates: the dense O(N²) Burton-Miller collocation operator of
PAPER.md Eq. (5) with piecewise-constant flat triangles and
centroid collocation, plus a dense LU / plain GMRES solver and the
analytic sphere solutions used to pin it.

Rules (task ③):
* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import anything here.
* It shares NO code with the CUDA path (``paper_1403_4747_b200``) and never
  imports it; the only shared module is ``fda_inputs`` (seeded meshes and
  vectors, no method arithmetic).
* Every function cites the PAPER.md passage (``P:n``) or the SURVEY.md reading
  (``C#``) it follows.  Where the paper is silent the SURVEY §8(c) readings are
  used; they are listed in DESIGN.md §3.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): static kernel values,
finite-difference derivatives, polynomial exactness of the rules, the disc
limit and off-surface limit of the self terms, the pulsating-sphere rows of
Table 2, the rigid-sphere series, the fictitious-frequency
conditioning, GMRES on closed-form systems.

Parity unpinned: none of the functions in this package (each has at least one
pin above); the FDA-specific constants are not part of the
oracle at all.
"""
from .geometry import element_geometry  # noqa: F401
from .kernels import (G, dG_dny, dG_dnx, d2G_dnxdny, lhs_kernel, rhs_kernel)  # noqa: F401
from .quadrature import RULE_Q3, RULE_Q6, RULE_Q7, subdivided_rule  # noqa: F401
from .selfterms import self_lhs, self_rhs, self_integrals  # noqa: F401
from .dense import (lhs_rows, rhs_rows, lhs_matvec_rows, lhs_dense, rhs_dense,  # noqa: F401
                    tier_of)
from .solvers import gmres, lu_solve  # noqa: F401
from .analytic import (rigid_sphere_total, pulsating_sphere_u, plane_wave_rhs,  # noqa: F401
                       point_source_rhs, rigid_sphere_point_source_total)
