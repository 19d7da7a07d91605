"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the paper's method (no kernels, no
quadrature, no geometry of elements): it only generates meshes (vertex and
triangle arrays), random densities, plane-wave directions and sampled row
indices, with fixed seeds.  It is the one module both ``oracle/`` and the CUDA
path's callers may import (task rule ③).

Workload recipe: SURVEY.md §8(d) (configs 1-5 of BASELINE.json) and the
pulsating-sphere family of PAPER.md §5.1 (octahedral spheres with
N = 8·4^n, k = π·2^(n-3)).
"""
from .meshes import icosphere, octasphere, graded_spheroid, geodesic_sphere  # noqa: F401
from .vectors import random_density, sampled_rows, plane_wave_direction  # noqa: F401
from .configs import CONFIGS, config_mesh, WorkloadConfig, POINT_SOURCE, point_source_mesh, bm_alpha  # noqa: F401
