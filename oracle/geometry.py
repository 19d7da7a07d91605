"""Element geometry for piecewise-constant flat triangles (oracle; fp64).

PAPER.md §5: collocation point x_i = centroid of triangle Δ_i.
Normal convention (SURVEY C1, P:153-158 / P:169-185): Eq. (2)/(4) as printed
hold with n pointing OUT of the acoustic domain Ω, i.e. INTO the scatterer;
meshes are CCW seen from outside, so the kernel normal is the negated CCW
normal: n = -(v2-v1)×(v3-v1)/‖·‖.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Elements:
    verts: np.ndarray     # (N,3,3) triangle vertices
    centroid: np.ndarray  # (N,3)
    normal: np.ndarray    # (N,3) kernel normal, into the body
    area: np.ndarray      # (N,)
    hmax: np.ndarray      # (N,) longest edge


def element_geometry(V: np.ndarray, F: np.ndarray) -> Elements:
    T = np.asarray(V, dtype=np.float64)[np.asarray(F)]
    a, b, c = T[:, 0], T[:, 1], T[:, 2]
    cr = np.cross(b - a, c - a)
    nrm = np.linalg.norm(cr, axis=1)
    area = 0.5 * nrm
    normal = -cr / nrm[:, None]
    centroid = (a + b + c) / 3.0
    hmax = np.max(np.stack([np.linalg.norm(b - a, axis=1), np.linalg.norm(c - b, axis=1),
                            np.linalg.norm(a - c, axis=1)]), axis=0)
    return Elements(T, centroid, normal, area, hmax)
