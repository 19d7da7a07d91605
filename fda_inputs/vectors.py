"""Seeded random densities, sampled row sets and plane-wave directions.

Recipes from SURVEY.md §8(d): x_j = (g1 + i g2)/√2 with g ~ N(0,1) from
``numpy.random.default_rng(1000+cfg)``; 2,000 sampled rows without
replacement from ``default_rng(2000+cfg)``; config-3 plane-wave direction
g ~ N(0, I3) from ``default_rng(3003)``, normalised.
"""
from __future__ import annotations

import numpy as np


def random_density(n: int, seed: int) -> np.ndarray:
    """Complex normal density, complex128 of length n (unit variance)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(2 * n).reshape(n, 2)
    return (g[:, 0] + 1j * g[:, 1]) / np.sqrt(2.0)


def sampled_rows(n: int, count: int, seed: int) -> np.ndarray:
    """Sorted distinct row indices (int64)."""
    rng = np.random.default_rng(seed)
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.int64)


def plane_wave_direction(seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(3)
    return g / np.linalg.norm(g)
