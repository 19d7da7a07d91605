"""Helmholtz kernels, written out as in SURVEY.md App. B (oracle; fp64).

G = e^{ikr}/(4πr)  (Eq. 3).  With d = x - y, r = ‖d‖,
∂r/∂n_x = d·n_x / r and ∂r/∂n_y = -d·n_y / r:
  G'  = e^{ikr}(ikr - 1)/(4π r²)
  G'' = e^{ikr}(2 - 2ikr - k²r²)/(4π r³)
  ∂G/∂n_y = G' ∂r/∂n_y ;  ∂G/∂n_x = G' ∂r/∂n_x
  ∂²G/∂n_x∂n_y = (G'' - G'/r)(∂r/∂n_x)(∂r/∂n_y) - G'(n_x·n_y)/r
LHS integrand of Eq. (5): ∂G/∂n_y + α ∂²G/∂n_x∂n_y.
RHS integrand of Eq. (4):  G + α ∂G/∂n_x.
All functions broadcast over leading dimensions; points/normals are (...,3).
"""
from __future__ import annotations

import numpy as np

FOUR_PI = 4.0 * np.pi


def _r(x, y):
    d = np.asarray(x, dtype=np.float64) - np.asarray(y, dtype=np.float64)
    r = np.sqrt(np.sum(d * d, axis=-1))
    return d, r


def G(x, y, k):
    _, r = _r(x, y)
    return np.exp(1j * k * r) / (FOUR_PI * r)


def _Gp(r, k):
    return np.exp(1j * k * r) * (1j * k * r - 1.0) / (FOUR_PI * r * r)


def _Gpp(r, k):
    return np.exp(1j * k * r) * (2.0 - 2.0j * k * r - (k * r) ** 2) / (FOUR_PI * r ** 3)


def dG_dny(x, y, ny, k):
    d, r = _r(x, y)
    drdny = -np.sum(d * ny, axis=-1) / r
    return _Gp(r, k) * drdny


def dG_dnx(x, y, nx, k):
    d, r = _r(x, y)
    drdnx = np.sum(d * nx, axis=-1) / r
    return _Gp(r, k) * drdnx


def d2G_dnxdny(x, nx, y, ny, k):
    d, r = _r(x, y)
    drdnx = np.sum(d * nx, axis=-1) / r
    drdny = -np.sum(d * ny, axis=-1) / r
    nxny = np.sum(np.asarray(nx) * np.asarray(ny), axis=-1)
    gp = _Gp(r, k)
    return (_Gpp(r, k) - gp / r) * drdnx * drdny - gp * nxny / r


def lhs_kernel(x, nx, y, ny, k, alpha):
    """∂G/∂n_y + α ∂²G/∂n_x∂n_y (Eq. 5 integrand)."""
    return dG_dny(x, y, ny, k) + alpha * d2G_dnxdny(x, nx, y, ny, k)


def rhs_kernel(x, nx, y, k, alpha):
    """G + α ∂G/∂n_x (Eq. 4 right side; also the L2T target kernel Eq. 12)."""
    return G(x, y, k) + alpha * dG_dnx(x, y, nx, k)
