"""Singular self-element integrals on a flat triangle, x = centroid (oracle).

The paper never states its singular integration; SURVEY reading C5:
  H_ii = (1/4π)·FP∫_Δ r⁻³ dS + ∫_Δ [e^{ikr}(1-ikr) - 1]/(4π r³) dS
  S_ii = (1/4π)·∫_Δ r⁻¹ dS   + ∫_Δ (e^{ikr} - 1)/(4π r) dS
  D_ii = K'_ii = 0  (d·n = 0 on a flat panel).
For coplanar x, y: ∂²G/∂n_x∂n_y = -G'(n_x·n_y)/r = e^{ikr}(1-ikr)/(4π r³)
(App. B).  Static parts in closed form (App. B), per edge e with perpendicular
distance δ_e, tangential endpoint coordinates t_a < t_b, endpoint distances
ρ_a, ρ_b:
  ∫_Δ r⁻¹ dS    =  Σ_e δ_e ln[(t_b+ρ_b)/(t_a+ρ_a)]
  FP∫_Δ r⁻³ dS  = -Σ_e (t_b/ρ_b - t_a/ρ_a)/δ_e
Remainders: polar Gauss-Legendre, n×n per edge sub-triangle (n = 20).
LHS diagonal: A_ii = ½ + D_ii + α H_ii (c = ½, reading C3; no jump on the
hypersingular term, C4).  RHS diagonal: B_ii = -α/2 + S_ii + α K'_ii.
Pins: disc limit FP∫ r⁻³ = -2π/a; off-surface limit of the hypersingular
integral; k → 0 continuity; polar-rule convergence (tests/test_oracle_self.py).
"""
from __future__ import annotations

import numpy as np

FOUR_PI = 4.0 * np.pi


def _edges(tri: np.ndarray, x: np.ndarray):
    """Per edge va→vb: (δ, t_a, t_b, ρ_a, ρ_b), each an array over the batch;
    t along the unit edge vector from the foot of the perpendicular through x,
    so t_b - t_a = |vb - va| > 0.  x must be interior (δ > 0 on every edge).
    tri: (M,3,3), x: (M,3)."""
    out = []
    nv = tri.shape[1]                      # 3 for triangles; any convex polygon works
    for e in range(nv):
        va, vb = tri[:, e], tri[:, (e + 1) % nv]
        u = (vb - va) / np.linalg.norm(vb - va, axis=1)[:, None]
        ta = np.sum((va - x) * u, axis=1)
        tb = np.sum((vb - x) * u, axis=1)
        delta = np.linalg.norm((va - x) - ta[:, None] * u, axis=1)
        out.append((delta, ta, tb, np.linalg.norm(va - x, axis=1), np.linalg.norm(vb - x, axis=1)))
    return out


def polygon_r1(tri, x):
    """∫_Δ r⁻¹ dS in closed form (App. B)."""
    return sum(d * np.log((tb + rb) / (ta + ra)) for (d, ta, tb, ra, rb) in _edges(tri, x))


def polygon_fp_r3(tri, x):
    """Hadamard finite part FP∫_Δ r⁻³ dS in closed form (App. B)."""
    return -sum((tb / rb - ta / ra) / d for (d, ta, tb, ra, rb) in _edges(tri, x))


def _polar_remainder(tri, x, g, n):
    """∫_Δ f dS with f·r = g(r) (smooth at r = 0), polar Gauss-Legendre n×n
    on each edge sub-triangle: ψ ∈ [atan(t_a/δ), atan(t_b/δ)], r ∈ [0, δ/cos ψ]."""
    gx, gw = np.polynomial.legendre.leggauss(n)
    total = np.zeros(tri.shape[0], dtype=np.complex128)
    for (d, ta, tb, _, _) in _edges(tri, x):
        pa, pb = np.arctan2(ta, d), np.arctan2(tb, d)                    # (M,)
        psi = 0.5 * (pb - pa)[:, None] * gx + 0.5 * (pb + pa)[:, None]  # (M,n)
        wpsi = 0.5 * (pb - pa)[:, None] * gw
        R = d[:, None] / np.cos(psi)                                     # (M,n)
        r = 0.5 * R[:, :, None] * (gx[None, None, :] + 1.0)             # (M,n,n)
        wr = 0.5 * R[:, :, None] * gw[None, None, :]
        total += np.sum(wpsi[:, :, None] * wr * g(r), axis=(1, 2))
    return total


def self_integrals(tri: np.ndarray, k: float, n: int = 20):
    """(S_ii, H_ii) at the centroid of each triangle; tri (3,3) or (M,3,3)."""
    tri = np.asarray(tri, dtype=np.float64)
    single = tri.ndim == 2
    T = tri[None] if single else tri
    x = T.mean(axis=1)
    s_static = polygon_r1(T, x) / FOUR_PI
    h_static = polygon_fp_r3(T, x) / FOUR_PI

    def g_s(r):
        return (np.exp(1j * k * r) - 1.0) / FOUR_PI

    def g_h(r):
        return (np.exp(1j * k * r) * (1.0 - 1j * k * r) - 1.0) / (FOUR_PI * r * r)

    S = s_static + _polar_remainder(T, x, g_s, n)
    H = h_static + _polar_remainder(T, x, g_h, n)
    return (S[0], H[0]) if single else (S, H)


def self_lhs(tri, k, alpha, n: int = 20):
    """A_ii = ½ + α H_ii  (Eq. 4 LHS diagonal at a centroid, C3-C5)."""
    _, H = self_integrals(tri, k, n)
    return 0.5 + alpha * H


def self_rhs(tri, k, alpha, n: int = 20):
    """B_ii = -α/2 + S_ii  (Eq. 4 RHS diagonal, C4-C5)."""
    S, _ = self_integrals(tri, k, n)
    return -0.5 * alpha + S
