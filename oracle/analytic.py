"""Closed-form sphere solutions and incident fields (oracle; fp64).

* Pulsating sphere (§5.1).  The printed u = 1/(1+ik) is
  the complex conjugate of the value consistent with G = e^{ikr}/4πr;
  reading C2: for ∂u/∂n = 1 with n into the body on a sphere of radius a,
  u = a/(1 - ika).
* Rigid (sound-hard) sphere, plane wave e^{ik d·x} (textbook partial-wave
  series, Wronskian form):
  u_tot(θ) = (i/(ka)²) Σ_n iⁿ(2n+1) P_n(cos θ) / h_n^{(1)'}(ka),  cos θ = d·x̂.
* Plane-wave BM right-hand side for the rigid problem (Eq. 4 with ∂u/∂n = 0,
  reading C22): b_i = u_inc(x_i) + α ∂u_inc/∂n(x_i) = e^{ik d·x_i}(1 + iαk d·n_i).
* Point source at x_s outside a rigid sphere (§5.2, P:1016-1019:
  "The point source is at (-2, 0, 0)"): u_inc(x) = G(x, x_s) = e^{ikR}/(4πR),
  R = |x - x_s| (Eq. 3); BM right-hand side
  b_i = u_inc + α ∂u_inc/∂n = G [1 + α (ik - 1/R) (x_i - x_s)·n_i / R].
  Total surface field (textbook addition theorem
  e^{ik|x-y|}/(4π|x-y|) = (ik/4π) Σ (2n+1) j_n(k r_<) h_n(k r_>) P_n(cos γ),
  Neumann condition, Wronskian j_n h_n' - j_n' h_n = i/(ka)²):
  u_tot(x̂) = -1/(4π k a²) Σ_n (2n+1) h_n(k r_s) / h_n'(ka) P_n(x̂·x̂_s).
"""
from __future__ import annotations

import numpy as np
from scipy.special import spherical_jn, spherical_yn


def pulsating_sphere_u(k: float, a: float = 1.0) -> complex:
    return a / (1.0 - 1j * k * a)


def _legendre_all(nmax: int, t: np.ndarray) -> np.ndarray:
    P = np.zeros((nmax + 1,) + t.shape)
    P[0] = 1.0
    if nmax >= 1:
        P[1] = t
    for n in range(1, nmax):
        P[n + 1] = ((2 * n + 1) * t * P[n] - n * P[n - 1]) / (n + 1)
    return P


def rigid_sphere_total(points: np.ndarray, k: float, a: float, d, tol: float = 1e-14,
                       return_terms: bool = False):
    """Total surface potential at ``points`` (projected to the sphere)."""
    d = np.asarray(d, dtype=np.float64)
    d = d / np.linalg.norm(d)
    pts = np.asarray(points, dtype=np.float64)
    cos_t = np.clip((pts @ d) / np.linalg.norm(pts, axis=1), -1.0, 1.0)
    ka = k * a
    nmax = int(ka + 12.0 * max(ka, 1.0) ** (1.0 / 3.0) + 40)
    P = _legendre_all(nmax, cos_t)
    total = np.zeros(cos_t.shape, dtype=np.complex128)
    small = 0
    nterms = 0
    for n in range(nmax + 1):
        hp = spherical_jn(n, ka, derivative=True) + 1j * spherical_yn(n, ka, derivative=True)
        if not np.isfinite(hp):
            break
        term = (1j ** n) * (2 * n + 1) * P[n] / hp
        total += term
        nterms = n + 1
        if np.max(np.abs(term)) < tol * max(np.max(np.abs(total)), 1e-300):
            small += 1
            if small >= 3:
                break
        else:
            small = 0
    u = (1j / ka ** 2) * total
    return (u, nterms) if return_terms else u


def plane_wave_rhs(centroid: np.ndarray, normal: np.ndarray, k: float, alpha: complex, d) -> np.ndarray:
    """b = u_inc + α ∂u_inc/∂n at the collocation points (n = kernel normal)."""
    d = np.asarray(d, dtype=np.float64)
    d = d / np.linalg.norm(d)
    phase = np.exp(1j * k * (centroid @ d))
    return phase * (1.0 + 1j * alpha * k * (normal @ d))


def point_source_rhs(centroid: np.ndarray, normal: np.ndarray, k: float, alpha: complex, xs) -> np.ndarray:
    """b = u_inc + α ∂u_inc/∂n for u_inc = e^{ikR}/(4πR) (n = kernel normal, into the body)."""
    d = np.asarray(centroid, dtype=np.float64) - np.asarray(xs, dtype=np.float64)
    R = np.linalg.norm(d, axis=1)
    G = np.exp(1j * k * R) / (4.0 * np.pi * R)
    dRdn = np.einsum("ij,ij->i", d, normal) / R
    return G * (1.0 + alpha * (1j * k - 1.0 / R) * dRdn)


def rigid_sphere_point_source_total(points: np.ndarray, k: float, a: float, xs, tol: float = 1e-14):
    """Total surface potential on a rigid sphere of radius a (centre 0) for a
    unit point source at xs (|xs| > a), at ``points`` projected to the sphere."""
    xs = np.asarray(xs, dtype=np.float64)
    rs = float(np.linalg.norm(xs))
    pts = np.asarray(points, dtype=np.float64)
    cos_g = np.clip((pts @ xs) / (np.linalg.norm(pts, axis=1) * rs), -1.0, 1.0)
    ka, krs = k * a, k * rs
    nmax = int(ka + 12.0 * max(ka, 1.0) ** (1.0 / 3.0) + 60)
    P = _legendre_all(nmax, cos_g)
    total = np.zeros(cos_g.shape, dtype=np.complex128)
    small = 0
    for n in range(nmax + 1):
        hs = spherical_jn(n, krs) + 1j * spherical_yn(n, krs)
        hp = spherical_jn(n, ka, derivative=True) + 1j * spherical_yn(n, ka, derivative=True)
        if not (np.isfinite(hs) and np.isfinite(hp)):
            break
        term = (2 * n + 1) * (hs / hp) * P[n]
        total += term
        if np.max(np.abs(term)) < tol * max(np.max(np.abs(total)), 1e-300):
            small += 1
            if small >= 3:
                break
        else:
            small = 0
    return -total / (4.0 * np.pi * k * a * a)
