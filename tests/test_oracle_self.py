"""Pins of oracle/selfterms.py (reading C5, closed forms of SURVEY App. B).

* disc limit: FP∫_disc r⁻³ = -2π/a and ∫_disc r⁻¹ = 2πa (regular polygons);
* off-surface limit: the hypersingular and single-layer self integrals equal
  the z → 0 limit of the regular integrals at x = centroid + z·n
  (Richardson-extrapolated; SURVEY A.10 reached ≤ 2.5e-5);
* polar-rule convergence and k → 0 continuity.
"""
import numpy as np
import pytest

import oracle as O
from oracle.selfterms import polygon_fp_r3, polygon_r1

FOUR_PI = 4 * np.pi


def _polygon(m, a):
    t = 2 * np.pi * np.arange(m) / m
    return np.stack([a * np.cos(t), a * np.sin(t), 0 * t], axis=1)[None]


def test_disc_limit():
    a = 0.37
    P = _polygon(4000, a)
    x = np.zeros((1, 3))
    assert abs(polygon_fp_r3(P, x)[0] - (-2 * np.pi / a)) < 1e-5 * 2 * np.pi / a
    assert abs(polygon_r1(P, x)[0] - 2 * np.pi * a) < 1e-5 * 2 * np.pi * a


TRIS = {
    "equilateral_h0.04": np.array([[0, 0, 0], [0.04, 0, 0], [0.02, 0.04 * np.sqrt(3) / 2, 0]]),
    "skewed": np.array([[0, 0, 0], [0.05, 0.004, 0.0], [0.013, 0.021, 0.0]]),
}


def _offsurface(tri, k, z, kind, nphi=200, nr=200):
    """∫_Δ K(x, y) dS_y at x = centroid + z·n by polar Gauss-Legendre around
    the foot point with a graded radial map ρ = z(e^t - 1): an independent,
    regular (non-singular) evaluation of the same integral for z > 0."""
    c = tri.mean(0)
    nrm = np.cross(tri[1] - tri[0], tri[2] - tri[0])
    nrm /= np.linalg.norm(nrm)
    x = c + z * nrm
    gx, gw = np.polynomial.legendre.leggauss(nphi)
    rx, rw = np.polynomial.legendre.leggauss(nr)
    total = 0j
    for e in range(3):
        va, vb = tri[e], tri[(e + 1) % 3]
        u = (vb - va) / np.linalg.norm(vb - va)
        ta, tb = np.dot(va - c, u), np.dot(vb - c, u)
        foot = (va - c) - ta * u
        d = np.linalg.norm(foot)
        pdir = foot / d
        pa, pb = np.arctan2(ta, d), np.arctan2(tb, d)
        psi = 0.5 * (pb - pa) * gx + 0.5 * (pb + pa)
        wpsi = 0.5 * (pb - pa) * gw
        for ps, wp in zip(psi, wpsi):
            R = d / np.cos(ps)
            dirv = np.cos(ps) * pdir + np.sin(ps) * u
            T = np.log1p(R / z)
            t = 0.5 * T * (rx + 1)
            rho = z * np.expm1(t)
            jac = z * np.exp(t) * 0.5 * T * rw
            y = c[None] + rho[:, None] * dirv[None]
            if kind == "H":
                val = O.d2G_dnxdny(x[None], nrm[None], y, nrm[None], k)
            else:
                val = O.G(x[None], y, k)
            total += wp * np.sum(val * rho * jac)
    return total


@pytest.mark.parametrize("name", list(TRIS))
@pytest.mark.parametrize("k", [0.0, 10.0])
def test_self_terms_match_offsurface_limit(name, k):
    tri = TRIS[name]
    S, H = O.self_integrals(tri, k)
    h = np.max([np.linalg.norm(tri[i] - tri[(i + 1) % 3]) for i in range(3)])
    zs = h * np.array([1 / 64, 1 / 128, 1 / 256])
    for kind, ref in (("H", H), ("S", S)):
        v = np.array([_offsurface(tri, k, z, kind) for z in zs])
        # quadratic Richardson in z (v(z) = v0 + c1 z + c2 z²)
        A = np.stack([np.ones(3), zs, zs ** 2], 1)
        v0 = np.linalg.solve(A, v)[0]
        assert abs(v0 - ref) / abs(ref) < 1e-4, (kind, v0, ref)


def test_polar_rule_converged_and_k0_continuity():
    tri = TRIS["skewed"]
    S20, H20 = O.self_integrals(tri, 1000.0 * 0 + 24.0, n=20)
    S40, H40 = O.self_integrals(tri, 24.0, n=40)
    assert abs(H20 - H40) < 1e-10 * abs(H40) and abs(S20 - S40) < 1e-10 * abs(S40)
    S0, H0 = O.self_integrals(tri, 0.0)
    Se, He = O.self_integrals(tri, 1e-4)
    assert abs(He - H0) < 1e-6 * abs(H0) and abs(Se - S0) < 1e-6 * abs(S0)


def test_self_lhs_structure():
    tri = TRIS["equilateral_h0.04"]
    _, H = O.self_integrals(tri, 3.0)
    assert abs(O.self_lhs(tri, 3.0, 0.0) - 0.5) == 0.0     # α = 0: CBIE diagonal ½ (C3)
    assert abs(O.self_lhs(tri, 3.0, 1j / 3) - (0.5 + 1j / 3 * H)) < 1e-15
    assert H.real < 0       # finite part of r⁻³ over a panel is negative (disc: -2π/a)
