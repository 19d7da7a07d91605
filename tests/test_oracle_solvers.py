"""Pins of oracle/solvers.py (GMRES, reading C20) and oracle/analytic.py."""
import numpy as np

import oracle as O


def test_gmres_identity_and_diag():
    b = np.array([1.0, 2.0, 3.0], dtype=complex)
    x, it, res, _ = O.gmres(lambda v: v, b, tol=1e-12)
    assert it == 1 and np.allclose(x, b)
    x, it, res, _ = O.gmres(lambda v: np.array([1.0, 2.0]) * v, np.array([1.0, 2.0]), tol=1e-12)
    assert it <= 2 and np.allclose(x, [1, 1])


def test_gmres_random_vs_lu_and_restart():
    rng = np.random.default_rng(1)
    n = 60
    A = np.eye(n) * 3 + (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    xs = O.lu_solve(A, b)
    x, it, res, hist = O.gmres(lambda v: A @ v, b, tol=1e-10, max_iter=200)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) < 1e-8
    assert abs(np.linalg.norm(b - A @ x) / np.linalg.norm(b) - res) < 1e-8
    assert all(hist[i + 1] <= hist[i] + 1e-15 for i in range(len(hist) - 1))
    x2, it2, res2, _ = O.gmres(lambda v: A @ v, b, tol=1e-10, max_iter=400, restart=10)
    assert np.linalg.norm(x2 - xs) / np.linalg.norm(xs) < 1e-8


def test_pulsating_closed_form():
    """u = a/(1-ika) satisfies ∂u/∂n = 1 (n = -r̂, into the body) for the
    radiating monopole u = A e^{ikr}/r — checked by finite differences."""
    for k, a in ((1.0, 1.0), (np.pi, 1.0), (10.0, 0.5)):
        u_a = O.pulsating_sphere_u(k, a)
        A = u_a * a / np.exp(1j * k * a)

        def u(r):
            return A * np.exp(1j * k * r) / r
        h = 1e-6
        dudn = -(u(a + h) - u(a - h)) / (2 * h)
        assert abs(dudn - 1.0) < 1e-7
    assert abs(O.pulsating_sphere_u(1.0, 1.0) - (1 + 1j) / 2) < 1e-15


def test_rigid_series_limits():
    rng = np.random.default_rng(2)
    pts = rng.normal(size=(20, 3))
    pts = 0.5 * pts / np.linalg.norm(pts, axis=1, keepdims=True)
    u = O.rigid_sphere_total(pts, 1e-3, 0.5, [0, 0, 1])
    assert np.abs(u - 1).max() < 1e-3                  # k → 0: u → 1
    d = np.array([0, 0, 1.0])
    lit, shadow = O.rigid_sphere_total(np.array([[0, 0, -0.5], [0, 0, 0.5]]), 4 * np.pi, 0.5, d)
    assert abs(lit) > abs(shadow)
    _, nterms = O.rigid_sphere_total(pts, 10.0, 0.5, d, return_terms=True)
    assert 15 <= nterms <= 40                          # A.9: ka=5 needs ~23 terms


def test_rigid_series_satisfies_neumann_condition():
    """Independent check of the series: the total field u_inc + u_s built from
    the same coefficients has zero radial derivative at r = a."""
    from scipy.special import spherical_jn, spherical_yn, eval_legendre
    k, a = 7.0, 0.5
    ka = k * a
    th = np.linspace(0.1, 3.0, 7)
    def field(r):
        tot = 0j
        for n in range(60):
            jn_p = spherical_jn(n, ka, derivative=True)
            hn_p = jn_p + 1j * spherical_yn(n, ka, derivative=True)
            hn = spherical_jn(n, k * r) + 1j * spherical_yn(n, k * r)
            tot = tot + (1j ** n) * (2 * n + 1) * eval_legendre(n, np.cos(th)) * (
                spherical_jn(n, k * r) - jn_p / hn_p * hn)
        return tot
    h = 1e-6
    assert np.abs((field(a + h) - field(a - h)) / (2 * h)).max() < 1e-5
    pts = a * np.stack([np.sin(th), 0 * th, np.cos(th)], 1)
    assert np.abs(field(a) - O.rigid_sphere_total(pts, k, a, [0, 0, 1])).max() < 1e-10
