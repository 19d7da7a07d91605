"""Pins of the point-source workload of PAPER.md §5.2 (Table 3):
the incident field u_inc = e^{ikR}/(4πR) (Eq. 3), its BM
right-hand side and the rigid-sphere series (oracle/analytic.py).

Independent pins:
* far-field limit: a unit point source at distance r_s along -d is, near the
  origin, the plane wave e^{ik d·x} times e^{ik r_s}/(4π r_s), so both the
  series and the right-hand side must converge to the plane-wave ones
  (a separately written formula) with an O(1/r_s) error;
* the dense oracle's BM solve converges to the series under refinement.
"""
import numpy as np

import oracle as O
from oracle import fast
from fda_inputs import icosphere, geodesic_sphere, POINT_SOURCE


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_geodesic_sphere_is_closed_and_sized():
    for nu in (1, 2, 5):
        V, F = geodesic_sphere(nu, 1.0)
        assert len(F) == 20 * nu * nu and len(V) == 10 * nu * nu + 2
        e = np.sort(np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]]), axis=1)
        _, cnt = np.unique(e, axis=0, return_counts=True)
        assert set(cnt.tolist()) == {2}
        assert np.allclose(np.linalg.norm(V, axis=1), 1.0)
        el = O.element_geometry(V, F)
        # kernel normals point into the body (reading C1)
        assert np.all(np.einsum("ij,ij->i", el.normal, el.centroid) < 0)
    assert POINT_SOURCE["nu"] ** 2 * 20 == 106580


def test_point_source_series_far_limit():
    k, a = 10.0, 0.5
    V, F = icosphere(3, a)
    el = O.element_geometry(V, F)
    d = np.array([0.3, -0.4, np.sqrt(1 - 0.25)])
    u_pw = O.rigid_sphere_total(el.centroid, k, a, d)
    errs = []
    for rs in (1e3, 1e4, 1e5):
        xs = -rs * d
        amp = np.exp(1j * k * rs) / (4 * np.pi * rs)
        errs.append(_rel(O.rigid_sphere_point_source_total(el.centroid, k, a, xs) / amp, u_pw))
    assert errs[-1] < 5e-5
    assert 8 < errs[0] / errs[1] < 12 and 8 < errs[1] / errs[2] < 12     # O(1/r_s)


def test_point_source_rhs_far_limit():
    k = 7.0
    V, F = icosphere(2, 0.5)
    el = O.element_geometry(V, F)
    alpha = 1j / k
    d = np.array([1.0, 0.0, 0.0])
    b_pw = O.plane_wave_rhs(el.centroid, el.normal, k, alpha, d)
    errs = []
    for rs in (1e3, 1e4):
        amp = np.exp(1j * k * rs) / (4 * np.pi * rs)
        errs.append(_rel(O.point_source_rhs(el.centroid, el.normal, k, alpha, -rs * d) / amp, b_pw))
    assert errs[1] < 1e-3 and 8 < errs[0] / errs[1] < 12


def test_point_source_rhs_values():
    """Direct values: on the ray through the source, ∂R/∂n = ∓1."""
    k, alpha = 3.0, 1j / 3.0
    xs = np.array([-2.0, 0.0, 0.0])
    x = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    n = np.array([[-1.0, 0.0, 0.0], [1.0, 0.0, 0.0]])     # into the unit sphere
    b = O.point_source_rhs(x, n, k, alpha, xs)
    for i, (R, dRdn) in enumerate(((3.0, -1.0), (1.0, 1.0))):
        G = np.exp(1j * k * R) / (4 * np.pi * R)
        assert abs(b[i] - G * (1 + alpha * (1j * k - 1 / R) * dRdn)) < 1e-15


def test_point_source_dense_solve_converges_to_series():
    k, a = 5.0, 0.5
    xs = np.array([-1.0, 0.0, 0.0])          # the paper's geometry (source at 2 radii), scaled
    errs = []
    for s in (2, 3):
        V, F = icosphere(s, a)
        el = O.element_geometry(V, F)
        A = fast.dense(el, k, 1j / k, "lhs")
        b = O.point_source_rhs(el.centroid, el.normal, k, 1j / k, xs)
        u = O.lu_solve(A, b)
        errs.append(_rel(u, O.rigid_sphere_point_source_total(el.centroid, k, a, xs)))
    assert errs[1] < 0.6 * errs[0] and errs[1] < 3e-2, errs
