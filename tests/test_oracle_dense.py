"""Pins of the dense oracle operator (oracle/dense.py, oracle/fast.py):
the paper's own Table 2 rows, the rigid-sphere series, the fictitious
frequency conditioning, tier accuracy against brute-force quadrature, and the
C row evaluator against the numpy definition."""
import json
import os

import numpy as np
import pytest

import oracle as O
from oracle import fast
from oracle.quadrature import RULE_Q7, subdivided_rule
from fda_inputs import icosphere, octasphere, random_density

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_c_rows_equal_numpy_definition():
    V, F = icosphere(2, 0.5)
    el = O.element_geometry(V, F)
    rows = np.arange(0, 320, 7)
    for kind, f in (("lhs", O.lhs_rows), ("rhs", O.rhs_rows)):
        a = f(el, rows, 7.0, 1j / 7.0)
        b = fast.dense_rows(el, rows, 7.0, 1j / 7.0, kind)
        assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()
    x = random_density(320, 5)
    y = fast.matvec_rows(el, rows, x, 7.0, 1j / 7.0)
    assert np.abs(y - O.lhs_rows(el, rows, 7.0, 1j / 7.0) @ x).max() < 1e-12 * np.abs(y).max()


@pytest.mark.parametrize("row", [0, 1])
def test_table2_pulsating_rows(row):
    """PAPER.md Table 2: pulsating unit sphere, dense BM solve.
    Reading C2: exact u = a/(1-ika); the printed 1/(1+ik) is its conjugate."""
    g = json.load(open(os.path.join(GOLD, "table2_pulsating.json")))
    r = g["rows"][row]
    k = np.pi * r["k_over_pi"]
    V, F = octasphere(r["n"], 1.0)
    assert F.shape[0] == r["N"]
    el = O.element_geometry(V, F)
    A = fast.dense(el, k, 1j / k, "lhs")
    B = fast.dense(el, k, 1j / k, "rhs")
    u = O.lu_solve(A, B @ np.ones(r["N"]))
    ue = O.pulsating_sphere_u(k, 1.0)
    err = np.linalg.norm(u - ue) / (abs(ue) * np.sqrt(r["N"]))
    assert abs(err / r["l2_error_eps1e-3"] - 1) < g["tolerance_rel"], err
    # the printed (conjugate) form is far off: the reading matters
    err_printed = np.linalg.norm(u - 1 / (1 + 1j * k)) / (abs(ue) * np.sqrt(r["N"]))
    assert err_printed > 0.5
    if row == 0:
        # normal convention C1: with mesh-outward kernel normals the error is O(1)
        el2 = O.element_geometry(V, F)
        el2.normal = -el2.normal
        A2 = fast.dense(el2, k, 1j / k, "lhs")
        B2 = fast.dense(el2, k, 1j / k, "rhs")
        u2 = O.lu_solve(A2, B2 @ (-np.ones(r["N"])))
        assert np.linalg.norm(u2 - ue) / (abs(ue) * np.sqrt(r["N"])) > 0.5


def _rigid_err(s, k=10.0):
    V, F = icosphere(s, 0.5)
    el = O.element_geometry(V, F)
    A = fast.dense(el, k, 1j / k, "lhs")
    d = np.array([0, 0, 1.0])
    b = O.plane_wave_rhs(el.centroid, el.normal, k, 1j / k, d)
    u = O.lu_solve(A, b)
    ue = O.rigid_sphere_total(el.centroid, k, 0.5, d)
    return np.linalg.norm(u - ue) / np.linalg.norm(ue), A


def test_rigid_sphere_series_convergence():
    """Dense BM solve vs the partial-wave series, kD = 10 (config-1 family);
    SURVEY A.6: 5.2e-2 (N=320), 1.5e-2 (N=1280)."""
    e2, _ = _rigid_err(2)
    e3, A3 = _rigid_err(3)
    assert e2 < 7e-2 and e3 < 2e-2
    assert e2 / e3 > 2.5            # ~O(h²) convergence of the discretisation


def test_fictitious_frequency_conditioning():
    """At ka = π (kD = 2π) the CBIE (½I + D, i.e. α = 0) is near-singular
    while Burton-Miller is not (Eq. 4 purpose)."""
    V, F = icosphere(3, 0.5)
    el = O.element_geometry(V, F)
    k = 2 * np.pi
    c_bm = np.linalg.cond(fast.dense(el, k, 1j / k, "lhs"))
    c_cbie = np.linalg.cond(fast.dense(el, k, 0.0, "lhs"))
    assert c_cbie > 10 * c_bm, (c_cbie, c_bm)
    assert c_bm < 20


def test_tier_accuracy_against_brute_force():
    """Each tier's entry vs a depth-6 subdivided Radon rule (28,672 points) —
    SURVEY A.5 bounds: T1 ≤ 1e-5, T2 ≤ 2e-4, T3 ≤ 1e-3 (coplanar worst case,
    kh ≈ 1.2)."""
    h = 0.04
    k = 1.2 / h
    tri = np.array([[0, 0, 0], [h, 0, 0], [h / 2, h * np.sqrt(3) / 2, 0.0]])
    ny = np.array([0, 0, -1.0])
    area = 0.5 * h * h * np.sqrt(3) / 2
    c = tri.mean(0)
    brute = subdivided_rule(RULE_Q7, 6)

    def integ(x, rule):
        P, W = rule
        Y = P @ tri
        return area * np.sum(W * O.lhs_kernel(x[None], ny[None], Y, ny[None], k, 1j / k))

    for rho, bound in ((0.7, 1e-5), (1.2, 1e-5), (2.0, 2e-4), (3.2, 1e-3), (6.0, 1e-3)):
        x = c + np.array([rho * h, 0.0, 0.0])
        ref = integ(x, brute)
        tier = 1 if rho < 1.5 else (2 if rho < 3 else 3)
        rule = {1: subdivided_rule(RULE_Q7, 3), 2: O.RULE_Q6, 3: O.RULE_Q3}[tier]
        assert abs(integ(x, rule) - ref) / abs(ref) < bound, (rho, tier)


def test_bm_coupling_sign_reading_c25():
    """Reading C25: the paper's α = i/k is α = −i/k
    in this code's convention (G = e^{ikr}, normals into the body).  Both
    signs give a uniquely solvable system with the same solution, so the
    oracle's arithmetic does not depend on it; what the paper fixes is the
    GMRES behaviour.  Pinned (i) by Table 2 row N = 8,192, ε = tol = 1e-3
    (P:996): the paper needs N_it = 3 and prints L2 error 9.26e-3 — the dense
    oracle system with −i/k reproduces both (≤ 3 iterations, error within 1%),
    with +i/k it needs twice the iterations and stops 2.7% off; (ii) at higher
    frequency (N = 1,280, kD = 30) +i/k needs ≥ 3× the iterations of −i/k."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table2_pulsating.json")))
    r = [q for q in g["rows"] if q["N"] == 8192][0]
    V, F = octasphere(r["n"], 1.0)
    el = O.element_geometry(V, F)
    k = np.pi * r["k_over_pi"]
    ue = O.pulsating_sphere_u(k, 1.0)
    out = {}
    for sg in (-1, 1):
        a = sg * 1j / k
        A = fast.dense(el, k, a, "lhs")
        b = fast.matvec_rows(el, np.arange(len(F)), np.ones(len(F)), k, a, kind="rhs")
        u, it, _, _ = O.gmres(lambda v: A @ v, b, tol=1e-3, max_iter=100)
        out[sg] = (it, np.linalg.norm(u - ue) / (abs(ue) * np.sqrt(len(F))))
        del A
    (it_m, e_m), (it_p, e_p) = out[-1], out[1]
    assert it_m <= r["n_it_eps1e-3"] < it_p, out
    assert abs(e_m / r["l2_error_eps1e-3"] - 1) < 0.01, out
    assert abs(e_m / r["l2_error_eps1e-3"] - 1) < abs(e_p / r["l2_error_eps1e-3"] - 1), out
    V, F = icosphere(3, 0.5)
    el = O.element_geometry(V, F)
    k = 30.0
    its = {}
    for sg in (-1, 1):
        a = sg * 1j / k
        A = fast.dense(el, k, a, "lhs")
        b = O.plane_wave_rhs(el.centroid, el.normal, k, a, np.array([0.0, 0.0, 1.0]))
        its[sg] = O.gmres(lambda v: A @ v, b, tol=1e-4, max_iter=200)[1]
    assert its[-1] <= 15 and its[1] >= 3 * its[-1], its


def test_tier_uses_source_element_size():
    """Reading C6 pins ρ_ij = |x_i − c_j| / h_j with h_j the SOURCE element's
    longest edge.  A large source triangle (h = 1) and a tiny target triangle
    (h = 0.01) one unit apart: row i sees j at ρ = 1 (tier T1, 448 points), row
    j sees i at ρ = 100 (tier T3).  Swapping h_i for h_j (a misreading near-
    uniform spheres cannot expose) flips both tiers; the T1 entry must also
    match brute-force quadrature (depth-6 Radon, 28,672 points) where Q3 would
    be off by O(1e-2).  Both the numpy definition and the C evaluator."""
    V = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, np.sqrt(3) / 2, 0],          # big source j = 0
                  [0.0, 0, 1.0], [0.01, 0, 1.0], [0.005, 0.01 * np.sqrt(3) / 2, 1.0]])  # tiny target i = 1
    F = np.array([[0, 1, 2], [3, 4, 5]], dtype=np.int32)
    el = O.element_geometry(V, F)
    el.centroid[1] = el.centroid[0] + np.array([0.0, 0.0, 1.0])     # |x_i − c_j| = 1 exactly
    el.verts[1] = el.verts[1] - el.verts[1].mean(0) + el.centroid[1]
    assert O.tier_of(el, 1)[0] == 1 and O.tier_of(el, 0)[1] == 3
    k = 3.0
    brute = subdivided_rule(RULE_Q7, 6)
    P, W = brute
    Y = P @ el.verts[0]
    ref = el.area[0] * np.sum(W * O.lhs_kernel(el.centroid[1][None], el.normal[1][None], Y, el.normal[0][None],
                                               k, 1j / k))
    for a in (O.lhs_rows(el, [1], k, 1j / k)[0, 0], fast.dense_rows(el, [1], k, 1j / k, "lhs")[0, 0]):
        assert abs(a - ref) <= 1e-6 * abs(ref)
    P3, W3 = O.RULE_Q3
    q3 = el.area[0] * np.sum(W3 * O.lhs_kernel(el.centroid[1][None], el.normal[1][None], P3 @ el.verts[0],
                                               el.normal[0][None], k, 1j / k))
    assert abs(q3 - ref) > 1e-3 * abs(ref)      # the wrong tier would be visible
