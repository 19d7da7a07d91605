"""Pins of oracle/kernels.py (Eq. 3-4 kernels) and
oracle/quadrature.py (rule exactness, reading C6)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from oracle.quadrature import RULE_Q3, RULE_Q6, RULE_Q7, RULE_T1

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_static_values_golden():
    data = json.load(open(os.path.join(GOLD, "kernel_static.json")))
    for c in data["cases"]:
        x, y, k = np.array(c["x"], float), np.array(c["y"], float), c["k"]
        if c["kind"] == "G":
            v = O.G(x, y, k)
        elif c["kind"] == "dG_dny":
            v = O.dG_dny(x, y, np.array(c["ny"], float), k)
        else:
            v = O.d2G_dnxdny(x, np.array(c["nx"], float), y, np.array(c["ny"], float), k)
        assert abs(v - complex(*c["value"])) < 1e-12, c


def test_reciprocity_and_modulus():
    rng = np.random.default_rng(0)
    x, y = rng.normal(size=(50, 3)), rng.normal(size=(50, 3))
    k = 3.7
    assert np.allclose(O.G(x, y, k), O.G(y, x, k), rtol=0, atol=0)
    r = np.linalg.norm(x - y, axis=1)
    assert np.allclose(np.abs(O.G(x, y, k)), 1 / (4 * np.pi * r), rtol=1e-14)


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


@pytest.mark.parametrize("k", [0.0, 1.3, 25.0])
def test_derivatives_by_finite_differences(k):
    """∂G/∂n_y, ∂G/∂n_x from central differences of G; ∂²G/∂n_x∂n_y from
    central differences of ∂G/∂n_y along n_x — catches any dropped
    term, sign or index error in App. B."""
    rng = np.random.default_rng(7)
    x = rng.normal(size=(40, 3))
    y = x + _unit(rng.normal(size=(40, 3))) * rng.uniform(0.3, 2.0, size=(40, 1))
    nx, ny = _unit(rng.normal(size=(40, 3))), _unit(rng.normal(size=(40, 3)))
    r = np.linalg.norm(x - y, axis=1, keepdims=True)
    h = 1e-5 * r
    fd_ny = (O.G(x, y + h * ny, k) - O.G(x, y - h * ny, k)) / (2 * h[:, 0])
    fd_nx = (O.G(x + h * nx, y, k) - O.G(x - h * nx, y, k)) / (2 * h[:, 0])
    fd_h = (O.dG_dny(x + h * nx, y, ny, k) - O.dG_dny(x - h * nx, y, ny, k)) / (2 * h[:, 0])
    for fd, an in ((fd_ny, O.dG_dny(x, y, ny, k)), (fd_nx, O.dG_dnx(x, y, nx, k)),
                   (fd_h, O.d2G_dnxdny(x, nx, y, ny, k))):
        err = np.abs(fd - an) / np.maximum(np.abs(an), 1e-3 * np.abs(O.G(x, y, k)) / r[:, 0])
        assert err.max() < 1e-6


def test_hyper_symmetry():
    rng = np.random.default_rng(3)
    x, y = rng.normal(size=(30, 3)), rng.normal(size=(30, 3))
    nx, ny = _unit(rng.normal(size=(30, 3))), _unit(rng.normal(size=(30, 3)))
    a = O.d2G_dnxdny(x, nx, y, ny, 2.0)
    b = O.d2G_dnxdny(y, ny, x, nx, 2.0)
    assert np.allclose(a, b, rtol=1e-12)


def _monomial_integral(a, b):
    return math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)


@pytest.mark.parametrize("rule,degree", [(RULE_Q3, 2), (RULE_Q6, 4), (RULE_Q7, 5), (RULE_T1, 5)])
def test_rule_exactness(rule, degree):
    """∫_ref x^a y^b dA = a! b!/(a+b+2)! on (0,0),(1,0),(0,1) for a+b ≤ degree,
    and the rule is NOT exact one degree higher (it is the rule it claims)."""
    P, W = rule
    assert abs(W.sum() - 1.0) < 1e-14
    X, Y = P[:, 1], P[:, 2]            # barycentric (1-x-y, x, y)
    for a in range(degree + 1):
        for b in range(degree + 1 - a):
            q = 0.5 * np.sum(W * X ** a * Y ** b)
            assert abs(q - _monomial_integral(a, b)) < 1e-13, (a, b)
    if rule is not RULE_T1:
        worst = max(abs(0.5 * np.sum(W * X ** a * Y ** (degree + 1 - a))
                        - _monomial_integral(a, degree + 1 - a)) for a in range(degree + 2))
        assert worst > 1e-8


def test_t1_is_depth3_subdivision():
    P, W = RULE_T1
    assert P.shape == (448, 3) and np.all(P >= -1e-15) and abs(P.sum(1) - 1).max() < 1e-14
