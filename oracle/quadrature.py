"""Triangle quadrature rules (oracle; fp64, barycentric, weights sum to 1).

The paper never states its quadrature; SURVEY §8(c) reading C6
fixes the tier rules used here:
  Q3 = Strang-Fix 3-point rule, degree 2 (interior points (2/3,1/6,1/6));
  Q6 = Dunavant 6-point rule, degree 4;
  Q7 = Radon 7-point rule, degree 5;
  T1 = Q7 on the depth-3 uniform 1:4 subdivision (64 sub-triangles, 448 pts).
Pinned by polynomial exactness against ∫_ref x^a y^b = a! b!/(a+b+2)!.
"""
from __future__ import annotations

import numpy as np


def _sym3(a, w):
    """Three barycentric points (1-2a, a, a) and permutations, weight w each."""
    b = 1.0 - 2.0 * a
    P = np.array([[b, a, a], [a, b, a], [a, a, b]])
    return P, np.full(3, w)


def _rule_q3():
    P, W = _sym3(1.0 / 6.0, 1.0 / 3.0)
    return P, W


def _rule_q6():
    P1, W1 = _sym3(0.445948490915965, 0.223381589678011)
    P2, W2 = _sym3(0.091576213509771, 0.109951743655322)
    return np.vstack([P1, P2]), np.concatenate([W1, W2])


def _rule_q7():
    s15 = np.sqrt(15.0)
    P0 = np.array([[1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0]])
    P1, W1 = _sym3((6.0 - s15) / 21.0, (155.0 - s15) / 1200.0)
    P2, W2 = _sym3((6.0 + s15) / 21.0, (155.0 + s15) / 1200.0)
    return np.vstack([P0, P1, P2]), np.concatenate([[9.0 / 40.0], W1, W2])


RULE_Q3 = _rule_q3()
RULE_Q6 = _rule_q6()
RULE_Q7 = _rule_q7()


def subdivided_rule(rule, depth: int):
    """Apply ``rule`` on each of the 4^depth triangles of the uniform 1:4
    subdivision of the reference triangle; returns barycentric points w.r.t.
    the parent and weights summing to 1."""
    tris = [np.eye(3)]  # rows = barycentric coordinates of the sub-triangle corners
    for _ in range(depth):
        nxt = []
        for T in tris:
            a, b, c = T
            ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
            nxt += [np.array([a, ab, ca]), np.array([ab, b, bc]),
                    np.array([ca, bc, c]), np.array([ab, bc, ca])]
        tris = nxt
    P, W = rule
    pts = np.concatenate([P @ T for T in tris], axis=0)
    wts = np.concatenate([W / len(tris) for _ in tris])
    return pts, wts


RULE_T1 = subdivided_rule(RULE_Q7, 3)


def integrate(f, tri: np.ndarray, rule) -> complex:
    """∫_Δ f dS ≈ area Σ w_q f(y_q) for one triangle (3,3)."""
    P, W = rule
    Y = P @ tri
    area = 0.5 * np.linalg.norm(np.cross(tri[1] - tri[0], tri[2] - tri[0]))
    return area * np.sum(W * f(Y))
