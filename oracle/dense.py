"""Dense Burton-Miller collocation operator, row by row (oracle; fp64).

Definition (Eq. (5), specialised to collocation at
centroids and piecewise-constant elements):
  (A x)_i = ½ x_i + Σ_j A_ij x_j,
  A_ij = ∫_Δj [∂G/∂n_y + α ∂²G/∂n_x∂n_y](x_i, y) dS_y   (n_x = n_i, n_y = n_j)
and the RHS operator of Eq. (4) (NEXT-1 in SURVEY §8(f)):
  (B v)_i = -(α/2) v_i + Σ_j ∫_Δj [G + α ∂G/∂n_x](x_i, y) dS_y v_j.
Entries by the tier rule of SURVEY §8(c) (reading C6), with
ρ_ij = |x_i - c_j| / h_j and h_j the longest edge of Δ_j:
  T0  i = j           closed-form self terms (selfterms.py, C5)
  T1  0 < ρ < 1.5     Radon 7-point on the depth-3 1:4 subdivision (448 pts)
  T2  1.5 ≤ ρ < 3     Dunavant 6-point
  T3  ρ ≥ 3           Strang-Fix 3-point
No blocking or reordering beyond this definition.
"""
from __future__ import annotations

import numpy as np

from .geometry import Elements
from .kernels import lhs_kernel, rhs_kernel
from .quadrature import RULE_Q3, RULE_Q6, RULE_T1
from .selfterms import self_lhs, self_rhs

TIER1_RHO = 1.5
TIER2_RHO = 3.0


def tier_of(el: Elements, i: int) -> np.ndarray:
    """Tier index (0..3) of every entry of row i."""
    rho = np.linalg.norm(el.centroid[i][None, :] - el.centroid, axis=1) / el.hmax
    t = np.full(rho.shape, 3, dtype=np.int8)
    t[rho < TIER2_RHO] = 2
    t[rho < TIER1_RHO] = 1
    t[i] = 0
    return t


def _rule_block(el: Elements, i: int, J: np.ndarray, rule, kernel):
    P, W = rule
    Y = np.einsum("qa,jad->jqd", P, el.verts[J])          # (|J|, q, 3)
    x = el.centroid[i][None, None, :]
    nx = el.normal[i][None, None, :]
    ny = el.normal[J][:, None, :]
    vals = kernel(x, nx, Y, ny)                               # (|J|, q)
    return el.area[J] * (vals @ W)


def _row(el: Elements, i: int, k: float, alpha: complex, kind: str) -> np.ndarray:
    if kind == "lhs":
        def kern(x, nx, Y, ny):
            return lhs_kernel(x, nx, Y, ny, k, alpha)
    else:
        def kern(x, nx, Y, ny):
            return rhs_kernel(x, nx, Y, k, alpha)
    t = tier_of(el, i)
    row = np.zeros(len(t), dtype=np.complex128)
    for tier, rule in ((3, RULE_Q3), (2, RULE_Q6), (1, RULE_T1)):
        J = np.nonzero(t == tier)[0]
        if J.size:
            row[J] = _rule_block(el, i, J, rule, kern)
    if kind == "lhs":
        row[i] = self_lhs(el.verts[i], k, alpha)
    else:
        row[i] = self_rhs(el.verts[i], k, alpha)
    return row


def lhs_rows(el: Elements, rows, k: float, alpha: complex) -> np.ndarray:
    """Rows of A = ½I + D + αH (dense, complex128, (len(rows), N))."""
    return np.stack([_row(el, int(i), k, alpha, "lhs") for i in rows])


def rhs_rows(el: Elements, rows, k: float, alpha: complex) -> np.ndarray:
    """Rows of B = -(α/2)I + S + αK'."""
    return np.stack([_row(el, int(i), k, alpha, "rhs") for i in rows])


def lhs_matvec_rows(el: Elements, rows, x: np.ndarray, k: float, alpha: complex) -> np.ndarray:
    """(A x)_i for i in rows, one row at a time (no N×N storage)."""
    x = np.asarray(x, dtype=np.complex128)
    return np.array([_row(el, int(i), k, alpha, "lhs") @ x for i in rows])


def lhs_dense(el: Elements, k: float, alpha: complex) -> np.ndarray:
    return lhs_rows(el, range(el.centroid.shape[0]), k, alpha)


def rhs_dense(el: Elements, k: float, alpha: complex) -> np.ndarray:
    return rhs_rows(el, range(el.centroid.shape[0]), k, alpha)
