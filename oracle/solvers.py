"""Dense LU and plain GMRES (oracle; fp64/complex128).

PAPER.md §5: "The resulting linear systems are solved by GMRES
solver"; tolerance = ε; no preconditioner.  Reading C20: relative
residual ‖b - Ax‖/‖b‖, x0 = 0, Arnoldi with modified Gram-Schmidt, Givens
rotations, optional restart.
"""
from __future__ import annotations

import numpy as np


def lu_solve(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Direct dense solve (LAPACK getrf/getrs via numpy) — library primitive."""
    return np.linalg.solve(A, b)


def gmres(matvec, b: np.ndarray, tol: float = 1e-4, max_iter: int = 200, restart: int = 0):
    """Returns (x, iterations, relative residual estimate, residual history)."""
    b = np.asarray(b, dtype=np.complex128)
    n = b.shape[0]
    m = restart if restart > 0 else max_iter
    x = np.zeros(n, dtype=np.complex128)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return x, 0, 0.0, [0.0]
    hist = [1.0]
    it = 0
    while it < max_iter:
        r = b - matvec(x) if it > 0 else b.copy()
        beta = np.linalg.norm(r)
        V = np.zeros((m + 1, n), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m, dtype=np.complex128)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        for j in range(m):
            w = matvec(V[j])
            for i in range(j + 1):              # modified Gram-Schmidt
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                  # apply previous rotations
                t = np.conj(cs[i]) * H[i, j] + np.conj(sn[i]) * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.sqrt(abs(H[j, j]) ** 2 + abs(H[j + 1, j]) ** 2)
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = np.conj(cs[j]) * g[j]
            it += 1
            j_done = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if hist[-1] <= tol or it >= max_iter:
                break
        y = np.linalg.solve(np.triu(H[:j_done, :j_done]), g[:j_done])
        x = x + V[:j_done].T @ y
        if hist[-1] <= tol:
            break
    return x, it, hist[-1], hist
