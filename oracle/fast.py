"""ctypes front-end of oracle/c/oracle_rows.c (oracle; test infrastructure).

Same operator as oracle/dense.py; the C code evaluates the off-diagonal
tiers T1-T3, the self entry (T0) comes from oracle/selfterms.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .geometry import Elements
from .selfterms import self_lhs, self_rhs

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "c", "oracle_rows.c")
_LIB = os.path.join(_HERE, "c", "liboracle_rows.so")
_lib = None


def build_oracle_c(force: bool = False) -> str:
    """Compile the plain-C oracle (gcc -O2 -fopenmp, fp64, no fast-math;
    -fcx-limited-range only drops the inf/NaN recovery of C99 complex * and /)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fcx-limited-range", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle_c()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_matvec_rows.argtypes = [ctypes.c_int, ctypes.c_int64, dp, dp, dp, dp, dp,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           dp, ip, ctypes.c_int64, dp]
        lib.oracle_rows.argtypes = [ctypes.c_int, ctypes.c_int64, dp, dp, dp, dp, dp,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ip, ctypes.c_int64, dp]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _geom_arrays(el: Elements):
    return (np.ascontiguousarray(el.verts.reshape(-1, 9)), np.ascontiguousarray(el.centroid),
            np.ascontiguousarray(el.normal), np.ascontiguousarray(el.area),
            np.ascontiguousarray(el.hmax))


def _self(el, rows, k, alpha, kind):
    out = np.empty(rows.size, dtype=np.complex128)
    for s in range(0, rows.size, 4096):       # batches bound the (M,20,20) temporaries
        R = rows[s:s + 4096]
        out[s:s + 4096] = (self_lhs(el.verts[R], k, alpha) if kind == "lhs"
                           else self_rhs(el.verts[R], k, alpha))
    return out


def matvec_rows(el: Elements, rows, x, k: float, alpha: complex, kind: str = "lhs") -> np.ndarray:
    """(A x)_i (kind 'lhs') or (B x)_i (kind 'rhs') for i in rows."""
    lib = _load()
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    xr = x.view(np.float64)
    n = el.centroid.shape[0]
    y = np.zeros(2 * rows.size, dtype=np.float64)
    g = _geom_arrays(el)
    lib.oracle_matvec_rows(0 if kind == "lhs" else 1, n, *(_p(a) for a in g), k,
                           float(np.real(alpha)), float(np.imag(alpha)), _p(xr),
                           rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), rows.size, _p(y))
    yc = y.view(np.complex128).copy()
    yc += _self(el, rows, k, alpha, kind) * x[rows]
    return yc


def dense_rows(el: Elements, rows, k: float, alpha: complex, kind: str = "lhs") -> np.ndarray:
    lib = _load()
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    n = el.centroid.shape[0]
    out = np.zeros((rows.size, n), dtype=np.complex128)
    g = _geom_arrays(el)
    lib.oracle_rows(0 if kind == "lhs" else 1, n, *(_p(a) for a in g), k,
                    float(np.real(alpha)), float(np.imag(alpha)),
                    rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), rows.size,
                    _p(out.view(np.float64)))
    out[np.arange(rows.size), rows] = _self(el, rows, k, alpha, kind)
    return out


def dense(el: Elements, k: float, alpha: complex, kind: str = "lhs") -> np.ndarray:
    return dense_rows(el, np.arange(el.centroid.shape[0]), k, alpha, kind)
